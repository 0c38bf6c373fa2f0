set -x
timeout 300 python -m pytest tests/test_gpu_large.py tests/test_gpu_reference_pin.py -x -q -m gpu > gpurun_out/r2_large_large_tests.log 2>&1; echo "large tests rc=$?"; tail -5 gpurun_out/r2_large_large_tests.log
timeout 120 python scripts/large_probe.py 0 128 4096 4 1 1; echo "rc=$?"
timeout 120 python scripts/large_probe.py 1 64 1024 64 2 1; echo "rc=$?"
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum"
timeout 600 ncu --metrics $M --clock-control none -c 300 --csv --log-file gpurun_out/r2_large_launches_c5.csv python scripts/large_probe.py 0 128 4096 4 1 1 > /dev/null 2>&1; echo "rc=$?"
timeout 600 ncu --metrics $M --clock-control none -c 400 --csv --log-file gpurun_out/r2_large_launches_c4.csv python scripts/large_probe.py 1 64 1024 64 2 1 > /dev/null 2>&1; echo "rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:bde_grad_ws -s 2 -c 1 -o gpurun_out/r2_large_grad_c5 -f python scripts/large_probe.py 0 128 4096 4 1 1 > /dev/null 2>&1; echo "rc=$?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:bde_grad_ws -s 2 -c 1 -o gpurun_out/r2_large_grad_c4 -f python scripts/large_probe.py 1 64 1024 64 2 1 > /dev/null 2>&1; echo "rc=$?"
