timeout 300 python -m pytest tests/test_gpu_large.py tests/test_gpu_reference_pin.py -x -q -m gpu 2>&1 | tail -2
timeout 120 python scripts/large_probe.py 1 64 1024 64 2 1 | head -1
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum"
timeout 600 ncu --metrics $M --clock-control none -c 400 --csv --log-file gpurun_out/s4_ws_launches_c4.csv python scripts/large_probe.py 1 64 1024 64 2 1 > /dev/null 2>&1; echo "rc=$?"
timeout 600 python bench.py --config c4 --steps 2 --warmup 2 --no-cpu > gpurun_out/s4c_bench_c4.json 2> gpurun_out/s4c_bench_c4.err; echo "c4 rc=$?"
