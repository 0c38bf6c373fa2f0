# BDE per-kernel times (configs 4, 5) and ncu --set full of the two DMMA kernels at config 5
set -x
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum"
python scripts/large_probe.py 0 128 4096 4 1 1 > gpurun_out/s4_probe_c5.txt 2>&1; echo "rc=$?"; cat gpurun_out/s4_probe_c5.txt
python scripts/large_probe.py 1 64 1024 64 2 1 > gpurun_out/s4_probe_c4.txt 2>&1; echo "rc=$?"; cat gpurun_out/s4_probe_c4.txt
timeout 900 ncu --metrics $M --clock-control none -c 300 --csv --log-file gpurun_out/s4_bde_launches_c5.csv python scripts/large_probe.py 0 128 4096 4 1 1 > gpurun_out/s4_ncu_c5.log 2>&1; echo "rc=$?"
timeout 900 ncu --metrics $M --clock-control none -c 400 --csv --log-file gpurun_out/s4_bde_launches_c4.csv python scripts/large_probe.py 1 64 1024 64 2 1 > gpurun_out/s4_ncu_c4.log 2>&1; echo "rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bde_gram -s 2 -c 1 -o gpurun_out/s4_bde_gram_c5 -f python scripts/large_probe.py 0 128 4096 4 1 1 > gpurun_out/s4_ncu_gram.log 2>&1; echo "rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:bde_grad -s 2 -c 1 -o gpurun_out/s4_bde_grad_c5 -f python scripts/large_probe.py 0 128 4096 4 1 1 > gpurun_out/s4_ncu_grad.log 2>&1; echo "rc=$?"
ls -la gpurun_out
