set -x
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/r2_gputests.log 2>&1; echo "gpu tests rc=$?"; tail -3 gpurun_out/r2_gputests.log
timeout 600 python bench.py --config c4 --steps 2 --warmup 3 --cpu-budget 20 > gpurun_out/r2_bench_c4.json 2> gpurun_out/r2_bench_c4.err; echo "c4 rc=$?"
cat gpurun_out/r2_bench_c4.json
timeout 900 python bench.py --config c5 --steps 1 --warmup 1 --no-cpu > gpurun_out/r2_bench_c5.json 2> gpurun_out/r2_bench_c5.err; echo "c5 rc=$?"
cat gpurun_out/r2_bench_c5.json
