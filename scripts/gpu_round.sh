# round-end check: GPU tests, then the driver's exact bench commands (reference arm first)
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
nproc; lscpu | head -20
timeout 1200 python -m pytest tests -x -q -m gpu > gpurun_out/r2_gputests.log 2>&1; echo "gpu tests rc=$?"
tail -3 gpurun_out/r2_gputests.log
( time timeout 1700 python bench.py --impl reference --gpus 1 --steps 20 --warmup 5 ) > gpurun_out/r2_ref.json 2> gpurun_out/r2_ref.err; echo "ref rc=$?"
( time timeout 1700 python bench.py --gpus 1 --steps 20 --warmup 5 ) > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err; echo "bench rc=$?"
cat gpurun_out/r2_ref.json gpurun_out/r2_bench.json; tail -n 5 gpurun_out/r2_ref.err; tail -n 5 gpurun_out/r2_bench.err
