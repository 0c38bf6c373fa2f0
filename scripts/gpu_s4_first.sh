# session-4 first GPU call: tests, BDE benches (c4, c5), C2 phase timers and per-stage timing
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/s4_gputests.log 2>&1; echo "gpu tests rc=$?"
tail -3 gpurun_out/s4_gputests.log
timeout 600 python bench.py --config c4 --steps 2 --warmup 3 --cpu-budget 20 > gpurun_out/s4_bench_c4.json 2> gpurun_out/s4_bench_c4.err; echo "c4 rc=$?"
cat gpurun_out/s4_bench_c4.json
timeout 900 python bench.py --config c5 --steps 1 --warmup 3 --no-cpu > gpurun_out/s4_bench_c5.json 2> gpurun_out/s4_bench_c5.err; echo "c5 rc=$?"
cat gpurun_out/s4_bench_c5.json
for dl in 0.1 0.01 0.001 1e-5 6e-9; do bash scripts/phase_timers.sh 0 2 100 $dl 512 1 1; done > gpurun_out/s4_phase_c2.txt 2>&1
cat gpurun_out/s4_phase_c2.txt
for ns in 1 2 3 4 6 8; do python scripts/run_solve.py 0 2 100 592 500 $ns; done > gpurun_out/s4_stage_times_c2.txt 2>&1
cat gpurun_out/s4_stage_times_c2.txt
