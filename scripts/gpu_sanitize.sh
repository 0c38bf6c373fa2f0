# compute-sanitizer passes over the kernels changed in round 2, session 5 (short runs).
set -x
export PATH=$PATH:/usr/local/cuda/bin
timeout 900 compute-sanitizer --tool racecheck --racecheck-report all python scripts/run_solve.py 0 2 100 2 2 1 > gpurun_out/sanitize_race_c2.log 2>&1; echo "racecheck c2 rc=$?"; tail -4 gpurun_out/sanitize_race_c2.log
timeout 900 compute-sanitizer --tool racecheck --racecheck-report all python scripts/run_solve.py 0 6 36 2 3 2 > gpurun_out/sanitize_race_c3.log 2>&1; echo "racecheck c3 rc=$?"; tail -4 gpurun_out/sanitize_race_c3.log
timeout 900 compute-sanitizer --tool memcheck python scripts/run_solve.py 0 2 100 2 2 1 > gpurun_out/sanitize_mem_c2.log 2>&1; echo "memcheck c2 rc=$?"; tail -4 gpurun_out/sanitize_mem_c2.log
timeout 900 compute-sanitizer --tool memcheck python -c "
from paper_2207_06374_b200 import baseline
r = baseline.solve_altproj(3, 9, baseline.AltProjConfig(max_iters=20), 2, 42); print(r.best_coherence)
r = baseline.solve_altproj(2, 33, baseline.AltProjConfig(max_iters=5), 2, 1); print(r.best_coherence)
" > gpurun_out/sanitize_mem_altproj.log 2>&1; echo "memcheck altproj rc=$?"; tail -4 gpurun_out/sanitize_mem_altproj.log
timeout 900 compute-sanitizer --tool racecheck --racecheck-report all python -c "
from paper_2207_06374_b200 import baseline
r = baseline.solve_altproj(3, 9, baseline.AltProjConfig(max_iters=10), 2, 42); print(r.best_coherence)
" > gpurun_out/sanitize_race_altproj.log 2>&1; echo "racecheck altproj rc=$?"; tail -4 gpurun_out/sanitize_race_altproj.log
