# Config-2 profiles of the round: launch list of a short bench run, ncu --set full of the anneal kernel, source page.
set -x
python bench.py --steps 2 --warmup 3 --no-cpu --trials 296 --slice 148 > gpurun_out/r2_c2_short_bench.json 2> gpurun_out/r2_c2_short_bench.err; echo "short bench rc=$?"
M="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum"
timeout 900 ncu --metrics $M --clock-control none -c 400 --csv --log-file gpurun_out/r2_launches_c2.csv python bench.py --steps 2 --warmup 3 --no-cpu --trials 296 --slice 148 > /dev/null 2>&1; echo "launch list rc=$?"
python scripts/launch_summary.py gpurun_out/r2_launches_c2.csv > gpurun_out/r2_launches_c2.txt 2>&1; cat gpurun_out/r2_launches_c2.txt
python scripts/run_solve.py 0 2 100 148 20 1; echo "run_solve rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:anneal_small -c 1 -o gpurun_out/r2_anneal_c2 -f python scripts/run_solve.py 0 2 100 148 20 1 > /dev/null 2>&1; echo "ncu full rc=$?"
ls -la gpurun_out/*.ncu-rep
