# quick GPU check: tests + micro probes (output under gpurun_out/)
set -x
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/gputests.log 2>&1; echo "gpu tests rc=$?"
tail -5 gpurun_out/gputests.log
timeout 300 ./scripts/micro/dmma > gpurun_out/dmma.txt 2>&1; echo "dmma rc=$?"
cat gpurun_out/dmma.txt
