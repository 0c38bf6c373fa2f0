# quick GPU check: tests (+ optional extra command in $1)
set -x
timeout 1200 python -m pytest tests -x -q -m gpu ${PYTEST_ARGS} > gpurun_out/gputests.log 2>&1; echo "gpu tests rc=$?"
tail -40 gpurun_out/gputests.log
