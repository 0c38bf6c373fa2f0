echo "== UW=5 only"; EXTRA="-DTRSTMI_EXP_UW=5" bash scripts/phase_timers.sh 0 2 100 0.1 512 1 1
echo "== UW=2 only, tiled"; EXTRA="-DTRSTMI_EXP_UW=2" bash scripts/phase_timers.sh 0 2 100 0.1 512 1 1
echo "== UW=2 only, untiled"; EXTRA="-DTRSTMI_EXP_UW=2 -DTRSTMI_TILED_MIN=1000" bash scripts/phase_timers.sh 0 2 100 0.1 512 1 1
echo "== UW=5 only, untiled"; EXTRA="-DTRSTMI_EXP_UW=5 -DTRSTMI_TILED_MIN=1000" bash scripts/phase_timers.sh 0 2 100 0.1 512 1 1
