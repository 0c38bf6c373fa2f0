M="gpu__time_duration.sum"
for v in "1 0" "0 1" "0 0"; do set -- $v
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false --expt-relaxed-constexpr -Xcompiler -fPIC,-ffp-contract=off,-O2 -I include -DTRSTMI_WS_NTW=$1 -DTRSTMI_WS_DEEP=$2 -c paper_2207_06374_b200/csrc/bde_engine.cu -o paper_2207_06374_b200/_build/bde_engine.o
  nvcc -gencode arch=compute_100a,code=sm_100a -shared -o paper_2207_06374_b200/_lib/libtrstmi_b200.so paper_2207_06374_b200/_build/*.o -cudart static -lnccl
  echo "== NTW=$1 DEEP=$2"
  python scripts/large_probe.py 1 64 1024 64 2 1 | head -1
  ncu --metrics $M --clock-control none -c 400 --csv --log-file gpurun_out/var_$1$2.csv python scripts/large_probe.py 1 64 1024 64 2 1 > /dev/null 2>&1
  python scripts/launch_summary.py gpurun_out/var_$1$2.csv | sed -n 2,2p
done
