#!/bin/bash
# Eval-throughput A/B on the GPU box: builds scripts/proto/gs_s.cu once per flag set and runs it.
# usage: scripts/proto/run_gs.sh N DELTA "FLAGS_A" "FLAGS_B" ...   (each FLAGS string = extra nvcc -D options)
cd "$(dirname "$0")/../.."
N=$1; DL=$2; shift 2
mkdir -p /tmp/gsp
i=0
for fl in "$@"; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false --expt-relaxed-constexpr -DSS=512 $fl \
    -I paper_2207_06374_b200/csrc -I include -o /tmp/gsp/gs_$i scripts/proto/gs_s.cu || { echo "build failed: $fl"; i=$((i+1)); continue; }
  echo "== [$fl]"
  for dl in $DL; do /tmp/gsp/gs_$i $N $dl; done
  i=$((i+1))
done
