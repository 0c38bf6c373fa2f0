#!/bin/bash
# Anneal-level A/B on the GPU box: builds scripts/proto/an_s.cu per flag set and runs it.
# usage: scripts/proto/run_an.sh "TRIALS STAGES [MAX_OUTER]" "FLAGS_A" "FLAGS_B" ...
cd "$(dirname "$0")/../.."
ARGS=$1; shift
mkdir -p /tmp/gsp
i=0
for fl in "$@"; do
  nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false --expt-relaxed-constexpr $fl \
    -I paper_2207_06374_b200/csrc -I include -o /tmp/gsp/an_$i scripts/proto/an_s.cu || { echo "build failed: $fl"; i=$((i+1)); continue; }
  echo "== [$fl]"
  /tmp/gsp/an_$i $ARGS
  i=$((i+1))
done
