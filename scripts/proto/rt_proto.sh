#!/bin/bash
# usage: scripts/proto/rt_proto.sh FIELD D N "DELTAS" [S] [V] [extra nvcc flags]
set -e
cd "$(dirname "$0")/../.."
mkdir -p /tmp/rtp
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -fmad=false --expt-relaxed-constexpr -DDD=$2 -DSS=${5:-512} -DVV=${6:-2} $7 \
  -I paper_2207_06374_b200/csrc -I scripts/proto -I include -o /tmp/rtp/rt_proto scripts/proto/rt_proto.cu
for dl in $4; do /tmp/rtp/rt_proto $1 $3 $dl; done
