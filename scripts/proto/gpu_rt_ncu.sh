set -x
bash scripts/proto/rt_proto.sh 0 2 100 "0.1" 512 1 "-DMINB=2" 2>&1
ncu --set full --clock-control none --import-source on -k regex:eval_rt_kernel -s 1 -c 1 -o gpurun_out/rt_proto_v1 -f /tmp/rtp/rt_proto 0 100 0.1 2 2>&1 | tail -3
bash scripts/proto/rt_proto.sh 0 2 100 "0.1" 512 2 "" 2>&1
ncu --set full --clock-control none --import-source on -k regex:eval_rt_kernel -s 1 -c 1 -o gpurun_out/rt_proto_v2 -f /tmp/rtp/rt_proto 0 100 0.1 2 2>&1 | tail -3
