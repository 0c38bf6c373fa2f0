set -x
bash scripts/proto/rt_proto.sh 0 2 100 "0.1 1e-5" 512 1 "-DMINB=2" 2>&1
bash scripts/proto/rt_proto.sh 0 2 100 "0.1 1e-5" 512 2 "-DMINB=3 -DNVEC=2" 2>&1
bash scripts/proto/rt_proto.sh 0 2 100 "0.1" 512 1 "-DMINB=2 -DPT" 2>&1
