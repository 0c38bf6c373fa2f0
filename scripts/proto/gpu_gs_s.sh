for U in 2 4 5; do nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -fmad=false --expt-relaxed-constexpr -DSS=512 -DTRSTMI_GS_UNROLL=$U -I paper_2207_06374_b200/csrc -I include -o /tmp/gs_u$U scripts/proto/gs_s.cu; echo "unroll $U"; for dl in 0.1 1e-5; do /tmp/gs_u$U 100 $dl; done; done
bash scripts/phase_timers.sh 0 2 100 0.1 512 1 1
