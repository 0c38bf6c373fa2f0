set -x
cd scripts/micro
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -o /tmp/dfma_ports dfma_ports.cu && /tmp/dfma_ports
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -fmad=false -o /tmp/fp64_ops fp64_ops.cu && /tmp/fp64_ops
