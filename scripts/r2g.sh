mkdir -p gpurun_out/r2g
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mufu_tp scripts/ubench/mufu_tp.cu && /tmp/mufu_tp > gpurun_out/r2g/mufu.txt 2>&1
