set -u
O=gpurun_out/r4c; mkdir -p $O
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/dfma_ilp tools/probe/dfma_ilp.cu && /tmp/dfma_ilp > $O/dfma_ilp.txt 2>&1; cat $O/dfma_ilp.txt
