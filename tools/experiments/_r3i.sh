# RED.ADD.F64 throughput by warp address pattern.
O=gpurun_out/r03i; mkdir -p $O
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/microbench/red_pattern tools/microbench/red_pattern.cu
timeout 120 tools/microbench/red_pattern > $O/red_pattern.txt 2>&1
cat $O/red_pattern.txt
