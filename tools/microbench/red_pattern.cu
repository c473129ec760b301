// RED.ADD.F64 throughput by address pattern (B200): does the L2 merge the
// lanes of one warp-level RED that fall into the same 32-B sector?
//   scattered : every lane its own random sector (the lane kernels' K updates)
//   triples   : lanes in groups of 3 on 3 consecutive doubles (a p-shell column
//               triple per ket, after a shuffle transpose), groups random
//   sextets   : groups of 6 (d-shell columns)
//   contiguous: 32 consecutive doubles per warp instruction
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o red_pattern red_pattern.cu
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned hash(unsigned x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16;
  return x;
}

template <int G>  // lanes per group on consecutive addresses (1 = scattered, 32 = contiguous)
__global__ void red_kernel(double* buf, size_t n, int iters) {
  const int lane = threadIdx.x & 31;
  const unsigned warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int grp = lane / G, pos = lane % G;
  for (int it = 0; it < iters; ++it) {
    const unsigned h = hash(warp * 1315423911u + it * 2654435761u + grp * 97u);
    size_t base = (static_cast<size_t>(h) * 8) % (n - 64);
    if (G == 32) base &= ~static_cast<size_t>(31);
    if (lane < (32 / G) * G) atomicAdd(buf + base + pos, 1.0);
  }
}

template <int G>
void run(double* buf, size_t n, const char* name) {
  const int blocks = 148 * 8, threads = 256, iters = 2000;
  red_kernel<G><<<blocks, threads>>>(buf, n, 10);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  red_kernel<G><<<blocks, threads>>>(buf, n, iters);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  const double ops = double(blocks) * threads / 32 * ((32 / G) * G) * iters;
  printf("%-12s %8.1f G element-REDs/s  %8.2f G warp-instr/s\n", name, ops / ms / 1e6,
         double(blocks) * threads / 32 * iters / ms / 1e6);
}

int main() {
  const size_t n = 4000000;  // 32 MB (the K matrix at N = 2000), L2-resident
  double* buf;
  cudaMalloc(&buf, n * sizeof(double));
  cudaMemset(buf, 0, n * sizeof(double));
  run<1>(buf, n, "scattered");
  run<2>(buf, n, "pairs");
  run<3>(buf, n, "triples");
  run<6>(buf, n, "sextets");
  run<32>(buf, n, "contiguous");
  cudaError_t e = cudaDeviceSynchronize();
  printf("%s\n", cudaGetErrorString(e));
  return 0;
}
