// Microbenchmarks that set the FP64 roofline denominator and the FP64 global
// atomic (RED.ADD.F64) throughput that bounds unaggregated J/K digestion.
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__);exit(1);}}while(0)

__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
  double x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  double s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
  if (s == 12345.678) out[0] = s;
}

__global__ void red_kernel(double* acc, unsigned mask, int iters, int stride_mode) {
  unsigned tid = blockIdx.x * blockDim.x + threadIdx.x;
  unsigned h = tid * 2654435761u;
  for (int i = 0; i < iters; ++i) {
    h = h * 1664525u + 1013904223u;
    unsigned idx = stride_mode == 0 ? (h & mask) : ((tid + i * 97) & mask);
    atomicAdd(acc + idx, 1.0);
  }
}

int main() {
  int dev = 0; cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  printf("{\"device\": \"%s\", \"sms\": %d, \"clock_khz\": %d", p.name, p.multiProcessorCount, p.clockRate);
  double* out; CK(cudaMalloc(&out, 8));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int blocks = p.multiProcessorCount * 8, threads = 256, iters = 4096;
  for (int w = 0; w < 3; ++w) dfma_kernel<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
  CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < 10; ++r) {
    cudaEventRecord(e0); dfma_kernel<<<blocks, threads>>>(out, iters, 0.999999, 1e-7); cudaEventRecord(e1);
    cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
  }
  double flops = 2.0 * 8 * 16 * (double)iters * blocks * threads;
  printf(", \"fp64_fma_tflops\": %.3f", flops / (best * 1e-3) / 1e12);
  // atomics: random addresses within a window (L2 resident), 4 window sizes
  size_t maxn = 1u << 25;  // 32M doubles = 256 MB
  double* acc; CK(cudaMalloc(&acc, maxn * 8)); CK(cudaMemset(acc, 0, maxn * 8));
  unsigned masks[4] = {(1u << 12) - 1, (1u << 19) - 1, (1u << 22) - 1, (1u << 25) - 1};
  const char* names[4] = {"32KB", "4MB", "32MB", "256MB"};
  for (int m = 0; m < 4; ++m) {
    int ab = p.multiProcessorCount * 16, at = 256, ai = 256;
    red_kernel<<<ab, at>>>(acc, masks[m], ai, 0); CK(cudaDeviceSynchronize());
    float bm = 1e30f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0); red_kernel<<<ab, at>>>(acc, masks[m], ai, 0); cudaEventRecord(e1);
      cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < bm) bm = ms;
    }
    double n = (double)ab * at * ai;
    printf(", \"red_f64_random_%s_Gops\": %.1f", names[m], n / (bm * 1e-3) / 1e9);
  }
  {
    int ab = p.multiProcessorCount * 16, at = 256, ai = 256;
    float bm = 1e30f;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0); red_kernel<<<ab, at>>>(acc, masks[2], ai, 1); cudaEventRecord(e1);
      cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < bm) bm = ms;
    }
    double n = (double)ab * at * ai;
    printf(", \"red_f64_coalesced_32MB_Gops\": %.1f", n / (bm * 1e-3) / 1e9);
  }
  printf("}\n");
  return 0;
}
