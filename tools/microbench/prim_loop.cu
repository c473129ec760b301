// Primitive-loop microbenchmark: how fast can the generated (ps|ss) / (ss|ss)
// primitive kernels (Cls*::prim_w1) run with no digestion, no item logic?
// Lanes = kets (ket record in registers), bra records from shared memory
// (warp-broadcast), as in the strip kernels. Also: dependent-chain latencies
// of DFMA / DMUL / MUFU.RSQ64H / LDS.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2412_13203_b200/csrc \
//        tools/microbench/prim_loop.cu -o /tmp/prim_loop
#include <cstdio>
#include <vector>
#include "generated/cls_0000.cu"
#include "generated/cls_1000.cu"
#define CKM(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__);exit(1);}}while(0)
using namespace eritile_b200;

__global__ void lat_kernel(long long* out, double a, int which) {
  double x = a + threadIdx.x;
  long long t0 = clock64();
  if (which == 0) {
#pragma unroll 1
    for (int i = 0; i < 1024; ++i) x = fma(x, a, 1e-9);
  } else if (which == 1) {
#pragma unroll 1
    for (int i = 0; i < 1024; ++i) x = x * a;
  } else {
#pragma unroll 1
    for (int i = 0; i < 1024; ++i) {
      double y;
      asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
      x = y;
    }
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) out[which] = t1 - t0;
  if (x == 1.2345) out[3] = 1;
}

// STYLE 0: one prim per inner step; 1: two bra prims per step (ILP 2)
template <class C, int NT, int STYLE>
__global__ void __launch_bounds__(NT, 1) loop_kernel(const PrimRec* __restrict__ bra_g, const double2* __restrict__ bw_g,
                                                     int kb, const PrimRec* __restrict__ ket_g, int kk, int reps,
                                                     const double* __restrict__ boys, double* out) {
  extern __shared__ __align__(16) double smem[];
  load_boys_for<C>(smem, boys);
  PrimRec* sb = reinterpret_cast<PrimRec*>(smem + BoysStage<C>::nsl * kBoysRows * kBoysCols);
  double2* sw = reinterpret_cast<double2*>(sb + 128);
  for (int t = threadIdx.x; t < kb; t += NT) { sb[t] = bra_g[t]; sw[t] = bw_g[t]; }
  __syncthreads();
  typename C::Acc acc;
  C::zero(acc);
  const int g = blockIdx.x * NT + threadIdx.x;
  for (int r = 0; r < reps; ++r) {
    for (int j = 0; j < kk; ++j) {
      const PrimRec kp = load_prim<C::KPA>(ket_g + ((g + j * 7 + r) & 1023));
      typename C::Acc s;
      C::zero(s);
      if constexpr (STYLE == 0) {
        for (int i = 0; i < kb; ++i) C::prim_w1(load_prim_gen<C::BPA>(sb + i), kp, smem, sw[i].x, s);
      } else {
        typename C::Acc s2;
        C::zero(s2);
        for (int i = 0; i < kb; i += 2) {
          C::prim_w1(load_prim_gen<C::BPA>(sb + i), kp, smem, sw[i].x, s);
          C::prim_w1(load_prim_gen<C::BPA>(sb + i + 1), kp, smem, sw[i + 1].x, s2);
        }
        C::fold(s, s2);
      }
      C::axpy(acc, 1.0, s);
    }
  }
  double o[C::NV];
  C::finish(acc, 0, 0, 0, 0, 0, 0, o);
  double t = 0;
  for (int v = 0; v < C::NV; ++v) t += o[v];
  if (t == 1.2345) out[0] = t;
}

template <class C, int NT, int STYLE>
void run(const char* name, const PrimRec* bra, const double2* bw, int kb, const PrimRec* ket, int kk, const double* boys,
         double* out) {
  auto fn = loop_kernel<C, NT, STYLE>;
  size_t smem = BoysStage<C>::bytes + (sizeof(PrimRec) + sizeof(double2)) * 128;
  CKM(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  cudaFuncAttributes at;
  cudaFuncGetAttributes(&at, fn);
  int bps = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, fn, NT, smem);
  int reps = 8;
  int grid = 148 * bps * 4;
  fn<<<grid, NT, smem>>>(bra, bw, kb, ket, kk, reps, boys, out);
  CKM(cudaDeviceSynchronize());
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  fn<<<grid, NT, smem>>>(bra, bw, kb, ket, kk, reps, boys, out);
  cudaEventRecord(e1);
  CKM(cudaEventSynchronize(e1));
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double prims = (double)grid * NT * reps * kk * kb;
  double per_sm_clk = prims / (ms * 1e-3) / (148 * 1.965e9);
  printf("%-28s NT=%4d regs=%3d bps=%d  %.3e prim/s  %.3f prim/SM/clk  %.2f ns/prim-lane\n", name, NT, at.numRegs, bps,
         prims / (ms * 1e-3), per_sm_clk, ms * 1e6 / prims * 148 * NT * bps);
}

int main() {
  long long* dlat; CKM(cudaMalloc(&dlat, 64));
  lat_kernel<<<1, 32>>>(dlat, 0.999, 0); lat_kernel<<<1, 32>>>(dlat, 0.999, 1); lat_kernel<<<1, 32>>>(dlat, 0.999, 2);
  CKM(cudaDeviceSynchronize());
  long long h[4]; cudaMemcpy(h, dlat, 32, cudaMemcpyDeviceToHost);
  printf("latency (cycles): DFMA %.1f  DMUL %.1f  MUFU.RSQ64H %.1f\n", h[0] / 1024.0, h[1] / 1024.0, h[2] / 1024.0);
  // synthetic records: water-like exponents, positions in a 20 bohr box
  std::vector<PrimRec> hb(128), hk(1024);
  std::vector<double2> hw(128);
  srand(1);
  auto fill = [](PrimRec& r) {
    r.p = 0.2 + 50.0 * (rand() / (double)RAND_MAX);
    r.U = 0.1; r.Px = 20.0 * rand() / RAND_MAX; r.Py = 20.0 * rand() / RAND_MAX; r.Pz = 20.0 * rand() / RAND_MAX;
    r.i2p = 0.5 / r.p; r.PAx = 0.1; r.PAy = -0.2; r.PAz = 0.05; r.pad = 0;
  };
  for (auto& r : hb) fill(r);
  for (auto& r : hk) fill(r);
  for (auto& w : hw) w = make_double2(0.3, 0.2);
  PrimRec *db, *dk; double2* dw; double* out;
  CKM(cudaMalloc(&db, sizeof(PrimRec) * 128)); CKM(cudaMalloc(&dk, sizeof(PrimRec) * 1024));
  CKM(cudaMalloc(&dw, sizeof(double2) * 128)); CKM(cudaMalloc(&out, 64));
  cudaMemcpy(db, hb.data(), sizeof(PrimRec) * 128, cudaMemcpyHostToDevice);
  cudaMemcpy(dk, hk.data(), sizeof(PrimRec) * 1024, cudaMemcpyHostToDevice);
  cudaMemcpy(dw, hw.data(), sizeof(double2) * 128, cudaMemcpyHostToDevice);
  // Boys table: any finite values (timing only)
  std::vector<double> tab((size_t)(kBoysMmax + 1) * kBoysRows * kBoysCols, 0.01);
  double* dtab; CKM(cudaMalloc(&dtab, tab.size() * 8));
  cudaMemcpy(dtab, tab.data(), tab.size() * 8, cudaMemcpyHostToDevice);
  for (int kb : {16, 80}) {
    printf("-- kb=%d kk=9\n", kb);
    run<Cls0000, 512, 0>("(ss|ss) plain", db, dw, kb, dk, 9, dtab, out);
    run<Cls0000, 768, 0>("(ss|ss) plain", db, dw, kb, dk, 9, dtab, out);
    run<Cls0000, 1024, 0>("(ss|ss) plain", db, dw, kb, dk, 9, dtab, out);
    run<Cls0000, 512, 1>("(ss|ss) ilp2", db, dw, kb, dk, 9, dtab, out);
    run<Cls0000, 768, 1>("(ss|ss) ilp2", db, dw, kb, dk, 9, dtab, out);
    run<Cls1000, 512, 0>("(ps|ss) plain", db, dw, kb, dk, 9, dtab, out);
    run<Cls1000, 768, 0>("(ps|ss) plain", db, dw, kb, dk, 9, dtab, out);
    run<Cls1000, 1024, 0>("(ps|ss) plain", db, dw, kb, dk, 9, dtab, out);
    run<Cls1000, 512, 1>("(ps|ss) ilp2", db, dw, kb, dk, 9, dtab, out);
    run<Cls1000, 768, 1>("(ps|ss) ilp2", db, dw, kb, dk, 9, dtab, out);
  }
  return 0;
}
