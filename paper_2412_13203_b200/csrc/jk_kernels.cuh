// Fused Schwarz-screened ERI + J/K digestion kernels (sm_100a, FP64).
//
// Work mapping: one warp per WorkItem = one bra pair x
// (warp-uniform) against up to 32 ket pairs y (one per lane). Kets of a
// work item come from one (class, contraction-degree) group sorted by
// Schwarz Q, so all lanes share the primitive trip count (Permutation).
// Each lane evaluates its contracted quartet with the class's generated
// straight-line plan (Cls*::eri), then digests it: J_ab is warp-reduced and
// flushed once per warp, J_cd and the four K blocks are FP64 atomics
// (RED.ADD.F64) into the accumulation matrices. The digestion follows the
// shell-level degeneracy rule of SPEC.md:350 with J weight deg/2 and K
// weight deg/4, so true J = sym(Jacc) and true K = sym(Kacc) after the
// finalize kernel.
#pragma once
#include <cuda_runtime.h>

#include "jk_api.h"

namespace eritile_b200 {

__device__ __forceinline__ PrimRec load_prim(const PrimRec* p) {
  const double2* q = reinterpret_cast<const double2*>(p);
  double2 a = __ldg(q), b = __ldg(q + 1), c = __ldg(q + 2), d = __ldg(q + 3), e = __ldg(q + 4);
  PrimRec r;
  r.p = a.x; r.Px = a.y; r.Py = b.x; r.Pz = b.y; r.PAx = c.x; r.PAy = c.y; r.PAz = d.x;
  r.U = d.y; r.i2p = e.x; r.pad = e.y;
  return r;
}

// Boys function F_0..F_M(T). T < 40: 8-term Taylor expansion of F_M about the
// nearest grid point T_i = i/16 (|d| <= 1/32, truncation < 3e-17 relative)
// from a table of F_{M+k}(T_i)/k! computed in extended precision at build
// time, exp(-T) = exp(-T_i) exp(-d) from the same table, then the stable
// downward recursion F_{m-1} = (2T F_m + e^-T)/(2m-1) (boys.hpp:40-41).
// T >= 40: F_0 = sqrt(pi/T)/2 (erf(sqrt T) = 1 - O(1e-19)) and the upward
// recursion F_{m+1} = ((2m+1) F_m - e^-T)/(2T) (boys.hpp:43), contractive
// for 2m+1 < 2T; e^-T is dropped above T = 80 where it is < 1e-34.
template <int M>
__device__ __forceinline__ void boys_eval(double T, const double* __restrict__ tab, double* F) {
  if (T < kBoysTmax) {
    const int i = __double2int_rn(T * 16.0);
    const double md = fma(static_cast<double>(i), 0.0625, -T);  // -(T - T_i)
    const double* r = tab + i * kBoysCols;
    double f = r[7];
#pragma unroll
    for (int k = 6; k >= 0; --k) f = fma(f, md, r[k]);
    F[M] = f;
    if (M > 0) {
      // exp(-d) = sum_k (-d)^k / k!, k <= 8
      double e = 2.48015873015873016e-05;
      e = fma(e, md, 1.98412698412698413e-04);
      e = fma(e, md, 1.38888888888888889e-03);
      e = fma(e, md, 8.33333333333333333e-03);
      e = fma(e, md, 4.16666666666666667e-02);
      e = fma(e, md, 1.66666666666666667e-01);
      e = fma(e, md, 0.5);
      e = fma(e, md, 1.0);
      e = fma(e, md, 1.0);
      e *= r[8];
      const double T2 = 2.0 * T;
#pragma unroll
      for (int m = M; m > 0; --m) F[m - 1] = fma(T2, F[m], e) * (1.0 / (2 * m - 1));
    }
  } else {
    const double rt = rsqrt(T);
    F[0] = 0.88622692545275801365 * rt;  // sqrt(pi)/2
    if (M > 0) {
      const double e = T < 80.0 ? exp(-T) : 0.0;
      const double h = 0.5 * rt * rt;  // 1/(2T)
#pragma unroll
      for (int m = 0; m < M; ++m) F[m + 1] = fma(static_cast<double>(2 * m + 1), F[m], -e) * h;
    }
  }
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Component normalisation (molecule.hpp:207-213) for L <= 4, x-major order.
__device__ __forceinline__ double comp_scale(int L, int i) {
  // sqrt((2L-1)!! / prod (2a_k-1)!!)
  constexpr double s2[6] = {1.0, 1.7320508075688772, 1.7320508075688772, 1.0, 1.7320508075688772, 1.0};
  constexpr double s3[10] = {1.0, 2.23606797749979, 2.23606797749979, 2.23606797749979,
                             3.872983346207417, 2.23606797749979, 1.0, 2.23606797749979,
                             2.23606797749979, 1.0};
  constexpr double s4[15] = {1.0, 2.6457513110645907, 2.6457513110645907, 3.415650255319866,
                             5.916079783099616, 3.415650255319866, 2.6457513110645907,
                             5.916079783099616, 5.916079783099616, 2.6457513110645907, 1.0,
                             2.6457513110645907, 3.415650255319866, 2.6457513110645907, 1.0};
  if (L <= 1) return 1.0;
  if (L == 2) return s2[i];
  if (L == 3) return s3[i];
  return s4[i];
}

template <class C>
__global__ void __launch_bounds__(128) jk_kernel(const WorkItem* __restrict__ items, long long nitems,
                                                 const PairMeta* __restrict__ pm,
                                                 const PrimRec* __restrict__ prims,
                                                 const double* __restrict__ D, double* __restrict__ J,
                                                 double* __restrict__ K, int N,
                                                 const double* __restrict__ boys_tab) {
  extern __shared__ double s_boys[];
  const double* gt = boys_tab + static_cast<size_t>(C::M) * kBoysRows * kBoysCols;
  for (int t = threadIdx.x; t < kBoysRows * kBoysCols; t += blockDim.x) s_boys[t] = gt[t];
  __syncthreads();

  const int lane = threadIdx.x & 31;
  const long long warps = static_cast<long long>(gridDim.x) * (blockDim.x >> 5);
  for (long long w = static_cast<long long>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
       w < nitems; w += warps) {
    const WorkItem it = items[w];
    const PairMeta bm = pm[it.bra];
    const bool active = lane < it.kcnt;
    const int y = it.kbeg + (active ? lane : 0);
    const PairMeta km = pm[y];
    double v[C::NV];
    C::eri(prims + bm.prim_off, bm.K, prims + km.prim_off, active ? km.K : 0, bm.ABx, bm.ABy, bm.ABz,
           km.ABx, km.ABy, km.ABz, s_boys, v);
    const double deg = (bm.sha != bm.shb ? 2.0 : 1.0) * (km.sha != km.shb ? 2.0 : 1.0) *
                       (it.bra != y ? 2.0 : 1.0);
    const double wj = active ? 0.5 * deg : 0.0;
    const double wk = active ? 0.25 * deg : 0.0;
    const size_t n = static_cast<size_t>(N);
    const double* Dab = D + bm.bfa * n + bm.bfb;
    const double* Dcd = D + km.bfa * n + km.bfb;
    const double* Dac = D + bm.bfa * n + km.bfa;
    const double* Dad = D + bm.bfa * n + km.bfb;
    const double* Dbc = D + bm.bfb * n + km.bfa;
    const double* Dbd = D + bm.bfb * n + km.bfb;
    // J_ab: warp-uniform bra -> reduce over lanes, one flush per warp
#pragma unroll
    for (int a = 0; a < C::NA; ++a)
#pragma unroll
      for (int b = 0; b < C::NB; ++b) {
        double s = 0.0;
#pragma unroll
        for (int c = 0; c < C::NC; ++c)
#pragma unroll
          for (int d = 0; d < C::ND; ++d)
            s = fma(v[((a * C::NB + b) * C::NC + c) * C::ND + d], __ldg(Dcd + c * n + d), s);
        s = warp_sum(s * wj);
        if (lane == 0) atomicAdd(J + (bm.bfa + a) * n + bm.bfb + b, s);
      }
    if (active) {
#pragma unroll
      for (int c = 0; c < C::NC; ++c)
#pragma unroll
        for (int d = 0; d < C::ND; ++d) {
          double s = 0.0;
#pragma unroll
          for (int a = 0; a < C::NA; ++a)
#pragma unroll
            for (int b = 0; b < C::NB; ++b)
              s = fma(v[((a * C::NB + b) * C::NC + c) * C::ND + d], __ldg(Dab + a * n + b), s);
          atomicAdd(J + (km.bfa + c) * n + km.bfb + d, s * wj);
        }
      // K_ac += sum_bd v D_bd ; K_bd += sum_ac v D_ac
#pragma unroll
      for (int a = 0; a < C::NA; ++a)
#pragma unroll
        for (int c = 0; c < C::NC; ++c) {
          double s = 0.0;
#pragma unroll
          for (int b = 0; b < C::NB; ++b)
#pragma unroll
            for (int d = 0; d < C::ND; ++d)
              s = fma(v[((a * C::NB + b) * C::NC + c) * C::ND + d], __ldg(Dbd + b * n + d), s);
          atomicAdd(K + (bm.bfa + a) * n + km.bfa + c, s * wk);
        }
#pragma unroll
      for (int b = 0; b < C::NB; ++b)
#pragma unroll
        for (int d = 0; d < C::ND; ++d) {
          double s = 0.0;
#pragma unroll
          for (int a = 0; a < C::NA; ++a)
#pragma unroll
            for (int c = 0; c < C::NC; ++c)
              s = fma(v[((a * C::NB + b) * C::NC + c) * C::ND + d], __ldg(Dac + a * n + c), s);
          atomicAdd(K + (bm.bfb + b) * n + km.bfb + d, s * wk);
        }
      // K_ad += sum_bc v D_bc ; K_bc += sum_ad v D_ad
#pragma unroll
      for (int a = 0; a < C::NA; ++a)
#pragma unroll
        for (int d = 0; d < C::ND; ++d) {
          double s = 0.0;
#pragma unroll
          for (int b = 0; b < C::NB; ++b)
#pragma unroll
            for (int c = 0; c < C::NC; ++c)
              s = fma(v[((a * C::NB + b) * C::NC + c) * C::ND + d], __ldg(Dbc + b * n + c), s);
          atomicAdd(K + (bm.bfa + a) * n + km.bfb + d, s * wk);
        }
#pragma unroll
      for (int b = 0; b < C::NB; ++b)
#pragma unroll
        for (int c = 0; c < C::NC; ++c) {
          double s = 0.0;
#pragma unroll
          for (int a = 0; a < C::NA; ++a)
#pragma unroll
            for (int d = 0; d < C::ND; ++d)
              s = fma(v[((a * C::NB + b) * C::NC + c) * C::ND + d], __ldg(Dad + a * n + d), s);
          atomicAdd(K + (bm.bfb + b) * n + km.bfa + c, s * wk);
        }
    }
  }
}

// Schwarz diagonal: Q_x = sqrt(max_{mu,nu} |(mu nu|mu nu)|) over normalised
// components, one lane per pair.
template <class C>
__global__ void __launch_bounds__(128) schwarz_kernel(const int* __restrict__ list, long long n,
                                                      const PairMeta* __restrict__ pm,
                                                      const PrimRec* __restrict__ prims,
                                                      double* __restrict__ Q,
                                                      const double* __restrict__ boys_tab) {
  extern __shared__ double s_boys[];
  const double* gt = boys_tab + static_cast<size_t>(C::M) * kBoysRows * kBoysCols;
  for (int t = threadIdx.x; t < kBoysRows * kBoysCols; t += blockDim.x) s_boys[t] = gt[t];
  __syncthreads();
  for (long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<long long>(gridDim.x) * blockDim.x) {
    const int x = list[i];
    const PairMeta m = pm[x];
    double v[C::NV];
    C::eri(prims + m.prim_off, m.K, prims + m.prim_off, m.K, m.ABx, m.ABy, m.ABz, m.ABx, m.ABy,
           m.ABz, s_boys, v);
    double mx = 0.0;
#pragma unroll
    for (int a = 0; a < C::NA; ++a)
#pragma unroll
      for (int b = 0; b < C::NB; ++b) {
        const double s = comp_scale(C::LA, a) * comp_scale(C::LB, b);
        const double val = fabs(v[((a * C::NB + b) * C::NC + a) * C::ND + b]) * (s * s);
        mx = fmax(mx, val);
      }
    Q[x] = sqrt(mx);
  }
}

// Raw (unscaled) integrals of explicit quartets, one thread each (tests and
// the eritile_gpu_eri_quartet entry point).
template <class C>
__global__ void __launch_bounds__(128) quartet_kernel(const int* __restrict__ qp, long long n,
                                                      const PairMeta* __restrict__ pm,
                                                      const PrimRec* __restrict__ prims,
                                                      double* __restrict__ out,
                                                      const double* __restrict__ boys_tab) {
  extern __shared__ double s_boys[];
  const double* gt = boys_tab + static_cast<size_t>(C::M) * kBoysRows * kBoysCols;
  for (int t = threadIdx.x; t < kBoysRows * kBoysCols; t += blockDim.x) s_boys[t] = gt[t];
  __syncthreads();
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const PairMeta b = pm[qp[2 * i]], k = pm[qp[2 * i + 1]];
  double v[C::NV];
  C::eri(prims + b.prim_off, b.K, prims + k.prim_off, k.K, b.ABx, b.ABy, b.ABz, k.ABx, k.ABy, k.ABz,
         s_boys, v);
#pragma unroll
  for (int t = 0; t < C::NV; ++t) out[i * C::NV + t] = v[t];
}

template <class C>
void launch_class(const LaunchArgs& a) {
  const size_t smem = sizeof(double) * kBoysRows * kBoysCols;
  const int block = a.block > 0 ? a.block : 128;
  if (a.mode == 0) {
    if (a.nitems <= 0) return;
    cudaFuncSetAttribute(jk_kernel<C>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    long long want = (a.nitems + (block / 32) - 1) / (block / 32);
    int grid = a.grid > 0 ? a.grid : static_cast<int>(want < 148LL * 16 ? want : 148LL * 16);
    jk_kernel<C><<<grid, block, smem, a.stream>>>(a.items, a.nitems, a.pm, a.prims, a.D, a.J, a.K,
                                                  a.N, a.boys_tab);
  } else if (a.mode == 2) {
    if (a.nq <= 0) return;
    cudaFuncSetAttribute(quartet_kernel<C>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    const int grid = static_cast<int>((a.nq + block - 1) / block);
    quartet_kernel<C><<<grid, block, smem, a.stream>>>(a.qpairs, a.nq, a.pm, a.prims, a.qout, a.boys_tab);
  } else {
    if (a.npair_list <= 0) return;
    cudaFuncSetAttribute(schwarz_kernel<C>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    long long want = (a.npair_list + block - 1) / block;
    int grid = static_cast<int>(want < 148LL * 16 ? want : 148LL * 16);
    schwarz_kernel<C><<<grid, block, smem, a.stream>>>(a.pair_list, a.npair_list, a.pm, a.prims,
                                                       a.Qout, a.boys_tab);
  }
}

}  // namespace eritile_b200
