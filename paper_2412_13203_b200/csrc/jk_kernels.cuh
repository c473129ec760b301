// Fused Schwarz-screened ERI + J/K digestion kernels (sm_100a, FP64).
//
// Work mapping: the surviving quartets of one
// (bra group X, ket group Y) pair are the concatenation, over bras x in X,
// of a prefix of Y (Y is sorted by Schwarz Q, so survivors of x are the
// first cnt[x] kets). A warp takes 32 consecutive quartets of that flat
// sequence (WorkItem = first bra, offset, counts pointer): lanes are kets,
// runs of lanes share a bra, every lane has the same primitive trip counts
// (groups are contraction-homogeneous — Permutation). Each
// lane evaluates its contracted quartet with the class's generated
// straight-line plan (Cls*::eri), then digests it: J_ab is reduced over the
// lanes sharing the bra (segmented warp scan) and flushed once per segment;
// J_cd and the four K blocks are FP64 atomics (RED.ADD.F64). Digestion
// follows the shell-level degeneracy rule of SPEC.md:350 with J weight
// deg/2 and K weight deg/4, so true J = sym(Jacc) and K = sym(Kacc) after
// the finalize kernel.
#pragma once
#include <cuda_runtime.h>

#include "jk_api.h"

namespace eritile_b200 {


// Primitive-pair record loads (read-only path). WithPA = false skips the
// PA/QC half for plans that never read it on that side.
template <bool WithPA = true>
__device__ __forceinline__ PrimRec load_prim(const PrimRec* p) {
  const double2* q = reinterpret_cast<const double2*>(p);
  const double2 a = __ldg(q), b = __ldg(q + 1), c = __ldg(q + 2);
  PrimRec r;
  r.p = a.x; r.U = a.y; r.Px = b.x; r.Py = b.y; r.Pz = c.x; r.i2p = c.y;
  if (WithPA) {
    const double2 d = __ldg(q + 3), e = __ldg(q + 4);
    r.PAx = d.x; r.PAy = d.y; r.PAz = e.x;
  } else {
    r.PAx = r.PAy = r.PAz = 0.0;
  }
  r.pad = 0.0;
  return r;
}

// 1/sqrt(x) for positive normal x: MUFU seed (rsqrt.approx.f64) and one
// third-order Newton step y' = y + y e (1/2 + 3/8 e), e = 1 - x y^2
// (seed error ~2^-23 -> < 1 ulp); no special-case branch (inputs are
// exponent sums and T > 0 here).
__device__ __forceinline__ double rsqrt_pos(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double e = fma(-x, y * y, 1.0);
  return fma(fma(e, 0.375, 0.5), y * e, y);
}

// Boys function F_0..F_M(T) (boys.hpp:23-44 semantics, table-driven).
// T < 40: 8-term Taylor expansion of F_M about the nearest grid point
// T_i = i/16 (|d| <= 1/32, truncation < 3e-17 relative) from a table of
// F_{M+k}(T_i)/k! computed in extended precision when the context is
// created, then the stable downward recursion F_{m-1} = (2T F_m + e^-T)/(2m-1)
// (boys.hpp:40-41). T >= 40: F_0 = sqrt(pi/T)/2 (erf(sqrt T) = 1 - O(1e-19))
// and the upward recursion F_{m+1} = ((2m+1) F_m - e^-T)/(2T) (boys.hpp:43),
// contractive for 2m+1 < 2T. e^-T = e^-T_i e^-d uses the table's exp column
// (for 40 <= T < 80 shifted by e^-40; 0 above 80, < 2e-35), so both branches
// share one short polynomial. Rows are kBoysCols = 10 doubles, 16-byte
// aligned, read as double2.
template <int M>
__device__ __forceinline__ void boys_eval(double T, const double* __restrict__ tab, double* F) {
  const bool small = T < kBoysTmax;
  double e = 0.0;
  const double* row;
  double md;
  {
    const double Tt = small ? T : (T < 2.0 * kBoysTmax ? T - kBoysTmax : 0.0);
    const int i = __double2int_rn(Tt * 16.0);
    md = fma(static_cast<double>(i), 0.0625, -Tt);  // -(Tt - T_i)
    row = tab + i * kBoysCols;
    if (M > 0) {
      // exp(-d) = sum_k (-d)^k / k!, k <= 8 (|d| <= 1/32)
      e = 2.48015873015873016e-05;
      e = fma(e, md, 1.98412698412698413e-04);
      e = fma(e, md, 1.38888888888888889e-03);
      e = fma(e, md, 8.33333333333333333e-03);
      e = fma(e, md, 4.16666666666666667e-02);
      e = fma(e, md, 1.66666666666666667e-01);
      e = fma(e, md, 0.5);
      e = fma(e, md, 1.0);
      e = fma(e, md, 1.0);
      const double scale = small ? 1.0 : (T < 2.0 * kBoysTmax ? 4.24835425529158899e-18 : 0.0);  // e^-40
      e *= row[8] * scale;
    }
  }
  if (small) {
    const double2* r = reinterpret_cast<const double2*>(row);
    const double2 c01 = r[0], c23 = r[1], c45 = r[2], c67 = r[3];
    double f = fma(c67.y, md, c67.x);
    f = fma(f, md, c45.y);
    f = fma(f, md, c45.x);
    f = fma(f, md, c23.y);
    f = fma(f, md, c23.x);
    f = fma(f, md, c01.y);
    f = fma(f, md, c01.x);
    F[M] = f;
    const double T2 = 2.0 * T;
#pragma unroll
    for (int m = M; m > 0; --m) F[m - 1] = fma(T2, F[m], e) * (1.0 / (2 * m - 1));
  } else {
    const double rt = rsqrt_pos(T);
    F[0] = 0.88622692545275801365 * rt;  // sqrt(pi)/2
    if (M > 0) {
      const double h = 0.5 * rt * rt;  // 1/(2T)
#pragma unroll
      for (int m = 0; m < M; ++m) F[m + 1] = fma(static_cast<double>(2 * m + 1), F[m], -e) * h;
    }
  }
}

// Component normalisation (molecule.hpp:207-213) for L <= 4, x-major order.
__device__ __forceinline__ double comp_scale(int L, int i) {
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

// Inclusive segmented sum over lanes with equal non-decreasing key; lanes
// whose key differs from lane+1 (segment tails) end holding the segment sum.
__device__ __forceinline__ double seg_sum(double v, int key, int lane) {
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const double u = __shfl_up_sync(0xffffffffu, v, o);
    const int k = __shfl_up_sync(0xffffffffu, key, o);
    if (lane >= o && k == key) v += u;
  }
  return v;
}

__device__ __forceinline__ void load_boys_slice(double* s_boys, const double* boys_tab, int M) {
  const double2* gt = reinterpret_cast<const double2*>(boys_tab + static_cast<size_t>(M) * kBoysRows * kBoysCols);
  double2* st = reinterpret_cast<double2*>(s_boys);
  for (int t = threadIdx.x; t < kBoysRows * kBoysCols / 2; t += blockDim.x) st[t] = gt[t];
  __syncthreads();
}

constexpr int kJkThreads = 256;

// U = 1: C::eri (one primitive quartet per step); U = 2: C::eri2 (two ket
// primitives per step sharing the bra record, two independent FMA chains).
template <class C, int MINB, int U = 1, int NT = kJkThreads>
__global__ void __launch_bounds__(NT, MINB) jk_kernel(const WorkItem* __restrict__ items, long long nitems,
                                                       const int* __restrict__ cnt,
                                                       const PairMeta* __restrict__ pm,
                                                       const PrimRec* __restrict__ prims,
                                                       const double* __restrict__ D, double* __restrict__ J,
                                                       double* __restrict__ K, int N,
                                                       const double* __restrict__ boys_tab) {
  extern __shared__ __align__(16) double s_boys[];
  load_boys_slice(s_boys, boys_tab, C::M);

  const int lane = threadIdx.x & 31;
  const long long warps = static_cast<long long>(gridDim.x) * (blockDim.x >> 5);
  for (long long w = static_cast<long long>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5);
       w < nitems; w += warps) {
    const WorkItem it = items[w];
    const int nq = it.r0nq >> 24;
    const bool active = lane < nq;
    // walk the per-bra survivor counts to this lane's (bra, ket)
    int q = (it.r0nq & 0xffffff) + (active ? lane : 0);
    int x = it.bra0, c = it.cntp;
    for (int n = __ldg(cnt + c); q >= n; n = __ldg(cnt + c)) {
      q -= n;
      ++x;
      ++c;
    }
    const int y = it.yfirst + q;
    const PairMeta bm = pm[x];
    const PairMeta km = pm[y];
    double v[C::NV];
    if constexpr (U == 2)
      C::eri2(prims + bm.prim_off, bm.K, prims + km.prim_off, active ? km.K : 0, bm.ABx, bm.ABy, bm.ABz,
              km.ABx, km.ABy, km.ABz, s_boys, v);
    else
      C::eri(prims + bm.prim_off, bm.K, prims + km.prim_off, active ? km.K : 0, bm.ABx, bm.ABy, bm.ABz,
             km.ABx, km.ABy, km.ABz, s_boys, v);
    const double deg = (bm.sha != bm.shb ? 2.0 : 1.0) * (km.sha != km.shb ? 2.0 : 1.0) * (x != y ? 2.0 : 1.0);
    const double wj = active ? 0.5 * deg : 0.0;
    const double wk = active ? 0.25 * deg : 0.0;
    const size_t n = static_cast<size_t>(N);
    const double* Dab = D + bm.bfa * n + bm.bfb;
    const double* Dcd = D + km.bfa * n + km.bfb;
    const double* Dac = D + bm.bfa * n + km.bfa;
    const double* Dad = D + bm.bfa * n + km.bfb;
    const double* Dbc = D + bm.bfb * n + km.bfa;
    const double* Dbd = D + bm.bfb * n + km.bfb;
    // J_ab: lanes sharing the bra form a segment -> one flush per segment
    const int xkey = active ? x : -1;
    const int xnext = __shfl_down_sync(0xffffffffu, xkey, 1);
    const bool tail = active && (lane == 31 || xnext != xkey);
#pragma unroll
    for (int a = 0; a < C::NA; ++a)
#pragma unroll
      for (int b = 0; b < C::NB; ++b) {
        double s = 0.0;
#pragma unroll
        for (int c2 = 0; c2 < C::NC; ++c2)
#pragma unroll
          for (int d = 0; d < C::ND; ++d)
            s = fma(v[((a * C::NB + b) * C::NC + c2) * C::ND + d], __ldg(Dcd + c2 * n + d), s);
        s = seg_sum(s * wj, xkey, lane);
        if (tail) atomicAdd(J + (bm.bfa + a) * n + bm.bfb + b, s);
      }
    if (active) {
#pragma unroll
      for (int c2 = 0; c2 < C::NC; ++c2)
#pragma unroll
        for (int d = 0; d < C::ND; ++d) {
          double s = 0.0;
#pragma unroll
          for (int a = 0; a < C::NA; ++a)
#pragma unroll
            for (int b = 0; b < C::NB; ++b)
              s = fma(v[((a * C::NB + b) * C::NC + c2) * C::ND + d], __ldg(Dab + a * n + b), s);
          atomicAdd(J + (km.bfa + c2) * n + km.bfb + d, s * wj);
        }
      // K_ac += sum_bd v D_bd ; K_bd += sum_ac v D_ac
#pragma unroll
      for (int a = 0; a < C::NA; ++a)
#pragma unroll
        for (int c2 = 0; c2 < C::NC; ++c2) {
          double s = 0.0;
#pragma unroll
          for (int b = 0; b < C::NB; ++b)
#pragma unroll
            for (int d = 0; d < C::ND; ++d)
              s = fma(v[((a * C::NB + b) * C::NC + c2) * C::ND + d], __ldg(Dbd + b * n + d), s);
          atomicAdd(K + (bm.bfa + a) * n + km.bfa + c2, s * wk);
        }
#pragma unroll
      for (int b = 0; b < C::NB; ++b)
#pragma unroll
        for (int d = 0; d < C::ND; ++d) {
          double s = 0.0;
#pragma unroll
          for (int a = 0; a < C::NA; ++a)
#pragma unroll
            for (int c2 = 0; c2 < C::NC; ++c2)
              s = fma(v[((a * C::NB + b) * C::NC + c2) * C::ND + d], __ldg(Dac + a * n + c2), s);
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
            for (int c2 = 0; c2 < C::NC; ++c2)
              s = fma(v[((a * C::NB + b) * C::NC + c2) * C::ND + d], __ldg(Dbc + b * n + c2), s);
          atomicAdd(K + (bm.bfa + a) * n + km.bfb + d, s * wk);
        }
#pragma unroll
      for (int b = 0; b < C::NB; ++b)
#pragma unroll
        for (int c2 = 0; c2 < C::NC; ++c2) {
          double s = 0.0;
#pragma unroll
          for (int a = 0; a < C::NA; ++a)
#pragma unroll
            for (int d = 0; d < C::ND; ++d)
              s = fma(v[((a * C::NB + b) * C::NC + c2) * C::ND + d], __ldg(Dad + a * n + d), s);
          atomicAdd(K + (bm.bfb + b) * n + km.bfa + c2, s * wk);
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
  extern __shared__ __align__(16) double s_boys[];
  load_boys_slice(s_boys, boys_tab, C::M);
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
  extern __shared__ __align__(16) double s_boys[];
  load_boys_slice(s_boys, boys_tab, C::M);
  const long long i = static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const PairMeta b = pm[qp[2 * i]], k = pm[qp[2 * i + 1]];
  double v[C::NV];
  C::eri(prims + b.prim_off, b.K, prims + k.prim_off, k.K, b.ABx, b.ABy, b.ABz, k.ABx, k.ABy, k.ABz,
         s_boys, v);
#pragma unroll
  for (int t = 0; t < C::NV; ++t) out[i * C::NV + t] = v[t];
}

// Lane kernels: MINB is the __launch_bounds__ residency target (2 -> up to
// 128 registers, 3 -> 80); the Workload Allocator picks per class.
// NT: threads per CTA. One Boys slice is staged per CTA, so 512/768-thread
// CTAs at MINB = 1 keep 16/24 warps per SM with a single 51 KB table and
// leave the rest of the 256 KB L1/shared array to L1 (primitive records).
template <class C, int MINB, int U = 1, int NT = kJkThreads>
void launch_class(const LaunchArgs& a) {
  const size_t smem = sizeof(double) * kBoysRows * kBoysCols;
  if (a.mode == 0) {
    if (a.nitems <= 0) return;
    static int blocks_per_sm = 0;
    static int sms = 0;
    if (!blocks_per_sm) {
      cudaFuncSetAttribute(jk_kernel<C, MINB, U, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks_per_sm, jk_kernel<C, MINB, U, NT>, NT, smem);
      int dev = 0;
      cudaGetDevice(&dev);
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
      if (blocks_per_sm < 1) blocks_per_sm = 1;
    }
    const long long want = (a.nitems + (NT / 32) - 1) / (NT / 32);
    const long long cap = static_cast<long long>(blocks_per_sm) * sms;
    const int grid = a.grid > 0 ? a.grid : static_cast<int>(want < cap ? want : cap);
    jk_kernel<C, MINB, U, NT><<<grid, NT, smem, a.stream>>>(a.items, a.nitems, a.cnt, a.pm, a.prims, a.D, a.J,
                                                       a.K, a.N, a.boys_tab);
  } else if (a.mode == 2) {
    if (a.nq <= 0) return;
    cudaFuncSetAttribute(quartet_kernel<C>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    const int grid = static_cast<int>((a.nq + 127) / 128);
    quartet_kernel<C><<<grid, 128, smem, a.stream>>>(a.qpairs, a.nq, a.pm, a.prims, a.qout, a.boys_tab);
  } else {
    if (a.npair_list <= 0) return;
    cudaFuncSetAttribute(schwarz_kernel<C>, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem));
    long long want = (a.npair_list + 127) / 128;
    int grid = static_cast<int>(want < 148LL * 16 ? want : 148LL * 16);
    schwarz_kernel<C><<<grid, 128, smem, a.stream>>>(a.pair_list, a.npair_list, a.pm, a.prims, a.Qout,
                                                     a.boys_tab);
  }
}

}  // namespace eritile_b200
