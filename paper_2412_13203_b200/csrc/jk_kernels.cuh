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

#include <map>
#include <mutex>
#include <tuple>

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
// Non-immediate FP64 constants of boys_eval live in the constant bank so
// DFMA/DMUL read them as c[][] operands instead of re-materialising them
// with register moves inside the primitive loop.
static __constant__ double kBoysK[10] = {
    1.66666666666666667e-01, 4.16666666666666667e-02, 8.33333333333333333e-03,
    1.38888888888888889e-03, 1.98412698412698413e-04, 2.48015873015873016e-05,
    6755399441055744.0 /* 1.5 * 2^52 */, 4.24835425529158899e-18 /* e^-40 */,
    0.88622692545275801365 /* sqrt(pi)/2 */, 0.0};

template <int M>
__device__ __forceinline__ void boys_eval_mixed(double T, const double* __restrict__ tab, double* F) {
  const bool small = T < kBoysTmax;
  double e = 0.0;
  const double* row;
  double md;
  {
    // T_i = round(16 Tt)/16 by the 1.5*2^52 shift (no F2I/I2F round trip):
    // the low word of the shifted value is the row index
    double Tt;
    if constexpr (M == 0)
      Tt = small ? T : 0.0;  // no e^-T needed above the table
    else
      Tt = small ? T : (T < 2.0 * kBoysTmax ? T - kBoysTmax : 0.0);
    const double sh = fma(Tt, 16.0, kBoysK[6]);
    const int i = __double2loint(sh);
    md = fma(sh - kBoysK[6], 0.0625, -Tt);  // -(Tt - T_i)
    row = tab + i * kBoysCols;
    if (M > 0) {
      // exp(-d) = sum_k (-d)^k / k!, k <= 8 (|d| <= 1/32), Estrin form
      // (dependency depth 4 instead of 8: the loop is latency-bound)
      const double m2 = md * md, m4 = m2 * m2;
      const double e01 = md + 1.0, e23 = fma(md, kBoysK[0], 0.5);
      const double e45 = fma(md, kBoysK[2], kBoysK[1]);
      const double e67 = fma(md, kBoysK[4], kBoysK[3]);
      const double e0123 = fma(m2, e23, e01), e4567 = fma(m2, e67, e45);
      e = fma(m4, fma(m4, kBoysK[5], e4567), e0123);
      const double scale = small ? 1.0 : (T < 2.0 * kBoysTmax ? kBoysK[7] : 0.0);  // e^-40
      e *= row[8] * scale;
    }
  }
  if (small) {
    const double2* r = reinterpret_cast<const double2*>(row);
    const double2 c01 = r[0], c23 = r[1], c45 = r[2], c67 = r[3];
    // Estrin: depth 3 FMAs after the loads instead of a 7-deep Horner chain
    const double m2 = md * md;
    const double p01 = fma(c01.y, md, c01.x), p23 = fma(c23.y, md, c23.x);
    const double p45 = fma(c45.y, md, c45.x), p67 = fma(c67.y, md, c67.x);
    const double q0 = fma(p23, m2, p01), q1 = fma(p67, m2, p45);
    F[M] = fma(q1, m2 * m2, q0);
    const double T2 = 2.0 * T;
#pragma unroll
    for (int m = M; m > 0; --m) F[m - 1] = fma(T2, F[m], e) * (1.0 / (2 * m - 1));
  } else {
    const double rt = rsqrt_pos(T);
    F[0] = kBoysK[8] * rt;  // sqrt(pi)/2
    if (M > 0) {
      const double h = 0.5 * rt * rt;  // 1/(2T)
#pragma unroll
      for (int m = 0; m < M; ++m) F[m + 1] = fma(static_cast<double>(2 * m + 1), F[m], -e) * h;
    }
  }
}

// Boys F_0..F_M(T) on every lane in one straight-line (if-converted) form.
// A warp-uniform dispatch (vote, then only the table or only the asymptotic
// branch) was measured slower: 450 vs 433 ms per (H2O)_80 build — lanes of
// a warp are kets at different distances, so warps mix both sides of T = 40
// and pay both branches plus the vote/reconvergence, and the branches split
// the primitive loop into basic blocks the scheduler cannot interleave.
template <int M>
__device__ __forceinline__ void boys_eval(double T, const double* __restrict__ tab, double* F) {
  boys_eval_mixed<M>(T, tab, F);
}

// F_0, F_1 for M = 1 classes from the slices 0 and 1 staged back to back
// (tab0 = slice 0): T < 40 each order by its own 8-term Taylor series about
// T_i (no exp(-T) polynomial, no recursion); T >= 40 F_0 = sqrt(pi/T)/2 and
// F_1 = F_0 / (2T), where the dropped e^-T / (2T) is < 3e-17 of F_1.
__device__ __forceinline__ void boys_eval_m1(double T, const double* __restrict__ tab0, double* F) {
  if (T < kBoysTmax) {
    const double sh = fma(T, 16.0, kBoysK[6]);
    const int i = __double2loint(sh);
    const double md = fma(sh - kBoysK[6], 0.0625, -T);
    const double m2 = md * md, m4 = m2 * m2;
    const double2* r0 = reinterpret_cast<const double2*>(tab0 + i * kBoysCols);
    const double2* r1 = reinterpret_cast<const double2*>(tab0 + (kBoysRows + i) * kBoysCols);
    {
      const double2 c01 = r0[0], c23 = r0[1], c45 = r0[2], c67 = r0[3];
      const double q0 = fma(fma(c23.y, md, c23.x), m2, fma(c01.y, md, c01.x));
      const double q1 = fma(fma(c67.y, md, c67.x), m2, fma(c45.y, md, c45.x));
      F[0] = fma(q1, m4, q0);
    }
    {
      const double2 c01 = r1[0], c23 = r1[1], c45 = r1[2], c67 = r1[3];
      const double q0 = fma(fma(c23.y, md, c23.x), m2, fma(c01.y, md, c01.x));
      const double q1 = fma(fma(c67.y, md, c67.x), m2, fma(c45.y, md, c45.x));
      F[1] = fma(q1, m4, q0);
    }
  } else {
    const double rt = rsqrt_pos(T);
    F[0] = kBoysK[8] * rt;
    F[1] = F[0] * (0.5 * rt * rt);
  }
}

// Primitive loop nests over the class's prim()/finish() (compiler/
// emit_cuda.py). Every style evaluates the same terms in the same order per
// accumulator; they differ in how bra records are staged in registers:
//  kLoopPlain     load each record where it is used (compiler schedules);
//  kLoopPrefetch  next bra record loaded one step ahead (register rotation);
//  kLoopSmemBra   plain loop; when all lanes of the warp share the bra, its
//                 primitive records are staged once in shared memory (per
//                 warp, reused while consecutive items keep the bra).
//  kLoopSmemBraPf as kLoopSmemBra, and the ket record of step j+1 is loaded
//                 during step j (hides the L2 trip of the ket gather).
//  kLoopSmemBra2K as kLoopSmemBra with two ket primitives per step sharing
//                 each bra record read (two independent chains per lane).
//  kLoopSmemBraL1 as kLoopSmemBra, and step j issues an L1 prefetch of the
//                 ket record of step j+1 (no registers held; ncu showed the
//                 first use of each ket record as the top long-scoreboard stall).
constexpr int kLoopPlain = 0, kLoopPrefetch = 1, kLoopSmemBra = 4, kLoopSmemBraPf = 8,
              kLoopSmemBra2K = 16, kLoopSmemBraL1 = 32;

__device__ __forceinline__ void prefetch_l1(const void* p) {
  asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
}
constexpr int kSmemBraMax = 81;  // records per warp buffer (cc-pVDZ s9 x s9)

// Generic-address record load (the pointer may be shared or global).
template <bool WithPA = true>
__device__ __forceinline__ PrimRec load_prim_gen(const PrimRec* p) {
  const double2* q = reinterpret_cast<const double2*>(p);
  const double2 a = q[0], b = q[1], c = q[2];
  PrimRec r;
  r.p = a.x; r.U = a.y; r.Px = b.x; r.Py = b.y; r.Pz = c.x; r.i2p = c.y;
  if (WithPA) {
    const double2 d = q[3], e = q[4];
    r.PAx = d.x; r.PAy = d.y; r.PAz = e.x;
  } else {
    r.PAx = r.PAy = r.PAz = 0.0;
  }
  r.pad = 0.0;
  return r;
}

template <class C, int STYLE>
__device__ __forceinline__ void eri_drive(const PrimRec* __restrict__ bra, int kb,
                                          const PrimRec* __restrict__ ket, int kk, int ks, double ABx, double ABy,
                                          double ABz, double CDx, double CDy, double CDz,
                                          const double* __restrict__ btab, double (&out)[C::NV]) {
  typename C::Acc a;
  if constexpr (STYLE == kLoopPlain && C::K1) {
    // one primitive quartet (d/f shells of cc-pVXZ are single primitives):
    // assign the boundary values instead of zeroing and accumulating them
    if (kk == 1 && kb == 1) {
      C::prim_set(load_prim<C::BPA>(bra), load_prim<C::KPA>(ket), btab, a);
      C::finish(a, ABx, ABy, ABz, CDx, CDy, CDz, out);
      return;
    }
  }
  C::zero(a);
  if constexpr (STYLE == kLoopPlain) {
    for (int j = 0; j < kk; ++j) {
      const PrimRec kp = load_prim<C::KPA>(ket + j * ks);
      for (int i = 0; i < kb; ++i) C::prim(load_prim<C::BPA>(bra + i), kp, btab, a);
    }
  } else if constexpr (STYLE == kLoopSmemBra || STYLE == kLoopSmemBraL1) {
    for (int j = 0; j < kk; ++j) {
      if constexpr (STYLE == kLoopSmemBraL1)
        if (j + 1 < kk) prefetch_l1(ket + (j + 1) * ks);
      const PrimRec kp = load_prim<C::KPA>(ket + j * ks);
      for (int i = 0; i < kb; ++i) C::prim(load_prim_gen<C::BPA>(bra + i), kp, btab, a);
    }
  } else if constexpr (STYLE == kLoopSmemBra2K) {
    typename C::Acc b;
    C::zero(b);
    int j = 0;
    for (; j + 1 < kk; j += 2) {
      const PrimRec k0 = load_prim<C::KPA>(ket + j * ks);
      const PrimRec k1 = load_prim<C::KPA>(ket + (j + 1) * ks);
      for (int i = 0; i < kb; ++i) {
        const PrimRec bq = load_prim_gen<C::BPA>(bra + i);
        C::prim(bq, k0, btab, a);
        C::prim(bq, k1, btab, b);
      }
    }
    if (j < kk) {
      const PrimRec kp = load_prim<C::KPA>(ket + j * ks);
      for (int i = 0; i < kb; ++i) C::prim(load_prim_gen<C::BPA>(bra + i), kp, btab, a);
    }
    C::fold(a, b);
  } else if constexpr (STYLE == kLoopSmemBraPf) {
    PrimRec kn = load_prim<C::KPA>(ket);
    for (int j = 0; j < kk; ++j) {
      const PrimRec kp = kn;
      if (j + 1 < kk) kn = load_prim<C::KPA>(ket + (j + 1) * ks);
      for (int i = 0; i < kb; ++i) C::prim(load_prim_gen<C::BPA>(bra + i), kp, btab, a);
    }
  } else if constexpr (STYLE == kLoopPrefetch) {
    for (int j = 0; j < kk; ++j) {
      const PrimRec kp = load_prim<C::KPA>(ket + j * ks);
      PrimRec bn = load_prim<C::BPA>(bra);
      for (int i = 0; i < kb; ++i) {
        const PrimRec bq = bn;
        bn = load_prim<C::BPA>(bra + (i + 1 < kb ? i + 1 : i));
        C::prim(bq, kp, btab, a);
      }
    }
  }
  C::finish(a, ABx, ABy, ABz, CDx, CDy, CDz, out);
}

// Two kets per lane in one loop nest (strip kernels, kStripDual): both kets
// have the same primitive count kk (same ket group); every bra record read
// from shared memory feeds two independent primitive chains.
template <class C>
__device__ __forceinline__ void eri_drive_dual(const PrimRec* bra, int kb, const PrimRec* __restrict__ ket1,
                                               const PrimRec* __restrict__ ket2, int kk, int ks, double ABx,
                                               double ABy, double ABz, double CDx1, double CDy1, double CDz1,
                                               double CDx2, double CDy2, double CDz2,
                                               const double* __restrict__ btab, double (&out1)[C::NV],
                                               double (&out2)[C::NV]) {
  typename C::Acc a1, a2;
  C::zero(a1);
  C::zero(a2);
  for (int j = 0; j < kk; ++j) {
    const PrimRec k1 = load_prim<C::KPA>(ket1 + j * ks);
    const PrimRec k2 = load_prim<C::KPA>(ket2 + j * ks);
    for (int i = 0; i < kb; ++i) {
      const PrimRec bq = load_prim_gen<C::BPA>(bra + i);
      C::prim(bq, k1, btab, a1);
      C::prim(bq, k2, btab, a2);
    }
  }
  C::finish(a1, ABx, ABy, ABz, CDx1, CDy1, CDz1, out1);
  C::finish(a2, ABx, ABy, ABz, CDx2, CDy2, CDz2, out2);
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

// Pair metadata re-read after the primitive loop (ints only: first basis
// functions and shells). asm volatile keeps the load where it is written.
__device__ __forceinline__ void ld_meta_late(const PairMeta* p, PairMeta& m) {
  int a, b, c, d, e, f, g, h;
  asm volatile("ld.global.nc.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(a), "=r"(b), "=r"(c), "=r"(d) : "l"(p));
  asm volatile("ld.global.nc.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(e), "=r"(f), "=r"(g), "=r"(h) : "l"(reinterpret_cast<const char*>(p) + 16));
  m.prim_off = a; m.K = b; m.bfa = c; m.bfb = d; m.sha = e; m.shb = f; m.ref = g; m.kstride = h;
}

// FP64 reduction into J/K. ERITILE_PROBE_NODIGEST (a measurement-only build,
// never the product) keeps the digestion arithmetic but drops the atomics.
__device__ __forceinline__ void red_add(double* p, double v, int det) {
#ifdef ERITILE_PROBE_NODIGEST
  if (v == 1.2345e-300) atomicAdd(p, v);
#else
  if (det)  // fixed point, exact integer sums: order-independent (kDetScale)
    atomicAdd(reinterpret_cast<unsigned long long*>(p),
              static_cast<unsigned long long>(__double2ll_rn(v * kDetScale)));
  else
    atomicAdd(p, v);
#endif
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

// Shared-memory Boys staging of a lane class: M = 1 classes stage slices 0
// and 1 and evaluate both orders by their own Taylor series (boys_eval_m1);
// every other class stages slice M.
template <class C>
struct BoysStage {
  static constexpr bool two = C::M == 1 && C::BOYS_M1_TWO;
  static constexpr int base = two ? 0 : C::M;
  static constexpr int nsl = two ? 2 : 1;
  static constexpr size_t bytes = sizeof(double) * kBoysRows * kBoysCols * nsl;
};

template <class C>
__device__ __forceinline__ void load_boys_for(double* s_boys, const double* boys_tab) {
  const double2* gt =
      reinterpret_cast<const double2*>(boys_tab + static_cast<size_t>(BoysStage<C>::base) * kBoysRows * kBoysCols);
  double2* st = reinterpret_cast<double2*>(s_boys);
  for (int t = threadIdx.x; t < BoysStage<C>::nsl * kBoysRows * kBoysCols / 2; t += blockDim.x) st[t] = gt[t];
  __syncthreads();
}

__device__ __forceinline__ void load_boys_slice(double* s_boys, const double* boys_tab, int M) {
  const double2* gt = reinterpret_cast<const double2*>(boys_tab + static_cast<size_t>(M) * kBoysRows * kBoysCols);
  double2* st = reinterpret_cast<double2*>(s_boys);
  for (int t = threadIdx.x; t < kBoysRows * kBoysCols / 2; t += blockDim.x) st[t] = gt[t];
  __syncthreads();
}

constexpr int kJkThreads = 256;

// Work items [i0, i1) in warp tasks of `gran` consecutive items (the
// Workload Allocator's Combine granularity), tasks dealt
// round-robin over the grid's warps; f(item) per item in order. The next
// item's descriptor is fetched one item ahead (hides its L2 trip).
template <class F>
__device__ __forceinline__ void for_warp_items(const WorkItem* __restrict__ items, long long i0, long long i1,
                                               int gran, long long wid, long long warps, F&& f) {
  const long long g = gran > 1 ? gran : 1;
  const long long ntask = (i1 - i0 + g - 1) / g;
  long long t = wid, w = i0 + t * g, e = w + g < i1 ? w + g : i1;
  WorkItem nxt = t < ntask ? items[w] : WorkItem{};
  while (t < ntask) {
    const WorkItem it = nxt;
    if (++w >= e) {
      t += warps;
      w = i0 + t * g;
      e = w + g < i1 ? w + g : i1;
    }
    if (t < ntask) nxt = items[w];
    f(it);
  }
}

// Shared-memory carveout just large enough for the resident CTAs, so the
// rest of the SM's 256 KB L1/shared array caches primitive records.
inline cudaError_t set_min_carveout(const void* fn, int blocks_per_sm, size_t smem) {
  const size_t need = static_cast<size_t>(blocks_per_sm) * (smem + 1024);
  int pct = static_cast<int>((need * 100 + 228 * 1024 - 1) / (228 * 1024));
  pct = pct < 1 ? 1 : (pct > 100 ? 100 : pct);
  return cudaFuncSetAttribute(fn, cudaFuncAttributePreferredSharedMemoryCarveout, pct);
}

// Per-(kernel, device) launch setup, done once per device: the dynamic
// shared-memory opt-in (> 48 KB for the Boys slice), the residency query and
// optionally the minimal carveout. Function attributes are per device, so a
// second device in the same process gets its own setup. On a CUDA error the
// result is {0, 0}, nothing is cached and the error stays pending for the
// caller's cudaGetLastError() check.
struct LaunchSetup {
  int bps;  // resident CTAs per SM
  int sms;
};
inline LaunchSetup launch_setup(const void* fn, int nt, size_t smem, bool min_carveout) {
  static std::mutex mu;
  static std::map<std::tuple<const void*, int, size_t>, LaunchSetup> cache;
  // the dynamic shared-memory opt-in is one attribute per (kernel, device):
  // it only ever grows, so a launch with a smaller size after a larger one
  // (another molecule, another class column count) never lowers it below a
  // size whose setup is already cached
  static std::map<std::pair<const void*, int>, size_t> attr;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return {0, 0};
  std::lock_guard<std::mutex> lk(mu);
  const auto key = std::make_tuple(fn, dev, smem);
  const auto it = cache.find(key);
  if (it != cache.end()) return it->second;
  LaunchSetup s{0, 0};
  size_t& cur = attr[std::make_pair(fn, dev)];
  if (smem > cur) {
    if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(smem)) != cudaSuccess)
      return {0, 0};
    cur = smem;
  }
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&s.bps, fn, nt, smem) != cudaSuccess ||
      cudaDeviceGetAttribute(&s.sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess)
    return {0, 0};
  if (s.bps < 1) s.bps = 1;
  if (min_carveout && set_min_carveout(fn, s.bps, cur) != cudaSuccess) return {0, 0};
  cache.emplace(key, s);
  return s;
}

// Sum x over the lanes of `peers` (lanes with equal key, this lane included);
// the lowest lane of the group ends with the total. All 32 lanes must call.
template <int NV>
__device__ __forceinline__ void reduce_peers(unsigned peers, double (&x)[NV], int lane) {
  int rel = __popc(peers & ((1u << lane) - 1u));  // rank within the group
  unsigned rest = peers & (0xfffffffeu << lane);  // group members above this lane
  while (__any_sync(0xffffffffu, rest != 0u)) {
    const int next = __ffs(rest);  // next remaining member (1-based), 0 if none
#pragma unroll
    for (int e = 0; e < NV; ++e) {
      const double t = __shfl_sync(0xffffffffu, x[e], next ? next - 1 : lane);
      if (next) x[e] += t;
    }
    rest &= ~__ballot_sync(0xffffffffu, rel & 1);
    rel >>= 1;
  }
}

// STYLE bit kLoopAggK (lane kernels): the four K blocks of a quartet are
// reduced over the lanes of the warp that hit the same block (same bra shell
// row, same ket shell column: __match_any_sync on the block origin), and only
// the group leader issues the RED.ADD.F64s. Global FP64 atomics bound the
// mid-L lane classes (measurement probe: (ds|ps) 37 -> 23 ms without them).
// Deterministic mode keeps the per-lane REDs (fixed-point rounding per
// contribution, identical across variants).
constexpr int kLoopAggK = 64;
// STYLE bit kLoopSplit (lane kernels): Deconstruction of each contracted
// quartet's primitive quartets over a lane pair (see the process lambda).
constexpr int kLoopSplit = 128;

template <class C, int MINB, int STYLE = kLoopPrefetch, int NT = kJkThreads>
__global__ void __launch_bounds__(NT, MINB) jk_kernel(const WorkItem* __restrict__ items, long long nitems,
                                                       const int* __restrict__ cnt,
                                                       const PairMeta* __restrict__ pm,
                                                       const PrimRec* __restrict__ prims,
                                                       const double* __restrict__ D, double* __restrict__ J,
                                                       double* __restrict__ K, int N,
                                                       const double* __restrict__ boys_tab,
                                                       const PrimRec* __restrict__ kprims, int det, int gran) {
  extern __shared__ __align__(16) double s_boys[];
  load_boys_for<C>(s_boys, boys_tab);

  const int lane = threadIdx.x & 31;
  PrimRec* sbra = reinterpret_cast<PrimRec*>(s_boys + BoysStage<C>::nsl * kBoysRows * kBoysCols) + (threadIdx.x >> 5) * kSmemBraMax;
  int staged = -1;  // bra pair whose records sit in sbra (warp-uniform)
  (void)sbra;
  (void)staged;
  const long long warps = static_cast<long long>(gridDim.x) * (blockDim.x >> 5);
  const size_t nK = static_cast<size_t>(N);
  auto process = [&](const WorkItem& it) {
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
    double v[C::NV];
    if constexpr ((STYLE & kLoopSplit) != 0) {
      // Deconstruction (compiler.hpp:371-390): each contracted
      // quartet's primitive quartets are split over a lane pair (ket
      // primitives j = s, s+2, ... on lane 2k+s), the pair's contracted
      // accumulators are summed with one shuffle per boundary value, and the
      // item's 32 quartets take two passes of 16; the integrals are then
      // handed to lane = quartet so the digestion below is unchanged.
      const int s2 = lane & 1;
#pragma unroll 1
      for (int pass = 0; pass < 2; ++pass) {
        const int qi = 16 * pass + (lane >> 1);
        const bool act = qi < nq;
        int qq = (it.r0nq & 0xffffff) + (act ? qi : 0);
        int xx = it.bra0, cc = it.cntp;
        for (int n2 = __ldg(cnt + cc); qq >= n2; n2 = __ldg(cnt + cc)) {
          qq -= n2;
          ++xx;
          ++cc;
        }
        const int yy = it.yfirst + qq;
        const int4 bh = __ldg(reinterpret_cast<const int4*>(pm + xx));
        const int4 kh = __ldg(reinterpret_cast<const int4*>(pm + yy));
        const int2 ks = __ldg(reinterpret_cast<const int2*>(&pm[yy].ksoa));
        const int kstride = __ldg(&pm[yy].kstride);
        typename C::Acc acc;
        C::zero(acc);
        const PrimRec* ket = kprims + ks.x;
        const int kk = act ? kh.y : 0;
        for (int j = s2; j < kk; j += 2) {
          const PrimRec kp = load_prim<C::KPA>(ket + j * kstride);
          for (int i = 0; i < bh.y; ++i) C::prim(load_prim<C::BPA>(prims + bh.x + i), kp, s_boys, acc);
        }
        double* av = reinterpret_cast<double*>(&acc);
#pragma unroll
        for (int e = 0; e < static_cast<int>(sizeof(acc) / sizeof(double)); ++e)
          av[e] += __shfl_xor_sync(0xffffffffu, av[e], 1);
        double ABx = 0.0, ABy = 0.0, ABz = 0.0, CDx = 0.0, CDy = 0.0, CDz = 0.0;
        if constexpr (C::LB > 0) {
          const double2 a2 = __ldg(reinterpret_cast<const double2*>(&pm[xx].ABx));
          ABx = a2.x; ABy = a2.y; ABz = __ldg(&pm[xx].ABz);
        }
        if constexpr (C::LD > 0) {
          const double2 a2 = __ldg(reinterpret_cast<const double2*>(&pm[yy].ABx));
          CDx = a2.x; CDy = a2.y; CDz = __ldg(&pm[yy].ABz);
        }
        double o[C::NV];
        C::finish(acc, ABx, ABy, ABz, CDx, CDy, CDz, o);
        // lane l < 16 takes quartet l from pass 0 (lane 2l), lane l >= 16
        // quartet l from pass 1 (lane 2(l - 16))
        const int src = lane < 16 ? 2 * lane : 2 * (lane - 16);
        const bool mine = (lane < 16) == (pass == 0);
#pragma unroll
        for (int e = 0; e < C::NV; ++e) {
          const double t = __shfl_sync(0xffffffffu, o[e], src);
          if (mine) v[e] = t;
        }
      }
    } else {
      // only what the integral loop needs is loaded here; the digestion
      // fields are re-read after it (asm volatile: not hoisted across the
      // loop), so they occupy no registers during the primitive loop
      const int4 bh = __ldg(reinterpret_cast<const int4*>(pm + x));
      const int4 kh = __ldg(reinterpret_cast<const int4*>(pm + y));
      double ABx = 0.0, ABy = 0.0, ABz = 0.0, CDx = 0.0, CDy = 0.0, CDz = 0.0;
      if constexpr (C::LB > 0) {
        const double2 a = __ldg(reinterpret_cast<const double2*>(&pm[x].ABx));
        ABx = a.x; ABy = a.y; ABz = __ldg(&pm[x].ABz);
      }
      if constexpr (C::LD > 0) {
        const double2 a = __ldg(reinterpret_cast<const double2*>(&pm[y].ABx));
        CDx = a.x; CDy = a.y; CDz = __ldg(&pm[y].ABz);
      }
      const PrimRec* brap = prims + bh.x;
      if constexpr ((STYLE & 63) == kLoopSmemBra) {
        const int x0 = __shfl_sync(0xffffffffu, x, 0);
        if (__all_sync(0xffffffffu, x == x0) && bh.y <= kSmemBraMax) {
          if (x0 != staged) {
            __syncwarp();
            const double2* src = reinterpret_cast<const double2*>(prims + bh.x);
            double2* dst = reinterpret_cast<double2*>(sbra);
            for (int t = lane; t < bh.y * 5; t += 32) dst[t] = __ldg(src + t);
            __syncwarp();
            staged = x0;
          }
          brap = sbra;
        }
      }
      // kets read from the group-transposed copy: record j of the warp's 32
      // consecutive kets are 32 consecutive records (coalesced)
      const int2 ks = __ldg(reinterpret_cast<const int2*>(&pm[y].ksoa));
      const int kstride = __ldg(&pm[y].kstride);
      eri_drive<C, (STYLE & 63)>(brap, bh.y, kprims + ks.x, active ? kh.y : 0, kstride, ABx, ABy, ABz, CDx, CDy, CDz,
                          s_boys, v);
    }
    PairMeta bm, km;
    ld_meta_late(pm + x, bm);
    ld_meta_late(pm + y, km);
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
    // common case: one bra for the whole warp -> plain butterfly sum
    const bool one_bra = __all_sync(0xffffffffu, !active || x == it.bra0);
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
        s *= wj;
        if (one_bra) {
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
          if (lane == 0) red_add(J + (bm.bfa + a) * n + bm.bfb + b, s, det);
        } else {
          s = seg_sum(s, xkey, lane);
          if (tail) red_add(J + (bm.bfa + a) * n + bm.bfb + b, s, det);
        }
      }
    if constexpr ((STYLE & kLoopAggK) != 0) {
      if (!det) {
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
              red_add(J + (km.bfa + c2) * n + km.bfb + d, s * wj, 0);
            }
        }
        const unsigned long long solo = 0xffffffff00000000ull | static_cast<unsigned>(lane);
        auto key = [&](int r, int c) {
          return active ? (static_cast<unsigned long long>(static_cast<unsigned>(r)) << 32) | static_cast<unsigned>(c)
                        : solo;
        };
        {  // K_ac += sum_bd v D_bd
          double kv[C::NA * C::NC];
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
              kv[a * C::NC + c2] = s * wk;
            }
          const unsigned pe = __match_any_sync(0xffffffffu, key(bm.bfa, km.bfa));
          reduce_peers<C::NA * C::NC>(pe, kv, lane);
          if (active && __ffs(pe) - 1 == lane)
#pragma unroll
            for (int a = 0; a < C::NA; ++a)
#pragma unroll
              for (int c2 = 0; c2 < C::NC; ++c2) red_add(K + (bm.bfa + a) * n + km.bfa + c2, kv[a * C::NC + c2], 0);
        }
        {  // K_bd += sum_ac v D_ac
          double kv[C::NB * C::ND];
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
              kv[b * C::ND + d] = s * wk;
            }
          const unsigned pe = __match_any_sync(0xffffffffu, key(bm.bfb, km.bfb));
          reduce_peers<C::NB * C::ND>(pe, kv, lane);
          if (active && __ffs(pe) - 1 == lane)
#pragma unroll
            for (int b = 0; b < C::NB; ++b)
#pragma unroll
              for (int d = 0; d < C::ND; ++d) red_add(K + (bm.bfb + b) * n + km.bfb + d, kv[b * C::ND + d], 0);
        }
        {  // K_ad += sum_bc v D_bc
          double kv[C::NA * C::ND];
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
              kv[a * C::ND + d] = s * wk;
            }
          const unsigned pe = __match_any_sync(0xffffffffu, key(bm.bfa, km.bfb));
          reduce_peers<C::NA * C::ND>(pe, kv, lane);
          if (active && __ffs(pe) - 1 == lane)
#pragma unroll
            for (int a = 0; a < C::NA; ++a)
#pragma unroll
              for (int d = 0; d < C::ND; ++d) red_add(K + (bm.bfa + a) * n + km.bfb + d, kv[a * C::ND + d], 0);
        }
        {  // K_bc += sum_ad v D_ad
          double kv[C::NB * C::NC];
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
              kv[b * C::NC + c2] = s * wk;
            }
          const unsigned pe = __match_any_sync(0xffffffffu, key(bm.bfb, km.bfa));
          reduce_peers<C::NB * C::NC>(pe, kv, lane);
          if (active && __ffs(pe) - 1 == lane)
#pragma unroll
            for (int b = 0; b < C::NB; ++b)
#pragma unroll
              for (int c2 = 0; c2 < C::NC; ++c2) red_add(K + (bm.bfb + b) * n + km.bfa + c2, kv[b * C::NC + c2], 0);
        }
        return;
      }
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
          red_add(J + (km.bfa + c2) * n + km.bfb + d, s * wj, det);
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
          red_add(K + (bm.bfa + a) * n + km.bfa + c2, s * wk, det);
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
          red_add(K + (bm.bfb + b) * n + km.bfb + d, s * wk, det);
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
          red_add(K + (bm.bfa + a) * n + km.bfb + d, s * wk, det);
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
          red_add(K + (bm.bfb + b) * n + km.bfa + c2, s * wk, det);
        }
    }
  };
  for_warp_items(items, 0, nitems, gran, static_cast<long long>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5),
                 warps, process);
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
  load_boys_for<C>(s_boys, boys_tab);
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
  load_boys_for<C>(s_boys, boys_tab);
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
// JK_ONLY: only the J/K kernel is instantiated (the Schwarz / raw-quartet
// modes of the big d/f classes run on their coop kernel instead: each
// instantiation of the straight-line plan costs minutes of nvcc).
template <class C, int MINB, int STYLE = kLoopPrefetch, int NT = kJkThreads, bool JK_ONLY = false>
void launch_class(const LaunchArgs& a) {
  const size_t smem = BoysStage<C>::bytes +
                      ((STYLE & 63) == kLoopSmemBra && a.mode == 0 ? sizeof(PrimRec) * kSmemBraMax * (NT / 32) : 0);
  if (a.mode == 0) {
    if (a.nitems <= 0) return;
    const LaunchSetup ls =
        launch_setup(reinterpret_cast<const void*>(jk_kernel<C, MINB, STYLE, NT>), NT, smem, true);
    if (!ls.bps) return;  // CUDA error pending for the caller's check
    const long long g = a.gran > 1 ? a.gran : 1;
    const long long want = ((a.nitems + g - 1) / g + (NT / 32) - 1) / (NT / 32);
    const long long cap = static_cast<long long>(ls.bps) * ls.sms;
    const int grid = a.grid > 0 ? a.grid : static_cast<int>(want < cap ? want : cap);
    jk_kernel<C, MINB, STYLE, NT><<<grid, NT, smem, a.stream>>>(a.items, a.nitems, a.cnt, a.pm, a.prims, a.D, a.J,
                                                       a.K, a.N, a.boys_tab, a.kprims, a.det, a.gran);
  } else if constexpr (JK_ONLY) {
    return;  // (callers route modes 1 and 2 elsewhere)
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
