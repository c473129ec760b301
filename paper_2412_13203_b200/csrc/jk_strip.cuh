// Bra-stationary strip kernels: on-chip J/K partial sums before global
// atomics (north_star (3); SURVEY.md §7 "Digestion").
//
// Every K update of a canonical quartet (ab|cd) lands in a row of the BRA:
//   K_ac += D_bd v, K_ad += D_bc v  (rows a)   K_bc += D_ad v, K_bd += D_ac v  (rows b)
// (the K_bd / K_bc blocks are written with the bra index as row,
// the finalize kernel symmetrises). The surviving kets of one bra are a long
// Q-sorted run (thousands of quartets at N = 2000), so a CTA that owns one bra
// pair (or bra unit) for a strip of its items keeps that bra's K rows in
// shared memory, restricted to the columns of the class's ket shells (the
// functions of shells with L = L_C, and L = L_D: 560 of 2000 columns for an
// s-shell ket at (H2O)_80), reads the matching D rows from shared memory, and
// accumulates J_ab in registers. Global traffic per quartet is then the J_cd
// block (one RED per component) and the ket data; the K rows are flushed once
// per strip (only non-zero entries). Shared FP64 adds are CAS loops on sm_100a
// (ATOMS.CAST.SPIN.64), but conflict-free in the common case and far cheaper
// than L2 RED.ADD.F64 on scattered addresses (211 G/s, profiles/r01_fp64_peak.json).
//
// Items of a strip are single-bra WorkItems (32 consecutive kets of one ket
// group); warps of the CTA take them round-robin. The bra's primitive records
// (and unit weights) are staged in shared memory once per strip; inner loops
// read them as warp-broadcast LDS (kLoopSmemBra). Integrals and degeneracy are
// exactly the lane kernel's (same generated prim()/finish(), same weights), so
// results differ from the other variants only by summation order.
#pragma once
#include "jk_family.cuh"
#ifndef ERITILE_PROBE_STRIP
#define ERITILE_PROBE_STRIP 0
#endif

namespace eritile_b200 {

// Shared memory of a strip kernel: Boys slice(s), bra records and weights,
// the K rows and (DSM) the D rows, each MB * (NA + NB) rows x ncols.
template <class C, int MB>
struct StripSmem {
  static constexpr int kRowsMax = MB * (C::NA + C::NB);
  static size_t bytes(int ncols, bool dsm) {
    return BoysStage<C>::bytes + (sizeof(PrimRec) + sizeof(double2)) * kStripBraMax +
           sizeof(double) * static_cast<size_t>(kRowsMax) * ncols * (dsm ? 2 : 1);
  }
};

// Shared-memory FP64 adds of one quartet's K-row updates, batched: sm_100a
// has no native shared FP64 atomic add (atomicAdd compiles to an
// LDS / DADD / ATOMS.CAST.SPIN.64 retry loop per element, one dependent
// chain after the other). Here all NE reads are issued, then all NE CAS,
// and only the (rare) losers of a race retry, so the NE chains overlap.
template <int NE>
__device__ __forceinline__ void smem_add_batch(double* sK, const int (&idx)[NE], const double (&val)[NE]) {
  unsigned long long old[NE];
#pragma unroll
  for (int e = 0; e < NE; ++e) old[e] = *reinterpret_cast<volatile unsigned long long*>(sK + idx[e]);
  bool lost[NE];  // (static indices: predicates, any NE)
  bool any = false;
#pragma unroll
  for (int e = 0; e < NE; ++e) {
    const unsigned long long nw = __double_as_longlong(__longlong_as_double(old[e]) + val[e]);
    const unsigned long long r = atomicCAS(reinterpret_cast<unsigned long long*>(sK + idx[e]), old[e], nw);
    lost[e] = r != old[e];
    any = any || lost[e];
  }
  if (any) {
#pragma unroll
    for (int e = 0; e < NE; ++e)
      if (lost[e]) atomicAdd(sK + idx[e], val[e]);
  }
}

// OPT bits: kStripKetPf (ket record of step j+1 loaded during step j),
// kStripCasBatch (smem_add_batch for the K rows), kStripItemPf (the warp's
// next item is claimed and loaded while it evaluates the current one).
// kStripTwoKet: two ket primitives per bra record read (kLoopSmemBra2K).
// kStripAgg: warp-aggregated K-row updates. Kets of one item often share a
// shell, so several lanes hit the same shared-memory K element and the CAS
// loops serialise (ncu: 2-4 ATOMS.CAST iterations per update, 8 threads
// active). Lanes with equal column are grouped (__match_any_sync), their
// values summed in log2(group) shuffle rounds (reduce_peers), and only the
// group leader issues the (batched) shared-memory add.
// kStripL1Pf: L1 prefetch of the next ket record (kLoopSmemBraL1) and, with
// kStripItemPf, of the next item's ket metadata and first ket record.
// kStripSplitK (with kStripAgg): the d-column K updates go to global memory.
// kStripDual: a warp claims items in pairs and, when both belong to one ket
// group (same K), runs each lane's two kets in one loop nest - two independent
// chains per bra record read and both items' load/digest latencies overlapped
// (ncu: the strip kernels are latency-bound, 0.7 eligible warps per scheduler).
constexpr int kStripKetPf = 1, kStripCasBatch = 2, kStripItemPf = 4, kStripTwoKet = 8, kStripAgg = 16,
              kStripL1Pf = 32, kStripSplitK = 64, kStripDual = 128;


template <class C, bool FAM, int MB, int MK, int NT, bool DSM, int OPT = 0>
__global__ void __launch_bounds__(NT, 1) jk_strip_kernel(LaunchArgs a, long long s0, long long s1) {
  constexpr int kLoop = (OPT & kStripTwoKet)  ? kLoopSmemBra2K
                        : (OPT & kStripKetPf) ? kLoopSmemBraPf
                        : (OPT & kStripL1Pf)  ? kLoopSmemBraL1
                                              : kLoopSmemBra;
  extern __shared__ __align__(16) double smem[];
  load_boys_for<C>(smem, a.boys_tab);
  constexpr int kBoysD = BoysStage<C>::nsl * kBoysRows * kBoysCols;
  PrimRec* sbra = reinterpret_cast<PrimRec*>(smem + kBoysD);
  double2* sbw = reinterpret_cast<double2*>(sbra + kStripBraMax);
  double* sK = reinterpret_cast<double*>(sbw + kStripBraMax);
  const int ncol = a.ncols;
  double* sD = sK + StripSmem<C, MB>::kRowsMax * ncol;
  __shared__ int s_rowg[StripSmem<C, MB>::kRowsMax];  // global basis function of each smem row
  __shared__ int s_bm[MB][4];                         // bra members: bfa, bfb, sha, shb
  __shared__ int s_next;                              // next item of the strip (dynamic hand-out)
  __shared__ double s_bq[MB];                         // Schwarz Q of the bra members
  __shared__ double s_bab[3];                         // bra AB vector
  __shared__ double s_dab[MB][C::NA * C::NB];         // D'_ab of the bra members (J_cd)
  (void)sD;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  constexpr int NW = NT / 32;
  const size_t n = static_cast<size_t>(a.N);
  constexpr int LDOFF = C::LC == C::LD ? 0 : 1;  // D-shell columns follow the C-shell list
  // Strips are handed out dynamically, heaviest first (the host sorts each
  // segment's strips by modelled cost): strips differ by orders of magnitude
  // in work (a bra's survivor run is cut at kStripMaxItems), so a static
  // stride leaves the CTAs that drew heavy strips running alone at the end.
  __shared__ long long s_strip;
  int* const sctr = a.sctr;
  auto next_strip = [&](long long cur) -> long long {
    if (sctr == nullptr) return cur < 0 ? s0 + blockIdx.x : cur + gridDim.x;
    __syncthreads();  // (every thread has read the previous s_strip)
    if (threadIdx.x == 0) s_strip = s0 + atomicAdd(sctr, 1);
    __syncthreads();
    return s_strip;
  };
  for (long long s = next_strip(-1); s < s1; s = next_strip(s)) {
    const Strip st = a.strips[s];
    const int nrows = st.nrows;
    if (threadIdx.x < 4) {  // (indexed through global memory: no local copy of st)
      const Strip* gs = a.strips + s;
      int r = 0;
      for (int k = 0; k < static_cast<int>(threadIdx.x); ++k) r += gs->rb_n[k];
      for (int t = 0; t < gs->rb_n[threadIdx.x]; ++t) s_rowg[r + t] = gs->rb_bf[threadIdx.x] + t;
    }
    // bra records (and unit weights): one copy per CTA for the whole strip
    // (strip bras have K <= kStripBraMax; the host keeps larger ones packed)
    int kb, boff;
    if constexpr (FAM) {
      kb = a.um[st.bra].K;
      boff = a.um[st.bra].prim_off;
    } else {
      kb = a.pm[st.bra].K;
      boff = a.pm[st.bra].prim_off;
    }
    {
      const double2* src = reinterpret_cast<const double2*>(a.prims + boff);
      double2* dst = reinterpret_cast<double2*>(sbra);
      for (int t = threadIdx.x; t < kb * 5; t += NT) dst[t] = __ldg(src + t);
      if constexpr (FAM)
        for (int t = threadIdx.x; t < kb; t += NT) sbw[t] = __ldg(a.uw + boff + t);
    }
    if (threadIdx.x < MB) {
      int px = st.bra;
      if constexpr (FAM) px = threadIdx.x == 0 ? a.um[st.bra].m0 : a.um[st.bra].m1;
      PairMeta bm;
      ld_meta_late(a.pm + px, bm);
      s_bm[threadIdx.x][0] = bm.bfa;
      s_bm[threadIdx.x][1] = bm.bfb;
      s_bm[threadIdx.x][2] = bm.sha;
      s_bm[threadIdx.x][3] = bm.shb;
      s_bq[threadIdx.x] = FAM ? __ldg(a.Qp + px) : 0.0;
    }
    if (threadIdx.x == 32) {
      if constexpr (FAM) {
        s_bab[0] = a.um[st.bra].ABx; s_bab[1] = a.um[st.bra].ABy; s_bab[2] = a.um[st.bra].ABz;
      } else {
        s_bab[0] = a.pm[st.bra].ABx; s_bab[1] = a.pm[st.bra].ABy; s_bab[2] = a.pm[st.bra].ABz;
      }
    }
    for (int e = threadIdx.x; e < MB * C::NA * C::NB; e += NT) {
      // (the bra members' first functions, read from global: s_bm is not yet visible)
      const int m = e / (C::NA * C::NB), ab = e % (C::NA * C::NB);
      int px = st.bra;
      if constexpr (FAM) px = m == 0 ? a.um[st.bra].m0 : a.um[st.bra].m1;
      const int bfa = __ldg(&a.pm[px].bfa), bfb = __ldg(&a.pm[px].bfb);
      s_dab[m][ab] = __ldg(a.D + static_cast<size_t>(bfa + ab / C::NB) * n + bfb + ab % C::NB);
    }
    if (threadIdx.x == 0) s_next = st.i0;
    for (int e = threadIdx.x; e < nrows * ncol; e += NT) sK[e] = 0.0;
    __syncthreads();
    if constexpr (DSM) {
      for (int e = threadIdx.x; e < nrows * ncol; e += NT) {
        const int r = e / ncol;
        sD[e] = __ldg(a.D + static_cast<size_t>(s_rowg[r]) * n + __ldg(a.cols + (e - r * ncol)));
      }
      __syncthreads();
    }
    const PrimRec* brap = sbra;
    const double2* bwp = sbw;
    (void)bwp;
    // J_ab partial sums, lane-private over all items of the strip
    double jab[MB][C::NA * C::NB];
#pragma unroll
    for (int m = 0; m < MB; ++m)
#pragma unroll
      for (int e = 0; e < C::NA * C::NB; ++e) jab[m][e] = 0.0;
    // bra members (pair strips: the pair itself)
    int bpx[MB];
    if constexpr (FAM) {
      bpx[0] = a.um[st.bra].m0;
      if constexpr (MB == 2) bpx[MB - 1] = a.um[st.bra].m1;
    } else {
      bpx[0] = st.bra;
    }
    (void)warp;
    // items are claimed in runs of g = a.gran consecutive items (the
    // Workload Allocator's Combine granularity); s_next may overshoot i1
    const int g0 = a.gran > 1 ? a.gran : 1;
    const int g = (OPT & kStripDual) && g0 < 2 ? 2 : g0;
    int lo = 0, hi = 0;  // this warp's claimed, not yet started items
    auto claim = [&]() -> bool {
      int c = 0;
      if (lane == 0) c = atomicAdd(&s_next, g);  // dynamic: items differ in primitive count
      c = __shfl_sync(0xffffffffu, c, 0);
      lo = c;
      hi = c + g < st.i1 ? c + g : st.i1;
      return c < st.i1;
    };
    int wn = st.i1;
    WorkItem nxt{};
    if constexpr (OPT & kStripItemPf) {
      if (claim()) wn = lo++;
      if (wn < st.i1) nxt = a.items[wn];
    }
    // digestion of one ket per lane (J_ab in registers, J_cd to global, K rows
    // in shared memory); called once per item, twice for dual items
    auto digest = [&](const int y, const bool active, double (&acc_v)[MB][MK][C::NV]) {
        // digestion metadata of this lane's ket: one 64-byte read (no registers
        // held across the primitive loop; measured slower when loaded up front)
        KetMeta km;
        {
          const int4* kq = reinterpret_cast<const int4*>(a.kmeta + y);
          int4 q0, q1, q2;
          double2 q3;
          asm volatile("ld.global.nc.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(q0.x), "=r"(q0.y), "=r"(q0.z), "=r"(q0.w) : "l"(kq));
          asm volatile("ld.global.nc.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(q1.x), "=r"(q1.y), "=r"(q1.z), "=r"(q1.w) : "l"(kq + 1));
          asm volatile("ld.global.nc.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(q2.x), "=r"(q2.y), "=r"(q2.z), "=r"(q2.w) : "l"(kq + 2));
          asm volatile("ld.global.nc.v2.f64 {%0,%1}, [%2];" : "=d"(q3.x), "=d"(q3.y) : "l"(kq + 3));
          km.bfa[0] = q0.x; km.bfa[1] = q0.y; km.bfb[0] = q0.z; km.bfb[1] = q0.w;
          km.colc[0] = q1.x; km.colc[1] = q1.y; km.cold[0] = q1.z; km.cold[1] = q1.w;
          km.offd[0] = q2.x; km.offd[1] = q2.y; km.m[0] = q2.z; km.m[1] = q2.w;
          km.q[0] = q3.x; km.q[1] = q3.y;
        }
  #pragma unroll
        for (int m = 0; m < MB; ++m) {
          PairMeta bm;
          bm.bfa = s_bm[m][0];
          bm.bfb = s_bm[m][1];
          bm.sha = s_bm[m][2];
          bm.shb = s_bm[m][3];
          const int rA = st.rowA[m], rB = st.rowB[m];
  #pragma unroll
          for (int k = 0; k < MK; ++k) {
            const int py = km.m[k];
            bool keep = active;
            if constexpr (FAM) keep = keep && !(st.bra == y && m > k) && (a.tau <= 0.0 || s_bq[m] * km.q[k] >= a.tau);
            constexpr bool AGG = (OPT & kStripAgg) != 0;
            if constexpr (AGG) {  // the whole warp digests (shuffle groups), non-kept lanes add zeros
              if (!__any_sync(0xffffffffu, keep)) continue;
            } else {
              if (!keep) continue;
            }
            const int kbfa = km.bfa[k], kbfb = km.bfb[k];
            const double* v = acc_v[m][k];
            const double deg =
                (bm.sha != bm.shb ? 2.0 : 1.0) * (km.offd[k] ? 2.0 : 1.0) * (bpx[m] != py ? 2.0 : 1.0);
            const double wj = keep ? 0.5 * deg : 0.0, wk = keep ? 0.25 * deg : 0.0;
            const int colC = km.colc[k];
            const int colD = km.cold[k] + (LDOFF ? a.ncolC : 0);
            const double* Dcd = a.D + kbfa * n + kbfb;
            auto dsm = [&](int row, int col, size_t grow, size_t gcol) -> double {
              if constexpr (DSM) return sD[row * ncol + col];
              else return __ldg(a.D + grow * n + gcol);
            };
  #pragma unroll
            for (int ia = 0; ia < C::NA; ++ia)
  #pragma unroll
              for (int ib = 0; ib < C::NB; ++ib) {
                double t = 0.0;
  #pragma unroll
                for (int ic = 0; ic < C::NC; ++ic)
  #pragma unroll
                  for (int id = 0; id < C::ND; ++id)
                    t = fma(v[((ia * C::NB + ib) * C::NC + ic) * C::ND + id], __ldg(Dcd + ic * n + id), t);
                jab[m][ia * C::NB + ib] = fma(t, wj, jab[m][ia * C::NB + ib]);
              }
  #pragma unroll
            for (int ic = 0; ic < C::NC; ++ic)
  #pragma unroll
              for (int id = 0; id < C::ND; ++id) {
                double t = 0.0;
  #pragma unroll
                for (int ia = 0; ia < C::NA; ++ia)
  #pragma unroll
                  for (int ib = 0; ib < C::NB; ++ib)
                    t = fma(v[((ia * C::NB + ib) * C::NC + ic) * C::ND + id], s_dab[m][ia * C::NB + ib], t);
                if (keep) red_add(a.J + (kbfa + ic) * n + kbfb + id, t * wj, 0);
              }
            // K_ac += sum_bd v D_bd ; K_ad += sum_bc v D_bc   (rows a of the bra)
            // K_bd += sum_ac v D_ac ; K_bc += sum_ad v D_ad   (rows b of the bra)
            constexpr int NKE = C::NA * (C::NC + C::ND) + C::NB * (C::NC + C::ND);
            int kidx[NKE];
            double kval[NKE];
            int ne = 0;
  #pragma unroll
            for (int ia = 0; ia < C::NA; ++ia) {
  #pragma unroll
              for (int ic = 0; ic < C::NC; ++ic) {
                double t = 0.0;
  #pragma unroll
                for (int ib = 0; ib < C::NB; ++ib)
  #pragma unroll
                  for (int id = 0; id < C::ND; ++id)
                    t = fma(v[((ia * C::NB + ib) * C::NC + ic) * C::ND + id],
                            dsm(rB + ib, colD + id, bm.bfb + ib, kbfb + id), t);
                kidx[ne] = (rA + ia) * ncol + colC + ic;
                kval[ne++] = t * wk;
              }
  #pragma unroll
              for (int id = 0; id < C::ND; ++id) {
                double t = 0.0;
  #pragma unroll
                for (int ib = 0; ib < C::NB; ++ib)
  #pragma unroll
                  for (int ic = 0; ic < C::NC; ++ic)
                    t = fma(v[((ia * C::NB + ib) * C::NC + ic) * C::ND + id],
                            dsm(rB + ib, colC + ic, bm.bfb + ib, kbfa + ic), t);
                kidx[ne] = (rA + ia) * ncol + colD + id;
                kval[ne++] = t * wk;
              }
            }
  #pragma unroll
            for (int ib = 0; ib < C::NB; ++ib) {
  #pragma unroll
              for (int id = 0; id < C::ND; ++id) {
                double t = 0.0;
  #pragma unroll
                for (int ia = 0; ia < C::NA; ++ia)
  #pragma unroll
                  for (int ic = 0; ic < C::NC; ++ic)
                    t = fma(v[((ia * C::NB + ib) * C::NC + ic) * C::ND + id],
                            dsm(rA + ia, colC + ic, bm.bfa + ia, kbfa + ic), t);
                kidx[ne] = (rB + ib) * ncol + colD + id;
                kval[ne++] = t * wk;
              }
  #pragma unroll
              for (int ic = 0; ic < C::NC; ++ic) {
                double t = 0.0;
  #pragma unroll
                for (int ia = 0; ia < C::NA; ++ia)
  #pragma unroll
                  for (int id = 0; id < C::ND; ++id)
                    t = fma(v[((ia * C::NB + ib) * C::NC + ic) * C::ND + id],
                            dsm(rA + ia, colD + id, bm.bfa + ia, kbfb + id), t);
                kidx[ne] = (rB + ib) * ncol + colC + ic;
                kval[ne++] = t * wk;
              }
            }
            if constexpr (AGG) {
              // c-keyed updates (K_ac, K_bc) and d-keyed updates (K_ad, K_bd)
              constexpr int NCK = (C::NA + C::NB) * C::NC, NDK = (C::NA + C::NB) * C::ND;
              int ci[NCK], di[NDK];
              double cv[NCK], dv[NDK];
              int nc = 0, nd = 0;
  #pragma unroll
              for (int ia = 0; ia < C::NA; ++ia) {
  #pragma unroll
                for (int ic = 0; ic < C::NC; ++ic) {
                  ci[nc] = kidx[ia * (C::NC + C::ND) + ic];
                  cv[nc++] = kval[ia * (C::NC + C::ND) + ic];
                }
  #pragma unroll
                for (int id = 0; id < C::ND; ++id) {
                  di[nd] = kidx[ia * (C::NC + C::ND) + C::NC + id];
                  dv[nd++] = kval[ia * (C::NC + C::ND) + C::NC + id];
                }
              }
  #pragma unroll
              for (int ib = 0; ib < C::NB; ++ib) {
                constexpr int b0 = C::NA * (C::NC + C::ND);
  #pragma unroll
                for (int id = 0; id < C::ND; ++id) {
                  di[nd] = kidx[b0 + ib * (C::NC + C::ND) + id];
                  dv[nd++] = kval[b0 + ib * (C::NC + C::ND) + id];
                }
  #pragma unroll
                for (int ic = 0; ic < C::NC; ++ic) {
                  ci[nc] = kidx[b0 + ib * (C::NC + C::ND) + C::ND + ic];
                  cv[nc++] = kval[b0 + ib * (C::NC + C::ND) + C::ND + ic];
                }
              }
              const unsigned pc = __match_any_sync(0xffffffffu, keep ? colC : -1 - lane);
              const unsigned pd = __match_any_sync(0xffffffffu, keep ? colD : -1 - lane);
              reduce_peers<NCK>(pc, cv, lane);
              reduce_peers<NDK>(pd, dv, lane);
              if (keep && __ffs(pc) - 1 == lane) smem_add_batch<NCK>(sK, ci, cv);
              if (keep && __ffs(pd) - 1 == lane) {
                if constexpr (OPT & kStripSplitK) {
                  // d-column updates straight to global K (L2 RED.ADD.F64): the
                  // shared-memory atomic unit (~2 cycles per lane) and the L2
                  // atomic units then each carry half of the K traffic
                  int e = 0;
  #pragma unroll
                  for (int ia = 0; ia < C::NA; ++ia)
  #pragma unroll
                    for (int id = 0; id < C::ND; ++id)
                      red_add(a.K + (bm.bfa + ia) * n + kbfb + id, dv[e++], 0);
  #pragma unroll
                  for (int ib = 0; ib < C::NB; ++ib)
  #pragma unroll
                    for (int id = 0; id < C::ND; ++id)
                      red_add(a.K + (bm.bfb + ib) * n + kbfb + id, dv[e++], 0);
                } else {
                  smem_add_batch<NDK>(sK, di, dv);
                }
              }
            } else if constexpr (OPT & kStripCasBatch) {
              smem_add_batch<NKE>(sK, kidx, kval);
            } else {
  #pragma unroll
              for (int e = 0; e < NKE; ++e) atomicAdd(sK + kidx[e], kval[e]);
            }
          }
        }
    };
    for (;;) {
      int w = 0;
      WorkItem it, it2{};
      bool dual = false;  // kStripDual: two consecutive items of one ket group
      if constexpr (OPT & kStripItemPf) {
        w = wn;
        if (w >= st.i1) break;
        it = nxt;
        wn = st.i1;
        if (lo < hi || claim()) wn = lo++;
        if (wn < st.i1) nxt = a.items[wn];  // in flight during this item
      } else {
        if (lo >= hi && !claim()) break;
        w = lo++;
        it = a.items[w];
        if constexpr (OPT & kStripDual) {
          if (lo < hi) {
            it2 = a.items[lo];
            dual = it2.yfirst == it.yfirst;
            if (dual) ++lo;
          }
        }
      }
      (void)w;
      (void)dual;
      const int nq = it.r0nq >> 24;
      const bool active = lane < nq;
      const int y = it.yfirst + (it.r0nq & 0xffffff) + (active ? lane : 0);  // single-bra item
      prefetch_l1(a.kmeta + y);  // read again after the primitive loop (digestion)
      const int nq2 = it2.r0nq >> 24;
      const bool active2 = dual && lane < nq2;
      const int y2 = dual ? it2.yfirst + (it2.r0nq & 0xffffff) + (active2 ? lane : 0) : y;
      if (dual) prefetch_l1(a.kmeta + y2);
      (void)y2;
      double acc_v[MB][MK][C::NV];
      double acc_v2[(OPT & kStripDual) ? MB : 1][(OPT & kStripDual) ? MK : 1][C::NV];
      (void)acc_v;
      (void)acc_v2;
      double ABx, ABy, ABz, CDx, CDy, CDz;
      if constexpr (FAM) {
        const UnitMeta ku = a.um[y];
        ABx = s_bab[0]; ABy = s_bab[1]; ABz = s_bab[2];
        CDx = ku.ABx; CDy = ku.ABy; CDz = ku.ABz;
        typename C::Acc acc[MB][MK];
        if constexpr (OPT & kStripDual) {
          if (dual) {  // both kets of the lane in one loop nest: two chains per bra record read
            const UnitMeta ku2 = a.um[y2];
            typename C::Acc acc2[MB][MK];
            fam_drive_dual<C, MB, MK>(brap, bwp, kb, a.ukprims + ku.ksoa, a.ukw + ku.ksoa, a.ukprims + ku2.ksoa,
                                      a.ukw + ku2.ksoa, ku.K, ku.kstride, smem, acc, acc2);
#pragma unroll
            for (int m = 0; m < MB; ++m)
#pragma unroll
              for (int k = 0; k < MK; ++k) {
                C::finish(acc[m][k], ABx, ABy, ABz, CDx, CDy, CDz, acc_v[m][k]);
                C::finish(acc2[m][k], ABx, ABy, ABz, ku2.ABx, ku2.ABy, ku2.ABz, acc_v2[m][k]);
              }
            digest(y, active, acc_v);
            digest(y2, active2, acc_v2);
            continue;
          }
        }
#if ERITILE_PROBE_STRIP == 2  // measurement build: no primitive loop
        fam_drive<C, MB, MK, kLoop>(brap, bwp, kb, a.ukprims + ku.ksoa, a.ukw + ku.ksoa, 0,
#else
        fam_drive<C, MB, MK, kLoop>(brap, bwp, kb, a.ukprims + ku.ksoa, a.ukw + ku.ksoa, active ? ku.K : 0,
#endif
                                           ku.kstride, smem, acc);
#pragma unroll
        for (int m = 0; m < MB; ++m)
#pragma unroll
          for (int k = 0; k < MK; ++k) C::finish(acc[m][k], ABx, ABy, ABz, CDx, CDy, CDz, acc_v[m][k]);
      } else {
        ABx = s_bab[0]; ABy = s_bab[1]; ABz = s_bab[2];
        const int4 kh = __ldg(reinterpret_cast<const int4*>(a.pm + y));
        const double2 cd = __ldg(reinterpret_cast<const double2*>(&a.pm[y].ABx));
        CDx = cd.x; CDy = cd.y; CDz = __ldg(&a.pm[y].ABz);
        const int2 ks = __ldg(reinterpret_cast<const int2*>(&a.pm[y].ksoa));
        const int kstride = __ldg(&a.pm[y].kstride);
        if constexpr (OPT & kStripDual) {
          if (dual) {
            const int ks2 = __ldg(&a.pm[y2].ksoa);
            const double2 cd2 = __ldg(reinterpret_cast<const double2*>(&a.pm[y2].ABx));
            const double cdz2 = __ldg(&a.pm[y2].ABz);
            eri_drive_dual<C>(brap, kb, a.kprims + ks.x, a.kprims + ks2, kh.y, kstride, ABx, ABy, ABz, CDx, CDy,
                              CDz, cd2.x, cd2.y, cdz2, smem, acc_v[0][0], acc_v2[0][0]);
            digest(y, active, acc_v);
            digest(y2, active2, acc_v2);
            continue;
          }
        }
        eri_drive<C, kLoop>(brap, kb, a.kprims + ks.x, active ? kh.y : 0, kstride, ABx, ABy, ABz, CDx, CDy,
                                   CDz, smem, acc_v[0][0]);
      }
#if ERITILE_PROBE_STRIP == 1  // measurement build: no digestion (keep the integrals live)
      {
        double t = 0.0;
#pragma unroll
        for (int m = 0; m < MB; ++m)
#pragma unroll
          for (int k = 0; k < MK; ++k)
#pragma unroll
            for (int e = 0; e < C::NV; ++e) t += acc_v[m][k][e];
        if (t == 1.2345e-300) a.J[lane] = t;
        continue;
      }
#endif
      if constexpr ((OPT & kStripL1Pf) && (OPT & kStripItemPf)) {
        // the next item has arrived by now: warm L1 with its ket metadata
        if (wn < st.i1) {
          const int nqn = nxt.r0nq >> 24;
          const int yn = nxt.yfirst + (nxt.r0nq & 0xffffff) + (lane < nqn ? lane : 0);
          if constexpr (FAM) prefetch_l1(a.um + yn);
          else prefetch_l1(a.pm + yn);
        }
      }
      digest(y, active, acc_v);
    }
    // J_ab: one butterfly per strip and warp, one RED per element and warp
#pragma unroll
    for (int m = 0; m < MB; ++m) {
      const size_t bfa = s_bm[m][0], bfb = s_bm[m][1];
#pragma unroll
      for (int e = 0; e < C::NA * C::NB; ++e) {
        double t = jab[m][e];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
        if (lane == 0 && t != 0.0) red_add(a.J + (bfa + e / C::NB) * n + bfb + e % C::NB, t, 0);
      }
    }
    __syncthreads();
    // flush the K rows (non-zero entries only)
    for (int e = threadIdx.x; e < nrows * ncol; e += NT) {
      const double v = sK[e];
      if (v != 0.0) {
        const int r = e / ncol;
        red_add(a.K + static_cast<size_t>(s_rowg[r]) * n + __ldg(a.cols + (e - r * ncol)), v, 0);
      }
    }
    __syncthreads();
  }
}

// Strips of member segment (MB, MK) through the strip kernel; returns false
// (nothing launched) if its shared memory does not fit - the caller then runs
// those items through the lane kernel.
template <class C, bool FAM, int MB, int MK, int NT, int OPT = 0>
bool launch_strip_seg(const LaunchArgs& a0, long long s0, long long s1, int seg) {
  if (s1 <= s0) return true;
  LaunchArgs a = a0;
  a.sctr = a0.sctr ? a0.sctr + seg : nullptr;
  const size_t with_d = StripSmem<C, MB>::bytes(a.ncols, true);
  const size_t no_d = StripSmem<C, MB>::bytes(a.ncols, false);
  constexpr size_t kMax = 227 * 1024 - 1024;  // static s_rowg + reserve
  if (no_d > kMax) return false;
  const bool dsm = with_d <= kMax;
  const void* fn = dsm ? reinterpret_cast<const void*>(jk_strip_kernel<C, FAM, MB, MK, NT, true, OPT>)
                       : reinterpret_cast<const void*>(jk_strip_kernel<C, FAM, MB, MK, NT, false, OPT>);
  const size_t smem = dsm ? with_d : no_d;
  const LaunchSetup ls = launch_setup(fn, NT, smem, false);
  if (!ls.bps) return true;  // CUDA error pending for the caller's check
  const long long cap = static_cast<long long>(ls.bps) * ls.sms;
  const int grid = static_cast<int>(s1 - s0 < cap ? s1 - s0 : cap);
  if (dsm)
    jk_strip_kernel<C, FAM, MB, MK, NT, true, OPT><<<grid, NT, smem, a.stream>>>(a, s0, s1);
  else
    jk_strip_kernel<C, FAM, MB, MK, NT, false, OPT><<<grid, NT, smem, a.stream>>>(a, s0, s1);
  return true;
}

// Pair-list strip variant: strips through the strip kernel, the remaining
// (multi-bra packed) items through the lane kernel <MINB, STYLE, NTL>.
// Deterministic mode runs every item on the lane kernels (the shared-memory
// K rows would sum in scheduling order).
template <class C, int NT, int MINB, int STYLE, int NTL, int OPT = 0>
void launch_strip(const LaunchArgs& a) {
  if (a.mode != 0) return launch_class<C, 2, kLoopPrefetch>(a);
  if (a.nitems <= 0) return;
  if (a.det) return launch_class<C, MINB, STYLE, NTL>(a);
  LaunchArgs r = a;
  if (a.sctr) cudaMemsetAsync(a.sctr, 0, 4 * sizeof(int), a.stream);
  if (launch_strip_seg<C, false, 1, 1, NT, OPT>(a, a.sseg[0], a.sseg[1], 0)) {
    r.items = a.items + a.sitem[0];
    r.nitems = a.nitems - a.sitem[0];
  }
  launch_class<C, MINB, STYLE, NTL>(r);
}

// Unit-list strip variant: per member segment, strips through the strip
// kernel and the rest through the unit lane kernel.
template <class C, int NT, int MINB, int STYLE, int NTL, int NT11, int OPT = 0>
void launch_fstrip(const LaunchArgs& a) {
  if (a.mode != 0) return launch_class<C, 2, kLoopPrefetch>(a);
  if (a.det) {
    launch_fam_seg<C, 1, 1, MINB, STYLE, NT11>(a, a.seg[0], a.seg[1]);
    launch_fam_seg<C, 1, 2, MINB, STYLE, NTL>(a, a.seg[1], a.seg[2]);
    launch_fam_seg<C, 2, 1, MINB, STYLE, NTL>(a, a.seg[2], a.seg[3]);
    launch_fam_seg<C, 2, 2, MINB, STYLE, NTL>(a, a.seg[3], a.seg[4]);
    return;
  }
  long long rest0[4];
  for (int sg = 0; sg < 4; ++sg) rest0[sg] = a.seg[sg];
  if (a.sctr) cudaMemsetAsync(a.sctr, 0, 4 * sizeof(int), a.stream);
  if (launch_strip_seg<C, true, 1, 1, NT, OPT>(a, a.sseg[0], a.sseg[1], 0)) rest0[0] = a.sitem[0];
  if (launch_strip_seg<C, true, 1, 2, NT, OPT>(a, a.sseg[1], a.sseg[2], 1)) rest0[1] = a.sitem[1];
  if (launch_strip_seg<C, true, 2, 1, NT, OPT>(a, a.sseg[2], a.sseg[3], 2)) rest0[2] = a.sitem[2];
  if (launch_strip_seg<C, true, 2, 2, NT, OPT>(a, a.sseg[3], a.sseg[4], 3)) rest0[3] = a.sitem[3];
  launch_fam_seg<C, 1, 1, MINB, STYLE, NT11>(a, rest0[0], a.seg[1]);
  launch_fam_seg<C, 1, 2, MINB, STYLE, NTL>(a, rest0[1], a.seg[2]);
  launch_fam_seg<C, 2, 1, MINB, STYLE, NTL>(a, rest0[2], a.seg[3]);
  launch_fam_seg<C, 2, 2, MINB, STYLE, NTL>(a, rest0[3], a.seg[4]);
}

}  // namespace eritile_b200
