// Shared-primitive ("family") lane kernels for generally contracted shells.
//
// cc-pVDZ writes the O/C/N 1s and 2s functions as two segmented shells with
// the same nine exponents (the reference's Shell, molecule.hpp:39-50, holds
// one contraction each). Shell pairs that differ only by such a sibling have
// bit-identical primitive-pair records except the contraction weight U
// (block.hpp:73-82: p, P, PA, kappa depend on exponents and centres only).
// The host groups them into units of <= 2 member pairs (engine.cu
// build_units); a lane evaluates one (bra unit, ket unit) pair: every
// primitive quartet is bound and recursed ONCE with the U-free prefactor
// 1/sqrt(p+q), and folded into the four member combinations with the member
// weights U_m(bra prim) U_n(ket prim). Each member quartet is then screened
// (Q_m Q_n >= tau, the same rule as the pair path) and digested exactly as
// SPEC.md:350 prescribes, so the surviving quartet set, the integrals and
// J/K are those of the per-pair path up to rounding.
#pragma once
#include "jk_kernels.cuh"

namespace eritile_b200 {

constexpr int kFamMax = 2;  // members per unit

// Primitive loop of one unit pair: acc[m][n] accumulates member combo (m, n).
// kw/bw: per-primitive member weights (U of member 0 / 1; 0 if absent).
template <class C, int MB, int MK, int STYLE>
__device__ __forceinline__ void fam_drive(const PrimRec* __restrict__ bra, const double2* __restrict__ bw, int kb,
                                          const PrimRec* __restrict__ ket, const double2* __restrict__ kw, int kk,
                                          int ks,
                                          const double* __restrict__ btab, typename C::Acc (&acc)[MB][MK]) {
#pragma unroll
  for (int m = 0; m < MB; ++m)
#pragma unroll
    for (int n = 0; n < MK; ++n) C::zero(acc[m][n]);
  if constexpr (STYLE == kLoopSmemBra2K) {  // two ket primitives per bra record read
    int j = 0;
    for (; j + 1 < kk; j += 2) {
      const PrimRec k0 = load_prim<C::KPA>(ket + j * ks);
      const PrimRec k1 = load_prim<C::KPA>(ket + (j + 1) * ks);
      typename C::Acc s0[MB], s1[MB];
#pragma unroll
      for (int m = 0; m < MB; ++m) {
        C::zero(s0[m]);
        C::zero(s1[m]);
      }
      for (int i = 0; i < kb; ++i) {
        const PrimRec bq = load_prim_gen<C::BPA>(bra + i);
        const double2 wq = bw[i];
        if constexpr (MB == 2) {
          C::prim_w(bq, k0, btab, wq.x, wq.y, s0[0], s0[MB - 1]);
          C::prim_w(bq, k1, btab, wq.x, wq.y, s1[0], s1[MB - 1]);
        } else {
          C::prim_w1(bq, k0, btab, wq.x, s0[0]);
          C::prim_w1(bq, k1, btab, wq.x, s1[0]);
        }
      }
      const double2 w0 = __ldg(kw + j * ks), w1 = __ldg(kw + (j + 1) * ks);
#pragma unroll
      for (int m = 0; m < MB; ++m) {
        C::axpy(acc[m][0], w0.x, s0[m]);
        C::axpy(acc[m][0], w1.x, s1[m]);
        if constexpr (MK == 2) {
          C::axpy(acc[m][MK - 1], w0.y, s0[m]);
          C::axpy(acc[m][MK - 1], w1.y, s1[m]);
        }
      }
    }
    if (j < kk) {
      const PrimRec kp = load_prim<C::KPA>(ket + j * ks);
      typename C::Acc s0[MB];
#pragma unroll
      for (int m = 0; m < MB; ++m) C::zero(s0[m]);
      for (int i = 0; i < kb; ++i) {
        const double2 wq = bw[i];
        if constexpr (MB == 2) C::prim_w(load_prim_gen<C::BPA>(bra + i), kp, btab, wq.x, wq.y, s0[0], s0[MB - 1]);
        else C::prim_w1(load_prim_gen<C::BPA>(bra + i), kp, btab, wq.x, s0[0]);
      }
      const double2 w0 = __ldg(kw + j * ks);
#pragma unroll
      for (int m = 0; m < MB; ++m) {
        C::axpy(acc[m][0], w0.x, s0[m]);
        if constexpr (MK == 2) C::axpy(acc[m][MK - 1], w0.y, s0[m]);
      }
    }
    return;
  }
  PrimRec kn;
  double2 kwn;
  if constexpr (STYLE == kLoopSmemBraPf) {  // ket record of step j+1 in flight during step j
    kn = load_prim<C::KPA>(ket);
    kwn = __ldg(kw);
  }
  for (int j = 0; j < kk; ++j) {
    PrimRec kp;
    double2 kwj;
    if constexpr (STYLE == kLoopSmemBraPf) {
      kp = kn;
      kwj = kwn;
      if (j + 1 < kk) {
        kn = load_prim<C::KPA>(ket + (j + 1) * ks);
        kwn = __ldg(kw + (j + 1) * ks);
      }
    } else {
      if constexpr (STYLE == kLoopSmemBraL1)
        if (j + 1 < kk) {
          prefetch_l1(ket + (j + 1) * ks);
          prefetch_l1(kw + (j + 1) * ks);
        }
      kp = load_prim<C::KPA>(ket + j * ks);
      kwj = __ldg(kw + j * ks);
    }
    typename C::Acc s[MB];  // sum over bra prims of U_m(bra) * g, per bra member
#pragma unroll
    for (int m = 0; m < MB; ++m) C::zero(s[m]);
    if constexpr (STYLE == kLoopPrefetch) {
      PrimRec bn = load_prim<C::BPA>(bra);
      double2 wn = __ldg(bw);
      for (int i = 0; i < kb; ++i) {
        const PrimRec bq = bn;
        const double2 wq = wn;
        bn = load_prim<C::BPA>(bra + (i + 1 < kb ? i + 1 : i));
        wn = __ldg(bw + (i + 1 < kb ? i + 1 : i));
        if constexpr (MB == 2) C::prim_w(bq, kp, btab, wq.x, wq.y, s[0], s[MB - 1]);
        else C::prim_w1(bq, kp, btab, wq.x, s[0]);
      }
    } else if constexpr (STYLE == kLoopSmemBra || STYLE == kLoopSmemBraPf || STYLE == kLoopSmemBraL1) {  // bra records / weights may sit in shared memory
      for (int i = 0; i < kb; ++i) {
        const double2 wq = bw[i];
        if constexpr (MB == 2) C::prim_w(load_prim_gen<C::BPA>(bra + i), kp, btab, wq.x, wq.y, s[0], s[MB - 1]);
        else C::prim_w1(load_prim_gen<C::BPA>(bra + i), kp, btab, wq.x, s[0]);
      }
    } else {
      for (int i = 0; i < kb; ++i) {
        const double2 wq = __ldg(bw + i);
        if constexpr (MB == 2) C::prim_w(load_prim<C::BPA>(bra + i), kp, btab, wq.x, wq.y, s[0], s[MB - 1]);
        else C::prim_w1(load_prim<C::BPA>(bra + i), kp, btab, wq.x, s[0]);
      }
    }
#pragma unroll
    for (int m = 0; m < MB; ++m) {
      C::axpy(acc[m][0], kwj.x, s[m]);
      if constexpr (MK == 2) C::axpy(acc[m][MK - 1], kwj.y, s[m]);
    }
  }
}

// Two ket units per lane in one loop nest (strip kernels, kStripDual): same
// unit group (same K and stride); every bra record / weight read from shared
// memory feeds two independent primitive chains.
template <class C, int MB, int MK>
__device__ __forceinline__ void fam_drive_dual(const PrimRec* bra, const double2* bw, int kb,
                                               const PrimRec* __restrict__ ket1, const double2* __restrict__ kw1,
                                               const PrimRec* __restrict__ ket2, const double2* __restrict__ kw2,
                                               int kk, int ks, const double* __restrict__ btab,
                                               typename C::Acc (&acc1)[MB][MK], typename C::Acc (&acc2)[MB][MK]) {
#pragma unroll
  for (int m = 0; m < MB; ++m)
#pragma unroll
    for (int n = 0; n < MK; ++n) {
      C::zero(acc1[m][n]);
      C::zero(acc2[m][n]);
    }
  for (int j = 0; j < kk; ++j) {
    const PrimRec k1 = load_prim<C::KPA>(ket1 + j * ks);
    const PrimRec k2 = load_prim<C::KPA>(ket2 + j * ks);
    const double2 w1 = __ldg(kw1 + j * ks), w2 = __ldg(kw2 + j * ks);
    typename C::Acc s1[MB], s2[MB];
#pragma unroll
    for (int m = 0; m < MB; ++m) {
      C::zero(s1[m]);
      C::zero(s2[m]);
    }
    for (int i = 0; i < kb; ++i) {
      const PrimRec bq = load_prim_gen<C::BPA>(bra + i);
      const double2 wq = bw[i];
      if constexpr (MB == 2) {
        C::prim_w(bq, k1, btab, wq.x, wq.y, s1[0], s1[MB - 1]);
        C::prim_w(bq, k2, btab, wq.x, wq.y, s2[0], s2[MB - 1]);
      } else {
        C::prim_w1(bq, k1, btab, wq.x, s1[0]);
        C::prim_w1(bq, k2, btab, wq.x, s2[0]);
      }
    }
#pragma unroll
    for (int m = 0; m < MB; ++m) {
      C::axpy(acc1[m][0], w1.x, s1[m]);
      C::axpy(acc2[m][0], w2.x, s2[m]);
      if constexpr (MK == 2) {
        C::axpy(acc1[m][MK - 1], w1.y, s1[m]);
        C::axpy(acc2[m][MK - 1], w2.y, s2[m]);
      }
    }
  }
}

// MB / MK: members per bra / ket unit of this launch segment (items are
// sorted by (MB, MK) within the class, csrc/host/engine.cu set_screening).
template <class C, int MB, int MK, int MINB, int STYLE, int NT>
__global__ void __launch_bounds__(NT, MINB) jk_fam_kernel(LaunchArgs a, long long i0, long long i1) {
  extern __shared__ __align__(16) double s_boys[];
  load_boys_for<C>(s_boys, a.boys_tab);
  const int lane = threadIdx.x & 31;
  PrimRec* sbra = reinterpret_cast<PrimRec*>(s_boys + BoysStage<C>::nsl * kBoysRows * kBoysCols) +
                  (threadIdx.x >> 5) * kSmemBraMax;
  double2* sbw = reinterpret_cast<double2*>(reinterpret_cast<PrimRec*>(s_boys + BoysStage<C>::nsl * kBoysRows *
                                                                                    kBoysCols) +
                                            (NT / 32) * kSmemBraMax) +
                 (threadIdx.x >> 5) * kSmemBraMax;
  int staged = -1;
  (void)sbra;
  (void)sbw;
  (void)staged;
  const size_t n = static_cast<size_t>(a.N);
  const long long warps = static_cast<long long>(gridDim.x) * (blockDim.x >> 5);
  auto process = [&](const WorkItem& it) {
    const int nq = it.r0nq >> 24;
    const bool active = lane < nq;
    int q = (it.r0nq & 0xffffff) + (active ? lane : 0);
    int x = it.bra0, c = it.cntp;
    for (int cn = __ldg(a.cnt + c); q >= cn; cn = __ldg(a.cnt + c)) {
      q -= cn;
      ++x;
      ++c;
    }
    const int y = it.yfirst + q;
    const UnitMeta bu = a.um[x];
    const UnitMeta ku = a.um[y];
    typename C::Acc acc[MB][MK];
    const PrimRec* brap = a.prims + bu.prim_off;
    const double2* bwp = a.uw + bu.prim_off;
    if constexpr (STYLE == kLoopSmemBra) {  // stage the warp's bra unit once while it stays
      const int x0 = __shfl_sync(0xffffffffu, x, 0);
      if (__all_sync(0xffffffffu, x == x0) && bu.K <= kSmemBraMax) {
        if (x0 != staged) {
          __syncwarp();
          const double2* src = reinterpret_cast<const double2*>(a.prims + bu.prim_off);
          double2* dst = reinterpret_cast<double2*>(sbra);
          for (int t = lane; t < bu.K * 5; t += 32) dst[t] = __ldg(src + t);
          for (int t = lane; t < bu.K; t += 32) sbw[t] = __ldg(a.uw + bu.prim_off + t);
          __syncwarp();
          staged = x0;
        }
        brap = sbra;
        bwp = sbw;
      }
    }
    fam_drive<C, MB, MK, STYLE>(brap, bwp, bu.K, a.ukprims + ku.ksoa, a.ukw + ku.ksoa, active ? ku.K : 0,
                                ku.kstride, s_boys, acc);
    constexpr int nmb = MB, nmk = MK;
    const int xkey = active ? x : -1;
    const int xnext = __shfl_down_sync(0xffffffffu, xkey, 1);
    const bool tail = active && (lane == 31 || xnext != xkey);
#pragma unroll
    for (int mb = 0; mb < nmb; ++mb) {
      const int px = mb == 0 ? bu.m0 : bu.m1;
      PairMeta bm;
      ld_meta_late(a.pm + px, bm);
      const double qb = __ldg(a.Qp + px);
      // J_ab of bra member mb: sum over ket members, then a segmented warp
      // reduction over the lanes sharing the bra unit (one atomic per segment)
      double jab[C::NA * C::NB];
#pragma unroll
      for (int e = 0; e < C::NA * C::NB; ++e) jab[e] = 0.0;
#pragma unroll
      for (int nk = 0; nk < nmk; ++nk) {
        const int py = nk == 0 ? ku.m0 : ku.m1;
        const bool keep = active && !(x == y && mb > nk) && (a.tau <= 0.0 || qb * __ldg(a.Qp + py) >= a.tau);
        if (!__any_sync(0xffffffffu, keep)) continue;
        PairMeta km;
        ld_meta_late(a.pm + py, km);
        double v[C::NV];
        C::finish(acc[mb][nk], bu.ABx, bu.ABy, bu.ABz, ku.ABx, ku.ABy, ku.ABz, v);
        const double deg =
            (bm.sha != bm.shb ? 2.0 : 1.0) * (km.sha != km.shb ? 2.0 : 1.0) * (px != py ? 2.0 : 1.0);
        const double wj = keep ? 0.5 * deg : 0.0, wk = keep ? 0.25 * deg : 0.0;
        const double* Dab = a.D + bm.bfa * n + bm.bfb;
        const double* Dcd = a.D + km.bfa * n + km.bfb;
        const double* Dac = a.D + bm.bfa * n + km.bfa;
        const double* Dad = a.D + bm.bfa * n + km.bfb;
        const double* Dbc = a.D + bm.bfb * n + km.bfa;
        const double* Dbd = a.D + bm.bfb * n + km.bfb;
#pragma unroll
        for (int ia = 0; ia < C::NA; ++ia)
#pragma unroll
          for (int ib = 0; ib < C::NB; ++ib) {
            double s = 0.0;
#pragma unroll
            for (int ic = 0; ic < C::NC; ++ic)
#pragma unroll
              for (int id = 0; id < C::ND; ++id)
                s = fma(v[((ia * C::NB + ib) * C::NC + ic) * C::ND + id], keep ? __ldg(Dcd + ic * n + id) : 0.0, s);
            jab[ia * C::NB + ib] = fma(s, wj, jab[ia * C::NB + ib]);
          }
        if (keep) {
#pragma unroll
          for (int ic = 0; ic < C::NC; ++ic)
#pragma unroll
            for (int id = 0; id < C::ND; ++id) {
              double s = 0.0;
#pragma unroll
              for (int ia = 0; ia < C::NA; ++ia)
#pragma unroll
                for (int ib = 0; ib < C::NB; ++ib)
                  s = fma(v[((ia * C::NB + ib) * C::NC + ic) * C::ND + id], __ldg(Dab + ia * n + ib), s);
              red_add(a.J + (km.bfa + ic) * n + km.bfb + id, s * wj, a.det);
            }
#pragma unroll
          for (int ia = 0; ia < C::NA; ++ia)
#pragma unroll
            for (int ic = 0; ic < C::NC; ++ic) {
              double s = 0.0;
#pragma unroll
              for (int ib = 0; ib < C::NB; ++ib)
#pragma unroll
                for (int id = 0; id < C::ND; ++id)
                  s = fma(v[((ia * C::NB + ib) * C::NC + ic) * C::ND + id], __ldg(Dbd + ib * n + id), s);
              red_add(a.K + (bm.bfa + ia) * n + km.bfa + ic, s * wk, a.det);
            }
#pragma unroll
          for (int ib = 0; ib < C::NB; ++ib)
#pragma unroll
            for (int id = 0; id < C::ND; ++id) {
              double s = 0.0;
#pragma unroll
              for (int ia = 0; ia < C::NA; ++ia)
#pragma unroll
                for (int ic = 0; ic < C::NC; ++ic)
                  s = fma(v[((ia * C::NB + ib) * C::NC + ic) * C::ND + id], __ldg(Dac + ia * n + ic), s);
              red_add(a.K + (bm.bfb + ib) * n + km.bfb + id, s * wk, a.det);
            }
#pragma unroll
          for (int ia = 0; ia < C::NA; ++ia)
#pragma unroll
            for (int id = 0; id < C::ND; ++id) {
              double s = 0.0;
#pragma unroll
              for (int ib = 0; ib < C::NB; ++ib)
#pragma unroll
                for (int ic = 0; ic < C::NC; ++ic)
                  s = fma(v[((ia * C::NB + ib) * C::NC + ic) * C::ND + id], __ldg(Dbc + ib * n + ic), s);
              red_add(a.K + (bm.bfa + ia) * n + km.bfb + id, s * wk, a.det);
            }
#pragma unroll
          for (int ib = 0; ib < C::NB; ++ib)
#pragma unroll
            for (int ic = 0; ic < C::NC; ++ic) {
              double s = 0.0;
#pragma unroll
              for (int ia = 0; ia < C::NA; ++ia)
#pragma unroll
                for (int id = 0; id < C::ND; ++id)
                  s = fma(v[((ia * C::NB + ib) * C::NC + ic) * C::ND + id], __ldg(Dad + ia * n + id), s);
              red_add(a.K + (bm.bfb + ib) * n + km.bfa + ic, s * wk, a.det);
            }
        }
      }
#pragma unroll
      for (int ia = 0; ia < C::NA; ++ia)
#pragma unroll
        for (int ib = 0; ib < C::NB; ++ib) {
          const double s = seg_sum(jab[ia * C::NB + ib], xkey, lane);
          if (tail && s != 0.0) red_add(a.J + (bm.bfa + ia) * n + bm.bfb + ib, s, a.det);
        }
    }
  };
  for_warp_items(a.items, i0, i1, a.gran, static_cast<long long>(blockIdx.x) * (blockDim.x >> 5) + (threadIdx.x >> 5),
                 warps, process);
}

template <class C, int MB, int MK, int MINB, int STYLE, int NT>
void launch_fam_seg(const LaunchArgs& a, long long i0, long long i1) {
  if (i1 <= i0) return;
  const size_t smem =
      BoysStage<C>::bytes + (STYLE == kLoopSmemBra ? (sizeof(PrimRec) + sizeof(double2)) * kSmemBraMax * (NT / 32) : 0);
  const LaunchSetup ls =
      launch_setup(reinterpret_cast<const void*>(jk_fam_kernel<C, MB, MK, MINB, STYLE, NT>), NT, smem, true);
  if (!ls.bps) return;  // CUDA error pending for the caller's check
  const long long g = a.gran > 1 ? a.gran : 1;
  const long long want = ((i1 - i0 + g - 1) / g + (NT / 32) - 1) / (NT / 32);
  const long long cap = static_cast<long long>(ls.bps) * ls.sms;
  const int grid = static_cast<int>(want < cap ? want : cap);
  jk_fam_kernel<C, MB, MK, MINB, STYLE, NT><<<grid, NT, smem, a.stream>>>(a, i0, i1);
}

// NT11: CTA size of the (1,1) segment (fewest live accumulators: it fits
// the tighter register budget of larger CTAs).
template <class C, int MINB, int STYLE, int NT, int NT11 = NT>
void launch_fam(const LaunchArgs& a) {
  if (a.mode != 0) {  // Schwarz / raw quartets are per pair: the lane kernel serves them
    launch_class<C, 2, kLoopPrefetch>(a);
    return;
  }
  // segments (1,1) (1,2) (2,1) (2,2) of the class's items
  launch_fam_seg<C, 1, 1, MINB, STYLE, NT11>(a, a.seg[0], a.seg[1]);
  launch_fam_seg<C, 1, 2, MINB, STYLE, NT>(a, a.seg[1], a.seg[2]);
  launch_fam_seg<C, 2, 1, MINB, STYLE, NT>(a, a.seg[2], a.seg[3]);
  launch_fam_seg<C, 2, 2, MINB, STYLE, NT>(a, a.seg[3], a.seg[4]);
}

}  // namespace eritile_b200
