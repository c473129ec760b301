// CTA-cooperative ERI + J/K kernel for high-L classes (Deconstruction).
//
// One CTA evaluates one contracted quartet at a time from the level-scheduled
// plan tables of compiler/coop.py: per primitive quartet warp 0 binds the
// geometry and Boys values (boys.hpp:23-44 semantics,
// boys_eval) into a small coefficient table, then all threads sweep the
// primitive-segment levels (vertical recurrences), fold the boundary into the
// contracted accumulators (compiler.hpp:143), and after the primitive loop
// sweep the horizontal levels (compiler.hpp:144). All values live in shared
// memory; one barrier per level. Digestion then spreads the six J/K blocks
// of SPEC.md:350 over the threads, one FP64 atomic per output element.
#pragma once
#include "jk_kernels.cuh"

namespace eritile_b200 {

// base coefficient ids (compiler/coop.py)
constexpr int kB_PA = 1, kB_QC = 4, kB_WP = 7, kB_WQ = 10, kB_I2P = 13, kB_I2Q = 14, kB_I2PQ = 15,
              kB_ITP = 16, kB_ITQ = 17, kB_AB = 18, kB_CD = 21, kB_PF = 24;
constexpr int kCoopMaxCombo = 64;
constexpr int kCoopBase = 48;  // >= kB_PF + M + 1 for M <= 16

struct CoopTables {
  const unsigned* lo;
  const int* lo_lvl;
  int nlo_lvl;
  const unsigned* bd;
  int nb;
  const unsigned* up;
  const int* up_lvl;
  int nup_lvl;
  const unsigned* combo;
  int ncombo;
  const unsigned short* tgt;
  int nslots;
  int tgt0;  // outputs occupy slots [tgt0, tgt0 + NV) in kernel order (final copy level)
};

// C::BOYS_SMEM: stage the class's Boys slice in shared memory (51 KB) or read
// it through L1 from global memory (classes whose value slots need the room).
template <class C>
struct CoopSmem {
  static constexpr size_t boys = C::BOYS_SMEM ? sizeof(double) * kBoysRows * kBoysCols : 0;
  static size_t bytes(int nslots) {
    return boys + sizeof(double) * (kCoopBase + kCoopMaxCombo + nslots) +
           ((sizeof(unsigned short) * C::NV + 15) & ~size_t(15));
  }
};

// One level of the plan: ops [o0, o1) dealt to this thread with stride `step`.
// The next op's table entry is loaded while the current one is evaluated (the
// entry loads were the top long-scoreboard stall of the interpreter, ncu
// profiles/r02_ncu_coop.txt). lo ops: 2 uint4 per op (up to 5 terms);
// up ops: 1 uint4 (up to 3 terms).
template <bool LO>
__device__ __forceinline__ void coop_level(const uint4* __restrict__ tab, int o0, int o1, int step,
                                           const double* cf, double* val) {
  int o = o0;
  if (o >= o1) return;
  uint4 h = __ldg(tab + (LO ? 2 * o : o));
  uint4 g = LO ? __ldg(tab + 2 * o + 1) : make_uint4(0, 0, 0, 0);
  while (true) {
    const int on = o + step;
    uint4 hn = h, gn = g;
    if (on < o1) {
      hn = __ldg(tab + (LO ? 2 * on : on));
      if (LO) gn = __ldg(tab + 2 * on + 1);
    }
    const int nt = h.x >> 16;
    double acc = cf[h.y >> 16] * val[h.y & 0xffff];
    if (nt > 1) acc = fma(cf[h.z >> 16], val[h.z & 0xffff], acc);
    if (nt > 2) acc = fma(cf[h.w >> 16], val[h.w & 0xffff], acc);
    if (LO && nt > 3) {
      acc = fma(cf[g.x >> 16], val[g.x & 0xffff], acc);
      if (nt > 4) acc = fma(cf[g.y >> 16], val[g.y & 0xffff], acc);
    }
    val[h.x & 0xffff] = acc;
    if (on >= o1) break;
    o = on;
    h = hn;
    g = gn;
  }
}

// Evaluate one contracted quartet; outputs end in val[tgt[k]], kernel order.
template <class C>
__device__ __forceinline__ void coop_eval(const CoopTables& tb, const PairMeta& bm, const PairMeta& km,
                                          const PrimRec* __restrict__ prims, const double* s_boys,
                                          double* coefb, double* cf, double* val) {
  const int tid = threadIdx.x;
  for (int s = tid; s < tb.nb; s += C::NT) val[1 + s] = 0.0;
  const PrimRec* bra = prims + bm.prim_off;
  const PrimRec* ket = prims + km.prim_off;
  const int np = bm.K * km.K;
  for (int pq = 0; pq < np; ++pq) {
    if (tid < 32) {
      const PrimRec bp = load_prim<true>(bra + pq / km.K);
      const PrimRec kp = load_prim<true>(ket + pq % km.K);
      const double s = bp.p + kp.p;
      const double rs = rsqrt_pos(s);
      const double inv = rs * rs;
      const double PQx = bp.Px - kp.Px, PQy = bp.Py - kp.Py, PQz = bp.Pz - kp.Pz;
      const double pinv = bp.p * inv, qinv = kp.p * inv;
      const double rho = bp.p * qinv;
      const double T = rho * fma(PQx, PQx, fma(PQy, PQy, PQz * PQz));
      const double pref = bp.U * kp.U * rs;
      double F[C::M + 1];
      boys_eval<C::M>(T, s_boys, F);
      const int lane = tid;
      if (lane == 0) {
        coefb[0] = 1.0;
        coefb[kB_PA] = bp.PAx; coefb[kB_PA + 1] = bp.PAy; coefb[kB_PA + 2] = bp.PAz;
        coefb[kB_QC] = kp.PAx; coefb[kB_QC + 1] = kp.PAy; coefb[kB_QC + 2] = kp.PAz;
        coefb[kB_WP] = -qinv * PQx; coefb[kB_WP + 1] = -qinv * PQy; coefb[kB_WP + 2] = -qinv * PQz;
        coefb[kB_WQ] = pinv * PQx; coefb[kB_WQ + 1] = pinv * PQy; coefb[kB_WQ + 2] = pinv * PQz;
      } else if (lane == 1) {
        coefb[kB_I2P] = bp.i2p;
        coefb[kB_I2Q] = kp.i2p;
        coefb[kB_I2PQ] = 0.5 * inv;
        coefb[kB_ITP] = bp.i2p * qinv;
        coefb[kB_ITQ] = kp.i2p * pinv;
        coefb[kB_AB] = bm.ABx; coefb[kB_AB + 1] = bm.ABy; coefb[kB_AB + 2] = bm.ABz;
        coefb[kB_CD] = km.ABx; coefb[kB_CD + 1] = km.ABy; coefb[kB_CD + 2] = km.ABz;
      } else if (lane == 2) {
#pragma unroll
        for (int m = 0; m <= C::M; ++m) coefb[kB_PF + m] = pref * F[m];
      }
      __syncwarp();
      for (int k = lane; k < tb.ncombo; k += 32) {
        const unsigned w = __ldg(tb.combo + k);
        cf[k] = static_cast<double>(static_cast<int>(w >> 8) - 128) * coefb[w & 0xff];
      }
    }
    __syncthreads();
    // primitive segment, level by level
    for (int L = 0; L < tb.nlo_lvl; ++L) {
      coop_level<true>(reinterpret_cast<const uint4*>(tb.lo), __ldg(tb.lo_lvl + L) + tid, __ldg(tb.lo_lvl + L + 1),
                       C::NT, cf, val);
      __syncthreads();
    }
    for (int k = tid; k < tb.nb; k += C::NT) {
      const unsigned w = __ldg(tb.bd + k);
      val[w >> 16] += val[w & 0xffff];
    }
    __syncthreads();
  }
  // contracted horizontal segment
  for (int L = 0; L < tb.nup_lvl; ++L) {
    coop_level<false>(reinterpret_cast<const uint4*>(tb.up), __ldg(tb.up_lvl + L) + tid, __ldg(tb.up_lvl + L + 1),
                      C::NT, cf, val);
    __syncthreads();
  }
}

template <class C>
__global__ void __launch_bounds__(C::NT) coop_kernel(CoopTables tb, LaunchArgs a) {
  extern __shared__ __align__(16) double smem[];
  const double* s_boys = C::BOYS_SMEM ? smem : a.boys_tab + static_cast<size_t>(C::M) * kBoysRows * kBoysCols;
  double* coefb = smem + (C::BOYS_SMEM ? kBoysRows * kBoysCols : 0);
  double* cf = coefb + kCoopBase;
  double* val = cf + kCoopMaxCombo;
  unsigned short* tgt = reinterpret_cast<unsigned short*>(val + tb.nslots);
  if (C::BOYS_SMEM) load_boys_slice(smem, a.boys_tab, C::M);
  for (int k = threadIdx.x; k < C::NV; k += C::NT) tgt[k] = __ldg(tb.tgt + k);
  if (threadIdx.x == 0) val[0] = 1.0;
  __syncthreads();
  const int tid = threadIdx.x;

  if (a.mode == 1 || a.mode == 2) {  // Schwarz diagonal / raw quartets
    const long long n = a.mode == 1 ? a.npair_list : a.nq;
    for (long long i = blockIdx.x; i < n; i += gridDim.x) {
      const int xb = a.mode == 1 ? a.pair_list[i] : a.qpairs[2 * i];
      const int xk = a.mode == 1 ? xb : a.qpairs[2 * i + 1];
      const PairMeta bm = a.pm[xb], km = a.pm[xk];
      coop_eval<C>(tb, bm, km, a.prims, s_boys, coefb, cf, val);
      if (a.mode == 2) {
        for (int k = tid; k < C::NV; k += C::NT) a.qout[i * C::NV + k] = val[tgt[k]];
      } else if (tid < 32) {
        double mx = 0.0;
        for (int ab = tid; ab < C::NA * C::NB; ab += 32) {
          const int ia = ab / C::NB, ib = ab % C::NB;
          const double s = comp_scale(C::LA, ia) * comp_scale(C::LB, ib);
          mx = fmax(mx, fabs(val[tgt[(ab * C::NC + ia) * C::ND + ib]]) * (s * s));
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        if (tid == 0) a.Qout[xb] = sqrt(mx);
      }
      __syncthreads();
    }
    return;
  }

  const size_t n = static_cast<size_t>(a.N);
  constexpr int NA = C::NA, NB = C::NB, NC = C::NC, ND = C::ND;
  constexpr int O1 = NA * NB, O2 = O1 + NC * ND, O3 = O2 + NA * NC, O4 = O3 + NB * ND, O5 = O4 + NA * ND,
                O6 = O5 + NB * NC;
  for (long long w = blockIdx.x; w < a.nitems; w += gridDim.x) {
    const WorkItem it = a.items[w];
    const int nq = it.r0nq >> 24;
    int q = it.r0nq & 0xffffff, x = it.bra0, c = it.cntp;
    for (int l = 0; l < nq; ++l, ++q) {
      for (int cn = __ldg(a.cnt + c); q >= cn; cn = __ldg(a.cnt + c)) {
        q -= cn;
        ++x;
        ++c;
      }
      const int y = it.yfirst + q;
      const PairMeta bm = a.pm[x], km = a.pm[y];
      coop_eval<C>(tb, bm, km, a.prims, s_boys, coefb, cf, val);
      const double deg = (bm.sha != bm.shb ? 2.0 : 1.0) * (km.sha != km.shb ? 2.0 : 1.0) * (x != y ? 2.0 : 1.0);
      const double wj = 0.5 * deg, wk = 0.25 * deg;
      for (int o = tid; o < O6; o += C::NT) {
        double s = 0.0;
        double* dst;
        if (o < O1) {  // J_ab += sum_cd v D_cd
          const int ia = o / NB, ib = o % NB;
          for (int ic = 0; ic < NC; ++ic)
            for (int id = 0; id < ND; ++id)
              s = fma(val[tgt[((ia * NB + ib) * NC + ic) * ND + id]], __ldg(a.D + (km.bfa + ic) * n + km.bfb + id), s);
          dst = a.J + (bm.bfa + ia) * n + bm.bfb + ib;
          s *= wj;
        } else if (o < O2) {  // J_cd += sum_ab v D_ab
          const int ic = (o - O1) / ND, id = (o - O1) % ND;
          for (int ia = 0; ia < NA; ++ia)
            for (int ib = 0; ib < NB; ++ib)
              s = fma(val[tgt[((ia * NB + ib) * NC + ic) * ND + id]], __ldg(a.D + (bm.bfa + ia) * n + bm.bfb + ib), s);
          dst = a.J + (km.bfa + ic) * n + km.bfb + id;
          s *= wj;
        } else if (o < O3) {  // K_ac += sum_bd v D_bd
          const int ia = (o - O2) / NC, ic = (o - O2) % NC;
          for (int ib = 0; ib < NB; ++ib)
            for (int id = 0; id < ND; ++id)
              s = fma(val[tgt[((ia * NB + ib) * NC + ic) * ND + id]], __ldg(a.D + (bm.bfb + ib) * n + km.bfb + id), s);
          dst = a.K + (bm.bfa + ia) * n + km.bfa + ic;
          s *= wk;
        } else if (o < O4) {  // K_bd += sum_ac v D_ac
          const int ib = (o - O3) / ND, id = (o - O3) % ND;
          for (int ia = 0; ia < NA; ++ia)
            for (int ic = 0; ic < NC; ++ic)
              s = fma(val[tgt[((ia * NB + ib) * NC + ic) * ND + id]], __ldg(a.D + (bm.bfa + ia) * n + km.bfa + ic), s);
          dst = a.K + (bm.bfb + ib) * n + km.bfb + id;
          s *= wk;
        } else if (o < O5) {  // K_ad += sum_bc v D_bc
          const int ia = (o - O4) / ND, id = (o - O4) % ND;
          for (int ib = 0; ib < NB; ++ib)
            for (int ic = 0; ic < NC; ++ic)
              s = fma(val[tgt[((ia * NB + ib) * NC + ic) * ND + id]], __ldg(a.D + (bm.bfb + ib) * n + km.bfa + ic), s);
          dst = a.K + (bm.bfa + ia) * n + km.bfb + id;
          s *= wk;
        } else {  // K_bc += sum_ad v D_ad
          const int ib = (o - O5) / NC, ic = (o - O5) % NC;
          for (int ia = 0; ia < NA; ++ia)
            for (int id = 0; id < ND; ++id)
              s = fma(val[tgt[((ia * NB + ib) * NC + ic) * ND + id]], __ldg(a.D + (bm.bfa + ia) * n + km.bfb + id), s);
          dst = a.K + (bm.bfb + ib) * n + km.bfa + ic;
          s *= wk;
        }
        red_add(dst, s, a.det);
      }
      __syncthreads();
    }
  }
}

template <class C>
void launch_coop(const CoopTables& tb, const LaunchArgs& a) {
  const size_t smem = CoopSmem<C>::bytes(tb.nslots);
  const long long n = a.mode == 0 ? a.nitems : (a.mode == 1 ? a.npair_list : a.nq);
  if (n <= 0) return;
  const LaunchSetup ls = launch_setup(reinterpret_cast<const void*>(coop_kernel<C>), C::NT, smem, false);
  if (!ls.bps) return;  // CUDA error pending for the caller's check
  const long long cap = static_cast<long long>(ls.bps) * ls.sms;
  const int grid = a.grid > 0 ? a.grid : static_cast<int>(n < cap ? n : cap);
  coop_kernel<C><<<grid, C::NT, smem, a.stream>>>(tb, a);
}


// ---------------------------------------------------------------------------
// Warp-cooperative form of the same tables: each warp owns one contracted
// quartet at a time in its own shared-memory slot region, so a level needs
// only __syncwarp() and a CTA holds kCoopWarps independent quartets (no CTA
// barriers). Suited to quartets with few primitive quartets (d/f shells are
// contracted over one primitive in cc-pVXZ), where the CTA form is barrier-
// and binding-bound. The Boys slice is read through L1 from global memory.
constexpr int kCoopWarps = 4;

template <class C>
__device__ __forceinline__ void coopw_eval(const CoopTables& tb, const PairMeta& bm, const PairMeta& km,
                                           const PrimRec* __restrict__ prims, const double* __restrict__ btab,
                                           const double* __restrict__ btab0, double* coefb, double* cf,
                                           double* val, int lane) {
  for (int s = lane; s < tb.nb; s += 32) val[1 + s] = 0.0;
  const PrimRec* bra = prims + bm.prim_off;
  const PrimRec* ket = prims + km.prim_off;
  const int np = bm.K * km.K;
  for (int pq = 0; pq < np; ++pq) {
    __syncwarp();
    {
      const PrimRec bp = load_prim<true>(bra + pq / km.K);
      const PrimRec kp = load_prim<true>(ket + pq % km.K);
      const double s = bp.p + kp.p;
      const double rs = rsqrt_pos(s);
      const double inv = rs * rs;
      const double PQx = bp.Px - kp.Px, PQy = bp.Py - kp.Py, PQz = bp.Pz - kp.Pz;
      const double pinv = bp.p * inv, qinv = kp.p * inv;
      const double rho = bp.p * qinv;
      const double T = rho * fma(PQx, PQx, fma(PQy, PQy, PQz * PQz));
      const double pref = bp.U * kp.U * rs;
      if (lane == 0) {
        coefb[0] = 1.0;
        coefb[kB_PA] = bp.PAx; coefb[kB_PA + 1] = bp.PAy; coefb[kB_PA + 2] = bp.PAz;
        coefb[kB_QC] = kp.PAx; coefb[kB_QC + 1] = kp.PAy; coefb[kB_QC + 2] = kp.PAz;
        coefb[kB_WP] = -qinv * PQx; coefb[kB_WP + 1] = -qinv * PQy; coefb[kB_WP + 2] = -qinv * PQz;
        coefb[kB_WQ] = pinv * PQx; coefb[kB_WQ + 1] = pinv * PQy; coefb[kB_WQ + 2] = pinv * PQz;
      } else if (lane == 1) {
        coefb[kB_I2P] = bp.i2p;
        coefb[kB_I2Q] = kp.i2p;
        coefb[kB_I2PQ] = 0.5 * inv;
        coefb[kB_ITP] = bp.i2p * qinv;
        coefb[kB_ITQ] = kp.i2p * pinv;
        coefb[kB_AB] = bm.ABx; coefb[kB_AB + 1] = bm.ABy; coefb[kB_AB + 2] = bm.ABz;
        coefb[kB_CD] = km.ABx; coefb[kB_CD + 1] = km.ABy; coefb[kB_CD + 2] = km.ABz;
      }
      if (T < kBoysTmax) {
        // warp-uniform (one primitive quartet per warp): lane 2 + m evaluates
        // F_m by its own 8-term Taylor series from table slice m (global,
        // L1-resident), so the M+1 orders are computed in parallel
        const int m = lane - 2;
        if (m >= 0 && m <= C::M) {
          const double sh = fma(T, 16.0, kBoysK[6]);
          const int i = __double2loint(sh);
          const double md = fma(sh - kBoysK[6], 0.0625, -T);
          const double m2 = md * md;
          const double2* r = reinterpret_cast<const double2*>(btab0 + (static_cast<size_t>(m) * kBoysRows + i) * kBoysCols);
          const double2 c01 = __ldg(r), c23 = __ldg(r + 1), c45 = __ldg(r + 2), c67 = __ldg(r + 3);
          const double q0 = fma(fma(c23.y, md, c23.x), m2, fma(c01.y, md, c01.x));
          const double q1 = fma(fma(c67.y, md, c67.x), m2, fma(c45.y, md, c45.x));
          coefb[kB_PF + m] = pref * fma(q1, m2 * m2, q0);
        }
      } else if (lane == 2) {
        double F[C::M + 1];
        boys_eval<C::M>(T, btab, F);
#pragma unroll
        for (int m = 0; m <= C::M; ++m) coefb[kB_PF + m] = pref * F[m];
      }
    }
    __syncwarp();
    for (int k = lane; k < tb.ncombo; k += 32) {
      const unsigned w = __ldg(tb.combo + k);
      cf[k] = static_cast<double>(static_cast<int>(w >> 8) - 128) * coefb[w & 0xff];
    }
    __syncwarp();
    for (int L = 0; L < tb.nlo_lvl; ++L) {
      coop_level<true>(reinterpret_cast<const uint4*>(tb.lo), __ldg(tb.lo_lvl + L) + lane, __ldg(tb.lo_lvl + L + 1),
                       32, cf, val);
      __syncwarp();
    }
    for (int k = lane; k < tb.nb; k += 32) {
      const unsigned w = __ldg(tb.bd + k);
      val[w >> 16] += val[w & 0xffff];
    }
  }
  __syncwarp();
  // coefb[kB_AB..] / [kB_CD..] are set per primitive quartet; the
  // horizontal combos only read UNIT, AB and CD, which are quartet constants
  for (int L = 0; L < tb.nup_lvl; ++L) {
    coop_level<false>(reinterpret_cast<const uint4*>(tb.up), __ldg(tb.up_lvl + L) + lane, __ldg(tb.up_lvl + L + 1),
                      32, cf, val);
    __syncwarp();
  }
}

template <class C>
__global__ void __launch_bounds__(32 * kCoopWarps) coopw_kernel(CoopTables tb, LaunchArgs a) {
  extern __shared__ __align__(16) double smem[];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  constexpr int DBLK = C::NA * C::NB + C::NC * C::ND + C::NA * C::NC + C::NB * C::ND + C::NA * C::ND +
                       C::NB * C::NC;
  const int region = kCoopBase + kCoopMaxCombo + tb.nslots + DBLK;
  double* coefb = smem + static_cast<size_t>(wid) * region;
  double* cf = coefb + kCoopBase;
  double* val = cf + kCoopMaxCombo;
  const double* btab = a.boys_tab + static_cast<size_t>(C::M) * kBoysRows * kBoysCols;
  if (lane == 0) val[0] = 1.0;
  __syncwarp();
  const long long gw = static_cast<long long>(blockIdx.x) * kCoopWarps + wid;
  const long long nw = static_cast<long long>(gridDim.x) * kCoopWarps;
  const size_t n = static_cast<size_t>(a.N);
  constexpr int NA = C::NA, NB = C::NB, NC = C::NC, ND = C::ND;
  constexpr int O1 = NA * NB, O2 = O1 + NC * ND, O3 = O2 + NA * NC, O4 = O3 + NB * ND, O5 = O4 + NA * ND,
                O6 = O5 + NB * NC;
  if (a.mode == 1 || a.mode == 2) {
    const long long cnt = a.mode == 1 ? a.npair_list : a.nq;
    for (long long i = gw; i < cnt; i += nw) {
      const int xb = a.mode == 1 ? a.pair_list[i] : a.qpairs[2 * i];
      const int xk = a.mode == 1 ? xb : a.qpairs[2 * i + 1];
      const PairMeta bm = a.pm[xb], km = a.pm[xk];
      coopw_eval<C>(tb, bm, km, a.prims, btab, a.boys_tab, coefb, cf, val, lane);
      if (a.mode == 2) {
        for (int k = lane; k < C::NV; k += 32) a.qout[i * C::NV + k] = val[__ldg(tb.tgt + k)];
      } else {
        double mx = 0.0;
        for (int ab = lane; ab < NA * NB; ab += 32) {
          const int ia = ab / NB, ib = ab % NB;
          const double sc = comp_scale(C::LA, ia) * comp_scale(C::LB, ib);
          mx = fmax(mx, fabs(val[__ldg(tb.tgt + (ab * NC + ia) * ND + ib)]) * (sc * sc));
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        if (lane == 0) a.Qout[xb] = sqrt(mx);
      }
      __syncwarp();
    }
    return;
  }
  for (long long w = gw; w < a.nitems; w += nw) {
    const WorkItem it = a.items[w];
    const int nq = it.r0nq >> 24;
    int q = it.r0nq & 0xffffff, x = it.bra0, c = it.cntp;
    for (int l = 0; l < nq; ++l, ++q) {
      for (int cn = __ldg(a.cnt + c); q >= cn; cn = __ldg(a.cnt + c)) {
        q -= cn;
        ++x;
        ++c;
      }
      const int y = it.yfirst + q;
      const PairMeta bm = a.pm[x], km = a.pm[y];
      coopw_eval<C>(tb, bm, km, a.prims, btab, a.boys_tab, coefb, cf, val, lane);
      const double deg = (bm.sha != bm.shb ? 2.0 : 1.0) * (km.sha != km.shb ? 2.0 : 1.0) * (x != y ? 2.0 : 1.0);
      const double wj = 0.5 * deg, wk = 0.25 * deg;
      // the six density blocks of this quartet, staged once per quartet:
      // [Dcd | Dab | Dbd | Dac | Dbc | Dad] feed [J_ab | J_cd | K_ac | K_bd | K_ad | K_bc]
      double* dsm = val + tb.nslots;
      constexpr int E1 = NC * ND, E2 = E1 + NA * NB, E3 = E2 + NB * ND, E4 = E3 + NA * NC, E5 = E4 + NB * NC,
                    E6 = E5 + NA * ND;
      for (int o = lane; o < E6; o += 32) {
        size_t r, cidx;
        if (o < E1) { r = km.bfa + o / ND; cidx = km.bfb + o % ND; }                     // Dcd
        else if (o < E2) { r = bm.bfa + (o - E1) / NB; cidx = bm.bfb + (o - E1) % NB; }  // Dab
        else if (o < E3) { r = bm.bfb + (o - E2) / ND; cidx = km.bfb + (o - E2) % ND; }  // Dbd
        else if (o < E4) { r = bm.bfa + (o - E3) / NC; cidx = km.bfa + (o - E3) % NC; }  // Dac
        else if (o < E5) { r = bm.bfb + (o - E4) / NC; cidx = km.bfa + (o - E4) % NC; }  // Dbc
        else { r = bm.bfa + (o - E5) / ND; cidx = km.bfb + (o - E5) % ND; }              // Dad
        dsm[o] = __ldg(a.D + r * n + cidx);
      }
      __syncwarp();
      const double* Dcd = dsm;             // NC x ND
      const double* Dab = dsm + E1;        // NA x NB
      const double* Dbd = dsm + E2;        // NB x ND
      const double* Dac = dsm + E3;        // NA x NC
      const double* Dbc = dsm + E4;        // NB x NC
      const double* Dad = dsm + E5;        // NA x ND
      for (int o = lane; o < O6; o += 32) {
        double s = 0.0;
        double* dst;
        if (o < O1) {
          const int ia = o / NB, ib = o % NB;
          for (int ic = 0; ic < NC; ++ic)
            for (int id = 0; id < ND; ++id) s = fma(val[__ldg(tb.tgt + ((ia * NB + ib) * NC + ic) * ND + id)], Dcd[ic * ND + id], s);
          dst = a.J + (bm.bfa + ia) * n + bm.bfb + ib;
          s *= wj;
        } else if (o < O2) {
          const int ic = (o - O1) / ND, id = (o - O1) % ND;
          for (int ia = 0; ia < NA; ++ia)
            for (int ib = 0; ib < NB; ++ib) s = fma(val[__ldg(tb.tgt + ((ia * NB + ib) * NC + ic) * ND + id)], Dab[ia * NB + ib], s);
          dst = a.J + (km.bfa + ic) * n + km.bfb + id;
          s *= wj;
        } else if (o < O3) {
          const int ia = (o - O2) / NC, ic = (o - O2) % NC;
          for (int ib = 0; ib < NB; ++ib)
            for (int id = 0; id < ND; ++id) s = fma(val[__ldg(tb.tgt + ((ia * NB + ib) * NC + ic) * ND + id)], Dbd[ib * ND + id], s);
          dst = a.K + (bm.bfa + ia) * n + km.bfa + ic;
          s *= wk;
        } else if (o < O4) {
          const int ib = (o - O3) / ND, id = (o - O3) % ND;
          for (int ia = 0; ia < NA; ++ia)
            for (int ic = 0; ic < NC; ++ic) s = fma(val[__ldg(tb.tgt + ((ia * NB + ib) * NC + ic) * ND + id)], Dac[ia * NC + ic], s);
          dst = a.K + (bm.bfb + ib) * n + km.bfb + id;
          s *= wk;
        } else if (o < O5) {
          const int ia = (o - O4) / ND, id = (o - O4) % ND;
          for (int ib = 0; ib < NB; ++ib)
            for (int ic = 0; ic < NC; ++ic) s = fma(val[__ldg(tb.tgt + ((ia * NB + ib) * NC + ic) * ND + id)], Dbc[ib * NC + ic], s);
          dst = a.K + (bm.bfa + ia) * n + km.bfb + id;
          s *= wk;
        } else {
          const int ib = (o - O5) / NC, ic = (o - O5) % NC;
          for (int ia = 0; ia < NA; ++ia)
            for (int id = 0; id < ND; ++id) s = fma(val[__ldg(tb.tgt + ((ia * NB + ib) * NC + ic) * ND + id)], Dad[ia * ND + id], s);
          dst = a.K + (bm.bfb + ib) * n + km.bfa + ic;
          s *= wk;
        }
        red_add(dst, s, a.det);
      }
      __syncwarp();
    }
  }
}

template <class C>
void launch_coopw(const CoopTables& tb, const LaunchArgs& a) {
  constexpr int DBLK = C::NA * C::NB + C::NC * C::ND + C::NA * C::NC + C::NB * C::ND + C::NA * C::ND +
                       C::NB * C::NC;
  const size_t smem = sizeof(double) * kCoopWarps * (kCoopBase + kCoopMaxCombo + tb.nslots + DBLK);
  const long long n = a.mode == 0 ? a.nitems : (a.mode == 1 ? a.npair_list : a.nq);
  if (n <= 0) return;
  const LaunchSetup ls =
      launch_setup(reinterpret_cast<const void*>(coopw_kernel<C>), 32 * kCoopWarps, smem, false);
  if (!ls.bps) return;  // CUDA error pending for the caller's check
  const long long cap = static_cast<long long>(ls.bps) * ls.sms;
  const long long want = (n + kCoopWarps - 1) / kCoopWarps;
  const int grid = a.grid > 0 ? a.grid : static_cast<int>(want < cap ? want : cap);
  coopw_kernel<C><<<grid, 32 * kCoopWarps, smem, a.stream>>>(tb, a);
}

}  // namespace eritile_b200
