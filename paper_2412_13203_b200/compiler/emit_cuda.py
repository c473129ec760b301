"""Emit per-class FP64 sm_100a device code from the Alg. 1 plans.

For every canonical ERI class (La>=Lb, Lc>=Ld, bra pair class >= ket pair
class in the key (L1+L2, L1, L2)) this writes ``csrc/generated/cls_<id>.cu``
holding

* ``struct Cls<id>``: compile-time sizes plus ``eri()``, the straight-line
  evaluation of one contracted quartet: per primitive quartet the binding
  (SPEC.md:290,316), the Boys values, the primitive (vertical) segment of the
  plan and the fold into contracted accumulators; then the contracted
  (horizontal) segment and the a-major target order (compiler.hpp:131-147,
  dag.hpp:221-229). Registers are SSA values; nvcc allocates them.
* explicit instantiations of the JK and Schwarz kernels of csrc/jk_kernels.cuh
  and C launchers registered in ``csrc/generated/registry.cpp``.

The plan is compiled in whichever orientation (bra|ket) or (ket|bra) has
fewer operations; targets are remapped at emission time so the device
function always returns values in the kernel's (bra|ket) a-major order.
The contraction weight and the 2 pi^(5/2)/(pq sqrt(p+q)) kappa_ab kappa_cd
prefactor are folded into one per-primitive-pair scalar U (csrc/host), so
the boundary fold is ``t += r``.
"""
from __future__ import annotations

import os
from pathlib import Path
from typing import Dict, List, Tuple

from .dag import (AB, CD, I2P, I2PQ, I2Q, ITP_RP, ITQ_RQ, PA, PB, QC, QD, UNIT, WP, WQ,
                  compile_class, components, is_base)

PAIR_CLASSES_L2 = [(0, 0), (1, 0), (1, 1), (2, 0), (2, 1), (2, 2)]


def pair_classes(lmax: int) -> List[Tuple[int, int]]:
    out = [(a, b) for a in range(lmax + 1) for b in range(a + 1)]
    return sorted(out, key=lambda t: (t[0] + t[1], t[0], t[1]))


def canonical_classes(lmax: int) -> List[Tuple[int, int, int, int]]:
    pcs = pair_classes(lmax)
    out = []
    for i, a in enumerate(pcs):
        for b in pcs[: i + 1]:
            out.append(a + b)
    return out


def class_id(c) -> str:
    return "%d%d%d%d" % tuple(c)


def ncart(L: int) -> int:
    return (L + 1) * (L + 2) // 2


DIRS = "xyz"


def _coef_expr(kind: int, d: int, side_swap: bool) -> str:
    """Symbolic coefficient -> device expression. With side_swap the plan's
    bra is the kernel's ket (roles of p/q, P/Q exchanged)."""
    if side_swap:
        kind = {PA: QC, QC: PA, WP: WQ, WQ: WP, I2P: I2Q, I2Q: I2P, ITP_RP: ITQ_RQ,
                ITQ_RQ: ITP_RP, AB: CD, CD: AB, PB: QD, QD: PB}.get(kind, kind)
    x = DIRS[d]
    return {
        UNIT: "1.0",
        PA: f"bPA{x}", QC: f"kPA{x}", WP: f"WP{x}", WQ: f"WQ{x}",
        I2P: "i2p", I2Q: "i2q", I2PQ: "i2pq", ITP_RP: "itp", ITQ_RQ: "itq",
        AB: f"AB{x}", CD: f"CD{x}",
    }[kind]


def _fmt_factor(f: float) -> str:
    if f == int(f):
        return "%d.0" % int(f)
    return repr(f)


def emit_class(cls) -> Tuple[str, Dict]:
    """Straight-line pieces of one class for the lane kernels.

    ``prim(bp, kp, btab, acc)`` is one primitive quartet: binding
    (SPEC.md:290,316), Boys, the plan's vertical segment, fold into the
    contracted accumulators ``acc`` (compiler.hpp:141-143). ``finish(acc, AB,
    CD, out)`` is the horizontal segment and the a-major targets
    (compiler.hpp:144-145, dag.hpp:221-229). The primitive loop nests that
    drive them (plain, prefetching, two-ket, ping-pong) are C++ templates in
    csrc/jk_kernels.cuh, so loop structure is a kernel variant, not codegen.
    """
    la, lb, lc, ld = cls
    p_fwd = compile_class(cls)
    p_swp = compile_class((lc, ld, la, lb))
    swap = p_swp.op_count < p_fwd.op_count
    plan = p_swp if swap else p_fwd
    cid = class_id(cls)
    M = plan.max_m
    na, nb, nc, nd = map(ncart, cls)

    lines: List[str] = []
    w = lines.append
    lower_name = {n: f"r{i}" for i, n in enumerate(plan.lower_order)}
    bnd_name = {n: f"t{i}" for i, n in enumerate(plan.boundary)}
    upper_name = {n: f"h{i}" for i, n in enumerate(plan.upper_order)}

    def val_after_contract(n):
        if n in upper_name:
            return upper_name[n]
        return bnd_name[n]

    body: List[str] = []
    b = body.append
    b("const double pq = bp.p + kp.p;")
    b("const double rs = rsqrt_pos(pq);")
    b("const double inv = rs * rs;")
    b("const double PQx = bp.Px - kp.Px, PQy = bp.Py - kp.Py, PQz = bp.Pz - kp.Pz;")
    b("const double pinv = bp.p * inv, qinv = kp.p * inv;")
    b("const double rho = bp.p * qinv;")
    b("const double T = rho * fma(PQx, PQx, fma(PQy, PQy, PQz * PQz));")
    b("const double pref = bp.U * kp.U * rs;")
    b(f"double F[{M + 1}];")
    b("boys_eval_m1(T, btab, F);" if (M == 1 and BOYS_M1_TWO_SLICES) else f"boys_eval<{M}>(T, btab, F);")
    if M > 0:
        b("const double WPx = -qinv * PQx, WPy = -qinv * PQy, WPz = -qinv * PQz;")
        b("const double WQx = pinv * PQx, WQy = pinv * PQy, WQz = pinv * PQz;")
        b("const double bPAx = bp.PAx, bPAy = bp.PAy, bPAz = bp.PAz;")
        b("const double kPAx = kp.PAx, kPAy = kp.PAy, kPAz = kp.PAz;")
        b("const double i2p = bp.i2p, i2q = kp.i2p, i2pq = 0.5 * inv;")
        b("const double itp = bp.i2p * qinv, itq = kp.i2p * pinv;")
        b("(void)WPx; (void)WPy; (void)WPz; (void)WQx; (void)WQy; (void)WQz;")
        b("(void)bPAx; (void)bPAy; (void)bPAz; (void)kPAx; (void)kPAy; (void)kPAz;")
        b("(void)i2p; (void)i2q; (void)i2pq; (void)itp; (void)itq;")
    for n in plan.lower_order:
        nm = lower_name[n]
        if is_base(n):
            b(f"const double {nm} = pref * F[{n[4]}];")
            continue
        expr = None
        for t in plan.deriv[n]:
            c = _coef_expr(t.kind, t.dir, swap)
            src = lower_name[t.node]
            if t.factor != 1.0:
                c = f"({_fmt_factor(t.factor)} * {c})"
            expr = f"{c} * {src}" if expr is None else f"fma({c}, {src}, {expr})"
        b(f"const double {nm} = {expr};")
    nhead = len(body)
    for n in plan.boundary:
        b(f"a.{bnd_name[n]} += {lower_name[n]};")
    btext = "\n".join(body[nhead - len(plan.boundary) - len([x for x in plan.lower_order]):])
    optext = "\n".join(ln for ln in body if ln.startswith("const double r"))

    w(f"// ERI class ({la},{lb},{lc},{ld}); plan orientation "
      f"{'(ket|bra)' if swap else '(bra|ket)'}; ops {plan.op_count}; "
      f"boundary {len(plan.boundary)}; max_m {M}")
    w(f"struct Cls{cid} {{")
    w(f"  static constexpr int LA = {la}, LB = {lb}, LC = {lc}, LD = {ld};")
    w(f"  static constexpr int NA = {na}, NB = {nb}, NC = {nc}, ND = {nd};")
    w(f"  static constexpr int NV = {na * nb * nc * nd};")
    w(f"  static constexpr int M = {M};")
    w(f"  static constexpr int OPS = {plan.op_count};")
    w(f"  static constexpr bool BOYS_M1_TWO = {'true' if (M == 1 and BOYS_M1_TWO_SLICES) else 'false'};")
    w(f"  static constexpr bool BPA = {'true' if 'bPA' in optext else 'false'};  // plan reads bra PA")
    w(f"  static constexpr bool KPA = {'true' if 'kPA' in optext else 'false'};  // plan reads ket PA (QC)")
    w("  struct Acc { double " + ", ".join(bnd_name[n] for n in plan.boundary) + "; };")
    w("  __device__ __forceinline__ static void zero(Acc& a) {")
    w("    " + " ".join(f"a.{bnd_name[n]} = 0.0;" for n in plan.boundary))
    w("  }")
    w("  __device__ __forceinline__ static void fold(Acc& a, const Acc& b) {")
    w("    " + " ".join(f"a.{bnd_name[n]} += b.{bnd_name[n]};" for n in plan.boundary))
    w("  }")
    w("  __device__ __forceinline__ static void prim(const PrimRec& bp, const PrimRec& kp,")
    w("                                              const double* __restrict__ btab, Acc& a) {")
    for ln in body:
        w("    " + ln)
    w("  }")
    # single-primitive contraction (K_bra = K_ket = 1: the d/f shells of
    # cc-pVXZ): the boundary values are the integrals themselves, so the
    # contracted accumulators are assigned, not zeroed and accumulated
    k1 = len(plan.boundary) >= K1_MIN_BOUNDARY
    w(f"  static constexpr bool K1 = {'true' if k1 else 'false'};")
    if k1:
        bset = {f"a.{bnd_name[n]} += {lower_name[n]};": n for n in plan.boundary}
        w("  __device__ __forceinline__ static void prim_set(const PrimRec& bp, const PrimRec& kp,")
        w("                                                  const double* __restrict__ btab, Acc& a) {")
        for ln in body:
            if ln in bset:
                n = bset[ln]
                w(f"    a.{bnd_name[n]} = {lower_name[n]};")
            else:
                w("    " + ln)
        w("  }")
    # family form (csrc/jk_family.cuh): U-free prefactor, two bra-member
    # weights; the ket-member weights are applied per ket primitive (axpy)
    w("  __device__ __forceinline__ static void prim_w(const PrimRec& bp, const PrimRec& kp,")
    w("                                                const double* __restrict__ btab, double w0, double w1,")
    w("                                                Acc& s0, Acc& s1) {")
    bnd_lines = {f"a.{bnd_name[n]} += {lower_name[n]};": n for n in plan.boundary}
    for ln in body:
        if ln == "const double pref = bp.U * kp.U * rs;":
            w("    const double pref = rs;")
        elif ln in bnd_lines:
            n = bnd_lines[ln]
            w(f"    s0.{bnd_name[n]} = fma(w0, {lower_name[n]}, s0.{bnd_name[n]}); "
              f"s1.{bnd_name[n]} = fma(w1, {lower_name[n]}, s1.{bnd_name[n]});")
        else:
            w("    " + ln)
    w("  }")
    w("  __device__ __forceinline__ static void prim_w1(const PrimRec& bp, const PrimRec& kp,")
    w("                                                 const double* __restrict__ btab, double w0, Acc& s0) {")
    for ln in body:
        if ln == "const double pref = bp.U * kp.U * rs;":
            w("    const double pref = rs * w0;")
        else:
            w("    " + ln.replace("a.t", "s0.t"))
    w("  }")
    w("  __device__ __forceinline__ static void axpy(Acc& a, double w, const Acc& s) {")
    w("    " + " ".join(f"a.{bnd_name[n]} = fma(w, s.{bnd_name[n]}, a.{bnd_name[n]});" for n in plan.boundary))
    w("  }")
    w("  __device__ __forceinline__ static void finish(const Acc& a, double ABx, double ABy, double ABz,")
    w("                                                double CDx, double CDy, double CDz, double (&out)[NV]) {")
    w("    (void)ABx; (void)ABy; (void)ABz; (void)CDx; (void)CDy; (void)CDz;")
    for n in plan.boundary:
        w(f"    const double {bnd_name[n]} = a.{bnd_name[n]};")
    for n in plan.upper_order:
        expr = None
        for t in plan.deriv[n]:
            c = _coef_expr(t.kind, t.dir, swap)
            src = val_after_contract(t.node)
            if t.kind == UNIT and t.factor == 1.0:
                expr = src if expr is None else f"({expr} + {src})"
            else:
                if t.factor != 1.0:
                    c = f"({_fmt_factor(t.factor)} * {c})"
                expr = f"{c} * {src}" if expr is None else f"fma({c}, {src}, {expr})"
        w(f"    const double {upper_name[n]} = {expr};")
    ca, cb, cc, cd = (components(L) for L in cls)
    k = 0
    for a in ca:
        for b_ in cb:
            for c in cc:
                for d in cd:
                    node = (c, d, a, b_, 0) if swap else (a, b_, c, d, 0)
                    w(f"    out[{k}] = {val_after_contract(node)};")
                    k += 1
    w("  }")
    w("  __device__ __forceinline__ static void eri(")
    w("      const PrimRec* __restrict__ bra, int kb, const PrimRec* __restrict__ ket, int kk,")
    w("      double ABx, double ABy, double ABz, double CDx, double CDy, double CDz,")
    w("      const double* __restrict__ btab, double (&out)[NV]) {")
    w(f"    eri_drive<Cls{cid}, kLoopPrefetch>(bra, kb, ket, kk, 1, ABx, ABy, ABz, CDx, CDy, CDz, btab, out);")
    w("  }")
    w("};")
    info = dict(cls=cls, swap=swap, ops=plan.op_count, M=M, nv=na * nb * nc * nd,
                boundary=len(plan.boundary), prim_terms=sum(len(i.terms) for i in plan.prim if i.base_m < 0),
                base=sum(1 for i in plan.prim if i.base_m >= 0), contract=len(plan.contract),
                hrr_terms=sum(len(i.terms) for i in plan.hrr))
    return "\n".join(lines) + "\n", info


# Variant policy (the Workload Allocator picks among these at run time,
# csrc/host/engine.cu tune()): one-lane-per-quartet straight-line kernels
# for plans up to LANE_MAX_OPS operations, in MINB_VARIANTS occupancy
# flavours for the small plans; CTA-cooperative table kernels (compiler/
# coop.py) for plans of at least COOP_MIN_OPS operations.
LANE_MAX_OPS = int(os.environ.get("ERITILE_LANE_MAX_OPS", "4000"))
# d/f classes above LANE_MAX_OPS (cc-pVTZ, config 5) also get one straight-line
# lane variant at the 255-register budget (values beyond the register file
# live in the thread's local memory): 1-4 minutes of nvcc per class
LANE_BIG_MAX_OPS = int(os.environ.get("ERITILE_LANE_BIG_MAX_OPS", "21000"))
COOP_MIN_OPS = int(os.environ.get("ERITILE_COOP_MIN_OPS", "250"))
MINB_SMALL_OPS = 700
MINB_VARIANTS = (2,)
# classes with at least this many boundary (contracted) values get a
# single-primitive fast path (prim_set, csrc/jk_kernels.cuh eri_drive)
K1_MIN_BOUNDARY = int(os.environ.get("ERITILE_K1_MIN_BOUNDARY", "48"))
COOP_SMEM_BUDGET = 110 * 1024
COOPW_MAX_SLOTS = 5500  # 4 warps x (slots + 112) doubles <= ~196 KB
# M = 1 classes evaluating F_0 and F_1 from two staged table slices: measured
# neutral-to-slower (the second 51 KB slice costs L1 capacity), off
BOYS_M1_TWO_SLICES = False
FAM_MAX_BOUNDARY = int(os.environ.get("ERITILE_FAM_MAX_BOUNDARY", "9"))  # keep >= 2 CTAs/SM when the Boys slice is staged


def variants(info) -> List[Tuple[str, str]]:
    """(name, launcher expression) per kernel variant of one class."""
    cid = class_id(info["cls"])
    out = []
    if info["ops"] <= LANE_MAX_OPS:
        mins = MINB_VARIANTS if info["ops"] <= MINB_SMALL_OPS else (2,)
        for m in mins:
            out.append((f"lane_m{m}", f"launch_class<Cls{cid}, {m}, kLoopPrefetch>"))
        if info["ops"] > 100:
            # up to 255 registers (1 CTA of 8 warps per SM): trades occupancy
            # for the spills of the large-NV plans
            out.append(("lane_plm1", f"launch_class<Cls{cid}, 1, kLoopPlain>"))
            out.append(("lane_pl384", f"launch_class<Cls{cid}, 1, kLoopPlain, 384>"))
            out.append(("lane_sbm2", f"launch_class<Cls{cid}, 2, kLoopSmemBra>"))
            # + warp-aggregated K REDs (kLoopAggK)
            out.append(("lane_plm1_a", f"launch_class<Cls{cid}, 1, kLoopPlain | kLoopAggK>"))
            out.append(("lane_pl384_a", f"launch_class<Cls{cid}, 1, kLoopPlain | kLoopAggK, 384>"))
        if info["ops"] <= MINB_SMALL_OPS:
            # one Boys table per SM: 512 (<=128 regs) / 768 (<=80 regs) threads
            out.append(("lane_pl512", f"launch_class<Cls{cid}, 1, kLoopPlain, 512>"))
            # Deconstruction: primitive quartets of one contracted quartet over 2 lanes
            out.append(("lane_ps512", f"launch_class<Cls{cid}, 1, kLoopPlain | kLoopSplit, 512>"))
            out.append(("lane_pl768", f"launch_class<Cls{cid}, 1, kLoopPlain, 768>"))
            out.append(("lane_sb512", f"launch_class<Cls{cid}, 1, kLoopSmemBra, 512>"))
        # bra-stationary strips (csrc/jk_strip.cuh): K rows in shared memory;
        # the packed multi-bra remainder runs on a lane kernel
        if info["ops"] <= MINB_SMALL_OPS:
            out.append(("strip_t512", f"launch_strip<Cls{cid}, 512, 1, kLoopPlain, 512>"))
            # + ket-record / item prefetch and batched shared-memory K adds (OPT 7)
            out.append(("strip_o7_t512", f"launch_strip<Cls{cid}, 512, 1, kLoopPlain, 512, 7>"))
            # two ket primitives per bra record read (+ batched K adds)
            # + warp-aggregated K-row updates (OPT 16)
            out.append(("strip_a_t512", f"launch_strip<Cls{cid}, 512, 1, kLoopPlain, 512, 18>"))
            out.append(("strip_a_t768", f"launch_strip<Cls{cid}, 768, 1, kLoopPlain, 768, 18>"))
            # + L1 prefetch of the next ket record / next item's metadata (OPT 32|4)
            out.append(("strip_p_t512", f"launch_strip<Cls{cid}, 512, 1, kLoopPlain, 512, 54>"))
            # + d-column K updates to global memory (OPT 64)
            out.append(("strip_s_t512", f"launch_strip<Cls{cid}, 512, 1, kLoopPlain, 512, 82>"))
            # + dual items: two kets per lane, one loop nest (OPT 128)
            out.append(("strip_d_t512", f"launch_strip<Cls{cid}, 512, 1, kLoopPlain, 512, 146>"))
    elif info["ops"] <= LANE_BIG_MAX_OPS and info["ops"] >= COOP_MIN_OPS:
        # J/K only; the Schwarz / raw-quartet modes go to the coop kernel
        out.append(("lane_plm1", f"launch_big_lane_cls{cid}"))
    if info["ops"] >= COOP_MIN_OPS:
        out.append(("coop", f"launch_coop_cls{cid}"))
        if info.get("coop_slots", 1 << 30) <= COOPW_MAX_SLOTS:
            out.append(("coopw", f"launch_coopw_cls{cid}"))
    if info["boundary"] <= FAM_MAX_BOUNDARY:
        # shared-primitive unit kernels (csrc/jk_family.cuh); kept last: the
        # engine uses these (and only these) when families are enabled
        out.append(("fam_pl512", f"launch_fam<Cls{cid}, 1, kLoopPlain, 512>"))
        out.append(("fam_x768", f"launch_fam<Cls{cid}, 1, kLoopPlain, 512, 768>"))
        out.append(("fstrip_t512", f"launch_fstrip<Cls{cid}, 512, 1, kLoopPlain, 512, 768>"))
        out.append(("fstrip_t768", f"launch_fstrip<Cls{cid}, 768, 1, kLoopPlain, 512, 768>"))
        out.append(("fstrip_o7_t512", f"launch_fstrip<Cls{cid}, 512, 1, kLoopPlain, 512, 768, 7>"))
        out.append(("fstrip_k2_t768", f"launch_fstrip<Cls{cid}, 768, 1, kLoopPlain, 512, 768, 10>"))
        out.append(("fstrip_a_t512", f"launch_fstrip<Cls{cid}, 512, 1, kLoopPlain, 512, 768, 18>"))
        out.append(("fstrip_a_t768", f"launch_fstrip<Cls{cid}, 768, 1, kLoopPlain, 512, 768, 18>"))
        out.append(("fstrip_ak2_t768", f"launch_fstrip<Cls{cid}, 768, 1, kLoopPlain, 512, 768, 26>"))
        out.append(("fstrip_p_t512", f"launch_fstrip<Cls{cid}, 512, 1, kLoopPlain, 512, 768, 54>"))
        out.append(("fstrip_s_t512", f"launch_fstrip<Cls{cid}, 512, 1, kLoopPlain, 512, 768, 82>"))
        out.append(("fstrip_sk2_t768", f"launch_fstrip<Cls{cid}, 768, 1, kLoopPlain, 512, 768, 90>"))
    assert len(out) <= 32, (info["cls"], out)  # kMaxVariants (csrc/jk_api.h)
    return out


def is_unit_variant(name: str) -> bool:
    """Variants that run the shared-primitive unit lists (kept last)."""
    return name.startswith("fam_") or name.startswith("fstrip")


def default_variant(info, vs) -> int:
    names = [v[0] for v in vs if not is_unit_variant(v[0])]
    if "coop" in names and (info["ops"] >= 2000 or len(names) == 1):
        return names.index("coop")
    return 0


def write_sources(outdir: Path, lmax: int = 2) -> List[Dict]:
    from .coop import emit_tables, schedule
    outdir.mkdir(parents=True, exist_ok=True)
    infos = []
    classes = canonical_classes(lmax)
    for idx, cls in enumerate(classes):
        body, info = emit_class(cls)
        cid = class_id(cls)
        info["index"] = idx
        sc = schedule(cls) if info["ops"] >= COOP_MIN_OPS else None
        if sc is not None:
            info["coop_slots"] = sc["nslots"]
        vs = variants(info)
        info["variants"] = vs
        info["default"] = default_variant(info, vs)
        infos.append(info)
        lane = any(n.startswith("lane") for n, _ in vs)
        coop = any(n == "coop" for n, _ in vs)
        src = ["// GENERATED by paper_2412_13203_b200/compiler/emit_cuda.py — do not edit.",
               '#include "../jk_coop.cuh"', '#include "../jk_strip.cuh"', "namespace eritile_b200 {"]
        if lane:
            src.append(body)
        else:  # sizes only; the straight-line body is not emitted
            na, nb, nc, nd = map(ncart, cls)
            src.append(f"struct Cls{cid} {{\n  static constexpr int LA = {cls[0]}, LB = {cls[1]}, "
                       f"LC = {cls[2]}, LD = {cls[3]};\n  static constexpr int NA = {na}, NB = {nb}, "
                       f"NC = {nc}, ND = {nd};\n  static constexpr int NV = {na * nb * nc * nd};\n"
                       f"  static constexpr int M = {info['M']};\n  static constexpr int OPS = {info['ops']};\n"
                       f"  static constexpr bool BOYS_M1_TWO = false;\n  static constexpr bool K1 = false;\n}};")
        if coop:
            width = max(b - a for a, b in zip(sc["lo_lvl"], sc["lo_lvl"][1:]))
            nt = 256 if width >= 192 else 128
            src.append(emit_tables(cid, sc))
            na, nb_, nc, nd = map(ncart, cls)
            need = 8 * (48 + 64 + sc["nslots"]) + 2 * na * nb_ * nc * nd
            boys_smem = need + 8 * 641 * 10 <= COOP_SMEM_BUDGET
            assert need <= 227 * 1024, (cls, need)
            src.append(f"struct CoopCls{cid} : Cls{cid} {{ static constexpr int NT = {nt}; "
                       f"static constexpr bool BOYS_SMEM = {'true' if boys_smem else 'false'}; }};")
            src.append(f"void launch_coop_cls{cid}(const LaunchArgs& a) {{")
            src.append("  CoopTables t{};")
            for fld, sym in [("lo", "kLo"), ("lo_lvl", "kLoLvl"), ("bd", "kBd"), ("up", "kUp"),
                             ("up_lvl", "kUpLvl"), ("combo", "kCombo"), ("tgt", "kTgt")]:
                src.append(f"  cudaGetSymbolAddress((void**)&t.{fld}, {sym}{cid});")
            src.append(f"  t.nlo_lvl = {len(sc['lo_lvl']) - 1}; t.nb = {sc['nb']}; "
                       f"t.nup_lvl = {len(sc['up_lvl']) - 1}; t.ncombo = {len(sc['combo'])}; "
                       f"t.nslots = {sc['nslots']}; t.tgt0 = {sc['tgt'][0]};")
            src.append(f"  launch_coop<CoopCls{cid}>(t, a);")
            src.append("}")
            if any(n == "coopw" for n, _ in vs):
                src.append(f"void launch_coopw_cls{cid}(const LaunchArgs& a) {{")
                src.append("  CoopTables t{};")
                for fld, sym in [("lo", "kLo"), ("lo_lvl", "kLoLvl"), ("bd", "kBd"), ("up", "kUp"),
                                 ("up_lvl", "kUpLvl"), ("combo", "kCombo"), ("tgt", "kTgt")]:
                    src.append(f"  cudaGetSymbolAddress((void**)&t.{fld}, {sym}{cid});")
                src.append(f"  t.nlo_lvl = {len(sc['lo_lvl']) - 1}; t.nb = {sc['nb']}; "
                           f"t.nup_lvl = {len(sc['up_lvl']) - 1}; t.ncombo = {len(sc['combo'])}; "
                           f"t.nslots = {sc['nslots']}; t.tgt0 = {sc['tgt'][0]};")
                src.append(f"  launch_coopw<CoopCls{cid}>(t, a);")
                src.append("}")
        if any(expr == f"launch_big_lane_cls{cid}" for _, expr in vs):
            src.append(f"void launch_big_lane_cls{cid}(const LaunchArgs& a) {{")
            src.append(f"  if (a.mode != 0) return launch_coop_cls{cid}(a);")
            src.append(f"  launch_class<Cls{cid}, 1, kLoopPlain, kJkThreads, true>(a);")
            src.append("}")
        for name, expr in vs:
            if name not in ("coop", "coopw"):
                src.append(f"void launch_{name}_cls{cid}(const LaunchArgs& a) {{ {expr}(a); }}")
        src += ["}  // namespace eritile_b200", ""]
        _write_if_changed(outdir / f"cls_{cid}.cu", "\n".join(src))
    reg = ["// GENERATED by paper_2412_13203_b200/compiler/emit_cuda.py — do not edit.",
           '#include "../jk_api.h"', "namespace eritile_b200 {"]
    def fn(name, cid):
        if name in ("coop", "coopw"):
            return f"launch_{name}_cls{cid}"
        return f"launch_{name}_cls{cid}"
    for info in infos:
        cid = class_id(info["cls"])
        for name, _ in info["variants"]:
            reg.append(f"void {fn(name, cid)}(const LaunchArgs&);")
    reg.append("const ClassEntry kClassTable[] = {")
    for info in infos:
        la, lb, lc, ld = info["cls"]
        cid = class_id(info["cls"])
        vs = info["variants"]
        fns = ", ".join(f"&{fn(n, cid)}" for n, _ in vs) + ", nullptr" * (16 - len(vs))
        names = ", ".join(f'"{n}"' for n, _ in vs) + ", nullptr" * (16 - len(vs))
        nfam = sum(1 for n, _ in vs if is_unit_variant(n))
        fam_def = len(vs) - nfam if nfam else -1
        reg.append(f"  {{{la}, {lb}, {lc}, {ld}, {info['M']}, {info['ops']}, {info['prim_terms']}, "
                   f"{info['base']}, {info['contract']}, {info['hrr_terms']}, {len(vs)}, {{{fns}}}, "
                   f"{{{names}}}, {info['default']}, {nfam}, {fam_def}}},")
    reg.append("};")
    reg.append(f"const int kNumClasses = {len(infos)};")
    reg.append(f"const int kMaxL = {lmax};")
    reg.append("}  // namespace eritile_b200")
    _write_if_changed(outdir / "registry.cpp", "\n".join(reg) + "\n")
    for stale in outdir.glob("cls_*.cu"):
        if stale.stem[4:] not in {class_id(i["cls"]) for i in infos}:
            stale.unlink()
    return infos


def _write_if_changed(path: Path, text: str) -> None:
    if path.exists() and path.read_text() == text:
        return
    tmp = path.with_suffix(path.suffix + ".tmp")
    tmp.write_text(text)
    os.replace(tmp, path)
