"""Level-scheduled plan tables for the CTA-cooperative (Deconstruction) kernels.

High-L classes do not fit the one-lane-per-quartet straight-line form: the
(2,2,2,2) plan has 2,256 primitive nodes, 961 contracted boundary values and
5,454 horizontal nodes, far beyond 255 registers, and
its straight-line source takes nvcc ~30 minutes. For those classes the plan of
``compile_class`` (the same Alg. 1 plan, compiler.hpp:193-301) is turned into
data: a CTA evaluates one contracted quartet at a time, the threads splitting
every dependency level of the plan, with all values in shared memory
(PAPER.md:253-308 splits high-L work the same way, "Deconstruction").

Tables (all little integers, emitted as ``__device__`` arrays):

* ``lo``: primitive-segment ops (vertical recurrences dag.hpp:125-140,
  148-163 and base loads pref*F_m), sorted by level, 8 words each:
  ``dst | nt << 16`` then up to 5 terms ``src | combo << 16``;
* ``bd``: contraction boundary ``t[ts] += r[rs]`` (compiler.hpp:143);
* ``up``: contracted horizontal ops (dag.hpp:141-147,164-170), 4 words each;
* ``combo``: the distinct (coefficient kind, direction, factor) triples of
  the plan, ``base_id | (factor + 128) << 8``; per primitive quartet the CTA
  forms ``factor * coef[base_id]`` once, so every plan term is one FMA;
* ``tgt``: slot of each output value, kernel a-major order (dag.hpp:221-229);
  a final copy level places them contiguously when shared memory allows.

Slot allocation is level-aware: a slot read at level L may be rewritten
from level L+1 on, so ops of one level never race. Slot 0 holds 1.0.
"""
from __future__ import annotations

import heapq
from typing import Dict, List, Tuple

from .dag import (AB, CD, I2P, I2PQ, I2Q, ITP_RP, ITQ_RQ, PA, PB, QC, QD, UNIT, WP, WQ,
                  compile_class, components, is_base)

# base coefficient ids (must match jk_coop.cuh)
B_UNIT = 0
B_PA, B_QC, B_WP, B_WQ = 1, 4, 7, 10
B_I2P, B_I2Q, B_I2PQ, B_ITP, B_ITQ = 13, 14, 15, 16, 17
B_AB, B_CD = 18, 21
B_PF = 24  # pref * F_m, m = 0..M
MAX_COMBO = 64
# contiguous output copy level: measured slower (the extra slots cost more
# occupancy than the indirection saves), off
COPY_TARGETS = False


def _base_id(kind: int, d: int, swap: bool) -> int:
    if swap:
        kind = {PA: QC, QC: PA, WP: WQ, WQ: WP, I2P: I2Q, I2Q: I2P, ITP_RP: ITQ_RQ,
                ITQ_RQ: ITP_RP, AB: CD, CD: AB, PB: QD, QD: PB}.get(kind, kind)
    if kind == UNIT:
        return B_UNIT
    table = {PA: B_PA, QC: B_QC, WP: B_WP, WQ: B_WQ, AB: B_AB, CD: B_CD}
    if kind in table:
        return table[kind] + d
    return {I2P: B_I2P, I2Q: B_I2Q, I2PQ: B_I2PQ, ITP_RP: B_ITP, ITQ_RQ: B_ITQ}[kind]


def _levels(order, deriv, base_level):
    lvl = {}
    for n in order:
        if n in base_level:
            lvl[n] = base_level[n]
            continue
        lvl[n] = 1 + max(lvl.get(t.node, 0) if t.node in lvl else base_level.get(t.node, 0)
                         for t in deriv[n])
    return lvl


class _Alloc:
    """Level-aware slot allocator (min-heap free list)."""

    def __init__(self, first: int):
        self.next = first
        self.free: List[int] = []
        self.pending: Dict[int, List[int]] = {}  # level -> slots freed after it
        self.high = first

    def release_after(self, slot: int, level: int):
        self.pending.setdefault(level, []).append(slot)

    def open_level(self, level: int):
        for lv in [k for k in self.pending if k < level]:
            for s in self.pending.pop(lv):
                heapq.heappush(self.free, s)

    def take(self) -> int:
        if self.free:
            return heapq.heappop(self.free)
        s = self.next
        self.next += 1
        self.high = max(self.high, self.next)
        return s


def schedule(cls) -> Dict:
    la, lb, lc, ld = cls
    p_fwd = compile_class(cls)
    p_swp = compile_class((lc, ld, la, lb))
    swap = p_swp.op_count < p_fwd.op_count
    plan = p_swp if swap else p_fwd
    deriv = plan.deriv
    M = plan.max_m

    combos: Dict[Tuple[int, int], int] = {}

    def combo(kind, d, factor) -> int:
        key = (_base_id(kind, d, swap), int(factor))
        assert factor == int(factor) and -128 < factor < 128
        if key not in combos:
            combos[key] = len(combos)
        return combos[key]

    def base_combo(m) -> int:
        key = (B_PF + m, 1)
        if key not in combos:
            combos[key] = len(combos)
        return combos[key]

    # ---- primitive segment
    lower = list(plan.lower_order)
    lset = set(lower)
    lvl: Dict = {}
    for n in lower:
        if is_base(n):
            lvl[n] = 0
        else:
            lvl[n] = 1 + max(lvl[t.node] for t in deriv[n])
    nlev = max(lvl.values()) + 1
    boundary = list(plan.boundary)
    bset = set(boundary)
    last_use: Dict = {}
    for n in lower:
        if not is_base(n):
            for t in deriv[n]:
                last_use[t.node] = max(last_use.get(t.node, -1), lvl[n])
    for n in boundary:
        last_use[n] = nlev  # read by the contraction phase
    # boundary slots: dedicated, 1..nb
    tslot = {n: 1 + i for i, n in enumerate(boundary)}
    nb = len(boundary)
    alloc = _Alloc(1 + nb)
    rslot = {}
    by_level: List[List] = [[] for _ in range(nlev)]
    for n in lower:
        by_level[lvl[n]].append(n)
    lo_ops: List[List[int]] = []
    lo_lvl = [0]
    for L in range(nlev):
        alloc.open_level(L)
        for n in by_level[L]:
            s = alloc.take()
            rslot[n] = s
            alloc.release_after(s, last_use.get(n, L))
            if is_base(n):
                terms = [(0, base_combo(n[4]))]
            else:
                terms = [(rslot[t.node], combo(t.kind, t.dir, t.factor)) for t in deriv[n]]
            assert len(terms) <= 5
            lo_ops.append([s | (len(terms) << 16)] + [src | (c << 16) for src, c in terms]
                          + [0] * (7 - len(terms)))
        lo_lvl.append(len(lo_ops))
    lo_high = alloc.high
    bd = [(tslot[n] << 16) | rslot[n] for n in boundary]

    # ---- contracted horizontal segment
    upper = list(plan.upper_order)
    ulvl: Dict = {n: 0 for n in boundary}
    for n in upper:
        ulvl[n] = 1 + max(ulvl[t.node] for t in deriv[n])
    unlev = (max(ulvl[n] for n in upper) + 1) if upper else 1
    ca, cb, cc, cd = (components(L) for L in cls)
    targets = []
    for a in ca:
        for b in cb:
            for c in cc:
                for d in cd:
                    targets.append((c, d, a, b, 0) if swap else (a, b, c, d, 0))
    tset = set(targets)
    ulast: Dict = {}
    for n in upper:
        for t in deriv[n]:
            ulast[t.node] = max(ulast.get(t.node, -1), ulvl[n])
    INF = 1 << 30
    for n in tset:
        ulast[n] = INF
    ualloc = _Alloc(1 + nb)  # the whole primitive region is free again
    # boundary values stay in their slots until their last upper use
    for n in boundary:
        if ulast.get(n, 0) != INF:
            ualloc.release_after(tslot[n], ulast.get(n, 0))
    uslot = dict(tslot)
    up_ops: List[List[int]] = []
    up_lvl = [0]
    ub: List[List] = [[] for _ in range(unlev)]
    for n in upper:
        ub[ulvl[n]].append(n)
    for L in range(1, unlev):
        ualloc.open_level(L)
        for n in ub[L]:
            s = ualloc.take()
            uslot[n] = s
            if ulast.get(n, L) != INF:
                ualloc.release_after(s, ulast.get(n, L))
            terms = [(uslot[t.node], combo(t.kind, t.dir, t.factor)) for t in deriv[n]]
            assert len(terms) <= 3
            up_ops.append([s | (len(terms) << 16)] + [src | (c << 16) for src, c in terms]
                          + [0] * (3 - len(terms)))
        up_lvl.append(len(up_ops))
    # final copy level: outputs into a contiguous region [t0, t0 + NV) in
    # kernel a-major order, so digestion indexes them without indirection
    # (only when it fits: the largest L=3 plans keep the indirect targets)
    base_slots = max(lo_high, ualloc.high, 1 + nb)
    if COPY_TARGETS and base_slots + len(targets) <= 20000:
        t0 = base_slots
        unit_combo = combo(UNIT, 0, 1.0)
        for k, n in enumerate(targets):
            up_ops.append([(t0 + k) | (1 << 16), uslot[n] | (unit_combo << 16), 0, 0])
        up_lvl.append(len(up_ops))
        nslots = t0 + len(targets)
        tgt = [t0 + k for k in range(len(targets))]
    else:
        nslots = base_slots
        tgt = [uslot[n] for n in targets]
    assert nslots < 65536 and len(combos) <= MAX_COMBO, (cls, nslots, len(combos))
    combo_words = [0] * len(combos)
    for (bid, fac), k in combos.items():
        combo_words[k] = bid | ((fac + 128) << 8)
    return dict(cls=cls, swap=swap, M=M, nslots=nslots, nb=nb, lo=lo_ops, lo_lvl=lo_lvl, bd=bd,
                up=up_ops, up_lvl=up_lvl, combo=combo_words, tgt=tgt,
                ops=plan.op_count)


def emit_tables(cid: str, s: Dict) -> str:
    def arr(name, ctype, vals, per=12):
        body = ",".join(str(v) for v in vals) if vals else "0"
        return f"__device__ const {ctype} {name}[] = {{{body}}};"

    lo_flat = [w for op in s["lo"] for w in op]
    up_flat = [w for op in s["up"] for w in op]
    out = [
        f"// cooperative tables: class {s['cls']} ({'ket|bra' if s['swap'] else 'bra|ket'} plan), "
        f"{len(s['lo'])} primitive ops in {len(s['lo_lvl']) - 1} levels, {s['nb']} boundary, "
        f"{len(s['up'])} contracted ops in {len(s['up_lvl']) - 1} levels, {s['nslots']} slots",
        arr(f"kLo{cid}", "unsigned", lo_flat),
        arr(f"kLoLvl{cid}", "int", s["lo_lvl"]),
        arr(f"kBd{cid}", "unsigned", s["bd"]),
        arr(f"kUp{cid}", "unsigned", up_flat),
        arr(f"kUpLvl{cid}", "int", s["up_lvl"]),
        arr(f"kCombo{cid}", "unsigned", s["combo"]),
        arr(f"kTgt{cid}", "unsigned short", s["tgt"]),
    ]
    return "\n".join(out) + "\n"
