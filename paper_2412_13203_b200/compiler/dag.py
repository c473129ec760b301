"""Recurrence DAG for one ERI class and the greedy path search (Alg. 1).

Semantics follow the reference graph compiler so that plan statistics agree
exactly (tests/test_compiler.py checks op/slot/node/reuse counts against
``compile_class`` through oracle/_ref):

* node ``[a b | c d]^(m)`` with Cartesian momenta (dag.hpp:16-30), ordered
  lexicographically on (a, b, c, d, m) like the reference's defaulted <=>;
* source rules of the four positions (dag.hpp:119-173): vertical on the bra
  (slot 0) and ket (slot 2) only for transferred nodes (b = d = 0), horizontal
  transfer b -> a (slot 1) and d -> c (slot 3);
* greedy cost (n - r) + lambda * ang, first minimum wins (compiler.hpp:27-42);
* depth-first derivation over a stack seeded with the a-major targets
  (compiler.hpp:52-81);
* plan emission (compiler.hpp:193-301): transferred nodes form the
  per-primitive segment, the rest the contracted horizontal segment, a
  boundary set is folded into contracted slots, topological order picks the
  smallest ready node, and primitive registers are reused after last use.

This module is the product's own implementation (Python, offline); the
emitted plans drive csrc code generation (compiler/emit_cuda.py).
"""
from __future__ import annotations

import functools
import heapq
import random
from dataclasses import dataclass, field
from typing import Callable, Dict, List, Sequence, Tuple

Mom = Tuple[int, int, int]
Node = Tuple[Mom, Mom, Mom, Mom, int]  # (a, b, c, d, m)

# coefficient kinds (dag.hpp:45-60)
UNIT, PA, PB, QC, QD, WP, WQ, I2P, I2Q, I2PQ, ITP_RP, ITQ_RQ, AB, CD = range(14)
KIND_NAMES = ["1", "PA", "PB", "QC", "QD", "WP", "WQ", "1/2p", "1/2q", "1/2(p+q)",
              "(1/2p)(rho/p)", "(1/2q)(rho/q)", "AB", "CD"]
DIRECTIONAL = {PA, PB, QC, QD, WP, WQ, AB, CD}


def components(L: int) -> List[Mom]:
    """Cartesian order x-major descending (molecule.hpp:176-183)."""
    return [(ax, ay, L - ax - ay) for ax in range(L, -1, -1) for ay in range(L - ax, -1, -1)]


def _tot(v: Mom) -> int:
    return v[0] + v[1] + v[2]


def _dec(v: Mom, i: int) -> Mom:
    w = list(v)
    w[i] -= 1
    return (w[0], w[1], w[2])


def _inc(v: Mom, i: int) -> Mom:
    w = list(v)
    w[i] += 1
    return (w[0], w[1], w[2])


def is_base(n: Node) -> bool:
    return _tot(n[0]) == 0 and _tot(n[1]) == 0 and _tot(n[2]) == 0 and _tot(n[3]) == 0


def is_transferred(n: Node) -> bool:
    return _tot(n[1]) == 0 and _tot(n[3]) == 0


@dataclass(frozen=True)
class Term:
    node: Node
    kind: int
    dir: int
    factor: float


def sources(n: Node, slot: int, d: int) -> List[Term]:
    a, b, c, dd, m = n
    out: List[Term] = []
    if slot == 0:  # vertical, bra
        e = _dec(a, d)
        out.append(Term((e, b, c, dd, m), PA, d, 1.0))
        out.append(Term((e, b, c, dd, m + 1), WP, d, 1.0))
        if e[d] > 0:
            e1 = _dec(e, d)
            out.append(Term((e1, b, c, dd, m), I2P, 0, float(e[d])))
            out.append(Term((e1, b, c, dd, m + 1), ITP_RP, 0, -float(e[d])))
        if c[d] > 0:
            out.append(Term((e, b, _dec(c, d), dd, m + 1), I2PQ, 0, float(c[d])))
    elif slot == 1:  # horizontal, bra
        b1 = _dec(b, d)
        out.append(Term((_inc(a, d), b1, c, dd, m), UNIT, 0, 1.0))
        out.append(Term((a, b1, c, dd, m), AB, d, 1.0))
    elif slot == 2:  # vertical, ket
        f = _dec(c, d)
        out.append(Term((a, b, f, dd, m), QC, d, 1.0))
        out.append(Term((a, b, f, dd, m + 1), WQ, d, 1.0))
        if f[d] > 0:
            f1 = _dec(f, d)
            out.append(Term((a, b, f1, dd, m), I2Q, 0, float(f[d])))
            out.append(Term((a, b, f1, dd, m + 1), ITQ_RQ, 0, -float(f[d])))
        if a[d] > 0:
            out.append(Term((_dec(a, d), b, f, dd, m + 1), I2PQ, 0, float(a[d])))
    else:  # horizontal, ket
        d1 = _dec(dd, d)
        out.append(Term((a, b, _inc(c, d), d1, m), UNIT, 0, 1.0))
        out.append(Term((a, b, c, d1, m), CD, d, 1.0))
    return out


@dataclass
class Position:
    slot: int
    dir: int
    ang: int
    r: int
    n: int
    srcs: List[Term]


def positions(n: Node, known: set) -> List[Position]:
    out = []
    tr = is_transferred(n)
    for slot in range(4):
        if slot in (0, 2) and not tr:
            continue
        v = n[slot]
        for d in range(3):
            if v[d] == 0:
                continue
            s = sources(n, slot, d)
            r = sum(1 for t in s if t.node in known)
            out.append(Position(slot, d, v[d], r, len(s) - r, s))
    return out


def greedy_choice(lam: float) -> Callable[[List[Position]], int]:
    def choose(ps: List[Position]) -> int:
        if not ps:
            raise ValueError("find_optimal_position: no candidates")
        best, opt = float("inf"), 0
        for i, p in enumerate(ps):
            cost = float(p.n - p.r) + lam * p.ang
            if cost < best:
                best, opt = cost, i
        return opt
    return choose


@dataclass
class DAG:
    cls: Tuple[int, int, int, int]
    nodes: set = field(default_factory=set)
    deriv: Dict[Node, List[Term]] = field(default_factory=dict)
    order: List[Node] = field(default_factory=list)
    targets: List[Node] = field(default_factory=list)
    reuse: int = 0

    def max_m(self) -> int:
        return max(n[4] for n in self.nodes)


def class_targets(cls) -> List[Node]:
    la, lb, lc, ld = cls
    return [(a, b, c, d, 0) for a in components(la) for b in components(lb)
            for c in components(lc) for d in components(ld)]


def search(cls, choose: Callable[[List[Position]], int]) -> DAG:
    g = DAG(tuple(cls))
    g.targets = class_targets(cls)
    stack: List[Node] = []
    for t in reversed(g.targets):
        if t not in g.nodes:
            g.nodes.add(t)
            stack.append(t)
    while stack:
        n = stack.pop()
        if is_base(n) or n in g.deriv:
            continue
        ps = positions(n, g.nodes)
        p = ps[choose(ps)]
        g.reuse += p.r
        for t in reversed(p.srcs):
            if t.node not in g.nodes:
                g.nodes.add(t.node)
                if not is_base(t.node):
                    stack.append(t.node)
        g.deriv[n] = p.srcs
        g.order.append(n)
    return g


def build_dag(cls, lam: float = 1.0) -> DAG:
    return search(cls, greedy_choice(lam))


def build_random_dag(cls, seed: int) -> DAG:
    rng = random.Random(seed)
    return search(cls, lambda ps: rng.randrange(len(ps)))


# ------------------------------------------------------------------ plans
@dataclass
class Instr:
    dst: int
    base_m: int  # >= 0: dst = pref * F[base_m]
    terms: List[Tuple[int, int, int, float]]  # (src, kind, dir, factor)


@dataclass
class Plan:
    cls: Tuple[int, int, int, int]
    lam: float
    max_m: int
    prim_slots: int
    cslots: int
    prim: List[Instr]
    contract: List[Tuple[int, int]]  # (prim register, contracted slot)
    hrr: List[Instr]
    targets: List[int]
    op_count: int
    node_count: int
    reuse_count: int
    # symbolic views used by the CUDA emitter
    lower_order: List[Node] = field(default_factory=list)
    boundary: List[Node] = field(default_factory=list)
    upper_order: List[Node] = field(default_factory=list)
    deriv: Dict[Node, List[Term]] = field(default_factory=dict)
    target_nodes: List[Node] = field(default_factory=list)

    @property
    def slot_count(self) -> int:
        return self.prim_slots + self.cslots


def _topo(g: DAG, wanted: set) -> List[Node]:
    indeg: Dict[Node, int] = {}
    deps: Dict[Node, List[Node]] = {}
    for n in sorted(wanted):
        deg = 0
        if n in g.deriv:
            for s in sorted({t.node for t in g.deriv[n]}):
                if s in wanted:
                    deg += 1
                    deps.setdefault(s, []).append(n)
        indeg[n] = deg
    ready = [n for n, d in indeg.items() if d == 0]
    heapq.heapify(ready)
    out = []
    while ready:
        n = heapq.heappop(ready)
        out.append(n)
        for dep in deps.get(n, []):
            indeg[dep] -= 1
            if indeg[dep] == 0:
                heapq.heappush(ready, dep)
    if len(out) != len(wanted):
        raise RuntimeError("plan generation: cycle in recurrence graph")
    return out


def generate_plan(g: DAG, lam: float = 1.0) -> Plan:
    lower = {n for n in g.nodes if is_transferred(n)}
    upper = g.nodes - lower
    boundary = set()
    for n in upper:
        for t in g.deriv[n]:
            if is_transferred(t.node):
                boundary.add(t.node)
    for t in g.targets:
        if is_transferred(t):
            boundary.add(t)
    cslot: Dict[Node, int] = {}
    for n in sorted(boundary):
        cslot.setdefault(n, len(cslot))
    for n in sorted(upper):
        cslot.setdefault(n, len(cslot))

    lower_order = _topo(g, lower)
    vreg: Dict[Node, int] = {}
    virt: List[Instr] = []
    for n in lower_order:
        v = len(vreg)
        vreg[n] = v
        if is_base(n):
            virt.append(Instr(v, n[4], []))
        else:
            virt.append(Instr(v, -1, [(vreg[t.node], t.kind, t.dir, t.factor) for t in g.deriv[n]]))
    last = [-1] * len(virt)
    for i, ins in enumerate(virt):
        for t in ins.terms:
            last[t[0]] = i
    live_end = {vreg[n] for n in boundary}
    phys = [-1] * len(virt)
    free: List[int] = []
    peak = 0
    prim: List[Instr] = []
    for i, ins in enumerate(virt):
        if free:
            slot = heapq.heappop(free)
        else:
            slot, peak = peak, peak + 1
        phys[i] = slot
        prim.append(Instr(slot, ins.base_m, [(phys[s], k, d, f) for (s, k, d, f) in ins.terms]))
        for v in range(i + 1):
            if last[v] == i and v not in live_end and phys[v] >= 0:
                heapq.heappush(free, phys[v])
                phys[v] = -phys[v] - 1000
    contract = [(phys[vreg[n]], cslot[n]) for n in sorted(boundary)]
    upper_order = _topo(g, upper)
    hrr = [Instr(cslot[n], -1, [(cslot[t.node], t.kind, t.dir, t.factor) for t in g.deriv[n]])
           for n in upper_order]
    ops = sum(1 if i.base_m >= 0 else len(i.terms) for i in prim) + sum(len(i.terms) for i in hrr)
    return Plan(cls=g.cls, lam=lam, max_m=g.max_m(), prim_slots=peak, cslots=len(cslot), prim=prim,
                contract=contract, hrr=hrr, targets=[cslot[t] for t in g.targets], op_count=ops,
                node_count=len(g.nodes), reuse_count=g.reuse, lower_order=lower_order,
                boundary=sorted(boundary), upper_order=upper_order, deriv=g.deriv,
                target_nodes=list(g.targets))


@functools.lru_cache(maxsize=None)
def compile_class(cls, lam: float = 1.0) -> Plan:
    """Plans are immutable after generation; cached per (class, lambda)."""
    return generate_plan(build_dag(tuple(cls), lam), lam)


def compile_random_class(cls, seed: int) -> Plan:
    return generate_plan(build_random_dag(cls, seed))
