"""Graph compiler (compiler/dag.py) against the reference's compile_class.

The product's Python implementation of Alg. 1 (§6, compiler.hpp)
must produce plans with exactly the reference's statistics; the emitted
CUDA must be deterministic and compile-time bounded.
"""
import json
import time
from pathlib import Path

import pytest

from paper_2412_13203_b200.compiler import dag
from paper_2412_13203_b200.compiler.emit_cuda import canonical_classes, emit_class

G = json.loads((Path(__file__).resolve().parent / "golden" / "reference_plans_boys.json").read_text())


def stats(p):
    return [p.op_count, p.slot_count, p.node_count, p.reuse_count,
            sum(len(i.terms) for i in p.prim if i.base_m < 0), sum(1 for i in p.prim if i.base_m >= 0),
            p.prim_slots, len(p.contract), sum(len(i.terms) for i in p.hrr), p.cslots, len(p.targets), p.max_m]


@pytest.mark.parametrize("key", sorted(G["plan_stats"]))
def test_plan_stats_match_reference(key):
    cls = tuple(int(c) for c in key)
    assert stats(dag.compile_class(cls)) == G["plan_stats"][key]


def test_find_optimal_position_examples():
    P = dag.Position
    choose = dag.greedy_choice(1.0)
    assert choose([P(0, 0, 1, 2, 3, [])]) == 0
    assert dag.greedy_choice(0.5)([P(0, 0, 2, 0, 2, []), P(0, 0, 1, 1, 1, [])]) == 1
    assert choose([P(0, 0, 1, 1, 2, []), P(0, 0, 1, 1, 2, [])]) == 0  # tie -> first
    with pytest.raises(ValueError):
        choose([])


def test_small_plans():
    p = dag.compile_class((0, 0, 0, 0))
    assert p.op_count == 1 and len(p.prim) == 1 and p.prim[0].base_m == 0
    p = dag.compile_class((1, 0, 0, 0))
    assert len(p.targets) == 3 and p.max_m == 1


def test_acyclic_and_base_reachable():
    for cls in canonical_classes(2):
        g = dag.build_dag(cls)
        order = {n: i for i, n in enumerate(g.order)}
        for n, srcs in g.deriv.items():
            for t in srcs:
                assert t.node in g.nodes
        assert all(dag.is_base(n) or n in g.deriv for n in g.nodes)


def test_emission_deterministic_and_fast():
    t = time.time()
    a = [emit_class(c)[0] for c in canonical_classes(2)]
    b = [emit_class(c)[0] for c in canonical_classes(2)]
    assert a == b
    assert time.time() - t < 20.0


def test_greedy_beats_random_on_average():
    # the reference's greedy is not <= every random path (12/900
    # exceptions with its RNG); the average advantage is the robust property.
    ratios = []
    for cls in canonical_classes(2):
        g = dag.compile_class(cls).op_count
        r = [dag.compile_random_class(cls, s).op_count for s in range(5)]
        ratios.append(sum(r) / len(r) / g)
    assert sum(ratios) / len(ratios) > 1.1
