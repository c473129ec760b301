"""Workload Allocator, Algorithm 2, against the SPEC's
mock-cost examples: the C++ loop (csrc/host/allocator.h)
runs on mock cost tables through eritile_alloc_simulate (no device)."""
import numpy as np
import pytest

from paper_2412_13203_b200.eritile import alloc_simulate

K = 13  # g = 1 .. 4096


def table(fn, ncls=1):
    return np.array([[fn(c, 2 ** k) for k in range(K)] for c in range(ncls)])


def test_cost_one_over_g_runs_to_cap():
    # SPEC: cost(g) = 1/g -> times halve per combine; all decreasing -> all g at cap
    g, acc, sweeps = alloc_simulate(table(lambda c, g: 1.0 / g, 3), [64, 4096, 8])
    assert list(g) == [64, 4096, 8]
    assert acc == 6 + 12 + 3
    assert sweeps == 12 + 1  # the longest class needs 12 accepted sweeps, then one that finds nothing


def test_minimum_at_four_converges_to_four():
    g, acc, _ = alloc_simulate(table(lambda c, g: (np.log2(g) - 2.0) ** 2 + 1.0), [4096])
    assert g[0] == 4 and acc == 2


def test_increasing_costs_leave_config_unchanged():
    g, acc, sweeps = alloc_simulate(table(lambda c, g: float(g), 4), [4096] * 4)
    assert list(g) == [1, 1, 1, 1] and acc == 0 and sweeps == 1  # immediate revert everywhere


def test_mixed_classes_are_isolated():
    # class A minimum at g = 4, class B minimum at g = 1
    cost = table(lambda c, g: (np.log2(g) - 2.0) ** 2 if c == 0 else float(g), 2)
    g, _, _ = alloc_simulate(cost, [4096, 4096])
    assert g[0] == 4 and g[1] == 1


def test_cap_bounds_combine():
    # g = cap: combine is a no-op (capped), nothing is measured or changed
    g, acc, sweeps = alloc_simulate(table(lambda c, g: 1.0 / g, 2), [1, 2])
    assert list(g) == [1, 2] and acc == 1 and sweeps == 2


def test_ties_revert():
    # the loop keeps a combine only on a strict improvement (t2 < t1)
    g, acc, _ = alloc_simulate(table(lambda c, g: 1.0), [4096])
    assert g[0] == 1 and acc == 0


@pytest.mark.parametrize("seed", range(5))
def test_termination_bound_on_random_costs(seed):
    # halts within log2(cap) * |classes| accepted steps plus one non-improving sweep
    rng = np.random.default_rng(seed)
    ncls = 6
    cost = rng.uniform(0.5, 2.0, (ncls, K))
    caps = [2 ** int(k) for k in rng.integers(0, K, ncls)]
    g, acc, sweeps = alloc_simulate(cost, caps)
    bound = sum(int(np.log2(c)) for c in caps)
    assert acc <= bound and sweeps <= bound + 1
    assert all(1 <= gi <= c and (gi & (gi - 1)) == 0 for gi, c in zip(g, caps))
    # every class sits at a point the greedy doubling cannot improve
    for c in range(ncls):
        k = int(np.log2(g[c]))
        if 2 * g[c] <= caps[c]:
            assert cost[c, k + 1] >= cost[c, k]


def test_memory_bound_kernel_gets_larger_granularity():
    # SPEC principle check ("allocate a larger workload per thread"): equal task
    # count N on P workers; a task costs its items plus a per-task overhead o
    # (latency of the task's loads: large when memory-bound), and a task of g
    # items leaves a tail of ~g items of imbalance.
    N, P, u = 2 ** 20, 4096, 1.0

    def model(o):
        return lambda c, g: (N / g) * o / P + N * u / P + g * u

    gm, _, _ = alloc_simulate(table(model(400.0)), [4096])  # memory-bound: long per-task latency
    gc, _, _ = alloc_simulate(table(model(4.0)), [4096])    # compute-bound
    assert gm[0] > gc[0]


def test_bad_table_rejected():
    with pytest.raises(ValueError):
        alloc_simulate(np.ones((1, 3)), [64])  # table does not reach g = cap
