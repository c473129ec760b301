"""Multi-rank product path on one GPU: n contexts on device 0 act as the n
ranks of a sharded build. Each takes its LPT share
(eritile_gpu_set_shard), runs build_jk_partial_device into its own
accumulator, the accumulators are summed (what the NCCL all-reduce does in
bench.py) and finalize_device gives J/K, compared with the CPU path. All
ranks share one variant table (rank 0's tuned table, as bench.py
broadcasts it)."""
import numpy as np
import pytest

from oracle_lib import Oracle
from systems import BASIS, geom

pytestmark = pytest.mark.gpu


def _density(n, seed):
    rng = np.random.default_rng(seed)
    A = rng.standard_normal((n, n))
    return (A + A.T) / np.sqrt(n)


@pytest.mark.parametrize("mol,kappa", [("w8", 0.0), ("w16", 1e-14)])
@pytest.mark.parametrize("nranks", [2, 4])
def test_sharded_partial_builds_sum_to_oracle(gpu, mol, kappa, nranks):
    import torch
    from paper_2412_13203_b200.eritile import Engine
    xyz, bas = geom(mol), BASIS["cc-pvdz"]
    tau = 1e-10
    full = Engine(0).load_molecule(xyz, bas).build_pairs(kappa)
    full.set_screening(tau)
    N = full.nbf
    D = _density(N, 17)
    full.tune(D, reps=1)
    table = full.get_variants()
    cf, hf, nf = full.pair_survivors()
    small = mol == "w8"  # explicit (x, y) sets there; per-pair counts + y-hashes everywhere
    if small:
        xf, yf = full.quartets()

    dev = torch.device("cuda", 0)
    Dd = torch.from_numpy(D).to(dev)
    acc = torch.zeros(2 * N * N, dtype=torch.float64, device=dev)
    ranks, seen, flops = [], set(), []
    csum = np.zeros_like(cf)
    hsum = np.zeros_like(hf)
    for r in range(nranks):
        e = Engine(0).load_molecule(xyz, bas).build_pairs(kappa)
        e.set_shard(r, nranks)
        e.set_screening(tau)
        e.set_variants(table)
        part = torch.empty(2 * N * N, dtype=torch.float64, device=dev)
        e.build_jk_partial_device(Dd.data_ptr(), part.data_ptr())
        torch.cuda.synchronize()
        acc += part
        c, h, _ = e.pair_survivors()
        csum += c
        hsum += h  # wraps mod 2^64 like the library's sums
        if small:
            xs, ys = e.quartets()
            s = set(zip(xs.tolist(), ys.tolist()))
            assert not (s & seen)  # disjoint shards
            seen |= s
        flops.append(e.stats()["model_flops"])
        ranks.append(e)
    # the shards' union is the canonical list: per-pair counts and y-hash sums
    # add up (a duplicated or missing quartet changes both)
    assert np.array_equal(csum, cf) and np.array_equal(hsum, hf)
    if small:
        assert seen == set(zip(xf.tolist(), yf.tolist()))
    assert max(flops) / (sum(flops) / nranks) < 1.05  # LPT balance of the model FLOPs
    J = torch.empty((N, N), dtype=torch.float64, device=dev)
    K = torch.empty_like(J)
    ranks[0].finalize_device(acc.data_ptr(), J.data_ptr(), K.data_ptr())
    torch.cuda.synchronize()
    Jo, Ko, nq = Oracle("orc").system(xyz, bas, kappa_screen=kappa).build_jk(D, tau)
    assert nq == nf
    assert np.max(np.abs(J.cpu().numpy() - Jo)) < 1e-10
    assert np.max(np.abs(K.cpu().numpy() - Ko)) < 1e-10
    Jf, Kf = full.build_jk(D)
    assert np.max(np.abs(J.cpu().numpy() - Jf)) < 1e-12 and np.max(np.abs(K.cpu().numpy() - Kf)) < 1e-12


def test_variant_table_round_trip_and_validation(gpu):
    from paper_2412_13203_b200.eritile import Engine
    e = Engine(0).load_molecule(geom("w4"), BASIS["cc-pvdz"]).build_pairs(0.0)
    e.set_screening(1e-10)
    t = e.get_variants()
    t2 = t.copy()
    t2[0] = 10_000
    with pytest.raises(ValueError):
        e.set_variants(t2)
    assert np.array_equal(e.get_variants(), t)
    with pytest.raises(ValueError):
        e.set_variants(t[:-1])
