"""Multi-rank host logic on CPU (gloo, world_size 2 and 3): the product's
LPT quartet sharding (eritile_gpu_set_shard, host-only contexts) is a
disjoint cover of the canonical list, and summing per-rank partial J/K
over exactly each rank's exported shard with one all-reduce reproduces the
full build (the path's only exchange step). The partial J/K arithmetic is
the CPU checker's (no GPU here); the GPU version of this test is
tests/test_gpu_multirank.py."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    sys.path[:0] = [str(root), str(root / "tests")]
    import torch
    from oracle_lib import Oracle
    from systems import BASIS, geom
    from paper_2412_13203_b200.eritile import Engine
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    xyz, bas = geom("w4"), BASIS["cc-pvdz"]
    O = Oracle("orc").system(xyz, bas)
    Q = O.schwarz()
    e = Engine(-1).load_molecule(xyz, bas).build_pairs(0.0)
    e.set_schwarz(Q)
    e.set_shard(rank, world)
    e.set_screening(1e-10)
    xs, ys = e.quartets()
    n = torch.tensor([len(xs)], dtype=torch.int64)
    dist.all_reduce(n)
    # partial J/K over exactly this rank's shard of the product's list
    rng = np.random.default_rng(3)
    A = rng.standard_normal((O.nbf, O.nbf))
    D = (A + A.T) / np.sqrt(O.nbf)
    J, K = O.build_jk_list(D, xs, ys, 2)
    JK = torch.from_numpy(np.concatenate([J.ravel(), K.ravel()]))
    dist.all_reduce(JK)
    if rank == 0:
        Jf, Kf, nqf = O.build_jk(D, 1e-10, 1)
        N = O.nbf * O.nbf
        q.put((int(n.item()), nqf, float(np.max(np.abs(JK[:N].numpy() - Jf.ravel()))),
               float(np.max(np.abs(JK[N:].numpy() - Kf.ravel()))), (xs.tolist(), ys.tolist())))
    else:
        q.put(("r%d" % rank, (xs.tolist(), ys.tolist())))
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_rank_shards_and_allreduce(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in ps:
        p.join(timeout=60)
    r0 = next(r for r in res if not isinstance(r[0], str))
    others = [r for r in res if isinstance(r[0], str)]
    total, full_nq, dj, dk, l0 = r0
    assert total == full_nq
    assert dj < 1e-12 and dk < 1e-12
    sets = [set(zip(*l0))] + [set(zip(*r[1])) for r in others]
    for a in range(world):
        for b in range(a + 1, world):
            assert not (sets[a] & sets[b])
    assert sum(len(s) for s in sets) == full_nq
