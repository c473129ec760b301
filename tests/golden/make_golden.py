"""Generate golden fixtures from the REFERENCE (oracle/_ref: the unmodified
headers in /root/reference/proj/include compiled with the Vec3 shim and the
SPEC executor). Run in the build container (the reference is absent on the
GPU box); the JSON outputs are committed.

  python tests/golden/make_golden.py
"""
import ctypes as C
import hashlib
import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parents[1]))
sys.path.insert(0, str(HERE.parent))

from oracle_lib import Oracle  # noqa: E402
from systems import BASIS, geom  # noqa: E402


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def seeded_density(n, seed):
    rng = np.random.default_rng(seed)
    A = rng.standard_normal((n, n))
    return (A + A.T) / np.sqrt(n)


def main():
    R = Oracle("ref")
    out = {}
    # Boys on the SPEC grid
    Ts = [0.0, 1e-6, 0.5, 1.0, 5.0, 20.0, 35.0, 36.0, 50.0, 200.0]
    out["boys"] = {"T": Ts, "F16": [R.boys(16, t).tolist() for t in Ts]}
    # plan statistics of compile_class (compiler.hpp:303-307)
    stats = {}
    classes = [(a, b, c, d) for a in range(3) for b in range(3) for c in range(3) for d in range(3)]
    classes += [(3, 0, 3, 0), (3, 1, 2, 0), (2, 2, 3, 3)]
    for cls in classes:
        buf = (C.c_longlong * 12)()
        R._plan_stats(*cls, 1.0, buf)
        stats["".join(map(str, cls))] = list(buf)
    out["plan_stats"] = stats
    out["plan_stats_fields"] = ["op_count", "slot_count", "node_count", "reuse_count", "primT", "base",
                                "prim_slots", "contract", "hrrT", "cslots", "targets", "max_m"]
    src = {}
    for cls in [(0, 0, 0, 0), (1, 0, 1, 0), (1, 1, 1, 1), (2, 1, 2, 1)]:
        n = R._emit_source(*cls, None, 0)
        b = C.create_string_buffer(n + 1)
        R._emit_source(*cls, b, n + 1)
        src["".join(map(str, cls))] = hashlib.sha256(b.value).hexdigest()
    out["emit_source_sha256"] = src
    rnd = {}
    for cls in [(1, 1, 0, 0), (0, 0, 1, 2), (2, 2, 2, 2)]:
        rnd["".join(map(str, cls))] = [R._random_plan_ops(*cls, s) for s in range(5)]
    out["random_plan_ops"] = rnd
    (HERE / "reference_plans_boys.json").write_text(json.dumps(out, indent=0))

    # water / STO-3G: pair store, every quartet, Schwarz, J/K
    S = R.system(geom("water"), BASIS["sto-3g"])
    i, j, k = S.pairs()
    w = {"nbf": S.nbf, "npairs": S.npairs, "ntiles": S.ntiles, "nblocks": S.nblocks,
         "pair_i": i.tolist(), "pair_j": j.tolist(), "pair_nprim": k.tolist(),
         "prims": [S.pair_prims(x, int(k[x])).ravel().tolist() for x in range(S.npairs)],
         "eri": {f"{x},{y}": S.eri(x, y).tolist() for x in range(S.npairs) for y in range(x, S.npairs)},
         "Q": S.schwarz().tolist()}
    D = seeded_density(S.nbf, 7)
    J, K, nq = S.build_jk(D, 0.0, 1)
    w.update({"D_seed": 7, "J": J.ravel().tolist(), "K": K.ravel().tolist(), "nquartets": nq})
    (HERE / "water_sto3g.json").write_text(json.dumps(w))

    # benzene / 6-31G*: block constructor sizes, Q, screened lists
    S = R.system(geom("benzene"), BASIS["6-31g*"])
    Q = S.schwarz()
    b = {"nbf": S.nbf, "npairs": S.npairs, "ntiles": S.ntiles, "nblocks": S.nblocks, "Q": Q.tolist(),
         "lists": {}}
    for tau in (1e-10, 1e-12):
        xs, ys = S.quartets(tau)
        o = np.lexsort((ys, xs))
        b["lists"][repr(tau)] = {"n": int(len(xs)), "sha256_sorted_xy": sha(np.stack([xs[o], ys[o]]))}
    (HERE / "benzene_631gs.json").write_text(json.dumps(b))

    # (H2O)_4 / cc-pVDZ: screened J/K with a seeded density
    S = R.system(geom("w4"), BASIS["cc-pvdz"])
    D = seeded_density(S.nbf, 11)
    J, K, nq = S.build_jk(D, 1e-10, 0)
    xs, ys = S.quartets(1e-10)
    o = np.lexsort((ys, xs))
    c = {"nbf": S.nbf, "npairs": S.npairs, "tau": 1e-10, "D_seed": 11, "nquartets": nq,
         "sha256_sorted_xy": sha(np.stack([xs[o], ys[o]])), "J": J.ravel().tolist(), "K": K.ravel().tolist()}
    (HERE / "w4_ccpvdz.json").write_text(json.dumps(c))
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
