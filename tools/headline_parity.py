"""Full headline J/K parity: the tuned GPU build of (H2O)_80/cc-pVDZ (N = 2000,
kappa 1e-14, tau 1e-10, the bench's synthetic density) against one complete
CPU build of the reference path (oracle/_ref: the unmodified reference headers
+ SPEC executor, all host threads; about 10 minutes on 16 cores).

  python tools/headline_parity.py --out profiles/r02_headline_parity.json

Test infrastructure: the CPU build is the checker, never the thing measured.
"""
import argparse
import json
import os
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
from bench import synthetic_density  # noqa: E402
from oracle_lib import Oracle, available  # noqa: E402
from paper_2412_13203_b200.eritile import Engine, read_fixture  # noqa: E402
from paper_2412_13203_b200.geometry import water_cluster  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--waters", type=int, default=80)
ap.add_argument("--tau", type=float, default=1e-10)
ap.add_argument("--kappa", type=float, default=1e-14)
ap.add_argument("--out", default="")
a = ap.parse_args()

xyz, basis = water_cluster(a.waters), read_fixture("basis", "cc-pvdz.txt")
e = Engine(0).load_molecule(xyz, basis).build_pairs(a.kappa)
e.set_screening(a.tau)
N = e.nbf
D = synthetic_density(N, e.nelectrons // 2)
t0 = time.perf_counter()
e.tune(D)
tune_s = time.perf_counter() - t0
J, K = e.build_jk(D)
st = e.stats()

kind = "ref" if available("ref") else "orc"
S = Oracle(kind).system(xyz, basis, kappa_screen=a.kappa)
cores = os.cpu_count() or 1
t0 = time.perf_counter()
Jo, Ko, nq = S.build_jk(D, a.tau, cores)
cpu_s = time.perf_counter() - t0
dj, dk = float(np.max(np.abs(J - Jo))), float(np.max(np.abs(K - Ko)))
rec = {
    "workload": f"(H2O)_{a.waters}/cc-pvdz, N={N}, tau={a.tau}, kappa={a.kappa}, bench synthetic density (C_occ C_occ^T, seeded QR)",
    "gpu": {"quartets": int(st["quartets"]), "variants": "tuned (Engine.tune)", "tune_s": round(tune_s, 1)},
    "cpu": {"kind": "reference (oracle/_ref)" if kind == "ref" else "port (oracle C restatement)",
            "quartets": int(nq), "threads": cores, "seconds": round(cpu_s, 1)},
    "max_abs_dJ": dj, "max_abs_dK": dk,
    "max_abs_J": float(np.max(np.abs(Jo))), "max_abs_K": float(np.max(np.abs(Ko))),
    "rms_dJ": float(np.sqrt(np.mean((J - Jo) ** 2))), "rms_dK": float(np.sqrt(np.mean((K - Ko) ** 2))),
    "tolerance": 1e-10, "pass": bool(nq == st["quartets"] and dj < 1e-10 and dk < 1e-10),
}
print(json.dumps(rec, indent=1))
if a.out:
    Path(a.out).write_text(json.dumps(rec, indent=1) + "\n")
sys.exit(0 if rec["pass"] else 1)
