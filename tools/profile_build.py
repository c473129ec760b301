"""Run a few Fock builds of one system (for ncu / nsys-less profiling).

  python tools/profile_build.py --waters 16 --builds 3
"""
import argparse
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))

from paper_2412_13203_b200.eritile import Engine, read_fixture  # noqa: E402
from paper_2412_13203_b200.geometry import alanine_chain, water_cluster  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--waters", type=int, default=16)
ap.add_argument("--geom", default="", help="ala<n>: H-(Ala)_n-OH strand instead of the water cluster")
ap.add_argument("--basis", default="cc-pvdz.txt")
ap.add_argument("--tau", type=float, default=1e-10)
ap.add_argument("--builds", type=int, default=2)
ap.add_argument("--kappa", type=float, default=1e-14)
ap.add_argument("--tune", action="store_true")
ap.add_argument("--set", action="append", default=[], help="CLS=VARIANT, e.g. 1000=fam_x768")
ap.add_argument("--variants-json", default="", help="write {class: chosen variant} here")
ap.add_argument("--profile-range", action="store_true",
                help="cudaProfilerStart/Stop around the measured builds only (ncu --profile-from-start off)")
a = ap.parse_args()
xyz = alanine_chain(int(a.geom[3:])) if a.geom.startswith("ala") else water_cluster(a.waters)
e = Engine(0).load_molecule(xyz, read_fixture("basis", a.basis)).build_pairs(a.kappa)
e.set_screening(a.tau)
N = e.nbf
rng = np.random.default_rng(0)
C, _ = np.linalg.qr(rng.standard_normal((N, e.nelectrons // 2)))
D = C @ C.T
if a.tune:
    e.tune(D, reps=1)
    print(e.variants())
if a.set:
    from paper_2412_13203_b200.eritile import class_table
    tab = ["".join(map(str, r[:4])) for r in class_table()]
    for kv in a.set:
        c, v = kv.split("=")
        e.set_variant(tab.index(c), v)
if a.variants_json:
    import json
    json.dump({"".join(map(str, k[:4])) if not isinstance(k, str) else k: v for k, v in e.variants().items()},
              open(a.variants_json, "w"))
if a.profile_range:
    import torch
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
for _ in range(a.builds):
    J, K = e.build_jk(D)
if a.profile_range:
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
print(e.stats())
