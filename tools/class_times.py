"""Per-class device times of one (H2O)_n build with fixed variants.

  python tools/class_times.py --waters 80 --set 1000=fstrip_a_t768 ...
"""
import argparse
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2412_13203_b200.eritile import Engine, class_table, read_fixture  # noqa: E402
from paper_2412_13203_b200.geometry import water_cluster  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--waters", type=int, default=80)
ap.add_argument("--basis", default="cc-pvdz.txt")
ap.add_argument("--set", action="append", default=[])
ap.add_argument("--builds", type=int, default=3)
a = ap.parse_args()
e = Engine(0).load_molecule(water_cluster(a.waters), read_fixture("basis", a.basis)).build_pairs(1e-14)
e.set_screening(1e-10)
N = e.nbf
rng = np.random.default_rng(0)
C, _ = np.linalg.qr(rng.standard_normal((N, e.nelectrons // 2)))
D = C @ C.T
tab = ["".join(map(str, r[:4])) for r in class_table()]
for kv in a.set:
    c, v = kv.split("=")
    e.set_variant(tab.index(c), v)
e.build_jk(D)
e.set_profiling(True)
best = {}
for _ in range(a.builds):
    e.build_jk(D)
    for r in e.class_profile():
        k = "".join(map(str, r["cls"]))
        best[k] = min(best.get(k, 1e9), r["ms"])
print(" ".join(f"{k}:{v:.2f}" for k, v in sorted(best.items(), key=lambda kv: -kv[1])[:12]))
