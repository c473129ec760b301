"""Per-class device time of chosen variants on one (H2O)_n build (min over builds).

  python tools/variant_compare.py --waters 80 --cls 1000,1010 --var fstrip_o7_t512,fstrip_w_t768
"""
import argparse
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2412_13203_b200.eritile import Engine, class_table, read_fixture, variant_names  # noqa: E402
from paper_2412_13203_b200.geometry import water_cluster  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--waters", type=int, default=80)
ap.add_argument("--basis", default="cc-pvdz.txt")
ap.add_argument("--cls", default="1000,1010,0000,1100,2000")
ap.add_argument("--var", default="fstrip_o7_t512,fstrip_a_t512,fstrip_p_t512,fstrip_sk2_t768")
ap.add_argument("--builds", type=int, default=3)
a = ap.parse_args()
e = Engine(0).load_molecule(water_cluster(a.waters), read_fixture("basis", a.basis)).build_pairs(1e-14)
e.set_screening(1e-10)
N = e.nbf
rng = np.random.default_rng(0)
C, _ = np.linalg.qr(rng.standard_normal((N, e.nelectrons // 2)))
D = C @ C.T
tab = ["".join(map(str, r[:4])) for r in class_table()]
e.build_jk(D)
e.set_profiling(True)
for c in a.cls.split(","):
    ci = tab.index(c)
    row = []
    for v in a.var.split(","):
        if v not in variant_names(ci):
            continue
        e.set_variant(ci, v)
        e.build_jk(D)
        best = 1e9
        for _ in range(a.builds):
            e.build_jk(D)
            for r in e.class_profile():
                if "".join(map(str, r["cls"])) == c:
                    best = min(best, r["ms"])
        row.append(f"{v}={best:.2f}")
    print(c, " ".join(row), flush=True)
