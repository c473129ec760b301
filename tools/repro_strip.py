"""Repro: strip kernels on (H2O)_8/cc-pVDZ with small strip thresholds."""
import sys
from pathlib import Path
import numpy as np
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
from systems import BASIS, geom
from paper_2412_13203_b200.eritile import Engine, class_table, variant_names

xyz, bas = geom(sys.argv[1] if len(sys.argv) > 1 else "w8"), BASIS["cc-pvdz"]
smin, smax = 64, 256
for fam in (False, True):
    e = Engine(0).load_molecule(xyz, bas).build_pairs(1e-14)
    e.set_families(fam).set_strips(smin, smax)
    e.set_screening(1e-10)
    N = e.nbf
    D = np.eye(N)
    for i in range(len(class_table())):
        names = variant_names(i)
        want = "fstrip" if fam else "strip"
        k = next((j for j, n in enumerate(names) if n.startswith(want)), None)
        if k is None:
            continue
        e.set_variant(i, k)
        try:
            e.build_jk(D)
            print("ok", fam, class_table()[i], names[k], flush=True)
        except Exception as ex:
            print("FAIL", fam, class_table()[i], names[k], ex, flush=True)
            e = Engine(0).load_molecule(xyz, bas).build_pairs(1e-14)
            e.set_families(fam).set_strips(smin, smax)
            e.set_screening(1e-10)
