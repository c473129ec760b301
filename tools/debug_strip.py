"""Which strip variants / classes disagree with the oracle (debug aid)."""
import sys
from pathlib import Path
import numpy as np
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
from oracle_lib import Oracle
from systems import BASIS, geom
from paper_2412_13203_b200.eritile import Engine, class_table, variant_names

mol = sys.argv[1] if len(sys.argv) > 1 else "w4"
xyz, bas = geom(mol), BASIS["cc-pvdz"]
O = Oracle("orc").system(xyz, bas, kappa_screen=1e-14)
rng = np.random.default_rng(7)
A = rng.standard_normal((O.nbf, O.nbf)); D = (A + A.T) / np.sqrt(O.nbf)
Jo, Ko, nq = O.build_jk(D, 1e-10)
tab = class_table()
for fam in (False, True):
    pre = "fstrip" if fam else "strip"
    for v in ("_t512", "_o7_t512", "_a_t512", "_p_t512", "_s_t512"):
        name = pre + v
        bad = []
        for i in range(len(tab)):
            if name not in variant_names(i):
                continue
            e = Engine(0).load_molecule(xyz, bas).build_pairs(1e-14)
            e.set_families(fam).set_strips(1, 64)
            e.set_screening(1e-10)
            e.set_variant(i, name)
            J, K = e.build_jk(D)
            dk = np.max(np.abs(K - Ko))
            if dk > 1e-10:
                bad.append(("".join(map(str, tab[i][:4])), f"{dk:.1e}"))
        print(name, "bad:", bad, flush=True)
