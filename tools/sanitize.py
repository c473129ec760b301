"""compute-sanitizer driver: one Fock build per kernel variant
name (set on every class that has it) on small systems, strips forced on, so
every kernel family (lane, unit, strip, coop/coopw) and the Schwarz / raw
quartet kernels run under memcheck / racecheck / synccheck.

  compute-sanitizer --tool memcheck python tools/sanitize.py [--quick]
"""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))
from systems import BASIS, geom  # noqa: E402
from paper_2412_13203_b200.eritile import Engine, class_table, variant_names  # noqa: E402

quick = "--quick" in sys.argv
systems = [("water", "cc-pvdz", 0.0), ("w2", "cc-pvdz", 1e-14)] if quick else \
    [("water", "cc-pvdz", 0.0), ("w2", "cc-pvdz", 1e-14), ("benzene", "6-31g*", 0.0), ("water", "cc-pvtz", 1e-14)]
ncls = len(class_table())
names = sorted({n for i in range(ncls) for n in variant_names(i)})
runs = 0
for mol, bas, kappa in systems:
    for fam in (False, True):
        e = Engine(0).load_molecule(geom(mol), BASIS[bas]).build_pairs(kappa)
        e.set_families(fam).set_strips(1, 16)
        e.set_screening(1e-10)
        N = e.nbf
        rng = np.random.default_rng(1)
        A = rng.standard_normal((N, N))
        D = (A + A.T) / np.sqrt(N)
        for vn in names:
            if vn.startswith(("fam_", "fstrip")) != fam:
                continue
            hit = False
            for i in range(ncls):
                if vn in variant_names(i):
                    e.set_variant(i, vn)
                    hit = True
            if not hit:
                continue
            for i in range(ncls):
                e.set_granularity(i, 2 if runs % 2 else 1)
            e.build_jk(D)
            runs += 1
        e.eri_quartet(0, e.npairs - 1)
    print(f"{mol}/{bas}: ok", flush=True)
print(f"sanitize: {runs} builds over {len(names)} variant names")
