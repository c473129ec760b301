"""Strip layout sweep on one tuned (H2O)_n build: device ms per build for
(min survivors per strip bra, max items per strip) settings, variants fixed
from one tune at the default layout.

  python tools/strip_sweep.py --waters 80 --set 1024,1024 --set 256,512 ...
"""
import argparse
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from bench import synthetic_density  # noqa: E402
from paper_2412_13203_b200.eritile import Engine, class_table, read_fixture  # noqa: E402
from paper_2412_13203_b200.geometry import water_cluster  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--waters", type=int, default=80)
ap.add_argument("--set", action="append", default=[])
ap.add_argument("--builds", type=int, default=5)
a = ap.parse_args()
e = Engine(0).load_molecule(water_cluster(a.waters), read_fixture("basis", "cc-pvdz.txt")).build_pairs(1e-14)
e.set_screening(1e-10)
N = e.nbf
Dh = synthetic_density(N, e.nelectrons // 2)
e.tune(Dh)
ncls = len(class_table())
var = [int(e._lib.eritile_gpu_get_variant(e._h, i)) for i in range(ncls)]
D = torch.from_numpy(Dh).cuda()
J = torch.empty_like(D)
K = torch.empty_like(D)
s = torch.cuda.current_stream()
for kv in a.set or ["1024,1024"]:
    smin, smax = (int(x) for x in kv.split(","))
    e.set_strips(smin, smax)
    e.set_screening(1e-10)
    e.set_variants(var)
    for _ in range(2):
        e.build_jk_device(D.data_ptr(), J.data_ptr(), K.data_ptr(), s.cuda_stream)
    ts = []
    for _ in range(a.builds):
        t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        t0.record(s)
        e.build_jk_device(D.data_ptr(), J.data_ptr(), K.data_ptr(), s.cuda_stream)
        t1.record(s)
        torch.cuda.synchronize()
        ts.append(t0.elapsed_time(t1))
    print(f"strips min={smin} max={smax}: {min(ts):.1f} ms (median {np.median(ts):.1f})", flush=True)
