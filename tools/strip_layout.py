"""Whole-build time (the bench's timed step, tuned per layout) for strip layouts
set_strips(min survivors per strip bra, max items per strip) on (H2O)_n.

  python tools/strip_layout.py --waters 80 --set 1024,1024 --set 256,4096
"""
import argparse
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from bench import synthetic_density  # noqa: E402
from paper_2412_13203_b200.eritile import Engine, read_fixture  # noqa: E402
from paper_2412_13203_b200.geometry import water_cluster  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--waters", type=int, default=80)
ap.add_argument("--set", action="append", default=[])
ap.add_argument("--builds", type=int, default=5)
a = ap.parse_args()
stream = torch.cuda.Stream()  # non-null: handle 0 would select the engine's own stream
sp = stream.cuda_stream
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for kv in a.set or ["1024,1024"]:
    smin, smax = (int(x) for x in kv.split(","))
    e = Engine(0).load_molecule(water_cluster(a.waters), read_fixture("basis", "cc-pvdz.txt")).build_pairs(1e-14)
    e.set_strips(smin, smax)
    e.set_screening(1e-10)
    N = e.nbf
    Dh = synthetic_density(N, e.nelectrons // 2)
    e.tune(Dh, reps=2)
    e.tune_granularity(Dh, reps=3)
    D = torch.from_numpy(Dh).cuda()
    JK = torch.zeros(2 * N * N, dtype=torch.float64, device="cuda")
    J, K = torch.empty_like(D), torch.empty_like(D)
    ts = []
    for i in range(a.builds + 2):
        with torch.cuda.stream(stream):
            flush.fill_(i & 255)
            t0, t1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t0.record(stream)
            e.build_jk_partial_device(D.data_ptr(), JK.data_ptr(), sp)
            e.finalize_device(JK.data_ptr(), J.data_ptr(), K.data_ptr(), sp)
            t1.record(stream)
        torch.cuda.synchronize()
        if i >= 2:
            ts.append(t0.elapsed_time(t1))
    print(f"strips min={smin:5d} max={smax:5d}: min {min(ts):.1f} ms  median {np.median(ts):.1f} ms", flush=True)
    del e
