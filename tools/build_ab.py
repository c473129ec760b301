"""A/B of whole concurrent builds (the bench's timed step) with variant
overrides on top of the tuned table: the tuner times each class alone, so it
cannot see how a variant loads the shared L2 atomic units while other classes
run concurrently.

  python tools/build_ab.py --waters 80 --ab 2010=strip_p_t512 --ab 2010=strip_p_t512,1110=lane_pl384
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
ap.add_argument("--ab", action="append", default=[])
ap.add_argument("--builds", type=int, default=7)
a = ap.parse_args()
e = Engine(0).load_molecule(water_cluster(a.waters), read_fixture("basis", "cc-pvdz.txt")).build_pairs(1e-14)
e.set_screening(1e-10)
N = e.nbf
Dh = synthetic_density(N, e.nelectrons // 2)
e.tune(Dh, reps=2)
table = e.get_variants().tolist()
e.tune_granularity(Dh, reps=3)
tab = ["".join(map(str, r[:4])) for r in class_table()]
D = torch.from_numpy(Dh).cuda()
JK = torch.zeros(2 * N * N, dtype=torch.float64, device="cuda")
J = torch.empty_like(D)
K = torch.empty_like(D)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
stream = torch.cuda.Stream()  # (a non-null stream: handle 0 would select the engine's own stream)
sp = stream.cuda_stream


def timed():
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
    return min(ts), float(np.median(ts))


for trial in range(2):
    e.set_variants(table)
    mn, md = timed()
    print(f"{'tuned':22s} min {mn:.1f} ms  median {md:.1f} ms", flush=True)
    for ab in a.ab:
        e.set_variants(table)
        for kv in ab.split(","):
            c, v = kv.split("=")
            e.set_variant(tab.index(c), v)
        mn, md = timed()
        print(f"{ab:22s} min {mn:.1f} ms  median {md:.1f} ms", flush=True)
