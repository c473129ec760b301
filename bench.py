#!/usr/bin/env python
"""Fock-build benchmark (BASELINE.json metric) — one JSON line on rank 0.

Workload: one closed-shell Fock build (Schwarz-screened ERI + J/K digestion)
of the (H2O)_80 water cluster in cc-pVDZ (N = 2000 Cartesian basis
functions; SURVEY.md Appendix D geometry), tau = 1e-10, synthetic density
D = C_occ C_occ^T from a seeded QR. A "step" is one Fock
build. ``value`` = surviving canonical quartets (all ranks) / device time per
build (max over ranks). Quartets are sharded across ranks; the partial J/K
are summed with one NCCL all-reduce per build (the path's real exchange).

  python bench.py [--gpus N --steps K --warmup W] [--impl reference]
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))

METRIC = "Fock-build ERI quartets/s ({mol} {basis}, Schwarz tau={tau:g})"
UNIT = "quartets/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--waters", type=int, default=80)
    ap.add_argument("--basis", default="cc-pvdz")
    ap.add_argument("--geom", default="", help="geometry fixture (e.g. benzene) or ala<n> (idealised "
                                                 "H-(Ala)_n-OH strand, config 5) instead of the water cluster")
    ap.add_argument("--tau", type=float, default=1e-10)
    ap.add_argument("--kappa", type=float, default=1e-14,
                    help="reference primitive-pair screen |coef|*kappa < thr (block.hpp:83-89; "
                         "SPEC.md:188 flag value 1e-14; 0 = off). Both arms use the same value.")
    ap.add_argument("--no-unscreened", action="store_true",
                    help="skip the secondary kappa-off measurement")
    ap.add_argument("--cpu-seconds", type=float, default=12.0, help="target CPU sample length")
    ap.add_argument("--no-cpu", action="store_true")
    return ap.parse_args()


BASIS_FILES = {"sto-3g": "sto-3g.txt", "6-31g*": "6-31gs.txt", "cc-pvdz": "cc-pvdz.txt", "cc-pvtz": "cc-pvtz.txt"}


def workload(args):
    from paper_2412_13203_b200.eritile import read_fixture
    from paper_2412_13203_b200.geometry import alanine_chain, water_cluster
    if args.geom.startswith("ala") and args.geom[3:].isdigit():
        xyz = alanine_chain(int(args.geom[3:]))
    else:
        xyz = read_fixture("geom", args.geom + ".xyz") if args.geom else water_cluster(args.waters)
    return xyz, read_fixture("basis", BASIS_FILES[args.basis])


def synthetic_density(N: int, nocc: int, seed: int = 2412) -> np.ndarray:
    rng = np.random.default_rng(seed)
    Cq, _ = np.linalg.qr(rng.standard_normal((N, nocc)))
    return np.ascontiguousarray(Cq @ Cq.T)


def config(args, nranks):
    mol = args.geom if args.geom else f"(H2O)_{args.waters}"
    return {"workload": f"{mol}/{args.basis} RHF Fock build (ERI + J/K), Schwarz tau={args.tau:g}, "
                        f"kappa screen {args.kappa:g}",
            "n_basis": None, "tau": args.tau, "kappa_screen": args.kappa, "basis": args.basis, "waters": args.waters,
            "density": "synthetic C_occ C_occ^T (seeded QR)", "parallelism": f"quartet-shard x{nranks} + NCCL allreduce(J,K)",
            "l2": "256 MiB buffer written between timed steps (L2 flush)"}


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [t.strip() for t in ln.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
            except ValueError:
                continue
            for n, v in zip(names, f[3:7]):
                if v.lower() == "active":
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        return {"sm_mhz": float(np.median(sm)), "sm_max_mhz": mx, "reasons": sorted(reasons), "samples": len(sm)}


FP64_DATASHEET_TFLOPS = 37.2  # 148 SM x 64 DFMA/clk x 2 x 1.965 GHz


def fp64_peak():
    """FP64 roofline denominator. MEASURED_PEAKS.json (driver-written) has no
    FP64 entry, so this is the FP64 FMA peak measured by this repo's own
    microbenchmark on a B200 of this pool (tools/microbench/fp64_peak.cu,
    profiles/*fp64_peak*.json); the datasheet figure is the fallback."""
    mp = ROOT / "MEASURED_PEAKS.json"
    try:
        v = json.loads(mp.read_text()).get("fp64_tflops")
        if v:
            return float(v), "MEASURED_PEAKS.json fp64_tflops"
    except Exception:
        pass
    for p in sorted((ROOT / "profiles").glob("*fp64_peak*.json")):
        try:
            return float(json.loads(p.read_text())["fp64_fma_tflops"]), (
                f"{p.relative_to(ROOT)}: measured FP64 FMA peak (tools/microbench/fp64_peak.cu); "
                "MEASURED_PEAKS.json has no FP64 entry")
        except Exception:
            pass
    return FP64_DATASHEET_TFLOPS, "fallback: B200 datasheet FP64 (148 SM x 64 DFMA x 2 x 1.965 GHz)"


def ncu_traffic(workload: str, cls: str):
    """DRAM bytes (read + write) of the dominant class launch (all its kernels)
    from an ncu capture of the same workload and class on the current tree
    (profiles/ncu_traffic.json, written by tools/ncu_traffic.sh, which names
    the kernel variant it measured). None when no capture matches."""
    p = ROOT / "profiles" / "ncu_traffic.json"
    if p.exists():
        try:
            for d in json.loads(p.read_text()):
                if d.get("workload") == workload and d.get("cls") == cls:
                    return d.get("dram_bytes_per_launch"), d.get("source")
        except Exception:
            pass
    return None, "no ncu capture of this workload/class on the current tree"


# ------------------------------------------------------------------ CPU arm
def cpu_model() -> str:
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def cpu_sample(args, steps: int, warmup: int, target_s: float, reference_arm: bool):
    """Reference CPU path on the host cores: oracle/_ref (unmodified reference
    headers + SPEC executor) when present, else the C restatement."""
    from oracle_lib import Oracle, available
    kind = "reference" if available("ref") else "port"
    o = Oracle("ref" if kind == "reference" else "orc")
    xyz, basis = workload(args)
    S = o.system(xyz, basis, kappa_screen=args.kappa)
    N = S.nbf
    D = synthetic_density(N, S.nelectrons // 2)
    cores = os.cpu_count() or 1
    t0 = time.perf_counter()
    S.schwarz()
    tq = time.perf_counter() - t0
    nblocks = S.nblocks
    # calibrate: a tiny systematic sample
    stride = max(1, nblocks // 200)
    for _ in range(3):  # calibrate the systematic sample to ~target_s
        _, _, nq, dt = S.build_jk_timed(D, args.tau, cores, stride, 0)
        dt = max(dt, 1e-3)
        if dt > 0.2 * target_s or stride == 1:
            break
        stride = max(1, int(stride * dt / (0.3 * target_s)))
    rate = nq / dt
    per_step = max(1, int(round(stride * dt / max(target_s, 0.5))))  # stride giving ~target_s
    per_step = max(1, min(per_step, nblocks))
    vals, qs, ts = [], 0, 0.0
    for s in range(warmup + steps):
        _, _, nq, dt = S.build_jk_timed(D, args.tau, cores, per_step, (s * 7919) % per_step)
        if s >= warmup:
            vals.append(nq / dt)
            qs += nq
            ts += dt
    value = qs / ts if ts > 0 else rate
    # one host thread on a smaller sample (~target_s / 4): the per-core rate
    st1 = max(per_step, int(per_step * cores * 4))
    st1 = min(st1, nblocks)
    _, _, nq1, dt1 = S.build_jk_timed(D, args.tau, 1, st1, 0)
    return {"value": value, "unit": UNIT, "cores": cores, "kind": kind, "cpu_model": cpu_model(),
            "value_1thread": nq1 / max(dt1, 1e-9),
            "sample_1thread": f"every {st1}-th QuadBlock, {nq1} quartets in {dt1:.1f} s on 1 thread",
            "sample": f"every {per_step}-th of {nblocks} QuadBlocks (M=32) per step, {steps} steps, "
                      f"{qs} quartets in {ts:.1f} s of parallel ERI+digestion time "
                      f"(partial-matrix merge and the {tq:.1f} s Schwarz diagonal excluded)",
            "n_basis": N}


# ------------------------------------------------------------------ GPU arm
def run_ours(args, rank, nranks, local_rank):
    import torch
    # ERITILE_DIST_BACKEND=gloo: test hook that runs N ranks on fewer GPUs
    # (ranks share devices round-robin; NCCL needs one GPU per rank)
    backend = os.environ.get("ERITILE_DIST_BACKEND", "nccl")
    if backend != "nccl":
        local_rank = local_rank % torch.cuda.device_count()
    torch.cuda.set_device(local_rank)
    dist = None
    if nranks > 1:
        import torch.distributed as dist
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        else:
            dist.init_process_group(backend)
    from paper_2412_13203_b200.eritile import Engine

    xyz, basis = workload(args)
    t0 = time.perf_counter()
    eng = Engine(local_rank).load_molecule(xyz, basis).build_pairs(args.kappa)
    eng.set_shard(rank, nranks)
    eng.set_screening(args.tau)
    setup_s = time.perf_counter() - t0
    N = eng.nbf
    Dh = synthetic_density(N, eng.nelectrons // 2)
    dev = torch.device("cuda", local_rank)
    stream = torch.cuda.Stream(dev)  # explicit stream: torch events and our kernels share it
    torch.cuda.set_stream(stream)
    sp = stream.cuda_stream
    D = torch.from_numpy(Dh).to(dev)
    JK = torch.empty(2 * N * N, dtype=torch.float64, device=dev)
    J = torch.empty((N, N), dtype=torch.float64, device=dev)
    K = torch.empty((N, N), dtype=torch.float64, device=dev)
    flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device=dev)

    # Workload Allocator: per-class kernel variant chosen on the live density
    # before the warm-up builds (untimed, like the reference's tune during
    # the first SCF iterations). Rank 0 tunes on the whole
    # lists and broadcasts its table: the LPT deal is a function of the
    # lists and the table, so all ranks must share it (disjoint cover).
    # Then Alg. 2 (combine / measure / revert of the work items per warp
    # task) on the chosen variants; g is broadcast too.
    t1 = time.perf_counter()
    table, gran, accepted = None, None, 0
    if rank == 0:
        eng.tune(Dh, reps=2)
        table = eng.get_variants().tolist()
        accepted = eng.tune_granularity(Dh, reps=3)
        gran = eng.granularity()
    if dist is not None:
        obj = [table, gran]
        dist.broadcast_object_list(obj, src=0)
        table, gran = obj
    eng.set_variants(table)
    from paper_2412_13203_b200.eritile import class_table
    tab = ["".join(map(str, r[:4])) for r in class_table()]
    for k, g in gran.items():
        eng.set_granularity(tab.index(k), g)
    tune_s = time.perf_counter() - t1
    chosen = eng.variants()
    tune_table = eng.tune_times() if rank == 0 else {}
    st = eng.stats()  # after tune: the lists and kernels the timed builds run

    def step():
        eng.build_jk_partial_device(D.data_ptr(), JK.data_ptr(), sp)
        if dist is not None:
            dist.all_reduce(JK)
        eng.finalize_device(JK.data_ptr(), J.data_ptr(), K.data_ptr(), sp)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    launches = eng.stats()["gpu_launches_last_build"] + 1  # + k_finalize (finalize_device)
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    if dist is not None:
        dist.barrier()
    torch.cuda.synchronize()
    prof_range = os.environ.get("ERITILE_PROFILE_RANGE") == "1"  # ncu --profile-from-start off
    if prof_range:
        torch.cuda.profiler.start()
    with ClockSampler(local_rank) as clk:
        for k in range(args.steps):
            flush.fill_(float(k))
            ev[k][0].record(stream)
            step()
            ev[k][1].record(stream)
        torch.cuda.synchronize()
    if prof_range:
        torch.cuda.profiler.stop()
    if dist is not None:
        dist.barrier()
    ms = sum(a.elapsed_time(b) for a, b in ev) / args.steps

    # e2e through the reference-facing C ABI with HOST buffers, every step:
    # eritile_gpu_build_jk(ctx, D, J, K) copies D in, builds, copies J and K
    # out and returns (synchronous), timed on the host clock. Multi-rank runs
    # time the device API + all-reduce with pinned host copies instead (a
    # single rank's build_jk is a partial sum there).
    if nranks == 1:
        e2e_api = "eritile_gpu_build_jk (host buffers: page-locked numpy arrays)"
        Dpin = torch.from_numpy(Dh).pin_memory().numpy()
        Jpin = torch.empty((N, N), dtype=torch.float64).pin_memory().numpy()
        Kpin = torch.empty((N, N), dtype=torch.float64).pin_memory().numpy()
        e2e_t = []
        for k in range(max(args.steps, 1)):
            flush.fill_(float(k))
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            Jh, Kh = eng.build_jk(Dpin, out=(Jpin, Kpin))
            e2e_t.append(time.perf_counter() - t0)
        e2e_ms = 1e3 * sum(e2e_t) / len(e2e_t)
    else:
        e2e_api = "build_jk_partial_device + NCCL all-reduce + finalize, pinned H2D/D2H"
        Dp = torch.from_numpy(Dh).pin_memory()
        Jp = torch.empty((N, N), dtype=torch.float64).pin_memory()
        Kp = torch.empty((N, N), dtype=torch.float64).pin_memory()
        e2e_ev = []
        for k in range(max(args.steps, 1)):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            flush.fill_(float(k))
            a.record(stream)
            D.copy_(Dp, non_blocking=True)
            step()
            Jp.copy_(J, non_blocking=True)
            Kp.copy_(K, non_blocking=True)
            b.record(stream)
            e2e_ev.append((a, b))
        torch.cuda.synchronize()
        e2e_ms = sum(a.elapsed_time(b) for a, b in e2e_ev) / len(e2e_ev)

    # per-class profile (separate, untimed pass)
    eng.set_profiling(True)
    step()
    torch.cuda.synchronize()
    prof = eng.class_profile()
    eng.set_profiling(False)

    # secondary: the same build with the primitive-pair screen off (the
    # reference's default), for transparency (not the headline)
    kappa_off = None
    if args.kappa > 0 and not args.no_unscreened and nranks == 1:
        del eng
        e0 = Engine(local_rank).load_molecule(xyz, basis).build_pairs(0.0)
        e0.set_screening(args.tau)
        e0.tune(Dh, reps=1)
        s0 = e0.stats()
        e0.build_jk_partial_device(D.data_ptr(), JK.data_ptr(), sp)
        ev0 = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(2)]
        for k in range(2):
            flush.fill_(float(k))
            ev0[k][0].record(stream)
            e0.build_jk_partial_device(D.data_ptr(), JK.data_ptr(), sp)
            e0.finalize_device(JK.data_ptr(), J.data_ptr(), K.data_ptr(), sp)
            ev0[k][1].record(stream)
        torch.cuda.synchronize()
        ms0 = sum(a.elapsed_time(b) for a, b in ev0) / 2
        kappa_off = {"kappa_screen": 0.0, "ms_per_step": ms0, "quartets_per_build": s0["quartets"],
                     "prim_quartets_per_build": s0["prim_quartets"], "value": s0["quartets"] / (ms0 * 1e-3),
                     "unit": UNIT, "steps": 2, "warmup": 1}
        del e0

    q_local = st["quartets"]
    pq_local = st["prim_quartets"]
    fl_local = st["model_flops"]
    pair_pq, pair_fl = st["pair_path_prim_quartets"], st["pair_path_model_flops"]
    vals = torch.tensor([ms, e2e_ms], dtype=torch.float64, device=dev)
    sums = torch.tensor([q_local, pq_local, fl_local], dtype=torch.float64, device=dev)
    if dist is not None:
        dist.all_reduce(vals, op=dist.ReduceOp.MAX)
        dist.all_reduce(sums)
    ms, e2e_ms = vals.tolist()
    q_tot, pq_tot, fl_tot = sums.tolist()
    if rank != 0:
        if dist is not None:
            dist.destroy_process_group()
        return None

    peak, peak_src = fp64_peak()
    top = max(prof, key=lambda r: r["ms"]) if prof else None
    total_prof_ms = sum(r["ms"] for r in prof) or 1.0
    roof = None
    if top:
        ach = top["flops"] / (top["ms"] * 1e-3) / 1e12
        kern = "class (%d%d%d%d) launch, variant %s" % (*top["cls"], chosen.get(tuple(top["cls"])))
        traffic, traffic_src = ncu_traffic(config(args, 1)["workload"], "".join(map(str, top["cls"])))
        roof = {"bound": "fp64", "achieved": ach, "peak": peak, "unit": "TFLOP/s", "frac": ach / peak,
                "frac_vs_datasheet": ach / FP64_DATASHEET_TFLOPS,
                "traffic": traffic, "traffic_source": traffic_src,
                "kernel": kern,
                "kernel_share_of_build": top["ms"] / total_prof_ms,
                "kernel_timing": "CUDA events on the launch stream, one serialised profiling build (rank 0)",
                "algorithmic_flops_per_launch": top["flops"],
                "build_frac": (fl_tot / (ms * 1e-3) / 1e12) / (peak * nranks),
                "build_flops_executed": fl_tot,
                "build_flops_pair_path": pair_fl,
                "peak_source": peak_src,
                "flops_model": "SURVEY.md 8d: F_c = Nprim(42+3m+2(P+B+X)) + Nq(2H+12n) with the plans and "
                               "primitive quartets the tuned kernels execute (build_flops_executed); "
                               "build_flops_pair_path counts the same quartets on the per-pair kernels"}
    out = {
        "metric": METRIC.format(mol=args.geom or f"(H2O)_{args.waters}", basis=args.basis, tau=args.tau), "value": q_tot / (ms * 1e-3), "unit": UNIT, "n_gpus": nranks, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (deterministic water-cluster geometry, seeded density)",
        "config": dict(config(args, nranks), n_basis=N),
        "s_per_build": ms * 1e-3,
        "quartets_per_build": int(q_tot), "prim_quartets_per_build": int(pq_tot),
        "prim_quartets_per_s": pq_tot / (ms * 1e-3),
        "prim_quartets_per_build_pair_path": int(pair_pq),
        "e2e": {"value": q_tot / (e2e_ms * 1e-3), "unit": UNIT, "h2d_bytes_per_step": 8 * N * N,
                "d2h_bytes_per_step": 16 * N * N, "ms_per_step": e2e_ms, "api": e2e_api},
        "gpu_launches": launches * args.steps,
        "kappa_off": kappa_off,
        "roofline": roof,
        "clocks": clk.summary(),
        "setup_s": setup_s,
        "tune_s": tune_s,
        "granularity": {"rule": "Alg. 2: work items per warp task, doubled while the class time drops",
                        "accepted_combines": accepted, "g": {k: v for k, v in gran.items() if v > 1}},
        "tune_ms": tune_table,
        "classes": [{"cls": "".join(map(str, r["cls"])), "ms": round(r["ms"], 4),
                     "variant": chosen.get(tuple(r["cls"])),
                     "tflops": r["flops"] / max(r["ms"], 1e-9) / 1e9, "quartets": r["quartets"],
                     "prim_quartets": r["prim_quartets"],
                     "ns_per_prim_quartet_sm": r["ms"] * 1e6 * 148 / max(r["prim_quartets"], 1)}
                    for r in sorted(prof, key=lambda r: -r["ms"])],
    }
    if not args.no_cpu and nranks == 1:
        try:
            cb = cpu_sample(args, steps=1, warmup=0, target_s=args.cpu_seconds, reference_arm=False)
            out["cpu_baseline"] = cb
        except Exception as e:  # the baseline is reported, never the product
            out["cpu_baseline"] = {"value": None, "error": str(e)}
    if dist is not None:
        dist.destroy_process_group()
    return out


def run_reference(args, rank):
    if rank != 0:
        return None
    cb = cpu_sample(args, steps=args.steps, warmup=args.warmup, target_s=args.cpu_seconds, reference_arm=True)
    return {"metric": METRIC.format(mol=args.geom or f"(H2O)_{args.waters}", basis=args.basis, tau=args.tau), "value": cb["value"], "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": None, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (deterministic water-cluster geometry, seeded density)",
            "config": dict(config(args, 1), n_basis=cb["n_basis"]), "impl": "reference",
            "cpu_baseline": cb,
            "e2e": {"value": cb["value"], "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def main():
    args = parse()
    rank = int(os.environ.get("RANK", "0"))
    nranks = int(os.environ.get("WORLD_SIZE", str(args.gpus if args.gpus else 1)))
    if "RANK" not in os.environ:
        nranks = 1
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if args.impl == "reference":
        out = run_reference(args, rank)
    else:
        out = run_ours(args, rank, nranks, local_rank)
    if out is not None:
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
