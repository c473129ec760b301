"""Python host mirror of the reference interface over the C ABI.

The reference (proj/include/eritile) is C++; its executor contract is
``build_g(blocks, plans, D, mode) -> G`` called by
``scf_iterate``. ``Engine`` exposes the same steps with the
reference's names — ``build_pairs`` (block.hpp:52), ``schwarz``,
``build_jk``/``build_g`` — over ``include/eritile_gpu.h``. Errors raise the
reference's exception kinds (ParseError, ValueError for invalid_argument,
ArithmeticError for domain_error, RuntimeError for device failures).

There is no CPU fallback: if the CUDA library is missing or no device is
present, construction raises.
"""
from __future__ import annotations

import ctypes as C
from pathlib import Path
from typing import Optional, Tuple

import numpy as np

from . import _native

_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_ip = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")

DATA = Path(__file__).resolve().parent / "data"


class ParseError(ValueError):
    """eritile::ParseError (molecule.hpp:72-74)."""


class Stats(C.Structure):
    _fields_ = [("nbf", C.c_int), ("nshells", C.c_int), ("npairs", C.c_int), ("nclasses", C.c_int),
                ("quartets", C.c_longlong), ("prim_quartets", C.c_longlong),
                ("work_items", C.c_longlong), ("model_flops", C.c_double),
                ("last_build_ms", C.c_double), ("last_schwarz_ms", C.c_double),
                ("gpu_launches_last_build", C.c_int),
                ("job_quartets", C.c_longlong), ("job_prim_quartets", C.c_longlong),
                ("job_model_flops", C.c_double),
                ("pair_path_prim_quartets", C.c_longlong), ("pair_path_model_flops", C.c_double)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


def _lib():
    lib = _native.load()
    if getattr(lib, "_eritile_bound", False):
        return lib
    sig = {
        "eritile_gpu_create": (C.c_int, [C.c_int, C.POINTER(C.c_void_p)]),
        "eritile_gpu_destroy": (None, [C.c_void_p]),
        "eritile_gpu_last_error": (C.c_char_p, [C.c_void_p]),
        "eritile_gpu_load_molecule": (C.c_int, [C.c_void_p, C.c_char_p, C.c_char_p]),
        "eritile_gpu_load_shells": (C.c_int, [C.c_void_p, C.c_int, _ip, _ip, _dp, _ip, _dp, _dp, C.c_int,
                                              _ip, _dp]),
        "eritile_gpu_nbf": (C.c_int, [C.c_void_p]),
        "eritile_gpu_nshells": (C.c_int, [C.c_void_p]),
        "eritile_gpu_shell_info": (C.c_int, [C.c_void_p, _ip, _ip, _ip]),
        "eritile_gpu_nelectrons": (C.c_int, [C.c_void_p]),
        "eritile_gpu_nuclear_repulsion": (C.c_double, [C.c_void_p]),
        "eritile_gpu_build_pairs": (C.c_int, [C.c_void_p, C.c_double]),
        "eritile_gpu_npairs": (C.c_int, [C.c_void_p]),
        "eritile_gpu_pair_shells": (C.c_int, [C.c_void_p, _ip, _ip]),
        "eritile_gpu_schwarz": (C.c_int, [C.c_void_p, C.c_void_p]),
        "eritile_gpu_set_schwarz": (C.c_int, [C.c_void_p, _dp]),
        "eritile_gpu_set_shard": (C.c_int, [C.c_void_p, C.c_int, C.c_int]),
        "eritile_gpu_set_screening": (C.c_int, [C.c_void_p, C.c_double]),
        "eritile_gpu_num_quartets": (C.c_longlong, [C.c_void_p]),
        "eritile_gpu_quartets": (C.c_longlong, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_longlong]),
        "eritile_gpu_pair_survivors": (C.c_longlong, [C.c_void_p, C.c_void_p, C.c_void_p]),
        "eritile_gpu_get_variants": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int]),
        "eritile_gpu_set_variants": (C.c_int, [C.c_void_p, _ip, C.c_int]),
        "eritile_gpu_build_jk": (C.c_int, [C.c_void_p, _dp, _dp, _dp]),
        "eritile_gpu_build_jk_partial_device": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p]),
        "eritile_gpu_finalize_device": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                                  C.c_void_p]),
        "eritile_gpu_build_jk_device": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                                  C.c_void_p]),
        "eritile_gpu_one_electron": (C.c_int, [C.c_void_p, _dp, _dp, _dp]),
        "eritile_gpu_boys": (C.c_int, [C.c_void_p, C.c_int, _dp, C.c_int, _dp]),
        "eritile_gpu_eri_quartet": (C.c_int, [C.c_void_p, C.c_int, C.c_int, _dp]),
        "eritile_gpu_get_stats": (C.c_int, [C.c_void_p, C.POINTER(Stats)]),
        "eritile_gpu_num_classes": (C.c_int, []),
        "eritile_gpu_set_profiling": (C.c_int, [C.c_void_p, C.c_int]),
        "eritile_gpu_class_profile": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p,
                                                C.c_void_p, C.c_void_p]),
        "eritile_gpu_class_info": (C.c_int, [C.c_int, _ip]),
        "eritile_gpu_tune": (C.c_int, [C.c_void_p, _dp, C.c_int]),
        "eritile_gpu_set_variant": (C.c_int, [C.c_void_p, C.c_int, C.c_int]),
        "eritile_gpu_tune_times": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_void_p]),
        "eritile_gpu_max_variants": (C.c_int, []),
        "eritile_gpu_tune_granularity": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_int]),
        "eritile_gpu_tune_step": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int]),
        "eritile_gpu_get_granularity": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int]),
        "eritile_gpu_set_granularity": (C.c_int, [C.c_void_p, C.c_int, C.c_int]),
        "eritile_gpu_granularity_history": (C.c_int, [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_void_p,
                                                      C.c_void_p, C.c_void_p]),
        "eritile_alloc_simulate": (C.c_int, [C.c_int, C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_void_p,
                                             C.c_void_p]),
        "eritile_gpu_set_families": (C.c_int, [C.c_void_p, C.c_int]),
        "eritile_gpu_set_concurrent": (C.c_int, [C.c_void_p, C.c_int]),
        "eritile_gpu_set_strips": (C.c_int, [C.c_void_p, C.c_longlong, C.c_int]),
        "eritile_gpu_set_mode": (C.c_int, [C.c_void_p, C.c_int]),
        "eritile_gpu_get_mode": (C.c_int, [C.c_void_p]),
        "eritile_gpu_pair_nprims": (C.c_int, [C.c_void_p, _ip]),
        "eritile_gpu_variant_range": (C.c_int, [C.c_void_p, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
        "eritile_gpu_get_variant": (C.c_int, [C.c_void_p, C.c_int]),
        "eritile_gpu_class_nvariants": (C.c_int, [C.c_int]),
        "eritile_gpu_variant_name": (C.c_char_p, [C.c_int, C.c_int]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    lib._eritile_bound = True
    return lib


def class_table():
    """Plan statistics of the generated class kernels (la lb lc ld max_m ops
    prim_terms base contract hrr_terms)."""
    lib = _lib()
    out = []
    for i in range(lib.eritile_gpu_num_classes()):
        v = np.zeros(10, np.int32)
        lib.eritile_gpu_class_info(i, v)
        out.append(tuple(int(t) for t in v))
    return out


def read_fixture(kind: str, name: str) -> str:
    return (DATA / kind / name).read_text()


class Engine:
    """One molecule + basis on one CUDA device (one rank of a sharded build)."""

    def __init__(self, device: int = 0):
        self._lib = _lib()
        h = C.c_void_p()
        rc = self._lib.eritile_gpu_create(device, C.byref(h))
        if rc != 0:
            raise RuntimeError("eritile_gpu_create failed: " + self._lib.eritile_gpu_last_error(None).decode())
        self._h = h
        self.device = device

    def close(self):
        if getattr(self, "_h", None):
            self._lib.eritile_gpu_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # -- error mapping (reference exception kinds)
    def _check(self, rc: int):
        if rc == 0:
            return
        msg = self._lib.eritile_gpu_last_error(self._h).decode()
        if rc == -2:
            raise ParseError(msg)
        if rc == -1:
            raise ValueError(msg)
        if rc == -5:
            raise ArithmeticError(msg)
        raise RuntimeError(msg)

    # -- input (molecule.hpp:105, basis_set.hpp:33,127)
    def load_molecule(self, xyz_text: str, basis_text: str) -> "Engine":
        self._check(self._lib.eritile_gpu_load_molecule(self._h, xyz_text.encode(), basis_text.encode()))
        return self

    @property
    def nbf(self) -> int:
        return self._lib.eritile_gpu_nbf(self._h)

    @property
    def nshells(self) -> int:
        return self._lib.eritile_gpu_nshells(self._h)

    @property
    def nelectrons(self) -> int:
        return self._lib.eritile_gpu_nelectrons(self._h)

    @property
    def npairs(self) -> int:
        return self._lib.eritile_gpu_npairs(self._h)

    def nuclear_repulsion(self) -> float:
        return self._lib.eritile_gpu_nuclear_repulsion(self._h)

    # -- block constructor (block.hpp:52-150)
    def build_pairs(self, kappa_screen: float = 0.0) -> "Engine":
        self._check(self._lib.eritile_gpu_build_pairs(self._h, kappa_screen))
        return self

    def pair_shells(self) -> Tuple[np.ndarray, np.ndarray]:
        n = self.npairs
        i, j = np.zeros(n, np.int32), np.zeros(n, np.int32)
        self._check(self._lib.eritile_gpu_pair_shells(self._h, i, j))
        return i, j

    def schwarz(self) -> np.ndarray:
        Q = np.zeros(self.npairs)
        self._check(self._lib.eritile_gpu_schwarz(self._h, Q.ctypes.data))
        return Q

    def set_schwarz(self, Q: np.ndarray):
        self._check(self._lib.eritile_gpu_set_schwarz(self._h, np.ascontiguousarray(Q, np.float64)))

    def set_shard(self, rank: int, nranks: int) -> "Engine":
        self._check(self._lib.eritile_gpu_set_shard(self._h, rank, nranks))
        return self

    def set_screening(self, tau: float) -> "Engine":
        self._check(self._lib.eritile_gpu_set_screening(self._h, tau))
        return self

    def num_quartets(self) -> int:
        return self._lib.eritile_gpu_num_quartets(self._h)

    def quartets(self) -> Tuple[np.ndarray, np.ndarray]:
        n = self._lib.eritile_gpu_quartets(self._h, None, None, 0)
        if n < 0:
            raise RuntimeError("quartets before set_screening")
        xs, ys = np.zeros(max(n, 1), np.int32), np.zeros(max(n, 1), np.int32)
        self._lib.eritile_gpu_quartets(self._h, xs.ctypes.data, ys.ctypes.data, n)
        return xs[:n], ys[:n]

    def pair_survivors(self):
        """(count, ysum, total): per reference pair x, this rank's canonical
        quartets (x, y >= x) and the wrapping sum of splitmix64(y) over them."""
        n = self.npairs
        cnt = np.zeros(n, np.int64)
        ysum = np.zeros(n, np.uint64)
        tot = self._lib.eritile_gpu_pair_survivors(self._h, cnt.ctypes.data, ysum.ctypes.data)
        if tot < 0:
            raise RuntimeError("pair_survivors before set_screening")
        return cnt, ysum, int(tot)

    def get_variants(self) -> np.ndarray:
        """The whole variant table (one index per class)."""
        n = self._lib.eritile_gpu_get_variants(self._h, None, 0)
        v = np.zeros(n, np.int32)
        self._lib.eritile_gpu_get_variants(self._h, v.ctypes.data, n)
        return v

    def set_variants(self, var) -> "Engine":
        v = np.ascontiguousarray(var, dtype=np.int32)
        self._check(self._lib.eritile_gpu_set_variants(self._h, v, len(v)))
        return self

    # -- executor
    def build_jk(self, D: np.ndarray, out: Optional[Tuple[np.ndarray, np.ndarray]] = None) -> Tuple[np.ndarray, np.ndarray]:
        """J, K of density D through eritile_gpu_build_jk (host buffers). ``out``:
        caller-owned (N, N) float64 C-contiguous arrays to write into (e.g.
        page-locked ones, for full-rate copies)."""
        N = self.nbf
        D = np.ascontiguousarray(D, dtype=np.float64)
        if D.shape != (N, N):
            raise ValueError(f"density must be {N}x{N}")
        if out is None:
            J, K = np.zeros((N, N)), np.zeros((N, N))
        else:
            J, K = out
            for M in (J, K):
                if M.shape != (N, N) or M.dtype != np.float64 or not M.flags.c_contiguous:
                    raise ValueError(f"out arrays must be C-contiguous float64 {N}x{N}")
        self._check(self._lib.eritile_gpu_build_jk(self._h, D, J, K))
        return J, K

    def build_g(self, D: np.ndarray) -> np.ndarray:
        """G = 2J - K for closed-shell RHF."""
        J, K = self.build_jk(D)
        return 2.0 * J - K

    def build_jk_device(self, D_ptr: int, J_ptr: int, K_ptr: int, stream: int = 0):
        self._check(self._lib.eritile_gpu_build_jk_device(self._h, C.c_void_p(D_ptr), C.c_void_p(J_ptr),
                                                          C.c_void_p(K_ptr), C.c_void_p(stream or None)))

    def build_jk_partial_device(self, D_ptr: int, JKacc_ptr: int, stream: int = 0):
        self._check(self._lib.eritile_gpu_build_jk_partial_device(self._h, C.c_void_p(D_ptr),
                                                                  C.c_void_p(JKacc_ptr),
                                                                  C.c_void_p(stream or None)))

    def finalize_device(self, JKacc_ptr: int, J_ptr: int, K_ptr: int, stream: int = 0):
        self._check(self._lib.eritile_gpu_finalize_device(self._h, C.c_void_p(JKacc_ptr), C.c_void_p(J_ptr),
                                                          C.c_void_p(K_ptr), C.c_void_p(stream or None)))

    def one_electron(self):
        N = self.nbf
        S, T, V = np.zeros((N, N)), np.zeros((N, N)), np.zeros((N, N))
        self._check(self._lib.eritile_gpu_one_electron(self._h, S, T, V))
        return S, T, V

    def boys(self, m_max: int, T) -> np.ndarray:
        T = np.ascontiguousarray(np.atleast_1d(T), dtype=np.float64)
        F = np.zeros(len(T) * (m_max + 1))
        self._check(self._lib.eritile_gpu_boys(self._h, m_max, T, len(T), F))
        return F.reshape(len(T), m_max + 1)

    def shell_info(self):
        n = self.nshells
        L, K, off = (np.zeros(n, np.int32) for _ in range(3))
        self._check(self._lib.eritile_gpu_shell_info(self._h, L, K, off))
        return L, K, off

    def eri_quartet(self, x: int, y: int) -> np.ndarray:
        """Scaled integrals of reference pairs (x, y), a-major over the
        components of (i, j, k, l) (dag.hpp:221-229)."""
        L, _, _ = self.shell_info()
        i, j = self.pair_shells()
        nc = lambda l: (l + 1) * (l + 2) // 2
        n = nc(L[i[x]]) * nc(L[j[x]]) * nc(L[i[y]]) * nc(L[j[y]])
        out = np.zeros(n)
        self._check(self._lib.eritile_gpu_eri_quartet(self._h, x, y, out))
        return out

    def set_profiling(self, on: bool = True):
        self._check(self._lib.eritile_gpu_set_profiling(self._h, int(on)))

    def class_profile(self):
        """Per-class launch records of the last build (profiling mode)."""
        n = self._lib.eritile_gpu_class_profile(self._h, 0, None, None, None, None, None)
        if n < 0:
            self._check(n)
        cls = np.zeros(4 * max(n, 1), np.int32)
        ms, fl = np.zeros(max(n, 1)), np.zeros(max(n, 1))
        q, pq = np.zeros(max(n, 1), np.int64), np.zeros(max(n, 1), np.int64)
        self._lib.eritile_gpu_class_profile(self._h, n, cls.ctypes.data, ms.ctypes.data, fl.ctypes.data,
                                            q.ctypes.data, pq.ctypes.data)
        return [dict(cls=tuple(int(v) for v in cls[4 * i:4 * i + 4]), ms=float(ms[i]), flops=float(fl[i]),
                     quartets=int(q[i]), prim_quartets=int(pq[i])) for i in range(n)]

    def tune(self, D: np.ndarray, reps: int = 3) -> "Engine":
        """Workload Allocator: pick the fastest kernel variant per class on
        density D."""
        D = np.ascontiguousarray(D, dtype=np.float64)
        self._check(self._lib.eritile_gpu_tune(self._h, D, int(reps)))
        return self

    def set_families(self, on: bool = True) -> "Engine":
        """Shared-primitive units for generally contracted sibling shells
        (csrc/jk_family.cuh); takes effect at the next set_screening."""
        self._check(self._lib.eritile_gpu_set_families(self._h, int(on)))
        return self

    def set_strips(self, min_quartets: int = 1024, max_items: int = 1024) -> "Engine":
        """Strip layout of the work lists (csrc/jk_strip.cuh); takes effect at
        the next set_screening."""
        self._check(self._lib.eritile_gpu_set_strips(self._h, int(min_quartets), int(max_items)))
        return self

    def set_mode(self, mode: str = "concurrent") -> "Engine":
        """build_g reduction mode (SPEC.md executor): "concurrent" (FP64
        atomics) or "deterministic" (fixed-point integer sums, bitwise
        reproducible)."""
        m = {"concurrent": 0, "deterministic": 1}[mode]
        self._check(self._lib.eritile_gpu_set_mode(self._h, m))
        return self

    @property
    def mode(self) -> str:
        return ["concurrent", "deterministic"][self._lib.eritile_gpu_get_mode(self._h)]

    def pair_nprims(self) -> np.ndarray:
        n = np.zeros(self.npairs, np.int32)
        self._check(self._lib.eritile_gpu_pair_nprims(self._h, n))
        return n

    def set_concurrent(self, on: bool = True) -> "Engine":
        """Class launches on 4 streams (default) or serialised on one."""
        self._check(self._lib.eritile_gpu_set_concurrent(self._h, int(on)))
        return self

    def variant_range(self, cls_index: int):
        lo, hi = C.c_int(), C.c_int()
        self._check(self._lib.eritile_gpu_variant_range(self._h, int(cls_index), C.byref(lo), C.byref(hi)))
        return lo.value, hi.value

    def set_variant(self, cls_index: int, var) -> "Engine":
        if isinstance(var, str):
            var = variant_names(cls_index).index(var)
        self._check(self._lib.eritile_gpu_set_variant(self._h, int(cls_index), int(var)))
        return self

    def tune_granularity(self, D: np.ndarray, reps: int = 3, max_sweeps: int = 64) -> int:
        """Workload Allocator Alg. 2: per
        class, double the work items per warp task while the measured class
        time drops (combine / measure / revert), to convergence. Returns the
        number of accepted combines."""
        D = np.ascontiguousarray(D, dtype=np.float64)
        rc = self._lib.eritile_gpu_tune_granularity(self._h, D.ctypes.data, reps, max_sweeps)
        if rc < 0:
            self._check(rc)
        return rc

    def tune_step(self, D: np.ndarray, reps: int = 3) -> bool:
        """One Alg. 2 sweep over the classes (SCF drivers interleave it with
        their first iterations). True if some class improved."""
        D = np.ascontiguousarray(D, dtype=np.float64)
        rc = self._lib.eritile_gpu_tune_step(self._h, D.ctypes.data, reps)
        if rc < 0:
            self._check(rc)
        return rc == 1

    def granularity(self) -> dict:
        """{class (la,lb,lc,ld) string: g} for every class."""
        n = self._lib.eritile_gpu_get_granularity(self._h, None, 0)
        g = np.zeros(n, np.int32)
        self._lib.eritile_gpu_get_granularity(self._h, g.ctypes.data, n)
        tab = class_table()
        return {"".join(map(str, tab[c][:4])): int(g[c]) for c in range(n)}

    def set_granularity(self, cls_index: int, g: int) -> "Engine":
        self._check(self._lib.eritile_gpu_set_granularity(self._h, cls_index, g))
        return self

    def granularity_history(self, cls_index: int):
        """[(g, median ms, spread ms, accepted)] of every Alg. 2 measurement."""
        n = self._lib.eritile_gpu_granularity_history(self._h, cls_index, 0, None, None, None, None)
        if n < 0:
            self._check(n)
        g = np.zeros(max(n, 1), np.int32)
        ms, sp = np.zeros(max(n, 1)), np.zeros(max(n, 1))
        acc = np.zeros(max(n, 1), np.int32)
        self._lib.eritile_gpu_granularity_history(self._h, cls_index, n, g.ctypes.data, ms.ctypes.data,
                                                  sp.ctypes.data, acc.ctypes.data)
        return [(int(g[k]), float(ms[k]), float(sp[k]), bool(acc[k])) for k in range(n)]

    def tune_times(self) -> dict:
        """{class: {variant name: median ms}} of the last tune."""
        n = self._lib.eritile_gpu_tune_times(self._h, 0, None, None)
        ci = np.zeros(max(n, 1), np.int32)
        nv = self._lib.eritile_gpu_max_variants()
        ms = np.zeros(nv * max(n, 1))
        self._lib.eritile_gpu_tune_times(self._h, n, ci.ctypes.data, ms.ctypes.data)
        tab = class_table()
        out = {}
        for w in range(n):
            names = variant_names(int(ci[w]))
            out["".join(map(str, tab[ci[w]][:4]))] = {nm: round(float(ms[nv * w + v]), 4) for v, nm in enumerate(names) if ms[nv * w + v] > 0}
        return out

    def variants(self) -> dict:
        """{class (la,lb,lc,ld): chosen variant name}."""
        out = {}
        for i, row in enumerate(class_table()):
            v = self._lib.eritile_gpu_get_variant(self._h, i)
            out[tuple(int(x) for x in row[:4])] = variant_names(i)[v]
        return out

    def stats(self) -> dict:
        s = Stats()
        self._check(self._lib.eritile_gpu_get_stats(self._h, C.byref(s)))
        return s.as_dict()


def alloc_simulate(cost, cap, max_sweeps: int = 64):
    """Run the Workload Allocator loop (Alg. 2, csrc/host/allocator.h) against
    a mock cost table: cost[c][k] = time of class c at g = 2**k (no device).
    Returns (g per class, accepted combines, sweeps)."""
    cost = np.ascontiguousarray(cost, dtype=np.float64)
    cap = np.ascontiguousarray(cap, dtype=np.int32)
    ncls, stride = cost.shape
    g = np.zeros(ncls, np.int32)
    sweeps = np.zeros(1, np.int32)
    acc = _lib().eritile_alloc_simulate(ncls, cap.ctypes.data, cost.ctypes.data, stride, max_sweeps, g.ctypes.data,
                                        sweeps.ctypes.data)
    if acc < 0:
        raise ValueError("alloc_simulate: bad arguments (the cost table must cover g = 1 .. cap)")
    return g, int(acc), int(sweeps[0])


def variant_names(cls_index: int):
    lib = _lib()
    return [lib.eritile_gpu_variant_name(cls_index, v).decode()
            for v in range(lib.eritile_gpu_class_nvariants(cls_index))]


def engine_for(xyz_text: str, basis_text: str, tau: float = 1e-10, device: int = 0,
               kappa_screen: float = 0.0, rank: int = 0, nranks: int = 1) -> Engine:
    """Convenience: load, build pairs, Schwarz, shard, screen."""
    e = Engine(device).load_molecule(xyz_text, basis_text).build_pairs(kappa_screen)
    e.set_shard(rank, nranks)
    e.set_screening(tau)
    return e
