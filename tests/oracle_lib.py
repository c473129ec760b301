"""ctypes loaders for the CPU checkers (TEST INFRASTRUCTURE ONLY).

* ``Oracle("orc")`` — oracle/_build/liboracle.so, the from-scratch C
  restatement of the reference path (oracle/eri_oracle.c).
* ``Oracle("ref")`` — oracle/_ref/libref_eritile.so, the unmodified reference
  headers (/root/reference/proj/include) compiled with oracle/ref_executor.cpp.

Both expose the same API; tests use them as checkers of the CUDA product and
the product never imports this module.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
LIBS = {
    "orc": ROOT / "oracle" / "_build" / "liboracle.so",
    "ref": ROOT / "oracle" / "_ref" / "libref_eritile.so",
}
_dp = np.ctypeslib.ndpointer(dtype=np.float64, flags="C_CONTIGUOUS")
_ip = np.ctypeslib.ndpointer(dtype=np.int32, flags="C_CONTIGUOUS")


def ensure_built(kind: str) -> bool:
    lib = LIBS[kind]
    if lib.exists():
        return True
    target = "oracle" if kind == "orc" else "ref"
    if kind == "ref" and not Path("/root/reference/proj/include").is_dir():
        return False
    subprocess.run(["make", "-s", "-C", str(ROOT / "oracle"), target], check=True)
    return lib.exists()


def available(kind: str) -> bool:
    try:
        return ensure_built(kind)
    except Exception:
        return False


class Oracle:
    def __init__(self, kind: str):
        if not ensure_built(kind):
            raise RuntimeError(f"checker library {LIBS[kind]} not built")
        self.kind = kind
        self.p = kind + "_"
        lib = C.CDLL(str(LIBS[kind]))
        self.lib = lib
        f = self._f
        f("last_error", C.c_char_p, [])
        f("create", C.c_void_p, [C.c_char_p, C.c_char_p, C.c_double, C.c_int])
        f("destroy", None, [C.c_void_p])
        for n in ("nbf", "nshells", "npairs", "ntiles", "natoms", "nelectrons"):
            f(n, C.c_int, [C.c_void_p])
        f("nblocks", C.c_longlong, [C.c_void_p])
        f("atoms", None, [C.c_void_p, _ip, _dp])
        f("shells", None, [C.c_void_p, _ip, _ip, _ip, _ip, _dp])
        f("shell_prims", None, [C.c_void_p, C.c_int, _dp, _dp])
        f("pairs", None, [C.c_void_p, _ip, _ip, _ip])
        f("pair_prims", None, [C.c_void_p, C.c_int, _dp])
        f("tiles", None, [C.c_void_p, _ip, _ip, _ip, _ip])
        f("boys", None, [C.c_int, C.c_double, _dp])
        f("eri_quartet", C.c_int, [C.c_void_p, C.c_int, C.c_int, _dp])
        f("schwarz", C.c_int, [C.c_void_p, _dp])
        f("set_schwarz", None, [C.c_void_p, _dp])
        f("quartets", C.c_longlong, [C.c_void_p, C.c_double, C.c_void_p, C.c_void_p, C.c_longlong])
        f("build_jk", C.c_int, [C.c_void_p, _dp, C.c_double, C.c_int, _dp, _dp, C.POINTER(C.c_longlong)])
        f("build_jk_sample", C.c_int, [C.c_void_p, _dp, C.c_double, C.c_int, C.c_longlong,
                                        C.c_longlong, _dp, _dp, C.POINTER(C.c_longlong)])
        f("build_jk_timed", C.c_int, [C.c_void_p, _dp, C.c_double, C.c_int, C.c_longlong, C.c_longlong,
                                       _dp, _dp, C.POINTER(C.c_longlong), C.POINTER(C.c_double)])
        f("pair_survivors", C.c_longlong, [C.c_void_p, C.c_double, C.c_void_p, C.c_void_p])
        if kind == "orc":
            f("build_jk_dsparse", C.c_int, [C.c_void_p, _dp, C.c_double, C.c_int, _dp, _dp,
                                            C.POINTER(C.c_longlong)])
            f("build_jk_list", C.c_int, [C.c_void_p, _dp, C.c_longlong, _ip, _ip, C.c_int, _dp, _dp])
            f("one_electron", C.c_int, [C.c_void_p, _dp, _dp, _dp])
            f("nuclear_repulsion", C.c_double, [C.c_void_p])
        else:
            f("plan_stats", None, [C.c_int] * 4 + [C.c_double, C.POINTER(C.c_longlong)])
            f("random_plan_ops", C.c_longlong, [C.c_int] * 4 + [C.c_ulonglong])
            f("emit_source", C.c_longlong, [C.c_int] * 4 + [C.c_char_p, C.c_longlong])

    def _f(self, name, res, args):
        fn = getattr(self.lib, self.p + name)
        fn.restype = res
        fn.argtypes = args
        setattr(self, "_" + name, fn)

    def boys(self, m: int, T: float) -> np.ndarray:
        F = np.zeros(m + 1)
        self._boys(m, T, F)
        return F

    def system(self, xyz: str, basis: str, kappa_screen: float = 0.0, tile_size: int = 32):
        return System(self, xyz, basis, kappa_screen, tile_size)


class System:
    """One molecule + basis inside a checker library."""

    def __init__(self, o: Oracle, xyz: str, basis: str, kappa_screen: float, tile_size: int):
        self.o = o
        self.h = o._create(xyz.encode(), basis.encode(), kappa_screen, tile_size)
        if not self.h:
            raise ValueError(o._last_error().decode())
        self.nbf = o._nbf(self.h)
        self.nshells = o._nshells(self.h)
        self.npairs = o._npairs(self.h)
        self.ntiles = o._ntiles(self.h)
        self.nblocks = o._nblocks(self.h)
        self.natoms = o._natoms(self.h)
        self.nelectrons = o._nelectrons(self.h)

    def __del__(self):
        if getattr(self, "h", None):
            self.o._destroy(self.h)
            self.h = None

    def shells(self):
        S = self.nshells
        L, K, atom, off = (np.zeros(S, np.int32) for _ in range(4))
        cen = np.zeros(3 * S)
        self.o._shells(self.h, L, K, atom, off, cen)
        return dict(L=L, K=K, atom=atom, bf_off=off, center=cen.reshape(S, 3))

    def shell_prims(self, s: int, K: int):
        e, c = np.zeros(K), np.zeros(K)
        self.o._shell_prims(self.h, s, e, c)
        return e, c

    def pairs(self):
        n = self.npairs
        i, j, k = (np.zeros(n, np.int32) for _ in range(3))
        self.o._pairs(self.h, i, j, k)
        return i, j, k

    def pair_prims(self, x: int, nprim: int) -> np.ndarray:
        rec = np.zeros(13 * max(nprim, 1))
        self.o._pair_prims(self.h, x, rec)
        return rec[: 13 * nprim].reshape(nprim, 13)

    def tiles(self):
        n = self.ntiles
        a = [np.zeros(n, np.int32) for _ in range(4)]
        self.o._tiles(self.h, *a)
        return a

    def eri(self, x: int, y: int) -> np.ndarray:
        out = np.zeros(50625)
        n = self.o._eri_quartet(self.h, x, y, out)
        if n < 0:
            raise ValueError(self.o._last_error().decode())
        return out[:n].copy()

    def schwarz(self) -> np.ndarray:
        Q = np.zeros(self.npairs)
        self.o._schwarz(self.h, Q)
        return Q

    def set_schwarz(self, Q: np.ndarray):
        self.o._set_schwarz(self.h, np.ascontiguousarray(Q, dtype=np.float64))

    def quartets(self, tau: float):
        n = self.o._quartets(self.h, tau, None, None, 0)
        xs = np.zeros(max(n, 1), np.int32)
        ys = np.zeros(max(n, 1), np.int32)
        self.o._quartets(self.h, tau, xs.ctypes.data, ys.ctypes.data, n)
        return xs[:n], ys[:n]

    def build_jk(self, D: np.ndarray, tau: float = 0.0, nthreads: int = 0, stride: int = 1,
                 offset: int = 0):
        N = self.nbf
        D = np.ascontiguousarray(D, dtype=np.float64)
        J = np.zeros((N, N))
        K = np.zeros((N, N))
        nq = C.c_longlong(0)
        rc = self.o._build_jk_sample(self.h, D, tau, nthreads, stride, offset, J, K, C.byref(nq))
        if rc != 0:
            raise RuntimeError(self.o._last_error().decode())
        return J, K, nq.value

    def build_jk_dsparse(self, D: np.ndarray, tau: float = 0.0, nthreads: int = 0):
        """True J, K for a density with zero shell blocks: quartets whose six D
        blocks are all zero are skipped (exactly zero contributions)."""
        N = self.nbf
        D = np.ascontiguousarray(D, dtype=np.float64)
        J, K = np.zeros((N, N)), np.zeros((N, N))
        nq = C.c_longlong(0)
        if self.o._build_jk_dsparse(self.h, D, tau, nthreads, J, K, C.byref(nq)) != 0:
            raise RuntimeError(self.o._last_error().decode())
        return J, K, nq.value

    def build_jk_list(self, D: np.ndarray, xs, ys, nthreads: int = 0):
        """True-J/K convention partial sums over an explicit canonical quartet
        list (x <= y): summing the results of a disjoint cover gives build_jk."""
        N = self.nbf
        D = np.ascontiguousarray(D, dtype=np.float64)
        xs = np.ascontiguousarray(xs, dtype=np.int32)
        ys = np.ascontiguousarray(ys, dtype=np.int32)
        J, K = np.zeros((N, N)), np.zeros((N, N))
        if self.o._build_jk_list(self.h, D, len(xs), xs, ys, nthreads, J, K) != 0:
            raise RuntimeError(self.o._last_error().decode())
        return J, K

    def pair_survivors(self, tau: float):
        """(count, ysum, total) per pair x over canonical survivors (x, y >= x)."""
        cnt = np.zeros(self.npairs, np.int64)
        ys = np.zeros(self.npairs, np.uint64)
        tot = self.o._pair_survivors(self.h, tau, cnt.ctypes.data, ys.ctypes.data)
        if tot < 0:
            raise RuntimeError(self.o._last_error().decode())
        return cnt, ys, int(tot)

    def build_jk_timed(self, D: np.ndarray, tau: float, nthreads: int, stride: int, offset: int):
        """(J, K, quartets, seconds of the parallel ERI+digestion phase)."""
        N = self.nbf
        D = np.ascontiguousarray(D, dtype=np.float64)
        J = np.zeros((N, N))
        K = np.zeros((N, N))
        nq = C.c_longlong(0)
        sec = C.c_double(0.0)
        rc = self.o._build_jk_timed(self.h, D, tau, nthreads, stride, offset, J, K, C.byref(nq), C.byref(sec))
        if rc != 0:
            raise RuntimeError(self.o._last_error().decode())
        return J, K, nq.value, sec.value

    def one_electron(self):
        N = self.nbf
        S, T, V = np.zeros((N, N)), np.zeros((N, N)), np.zeros((N, N))
        self.o._one_electron(self.h, S, T, V)
        return S, T, V

    def nuclear_repulsion(self) -> float:
        return self.o._nuclear_repulsion(self.h)

    def atoms(self):
        Z = np.zeros(self.natoms, np.int32)
        pos = np.zeros(3 * self.natoms)
        self.o._atoms(self.h, Z, pos)
        return Z, pos.reshape(-1, 3)
