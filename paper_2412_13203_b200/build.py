"""Build the sm_100a engine library in-tree.

1. Offline graph compiler: emit per-class CUDA from the Alg. 1 plans
   (compiler/emit_cuda.py) into csrc/generated/.
2. nvcc every translation unit for sm_100a (-gencode arch=compute_100a,
   code=sm_100a -lineinfo) in parallel, g++ the host-only units with
   -ffp-contract=off (bit-identical pair data / kappa), link
   ``_lib/liberitile_b200.so``.

Object files are cached by a hash of their inputs so a rebuild after a small
change recompiles only what changed.
"""
from __future__ import annotations

import concurrent.futures as cf
import hashlib
import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
GEN = CSRC / "generated"
_EXTRA = os.environ.get("ERITILE_NVFLAGS", "").strip()
# experiment builds (extra nvcc flags) keep their own object cache
OBJ = PKG / ("_build" if not _EXTRA else "_build_" + hashlib.sha256(_EXTRA.encode()).hexdigest()[:8])
LIBDIR = PKG / "_lib"
LIB = LIBDIR / os.environ.get("ERITILE_LIBNAME", "liberitile_b200.so")
ROOT = PKG.parent
INCLUDE = ROOT / "include"

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVFLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-ffp-contract=off",
                  "-I" + str(INCLUDE), "-I" + str(CSRC)] + os.environ.get("ERITILE_NVFLAGS", "").split()
CXXFLAGS = ["-O2", "-std=c++17", "-fPIC", "-ffp-contract=off", "-pthread", "-I" + str(INCLUDE),
            "-I" + str(CSRC), "-I/usr/local/cuda/include"]
LMAX = int(os.environ.get("ERITILE_LMAX", "3"))


def _digest(paths, extra: str) -> str:
    h = hashlib.sha256(extra.encode())
    for p in paths:
        h.update(Path(p).read_bytes())
    return h.hexdigest()[:16]


def _compile(src: Path, deps, flags, tool) -> Path:
    key = _digest([src, *deps], " ".join(flags) + tool)
    obj = OBJ / f"{src.stem}.{key}.o"
    if obj.exists():
        return obj
    tmp = obj.with_suffix(".tmp.o")
    cmd = [tool, *flags, "-c", str(src), "-o", str(tmp)]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"compile failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, obj)
    return obj


def generate() -> list:
    sys.path.insert(0, str(ROOT))
    from paper_2412_13203_b200.compiler.emit_cuda import write_sources
    return write_sources(GEN, LMAX)


def build(jobs: int | None = None, verbose: bool = True) -> Path:
    OBJ.mkdir(exist_ok=True)
    LIBDIR.mkdir(exist_ok=True)
    generate()
    kern_deps = [CSRC / "jk_kernels.cuh", CSRC / "jk_coop.cuh", CSRC / "jk_family.cuh", CSRC / "jk_strip.cuh",
                 CSRC / "jk_api.h"]
    host_deps = [CSRC / "host" / "molecule.h", CSRC / "host" / "onee.h", CSRC / "host" / "allocator.h", CSRC / "jk_api.h",
                 INCLUDE / "eritile_gpu.h"]
    units = []
    # biggest classes first so the long compiles start early
    gen = sorted(GEN.glob("cls_*.cu"), key=lambda p: -p.stat().st_size)
    for src in gen:
        units.append((src, kern_deps, NVFLAGS, NVCC))
    units.append((GEN / "registry.cpp", [CSRC / "jk_api.h"], CXXFLAGS, "g++"))
    units.append((CSRC / "host" / "engine.cu", host_deps + kern_deps, NVFLAGS, NVCC))
    units.append((CSRC / "host" / "molecule.cpp", host_deps, CXXFLAGS, "g++"))
    units.append((CSRC / "host" / "onee.cpp", host_deps, CXXFLAGS, "g++"))
    jobs = jobs or max(2, os.cpu_count() or 2)
    with cf.ThreadPoolExecutor(jobs) as ex:
        objs = list(ex.map(lambda u: _compile(*u), units))
    for stale in OBJ.glob("*.o"):  # objects of superseded sources
        if stale not in objs:
            stale.unlink()
    key = _digest(objs, "link")
    stamp = LIBDIR / (".link." + LIB.name)
    if LIB.exists() and stamp.exists() and stamp.read_text() == key:
        return LIB
    tmp = LIBDIR / "liberitile_b200.tmp.so"
    cmd = [NVCC, *ARCH, "-shared", "-o", str(tmp), *map(str, objs), "-lcudart", "-lpthread"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed: {' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    os.replace(tmp, LIB)
    stamp.write_text(key)
    if verbose:
        print(f"built {LIB}")
    return LIB


if __name__ == "__main__":
    build()
