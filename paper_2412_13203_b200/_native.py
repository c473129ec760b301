"""Locate and load the in-tree sm_100a engine library.

The library is built by ``paper_2412_13203_b200.build`` (or
``__graft_entry__.build()``) into ``_lib/liberitile_b200.so``. There is no
fallback: a missing library raises.
"""
from __future__ import annotations

import ctypes
from pathlib import Path

import os

LIB = Path(__file__).resolve().parent / "_lib" / os.environ.get("ERITILE_LIBNAME", "liberitile_b200.so")
_handle = None


def load() -> ctypes.CDLL:
    global _handle
    if _handle is None:
        if not LIB.exists():
            raise RuntimeError(f"eritile CUDA library not built: {LIB} (run __graft_entry__.build())")
        _handle = ctypes.CDLL(str(LIB))
    return _handle
