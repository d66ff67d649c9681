"""ctypes binding of the scalar C oracle (oracle/c/bicoptor_ref.c); test infrastructure only.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
use it.  It shares nothing with the CUDA path.  ``build()`` compiles it with gcc
(-O2 -fopenmp) in-tree; ``lib()`` builds on first use when the library is missing or
older than its source.

    fused(prm, x0, x1, j0, seeds, relu=False, transcript=False, threads=0)
        Alg 7 (DReLU) / Alg 8 (ReLU), all three parties, elements j0 .. j0 + n - 1:
        {"y0", "y1"} (+ "W0", "W1" as (n, S) uint64 with transcript=True).
    ladder_modswitch(prm, party, x, threads=0)
        Alg 7 steps 3-5 alone (config 2): v'_0 .. v'_lx, (n, S) uint64.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "c", "bicoptor_ref.c")
LIB = os.path.join(HERE, "c", "libbcref.so")
_lib = None


def build(force: bool = False) -> str:
    if not force and os.path.exists(LIB) and os.path.getmtime(LIB) >= os.path.getmtime(SRC):
        return LIB
    tmp = LIB + f".{os.getpid()}.tmp"
    cmd = ["gcc", "-O2", "-std=c11", "-fopenmp", "-shared", "-fPIC", "-o", tmp, SRC]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("gcc failed for the C oracle:\n" + r.stderr)
    os.replace(tmp, LIB)
    return LIB


def lib() -> ctypes.CDLL:
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build())
        u8p, u64p = ctypes.c_char_p, ctypes.c_void_p
        L.bcref_fused.argtypes = [ctypes.c_int] * 5 + [u8p] * 3 + [u64p] * 6 + [ctypes.c_int64, ctypes.c_uint64,
                                                                                ctypes.c_int, ctypes.c_int]
        L.bcref_fused.restype = ctypes.c_int
        L.bcref_ladder_modswitch.argtypes = [ctypes.c_int] * 5 + [u64p, u64p, ctypes.c_int64, ctypes.c_int]
        L.bcref_ladder_modswitch.restype = ctypes.c_int
        L.bcref_chacha_block.argtypes = [u8p, ctypes.c_uint64, ctypes.c_uint64, ctypes.c_int, ctypes.c_char_p]
        L.bcref_chacha_block.restype = None
        L.bcref_threads.restype = ctypes.c_int
        _lib = L
    return _lib


def threads() -> int:
    """OpenMP's default thread count (the host cores it will use)."""
    return int(lib().bcref_threads())


def chacha_block(key: bytes, label: int, counter: int, rounds: int = 20) -> bytes:
    out = ctypes.create_string_buffer(64)
    lib().bcref_chacha_block(key, label, counter, rounds, out)
    return out.raw


def _ptr(a: np.ndarray) -> int:
    return a.ctypes.data


def _prm_args(prm):
    return (prm.ell, prm.lx, prm.f, 1 if prm.mode == "literal" else 0, prm.rounds)


def fused(prm, x0, x1, j0: int, seeds, relu: bool = False, transcript: bool = False, threads: int = 0) -> dict:
    x0 = np.ascontiguousarray(x0, dtype=np.uint64)
    x1 = np.ascontiguousarray(x1, dtype=np.uint64)
    n = x0.size
    y0, y1 = np.empty(n, dtype=np.uint64), np.empty(n, dtype=np.uint64)
    W0 = np.empty((n, prm.slots), dtype=np.uint64) if transcript else None
    W1 = np.empty((n, prm.slots), dtype=np.uint64) if transcript else None
    rc = lib().bcref_fused(*_prm_args(prm), seeds.s01, seeds.s02, seeds.s12, _ptr(x0), _ptr(x1), _ptr(y0), _ptr(y1),
                           _ptr(W0) if transcript else None, _ptr(W1) if transcript else None, n, int(j0),
                           1 if relu else 0, int(threads))
    if rc:
        raise ValueError("bcref_fused: bad parameters")
    out = {"y0": y0, "y1": y1}
    if transcript:
        out.update(W0=W0, W1=W1)
    return out


def ladder_modswitch(prm, party: int, x, threads: int = 0) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.uint64)
    vp = np.empty((x.size, prm.slots), dtype=np.uint64)
    rc = lib().bcref_ladder_modswitch(prm.ell, prm.lx, prm.f, 1 if prm.mode == "literal" else 0, party, _ptr(x),
                                      _ptr(vp), x.size, int(threads))
    if rc:
        raise ValueError("bcref_ladder_modswitch: bad parameters")
    return vp
