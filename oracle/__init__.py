"""CPU oracle for the partial-evaluation hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its ``cpu_baseline`` leg and
``--impl reference``) may import this package.  The product path
(``paper_2004_11571_b200``) never does, and shares no code with it.

* ``oracle.c``  -- the direct definition with ``unsigned
  __int128`` square-and-multiply, OpenMP over points; and ``incr_eval``, Alg. 1
   as the incremental companion checker (``incr_eval_blocked``: the same
  checker with the points cut into blocks, each seeded at its first point, for load balance on
  Zipf-skewed rows).
* ``brute.py``  -- Python big-integer literal substitution for tiny inputs.

Pins: tests/test_oracle_pins.py (DESIGN.md "Oracle pins" P1-P13).
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lib = None


def build(force: bool = False) -> str:
    """Compile oracle.c with plain gcc (-O2, OpenMP) into oracle/liboracle.so."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c11",
                               "-o", tmp, _SRC])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    if _lib is None:
        lib = ctypes.CDLL(build())
        u64, u32, vp = ctypes.c_uint64, ctypes.c_uint32, ctypes.c_void_p
        lib.oracle_powmod.argtypes = [u64, u64, u64]
        lib.oracle_powmod.restype = u64
        lib.oracle_mulmod.argtypes = [u64, u64, u64]
        lib.oracle_mulmod.restype = u64
        lib.oracle_buckets.argtypes = [u64, u32, vp, vp]
        lib.oracle_buckets.restype = u64
        lib.oracle_eval.argtypes = [u64, u64, u32, vp, vp, vp, u64, vp, u64, vp]
        lib.oracle_eval.restype = ctypes.c_int
        lib.incr_eval.argtypes = [u64, u64, u32, vp, vp, vp, u64, u64, vp]
        lib.incr_eval.restype = ctypes.c_int
        lib.incr_eval_blocked.argtypes = [u64, u64, u32, vp, vp, vp, u64, u64, u64, vp]
        lib.incr_eval_blocked.restype = ctypes.c_int
        _lib = lib
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p) if a is not None and a.size else None


def _prep(coeffs, exps, alpha, n):
    coeffs = np.ascontiguousarray(coeffs, dtype=np.uint64)
    exps = np.ascontiguousarray(exps, dtype=np.uint32).reshape(-1, n)
    alpha = np.ascontiguousarray(alpha, dtype=np.uint64)
    return coeffs, exps, alpha


def powmod(b: int, e: int, p: int) -> int:
    return int(_load().oracle_powmod(b, e, p))


def mulmod(a: int, b: int, p: int) -> int:
    return int(_load().oracle_mulmod(a, b, p))


def buckets(exps: np.ndarray, n: int) -> np.ndarray:
    """Rows of the output: distinct (dx, dy), descending lex -> uint32 [G, 2]."""
    exps = np.ascontiguousarray(exps, dtype=np.uint32).reshape(-1, n)
    t = exps.shape[0]
    lib = _load()
    G = int(lib.oracle_buckets(t, n, _ptr(exps), None))
    dxdy = np.zeros((G, 2), np.uint32)
    lib.oracle_buckets(t, n, _ptr(exps), _ptr(dxdy))
    return dxdy


def eval_direct(p, n, coeffs, exps, alpha, j0, T=None, ks=None) -> np.ndarray:
    """out[g, c] for j = j0 + c (c < T), or j = j0 + ks[c] (sampled mode). uint64 [G, ncols]."""
    coeffs, exps, alpha = _prep(coeffs, exps, alpha, n)
    G = buckets(exps, n).shape[0]
    if ks is not None:
        ks = np.ascontiguousarray(ks, dtype=np.uint64)
        nk = ks.size
    else:
        nk = int(T)
    out = np.zeros((G, nk), np.uint64)
    if G and nk:
        rc = _load().oracle_eval(p, coeffs.size, n, _ptr(coeffs), _ptr(exps), _ptr(alpha),
                                 j0, _ptr(ks) if ks is not None else None, nk, _ptr(out))
        assert rc == 0
    return out


def eval_incremental(p, n, coeffs, exps, alpha, j0, T) -> np.ndarray:
    """Alg. 1 companion checker; uint64 [G, T]."""
    coeffs, exps, alpha = _prep(coeffs, exps, alpha, n)
    G = buckets(exps, n).shape[0]
    out = np.zeros((G, int(T)), np.uint64)
    if G and T:
        rc = _load().incr_eval(p, coeffs.size, n, _ptr(coeffs), _ptr(exps), _ptr(alpha), j0, T, _ptr(out))
        assert rc == 0
    return out


def eval_incremental_blocked(p, n, coeffs, exps, alpha, j0, T, block=512) -> np.ndarray:
    """Alg. 1 checker with the points split into blocks (each task seeded at its first point by
    exponentiation): same values as eval_incremental, balanced over (row, block) tasks."""
    coeffs, exps, alpha = _prep(coeffs, exps, alpha, n)
    G = buckets(exps, n).shape[0]
    out = np.zeros((G, int(T)), np.uint64)
    if G and T:
        rc = _load().incr_eval_blocked(p, coeffs.size, n, _ptr(coeffs), _ptr(exps), _ptr(alpha), j0, T, block,
                                       _ptr(out))
        assert rc == 0
    return out


def eval_workload(w, ks=None) -> np.ndarray:
    return eval_direct(w.p, w.n, w.coeffs, w.exps, w.alpha, w.j0, w.T, ks)
