"""B200-native partial modular evaluation of sparse polynomials (arXiv 2004.11571 hot path).

Thin ctypes binding over ``libpe.so`` (C ABI: ``include/pe.h``, ``include/pe_test.h``).
Argument marshalling only: every step of the evaluation runs in the CUDA kernels of
``csrc/``.  There is no CPU fallback -- if the library or a GPU is missing, calls raise.

    ctx = Context(p, coeffs, exps, alpha)          # pe_create  (host numpy arrays)
    out = ctx.eval(j0, T)                          # pe_eval -> numpy uint64 [G, T]
    ctx.eval_device(j0, T, d_out_ptr, ld, stream)  # pe_eval_device (device pointer)
    ctx.buckets()                                  # rows (dx, dy), descending lex
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libpe.so")
TEST_LIB_PATH = os.path.join(_PKG, "libpe_test.so")   # include/pe_test.h: probes, not the product

PE_OK, PE_EINVAL, PE_ENOTPRIME, PE_ERANGE, PE_ENOMEM, PE_ECUDA, PE_ENOTSUP = 0, -1, -2, -3, -4, -5, -6
PATH_AUTO, PATH_INT, PATH_FP64, PATH_INT32, PATH_TC, PATH_FAST = 0, 1, 2, 4, 5, 6
TC_FORM_AUTO, TC_FORM_PLAIN, TC_FORM_SWAPPED = 0, 1, 2
(CORE_SHOUP4, CORE_SHOUP2, CORE_MONT, CORE_FP64, CORE_FP64ADD, CORE_POW, CORE_SHOUP4RAW, CORE_HYB, CORE_HYBRAW,
 CORE_SHOUPW) = range(10)

#: every symbol include/pe.h declares (libpe.so)
EXPORTS = ["pe_create", "pe_create_ex", "pe_eval", "pe_eval_device", "pe_destroy", "pe_num_buckets",
           "pe_bucket_exps", "pe_info", "pe_monomials", "pe_last_error", "pe_strerror",
           "pe_interp_bound_ok", "pe_set_timing", "pe_kernel_stats",
           "pe_create_batch", "pe_num_polys", "pe_poly_rows", "pe_bm_device", "pe_bm", "pe_tc_info",
           "pe_rows_addmod", "pe_unshard_columns", "pe_eval_kernel", "pe_create_compact",
           "pe_eval_device_rows", "pe_row_split", "pe_tc_form"]
#: every symbol include/pe_test.h declares (libpe_test.so)
TEST_EXPORTS = ["pe_test_core", "pe_bench_core", "pe_bench_mma"]


class PEError(RuntimeError):
    def __init__(self, code: int, what: str):
        self.code = code
        super().__init__(f"{what}: {lib().pe_strerror(code).decode()} ({code})")


class Config(ctypes.Structure):
    _fields_ = [("path", ctypes.c_int32), ("R", ctypes.c_int32), ("warps", ctypes.c_int32),
                ("chunk", ctypes.c_int32), ("tc_form", ctypes.c_int32)]


_lib = None


def lib():
    """Load libpe.so (built in-tree by ``build.py``); raises if it is missing."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} missing: run `python -m paper_2004_11571_b200.build` "
                               "(there is no CPU fallback)")
        L = ctypes.CDLL(LIB_PATH)
        u64, u32, i32, vp = ctypes.c_uint64, ctypes.c_uint32, ctypes.c_int32, ctypes.c_void_p
        L.pe_create.argtypes = [u64, u64, u32, vp, vp, vp]
        L.pe_create.restype = vp
        L.pe_create_ex.argtypes = [u64, u64, u32, vp, vp, vp, ctypes.POINTER(Config)]
        L.pe_create_ex.restype = vp
        L.pe_eval.argtypes = [vp, u64, u64, vp]
        L.pe_eval.restype = ctypes.c_int
        L.pe_eval_device.argtypes = [vp, u64, u64, vp, u64, vp]
        L.pe_eval_device.restype = ctypes.c_int
        L.pe_destroy.argtypes = [vp]
        L.pe_destroy.restype = None
        L.pe_num_buckets.argtypes = [vp]
        L.pe_num_buckets.restype = u64
        L.pe_bucket_exps.argtypes = [vp, vp]
        L.pe_bucket_exps.restype = ctypes.c_int
        L.pe_info.argtypes = [vp, ctypes.POINTER(i32), ctypes.POINTER(i32), ctypes.POINTER(i32),
                              ctypes.POINTER(u64), ctypes.POINTER(u64)]
        L.pe_info.restype = ctypes.c_int
        L.pe_monomials.argtypes = [vp, vp]
        L.pe_monomials.restype = ctypes.c_int
        L.pe_last_error.argtypes = []
        L.pe_last_error.restype = ctypes.c_int
        L.pe_strerror.argtypes = [ctypes.c_int]
        L.pe_strerror.restype = ctypes.c_char_p
        L.pe_interp_bound_ok.argtypes = [u64, u64]
        L.pe_interp_bound_ok.restype = ctypes.c_int
        L.pe_set_timing.argtypes = [vp, ctypes.c_int]
        L.pe_set_timing.restype = ctypes.c_int
        L.pe_kernel_stats.argtypes = [vp, ctypes.POINTER(u64), ctypes.POINTER(ctypes.c_double),
                                      ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)]
        L.pe_kernel_stats.restype = ctypes.c_int
        L.pe_eval_device_rows.argtypes = [vp, u64, u64, u64, u64, vp, u64, vp]
        L.pe_eval_device_rows.restype = ctypes.c_int
        L.pe_row_split.argtypes = [vp]
        L.pe_row_split.restype = u64
        L.pe_create_compact.argtypes = [u64, u64, u32, vp, vp, vp, ctypes.POINTER(Config)]
        L.pe_create_compact.restype = vp
        L.pe_create_batch.argtypes = [u64, u32, vp, u32, vp, vp, vp, ctypes.POINTER(Config)]
        L.pe_create_batch.restype = vp
        L.pe_num_polys.argtypes = [vp]
        L.pe_num_polys.restype = u32
        L.pe_poly_rows.argtypes = [vp, vp]
        L.pe_poly_rows.restype = ctypes.c_int
        L.pe_bm_device.argtypes = [u64, u64, u64, vp, u64, vp, u64, vp, vp]
        L.pe_bm_device.restype = ctypes.c_int
        L.pe_bm.argtypes = [u64, u64, u64, vp, vp, vp]
        L.pe_bm.restype = ctypes.c_int
        L.pe_tc_info.argtypes = [vp, ctypes.POINTER(i32), ctypes.POINTER(u64), ctypes.POINTER(u64)]
        L.pe_tc_info.restype = ctypes.c_int
        L.pe_eval_kernel.argtypes = [vp, u64]
        L.pe_eval_kernel.restype = ctypes.c_int
        L.pe_tc_form.argtypes = [vp]
        L.pe_tc_form.restype = ctypes.c_int
        L.pe_rows_addmod.argtypes = [u64, vp, u64, vp, u64, u64, u64, vp]
        L.pe_rows_addmod.restype = ctypes.c_int
        L.pe_unshard_columns.argtypes = [vp, u64, vp, u64, u64, u64, u64, vp]
        L.pe_unshard_columns.restype = ctypes.c_int
        _lib = L
    return _lib


_test_lib = None


def test_lib():
    """Load libpe_test.so (include/pe_test.h: modular-core probes, roofline microbenchmarks)."""
    global _test_lib
    if _test_lib is None:
        if not os.path.exists(TEST_LIB_PATH):
            raise RuntimeError(f"{TEST_LIB_PATH} missing: run `python -m paper_2004_11571_b200.build`")
        L = ctypes.CDLL(TEST_LIB_PATH)
        u64, vp = ctypes.c_uint64, ctypes.c_void_p
        L.pe_test_core.argtypes = [ctypes.c_int, u64, u64, vp, vp, vp, vp]
        L.pe_test_core.restype = ctypes.c_int
        L.pe_bench_core.argtypes = [ctypes.c_int, u64, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int,
                                    ctypes.POINTER(ctypes.c_float), ctypes.POINTER(ctypes.c_double),
                                    ctypes.POINTER(ctypes.c_double)]
        L.pe_bench_core.restype = ctypes.c_int
        L.pe_bench_mma.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.POINTER(ctypes.c_float),
                                   ctypes.POINTER(ctypes.c_double)]
        L.pe_bench_mma.restype = ctypes.c_int
        _test_lib = L
    return _test_lib


def _ptr(a):
    return a.ctypes.data_as(ctypes.c_void_p) if a is not None and a.size else None


def _check(rc: int, what: str):
    if rc != PE_OK:
        raise PEError(rc, what)


class Context:
    """An evaluation handle (``pe_create_ex``).  Arrays are host numpy arrays."""

    def __init__(self, p: int, coeffs, exps, alpha, n: int | None = None, path: int = PATH_AUTO,
                 R: int = 0, warps: int = 0, chunk: int = 0, compact: bool = False, tc_form: int = 0):
        """compact=True: exponents passed as uint8 (pe_create_compact; every degree must be < 256).
        tc_form: TC_FORM_PLAIN / TC_FORM_SWAPPED (tensor-core form for p >= 2^54), 0 = automatic."""
        coeffs = np.ascontiguousarray(coeffs, dtype=np.uint64).ravel()
        if compact:
            e = np.asarray(exps)
            if e.size and int(e.max()) > 255:
                raise ValueError("compact exponents must be < 256")
            exps = np.ascontiguousarray(e, dtype=np.uint8)
        else:
            exps = np.ascontiguousarray(exps, dtype=np.uint32)
        n = exps.shape[1] if n is None else n
        exps = exps.reshape(-1, n) if exps.size else np.zeros((0, n), exps.dtype)
        alpha = np.ascontiguousarray(alpha, dtype=np.uint64).ravel()
        self.p, self.n, self.t = int(p), int(n), int(coeffs.size)
        cfg = Config(path, R, warps, chunk, tc_form)
        L = lib()
        create = L.pe_create_compact if compact else L.pe_create_ex
        h = create(self.p, self.t, self.n, _ptr(coeffs), _ptr(exps), _ptr(alpha), ctypes.byref(cfg))
        if not h:
            raise PEError(L.pe_last_error(), "pe_create")
        self._h = ctypes.c_void_p(h)

    @classmethod
    def batch(cls, p: int, polys, alpha, n: int, path: int = PATH_AUTO, R: int = 0, warps: int = 0,
              chunk: int = 0) -> "Context":
        """pe_create_batch: ``polys`` = [(coeffs, exps), ...] evaluated at the same points."""
        cs = [np.ascontiguousarray(c, dtype=np.uint64).ravel() for c, _ in polys]
        es = [np.ascontiguousarray(e, dtype=np.uint32).reshape(-1, n) for _, e in polys]
        tper = np.array([c.size for c in cs], np.uint64)
        coeffs = np.concatenate(cs) if cs else np.zeros(0, np.uint64)
        exps = np.concatenate(es) if es else np.zeros((0, n), np.uint32)
        alpha = np.ascontiguousarray(alpha, dtype=np.uint64).ravel()
        self = cls.__new__(cls)
        self.p, self.n, self.t = int(p), int(n), int(coeffs.size)
        cfg = Config(path, R, warps, chunk, 0)
        L = lib()
        h = L.pe_create_batch(self.p, len(polys), _ptr(tper), self.n, _ptr(coeffs), _ptr(exps), _ptr(alpha),
                              ctypes.byref(cfg))
        if not h:
            raise PEError(L.pe_last_error(), "pe_create_batch")
        self._h = ctypes.c_void_p(h)
        return self

    def poly_rows(self) -> np.ndarray:
        k = int(lib().pe_num_polys(self._h))
        out = np.zeros(k + 1, np.uint64)
        _check(lib().pe_poly_rows(self._h, _ptr(out)), "pe_poly_rows")
        return out

    @classmethod
    def from_workload(cls, w, **kw) -> "Context":
        return cls(w.p, w.coeffs, w.exps, w.alpha, n=w.n, **kw)

    def close(self):
        if getattr(self, "_h", None):
            lib().pe_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    @property
    def G(self) -> int:
        return int(lib().pe_num_buckets(self._h))

    def buckets(self) -> np.ndarray:
        out = np.zeros((self.G, 2), np.uint32)
        _check(lib().pe_bucket_exps(self._h, _ptr(out)), "pe_bucket_exps")
        return out

    def info(self) -> dict:
        path, R, W = ctypes.c_int32(), ctypes.c_int32(), ctypes.c_int32()
        tp, ns = ctypes.c_uint64(), ctypes.c_uint64()
        _check(lib().pe_info(self._h, ctypes.byref(path), ctypes.byref(R), ctypes.byref(W), ctypes.byref(tp),
                             ctypes.byref(ns)), "pe_info")
        name = {PATH_FP64: "fp64", PATH_INT32: "int32"}.get(path.value, "int")
        mode, pieces, min_t = ctypes.c_int32(), ctypes.c_uint64(), ctypes.c_uint64()
        _check(lib().pe_tc_info(self._h, ctypes.byref(mode), ctypes.byref(pieces), ctypes.byref(min_t)),
               "pe_tc_info")
        return {"path": name, "R": R.value, "warps": W.value,
                "t_padded": tp.value, "n_slots": ns.value,
                "tc_mode": mode.value, "tc_pieces": pieces.value, "tc_min_T": min_t.value}

    def eval_kernel(self, T: int) -> str:
        """Hot kernel an evaluation of T points runs (pe_eval_kernel): "k_step" or "k_tc"."""
        k = lib().pe_eval_kernel(self._h, T)
        if k < 0:
            raise PEError(k, "pe_eval_kernel")
        return {0: "k_step", 1: "k_tc", 2: "fast"}[k]

    def tc_form(self) -> int:
        """TC_FORM_PLAIN / TC_FORM_SWAPPED, or 0 without a tensor-core path (pe_tc_form)."""
        k = lib().pe_tc_form(self._h)
        if k < 0:
            raise PEError(k, "pe_tc_form")
        return k

    def uses_tc(self, T: int) -> bool:
        """True if an evaluation of T points runs the tensor-core kernel (PE_PATH_TC / auto)."""
        return self.eval_kernel(T) == "k_tc"

    def monomials(self) -> np.ndarray:
        out = np.zeros(self.t, np.uint64)
        _check(lib().pe_monomials(self._h, _ptr(out)), "pe_monomials")
        return out

    def eval(self, j0: int, T: int, out: np.ndarray | None = None) -> np.ndarray:
        """pe_eval: host result uint64 [G, T]."""
        if out is None:
            out = np.empty((self.G, T), np.uint64)
        assert out.dtype == np.uint64 and out.flags.c_contiguous and out.size == self.G * T
        _check(lib().pe_eval(self._h, j0, T, _ptr(out)), "pe_eval")
        return out

    def set_timing(self, enable: bool = True):
        _check(lib().pe_set_timing(self._h, int(enable)), "pe_set_timing")

    def kernel_stats(self) -> dict:
        n, s, f, tp = ctypes.c_uint64(), ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
        _check(lib().pe_kernel_stats(self._h, ctypes.byref(n), ctypes.byref(s), ctypes.byref(f), ctypes.byref(tp)),
               "pe_kernel_stats")
        return {"step_launches": n.value, "step_ms": s.value, "fixup_ms": f.value, "term_points": tp.value}

    def row_split(self) -> int:
        """pe_row_split: the row G1 splitting evaluations into two overlappable blocks (0: none)."""
        return int(lib().pe_row_split(self._h))

    def eval_device_rows(self, j0: int, T: int, g0: int, g1: int, d_out: int, ld: int | None = None,
                         stream: int = 0):
        """pe_eval_device_rows: rows [g0, g1) into the [G, ld] device matrix at d_out."""
        _check(lib().pe_eval_device_rows(self._h, j0, T, g0, g1, ctypes.c_void_p(d_out), T if ld is None else ld,
                                         ctypes.c_void_p(stream)), "pe_eval_device_rows")

    def eval_device(self, j0: int, T: int, d_out: int, ld: int | None = None, stream: int = 0):
        """pe_eval_device into a device pointer (e.g. ``torch_tensor.data_ptr()``)."""
        _check(lib().pe_eval_device(self._h, j0, T, ctypes.c_void_p(d_out), T if ld is None else ld,
                                    ctypes.c_void_p(stream)), "pe_eval_device")


def test_core(variant: int, p: int, a, b, extra=None) -> np.ndarray:
    a = np.ascontiguousarray(a, dtype=np.uint64)
    b = np.ascontiguousarray(b, dtype=np.uint64)
    out = np.zeros(a.size, np.uint64)
    x = None if extra is None else np.ascontiguousarray(extra, dtype=np.uint64)
    _check(test_lib().pe_test_core(variant, p, a.size, _ptr(a), _ptr(b), _ptr(x), _ptr(out)), "pe_test_core")
    return out


def bench_core(variant: int, p: int, R: int, blocks: int, threads: int, iters: int):
    ms, steps, cyc = ctypes.c_float(), ctypes.c_double(), ctypes.c_double()
    _check(test_lib().pe_bench_core(variant, p, R, blocks, threads, iters, ctypes.byref(ms), ctypes.byref(steps),
                               ctypes.byref(cyc)), "pe_bench_core")
    return ms.value, steps.value, cyc.value


def bench_mma(N: int = 128, iters: int = 20000):
    """pe_bench_mma: int8 tcgen05 MMA rate (M=128, N, K=32) -> int8 ops/s (2 per MAC)."""
    ms, macs = ctypes.c_float(), ctypes.c_double()
    _check(test_lib().pe_bench_mma(N, iters, ctypes.byref(ms), ctypes.byref(macs)), "pe_bench_mma")
    return 2 * macs.value / (ms.value * 1e-3)


def berlekamp_massey(p: int, seq: np.ndarray):
    """pe_bm on host rows seq[G, T] -> (lengths uint32[G], connection polys uint64[G, T+1])."""
    seq = np.ascontiguousarray(seq, dtype=np.uint64)
    G, T = seq.shape
    lam = np.zeros((G, T + 1), np.uint64)
    ln = np.zeros(G, np.uint32)
    _check(lib().pe_bm(p, G, T, _ptr(seq), _ptr(lam), _ptr(ln)), "pe_bm")
    return ln, lam


def interp_bound_ok(p: int, t: int) -> bool:
    return bool(lib().pe_interp_bound_ok(p, t))


def rows_addmod(p: int, d_dst: int, ld_dst: int, d_src: int, ld_src: int, rows: int, cols: int, stream: int = 0):
    """pe_rows_addmod on device pointers: dst = (dst + src) mod p, element-wise over rows x cols."""
    _check(lib().pe_rows_addmod(p, ctypes.c_void_p(d_dst), ld_dst, ctypes.c_void_p(d_src), ld_src, rows, cols,
                                ctypes.c_void_p(stream)), "pe_rows_addmod")


def unshard_columns(d_out: int, ld: int, d_blocks: int, P: int, G: int, Tr: int, T: int, stream: int = 0):
    """pe_unshard_columns: [P][G][Tr] point-range blocks -> rows of [G][ld]."""
    _check(lib().pe_unshard_columns(ctypes.c_void_p(d_out), ld, ctypes.c_void_p(d_blocks), P, G, Tr, T,
                                    ctypes.c_void_p(stream)), "pe_unshard_columns")
