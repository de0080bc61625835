"""C-ABI boundary checks that need no GPU: the library loads, exports every symbol the
headers declare, and host-side validation (done before any CUDA call) reports the documented
error codes.  No compute call is made here."""
import ctypes
import os
import re

import numpy as np
import pytest

import paper_2004_11571_b200 as pe
from paper_2004_11571_b200 import build as pe_build
from conftest import ROOT

P62 = (1 << 62) - 57


@pytest.fixture(scope="module")
def L():
    pe_build.build()
    return pe.lib()


def _declared(header):
    src = open(os.path.join(ROOT, "include", header)).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return set(re.findall(r"\b(pe_[a-z_0-9]+)\s*\(", src))


@pytest.mark.parametrize("header,names,path", [("pe.h", "EXPORTS", "LIB_PATH"),
                                               ("pe_test.h", "TEST_EXPORTS", "TEST_LIB_PATH")])
def test_exports_every_declared_symbol(L, header, names, path):
    """libpe.so exports exactly include/pe.h; the probes (include/pe_test.h) live in libpe_test.so."""
    declared = _declared(header)
    assert declared, "no declarations parsed"
    assert declared == set(getattr(pe, names))
    lib = L if header == "pe.h" else pe.test_lib()
    for name in declared:
        assert hasattr(lib, name), name           # dlsym succeeds
    out = os.popen(f"nm -D --defined-only {getattr(pe, path)}").read()
    for name in declared:
        assert re.search(rf"\bT {name}\b", out), f"{name} not exported as a text symbol"
    if header == "pe.h":                          # no probe or microbenchmark ships in the product
        for name in pe.TEST_EXPORTS:
            assert not re.search(rf"\bT {name}\b", out), name


def test_strerror_and_bound(L):
    assert L.pe_strerror(0) == b"ok"
    assert L.pe_strerror(-2) == b"p is not prime"
    assert pe.interp_bound_ok(1009, 1)          # SPEC.md:116 examples (PAPER.md:774 p > 100 s^2)
    assert not pe.interp_bound_ok(1009, 10)
    # SPEC.md:116 claims (2^49, 10^6) -> false, but 2^49 ~ 5.6e14 > 100 * 10^12: true.
    assert pe.interp_bound_ok(1 << 49, 10**6)
    assert not pe.interp_bound_ok(1 << 49, 10**7)
    assert not pe.interp_bound_ok(100 * 7**2, 7) and pe.interp_bound_ok(100 * 7**2 + 1, 7)


def _create(L, p, t, n, coeffs, exps, alpha):
    return L.pe_create(p, t, n, coeffs, exps, alpha)


def test_validation_before_cuda(L):
    c = np.array([1, 2], np.uint64)
    e = np.zeros((2, 4), np.uint32)
    a = np.array([2, 3], np.uint64)
    cp, ep, ap = (x.ctypes.data_as(ctypes.c_void_p) for x in (c, e, a))
    cases = [
        (dict(p=15, n=4), pe.PE_ENOTPRIME),           # composite
        (dict(p=2**61 - 1 + 2, n=4), pe.PE_ENOTPRIME),
        (dict(p=2, n=4), pe.PE_ERANGE),                # p < 3
        (dict(p=(1 << 63) + 29, n=4), pe.PE_ERANGE),   # p >= 2^63
        (dict(p=P62, n=1), pe.PE_EINVAL),              # n < 2
    ]
    for kw, code in cases:
        assert not _create(L, kw["p"], 2, kw["n"], cp, ep, ap)
        assert L.pe_last_error() == code, kw
    assert not _create(L, P62, 2, 4, None, ep, ap)
    assert L.pe_last_error() == pe.PE_EINVAL
    assert not _create(L, P62, 2, 4, cp, ep, None)       # alpha NULL with n > 2
    assert L.pe_last_error() == pe.PE_EINVAL
    # t > 2^31 - 1 (the device sort takes int counts): rejected before the arrays are read
    assert not _create(L, P62, 1 << 31, 4, cp, ep, ap)
    assert L.pe_last_error() == pe.PE_ERANGE
    z = np.array([2, P62 * 2], np.uint64)                 # alpha_2 == 0 mod p
    assert not _create(L, P62, 2, 4, cp, ep, z.ctypes.data_as(ctypes.c_void_p))
    assert L.pe_last_error() == pe.PE_ERANGE
    # NULL handles
    assert L.pe_eval(None, 1, 4, None) == pe.PE_EINVAL
    assert L.pe_eval_device(None, 1, 4, None, 4, None) == pe.PE_EINVAL
    assert L.pe_num_buckets(None) == 0
    L.pe_destroy(None)                                    # NULL-safe


def test_fp64_path_rejects_wide_prime(L):
    c = np.array([1], np.uint64)
    e = np.zeros((1, 3), np.uint32)
    a = np.array([2], np.uint64)
    with pytest.raises(pe.PEError) as ei:
        pe.Context(P62, c, e, a, path=pe.PATH_FP64)
    assert ei.value.code == pe.PE_ENOTSUP


def test_loud_failure_without_gpu(L):
    """The product path has no CPU fallback: on a box without a GPU a valid create fails with
    PE_ECUDA (on a GPU box this test is skipped; the gpu tests cover it)."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(pe.PEError) as ei:
        pe.Context(13, [3, 5], [[1, 0, 2], [0, 0, 1]], [2])
    assert ei.value.code == pe.PE_ECUDA
