"""CPU: the XB12 record format (kernels/xb12.hpp) restated in numpy round-trips bit for bit, and the
CPU baseline's on-the-fly XB12 decoder (baseline/cpu_ffn.c cpu_moe_layer_xb12) computes the same layer
as its bf16 path, bit for bit."""
import ctypes as C
import os

import numpy as np
import pytest

import xb12_ref as X

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bf16(a):
    u = np.ascontiguousarray(a, dtype=np.float32).view(np.uint32)
    return ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)


def test_roundtrip_gaussian_and_escapes():
    rng = np.random.default_rng(0)
    w = _bf16(rng.standard_normal(1 << 16) * 0.02)
    w[::997] = 0                      # zeros: escapes
    w[5] = 0x7F80                     # +inf: escape
    w[7] = 0x0001                     # denormal: escape
    rec, meta = X.encode(w)
    assert meta["format"] == 1 and meta["n_exc"] > 60
    assert len(rec) < 0.77 * 2 * w.size
    assert np.array_equal(X.decode(rec, meta, w.size), w)


def test_wide_exponent_tile_stays_raw():
    rng = np.random.default_rng(1)
    w = rng.integers(0, 1 << 16, 4096, dtype=np.uint16)  # uniform bits: exponents everywhere
    rec, meta = X.encode(w)
    assert meta["format"] == 0 and np.array_equal(X.decode(rec, meta, w.size), w)


@pytest.fixture(scope="module")
def lib():
    path = os.path.join(ROOT, "baseline", "libcpu_ffn.so")
    if not os.path.exists(path):
        pytest.skip("baseline/libcpu_ffn.so not built")
    L = C.CDLL(path)
    L.cpu_moe_layer.argtypes = [C.POINTER(C.c_void_p), C.POINTER(C.c_double), C.c_int, C.c_int, C.c_int, C.c_int,
                                C.POINTER(C.c_double), C.POINTER(C.c_float), C.c_int]
    L.cpu_moe_layer_xb12.argtypes = [C.POINTER(C.c_void_p), C.POINTER(C.c_int32), C.POINTER(C.c_uint32),
                                     C.POINTER(C.c_int64), C.POINTER(C.c_int64), C.POINTER(C.c_int64),
                                     C.POINTER(C.c_double), C.c_int, C.c_int, C.c_int, C.c_int,
                                     C.POINTER(C.c_double), C.POINTER(C.c_float), C.c_int]
    return L


def test_cpu_baseline_xb12_equals_bf16(lib):
    D, F, T = 256, 512, 4
    rng = np.random.default_rng(2)
    experts = [_bf16(rng.standard_normal(3 * F * D) / 16) for _ in range(2)]
    experts[1][1234] = 0
    x = rng.standard_normal(D)
    wts = (C.c_double * 2)(0.6, 0.4)
    out_raw = np.zeros(D, dtype=np.float32)
    keep = [np.ascontiguousarray(e) for e in experts]
    ptrs = (C.c_void_p * 2)(*[e.ctypes.data for e in keep])
    xp = x.ctypes.data_as(C.POINTER(C.c_double))
    assert lib.cpu_moe_layer(ptrs, wts, 2, D, F, T, xp, out_raw.ctypes.data_as(C.POINTER(C.c_float)), 3) == 0
    n = 3 * F * D // T
    recs, metas = [], []
    for e in experts:
        for t in range(T):
            r, m = X.encode(e[t * n:(t + 1) * n])
            recs.append(np.frombuffer(r, dtype=np.uint8).copy())
            metas.append(m)
    k = len(recs)
    out_x = np.zeros(D, dtype=np.float32)
    rc = lib.cpu_moe_layer_xb12((C.c_void_p * k)(*[r.ctypes.data for r in recs]),
                                (C.c_int32 * k)(*[m["format"] for m in metas]),
                                (C.c_uint32 * k)(*[m["base"] for m in metas]),
                                (C.c_int64 * k)(*[m["n_exc"] for m in metas]),
                                (C.c_int64 * k)(*[m.get("nib_off", 0) for m in metas]),
                                (C.c_int64 * k)(*[m.get("exc_off", 0) for m in metas]),
                                wts, 2, D, F, T, xp, out_x.ctypes.data_as(C.POINTER(C.c_float)), 3)
    assert rc == 0
    assert np.array_equal(out_raw, out_x)
