"""CPU: the XBH record format (kernels/xbh.hpp) restated in numpy round-trips bit for bit, its code
is a valid length-limited prefix code that reaches the Huffman optimum, and the CPU baseline's
on-the-fly XBH decoder (baseline/cpu_ffn.c) computes the same layer as its bf16 path, bit for bit."""
import ctypes as C
import heapq
import os

import numpy as np
import pytest

import xbh_ref as X

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _bf16(a):
    u = np.ascontiguousarray(a, dtype=np.float32).view(np.uint32)
    return ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)


def _huffman_cost(counts):
    """Unconstrained Huffman total bits (sum of merged weights)."""
    h = [c for c in counts if c]
    if len(h) == 1:
        return h[0]
    heapq.heapify(h)
    cost = 0
    while len(h) > 1:
        a, b = heapq.heappop(h), heapq.heappop(h)
        cost += a + b
        heapq.heappush(h, a + b)
    return cost


def test_roundtrip_gaussian_and_escapes():
    rng = np.random.default_rng(0)
    w = _bf16(rng.standard_normal(1 << 16) * 0.02)
    w[::997] = 0                      # zeros: escapes
    w[5] = 0x7F80                     # +inf: escape
    w[7] = 0x0001                     # denormal: escape
    rec, meta = X.encode(w)
    assert meta["format"] == 2 and meta["n_exc"] > 60
    assert np.array_equal(X.decode(rec, meta, w.size), w)


def test_ragged_blocks_and_single_symbol():
    rng = np.random.default_rng(3)
    w = _bf16(rng.standard_normal(3 * 12800 + 48) * 0.02)  # ~3 decode blocks, the last one partial
    rec, meta = X.encode(w)
    assert meta["format"] == 2 and np.array_equal(X.decode(rec, meta, w.size), w)
    one = np.full(1 << 17, 0x3F80, dtype=np.uint16)  # every exponent equal: one 1-bit code
    base, ln, code, lut, _ = X.build_code(np.bincount((one >> 7) & 0xFF, minlength=256))
    assert sorted(x for x in ln if x) == [1]
    rec, meta = X.encode(one)
    assert meta["total_bits"] == one.size and np.array_equal(X.decode(rec, meta, one.size), one)


def test_code_is_prefix_free_optimal_and_length_limited():
    rng = np.random.default_rng(4)
    for trial in range(200):
        k = int(rng.integers(2, 17))
        hist = np.zeros(256, dtype=np.int64)
        start = int(rng.integers(0, 240))
        # geometric-ish tails (deep codes) and random counts
        if trial % 2:
            hist[start:start + k] = (rng.random(k) ** 8 * 1e6).astype(np.int64) + 1
        else:
            hist[start:start + k] = (2.0 ** -np.arange(k) * 1e7).astype(np.int64) + 1
        base, ln, code, lut, mlut = X.build_code(hist)
        used = [s for s in range(16) if ln[s]]
        assert max(ln) <= X.MAX_LEN
        assert abs(sum(2.0 ** -ln[s] for s in used) - 1.0) < 1e-12  # complete prefix code
        for s in used:  # prefix-free: the table maps every code's range back to s
            sh = X.MAX_LEN - ln[s]
            ent = lut[code[s] << sh: (code[s] + 1) << sh]
            assert np.all(ent >> 8 == ln[s])
        # the multi-code table decodes the same symbols as the single-code walk, its first length and
        # its total length match
        sym_of = {((base + k) & 0xFF): k for k in range(15)}
        for i in rng.integers(0, 1 << X.MAX_LEN, 64):
            m = int(mlut[i])
            pos = 0
            for q in range((m >> 20) & 7):
                p12 = (int(i) << pos) & ((1 << X.MAX_LEN) - 1)
                e = int(lut[p12])
                s_ = 15 if (ln[15] and p12 >> (X.MAX_LEN - ln[15]) == code[15]) else sym_of[e & 0xFF]
                assert (m >> (4 * q)) & 15 == s_
                if q == 0:
                    assert (m >> 23) & 15 == e >> 8
                pos += e >> 8
            assert pos == m >> 27
        counts = list(hist[base:base + 15]) + [int(hist.sum() - hist[base:base + 15].sum())]
        cost = sum(counts[s] * ln[s] for s in used)
        ref = _huffman_cost(counts)
        if max(ln) < X.MAX_LEN:  # the limit did not bind: package-merge == Huffman
            assert cost == ref
        else:
            assert cost >= ref


def test_mixtral_like_tile_size():
    rng = np.random.default_rng(5)
    n = 1 << 22  # 8 MB of bf16: the 24 KB of tables are ~0.05 bits per value
    x = (rng.integers(0, 65536, (4, n)).sum(0) - 4 * 32767.5) / (37837.22 * 64)
    w = (x.astype(np.float32).view(np.uint32) >> 16).astype(np.uint16)
    rec, meta = X.encode(w)
    assert meta["format"] == 2
    assert 8 * len(rec) / n < 10.8            # ~66 % of bf16 (XB12: 12 bits)
    assert meta["total_bits"] / n < 2.6       # exponent entropy of these weights ~2.52 bits


def test_wide_exponent_tile_stays_raw():
    rng = np.random.default_rng(1)
    w = rng.integers(0, 1 << 16, 4096, dtype=np.uint16)
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


@pytest.mark.parametrize("D,F,T", [(256, 512, 4), (512, 1024, 2)])
def test_cpu_baseline_xbh_equals_bf16(lib, D, F, T):
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
            assert m["format"] == 2
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


def straddle_tile(n=122880, blocks=5, seed=9):
    """n values (a multiple of 16) whose codes total blocks * 32768 + 1 bits and whose last code runs
    into a final 128-bit chunk that starts a new decode block and holds no code start: exponent 120
    (1-bit code) first, then alternating 121 / 119 (2-bit codes)."""
    total = blocks * X.BLOCK + 1
    x = total - n  # 2-bit codes
    na = n - x
    assert n % 16 == 0 and na > 2 * x // 2
    rng = np.random.default_rng(seed)
    ex = np.concatenate([np.full(na, 120), np.tile([121, 119], x // 2 + 1)[:x]]).astype(np.uint16)
    return ((rng.integers(0, 2, n).astype(np.uint16) << 15) | (ex << 7) |
            rng.integers(0, 128, n).astype(np.uint16)).astype(np.uint16), total


def test_last_code_straddles_into_a_new_block():
    w, total = straddle_tile()
    rec, meta = X.encode(w)
    assert meta["format"] == 2 and meta["total_bits"] == total
    assert X.chunks(total) - 1 == 5 * 256  # the final chunk opens block 5
    assert np.array_equal(X.decode(rec, meta, w.size), w)  # decode asserts the block bases too
