"""Coded expert stores on the B200 (lossless exponent-coded bf16 over the host link): XB12
(MOE_STORE_XB12, 4-bit window codes) and XBH (MOE_STORE_XBH, per-tile Huffman codes).

* The GPU encoders produce exactly the records of the numpy restatements (tests/xb12_ref.py,
  tests/xbh_ref.py), and the store decodes (host and device) to the bf16 store's bits.
* A decode session over a coded store returns bit-identical layer outputs and the identical logical
  trace as over a bf16 store, while the copy engine moves ~75 % (XB12) / ~66 % (XBH) of the bytes.
* Real-weight uploads (moe_expert_set) encode too; tiles that would not shrink stay raw.
"""
import ctypes as C

import numpy as np
import pytest

import paper_2408_10284_b200 as P
import xb12_ref as X
import xbh_ref as XH
from conftest import load_golden
from helpers import oracle_inputs, sim_config
from oracle import oracle as O
from paper_2408_10284_b200 import timeline as TL

pytestmark = pytest.mark.gpu


def _record_bytes(eng, l, e, t):
    r = eng.expert_tile_record(l, e, t)
    return bytes((C.c_uint8 * r["bytes"]).from_address(r["ptr"])), r


# (restatement, format code, link-bytes ratio bound at Mixtral width; XBH's 24 KB of decode tables
# per tile weigh more on the tiny shape's 344 KB tiles)
FORMATS = {"xb12": (X, 1, 0.76), "xbh": (XH, 2, 0.675)}


@pytest.mark.parametrize("store", ["xb12", "xbh"])
@pytest.mark.parametrize("d,f,tiles", [(256, 896, 4), (4096, 14336, 4)])
def test_store_records_match_reference_encoder(d, f, tiles, store):
    ref_mod, code, ratio = FORMATS[store]
    with P.Engine(P.ModelSpec(2, 4, 2, d)) as eng:
        eng.experts_init(f, tiles, seed=5, store_format=store)
        fmt, link = eng.experts_format()
        assert fmt == store and link < (ratio if d >= 4096 else ratio + 0.08) * 8 * 3 * f * d * 2
        n = 3 * f * d // tiles
        for l, e in [(0, 0), (1, 3)]:
            raw = O.expert_init(5, l, e, d, f, tiles)
            assert np.array_equal(eng.expert_read(l, e), raw)
            for t in range(tiles):
                got, meta = _record_bytes(eng, l, e, t)
                ref, rmeta = ref_mod.encode(raw[t * n:(t + 1) * n])
                assert meta["format"] == rmeta["format"] == code
                assert (meta["base"], meta["n_escapes"]) == (rmeta["base"], rmeta["n_exc"])
                assert meta["esc_offset"] == rmeta["exc_off"] and meta["nib_offset"] == rmeta["nib_off"]
                assert got == ref


@pytest.mark.parametrize("store", ["xb12", "xbh"])
def test_expert_set_real_weights_encode_and_raw_fallback(store):
    d, f, tiles = 256, 512, 2
    rng = np.random.default_rng(7)
    w1 = X_bf16(rng.standard_normal((f, d)) * 0.05)
    w3 = X_bf16(rng.standard_normal((f, d)) * 0.05)
    w2 = rng.integers(0, 1 << 16, (d, f), dtype=np.uint16)  # exponents everywhere: tiles stay raw
    w2[:, : f // 2] = X_bf16(rng.standard_normal((d, f // 2)) * 0.05)
    with P.Engine(P.ModelSpec(1, 2, 2, d)) as raw_eng, P.Engine(P.ModelSpec(1, 2, 2, d)) as xb_eng:
        raw_eng.experts_alloc(f, tiles)
        xb_eng.experts_alloc(f, tiles, store_format=store)
        for eng in (raw_eng, xb_eng):
            eng.expert_set(0, 1, w1, w3, w2)
            eng.expert_set(0, 0, w1, w3, X_bf16(np.ones((d, f)) * 0.01))
        for e in (0, 1):
            assert np.array_equal(xb_eng.expert_read(0, e), raw_eng.expert_read(0, e))
        formats = [xb_eng.expert_tile_record(0, 1, t)["format"] for t in range(tiles)]
        assert 0 in formats  # the random-bit W2 columns make a tile not worth coding
        assert xb_eng.expert_tile_record(0, 0, 0)["format"] == FORMATS[store][1]


def X_bf16(a):
    u = np.ascontiguousarray(a, dtype=np.float32).view(np.uint32)
    return ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)


def _decode(g, fmt, T, batch=1, timeline=None):
    w, fg = oracle_inputs(g)
    cfg = sim_config(g)
    with P.Engine(P.ModelSpec(w.L, w.N, w.K, w.D)) as eng:
        eng.load_gates(w.gates, fg)
        eng.experts_init(224 * cfg.tile_count_per_expert, cfg.tile_count_per_expert, seed=4, store_format=fmt)
        eng.decode_begin(g["sim_capacities"], w.fisher, g["tau"], cfg, int(g["workload"]["seed"]), T)
        if timeline:
            eng.decode_record_timeline(True)
        hid = np.zeros((T, w.L, w.D), dtype=np.float32)
        eng.decode_tokens(w.acts[:T], w.scores[:T], hid)
        n = eng.decode_timeline_write(timeline) if timeline else 0
        st = eng.decode_stats()
        r = eng.decode_end(cfg, T)
    return hid, r, st, n


@pytest.mark.parametrize("store", ["xb12", "xbh"])
@pytest.mark.parametrize("name", ["tiny", "tiny_transfer_heavy", "tiny_budget0"])
def test_decode_over_coded_store_is_bit_identical(name, store, tmp_path):
    g = load_golden(name)
    T = 24
    h0, r0, s0, _ = _decode(g, "bf16", T)
    path = tmp_path / "tl.jsonl"
    h1, r1, s1, n = _decode(g, store, T, timeline=str(path))
    assert np.array_equal(h0, h1)
    assert r0.metrics == r1.metrics and np.array_equal(r0.timeline, r1.timeline)
    # how many queued prefetch tiles get cancelled before issue depends on physical timing, so
    # compare bytes per issued tile
    if s0["tile_copies"] and s1["tile_copies"]:
        assert s1["copy_bytes"] / s1["tile_copies"] < 0.8 * s0["copy_bytes"] / s0["tile_copies"]
    ev = TL.load(path)
    assert len(ev) == n
    assert not TL.check_causality(ev) and not TL.check_stream_exclusivity(ev)
    assert not TL.check_conservation(ev, r1.metrics, s1)


@pytest.mark.parametrize("store,lo,hi", [("xb12", 0.74, 0.76), ("xbh", 0.655, 0.675)])
def test_decode_mixtral_width_coded_vs_bf16(store, lo, hi):
    """88 MB tiles (66 / 58 MB records) through the staging ring and the decode stream: outputs and
    trace identical to the bf16 store, link bytes ~75 % (XB12) / ~66 % (XBH)."""
    from paper_2408_10284_b200 import workloads as W
    wl = W.mixtral_8x7b(tokens=4, budget=8)
    L = 3
    w = O.generate_trace(L, 8, 2, 4096, wl.tokens, wl.concentration, wl.drift, wl.gate_seed, wl.token_seed, False,
                         wl.fisher_scales[:L], wl.drift_scales[:L])
    tau = O.calibrate_threshold(w, wl.target_single_ratio)
    caps = [2, 2, 2]
    cfg = P.SimConfig()
    outs = []
    for fmt in ("bf16", store):
        with P.Engine(P.ModelSpec(L, 8, 2, 4096)) as eng:
            eng.load_gates(w.gates)
            eng.experts_init(wl.ffn, 4, seed=9, store_format=fmt)
            eng.decode_begin(caps, w.fisher, tau, cfg, 0, wl.tokens)
            hid = np.zeros((wl.tokens, L, 4096), dtype=np.float32)
            eng.decode_tokens(w.acts, w.scores, hid)
            st = eng.decode_stats()
            r = eng.decode_end(cfg, wl.tokens)
            outs.append((hid, r, st))
    (h0, r0, s0), (h1, r1, s1) = outs
    assert np.array_equal(h0, h1)
    assert r0.metrics == r1.metrics and np.array_equal(r0.timeline, r1.timeline)
    # bytes per issued tile (how many queued prefetches get cancelled depends on physical timing)
    assert lo < (s1["copy_bytes"] / s1["tile_copies"]) / (s0["copy_bytes"] / s0["tile_copies"]) < hi


@pytest.mark.parametrize("store", ["xb12", "xbh"])
def test_copy_tiles_decodes_coded(store):
    import torch
    d, f, tiles = 4096, 14336, 4
    with P.Engine(P.ModelSpec(1, 2, 2, d)) as eng:
        eng.experts_init(f, tiles, seed=3, store_format=store)
        buf = torch.empty(eng.expert_bytes() // 2, dtype=torch.int16, device="cuda")
        eng.copy_tiles(0, 1, 1, 2, buf.data_ptr())  # tiles 1..2 only
        torch.cuda.synchronize()
        got = buf.cpu().numpy().view(np.uint16)
        ref = O.expert_init(3, 0, 1, d, f, tiles)
        n = ref.size // tiles
        assert np.array_equal(got[n:3 * n], ref[n:3 * n])
        x = np.random.default_rng(0).standard_normal(d)
        y = eng.expert_ffn(0, 1, x)  # host helper uploads through the decode path too
        yr = O.swiglu(ref, d, f, tiles, x.astype(np.float32))
        assert np.abs(y - yr).max() / np.abs(yr).max() < 1e-4


@pytest.mark.parametrize("store", ["xb12", "xbh"])
def test_degenerate_exponent_tiles(store):
    """Edge cases of the codes: a tile with a single exponent (XBH: one 1-bit code, 128 codes per
    128-bit chunk — the decoder's slot capacity), two exponents, and exponents far outside any window
    (escapes past the raw-fallback cap): records match the restatement, decodes are exact."""
    d, f, tiles = 256, 512, 2
    rng = np.random.default_rng(11)
    one = np.full((f, d), 0x3F80, dtype=np.uint16)                       # every weight 1.0
    two = np.where(rng.random((f, d)) < 0.5, 0x3F80, 0x4000).astype(np.uint16)  # 1.0 / 2.0
    w2_one = np.full((d, f), 0xBF80, dtype=np.uint16)                    # -1.0
    spread = rng.integers(0, 1 << 16, (d, f), dtype=np.uint16)           # all exponents: raw fallback
    ref_mod, code, _ = FORMATS[store]
    with P.Engine(P.ModelSpec(1, 3, 2, d)) as raw_eng, P.Engine(P.ModelSpec(1, 3, 2, d)) as eng:
        raw_eng.experts_alloc(f, tiles)
        eng.experts_alloc(f, tiles, store_format=store)
        for e_ in (raw_eng, eng):
            e_.expert_set(0, 0, one, one, w2_one)
            e_.expert_set(0, 1, two, one, two.T.copy())
            e_.expert_set(0, 2, two, one, spread)
        n = 3 * f * d // tiles
        for e in range(3):
            raw = raw_eng.expert_read(0, e)
            assert np.array_equal(eng.expert_read(0, e), raw)
            for t in range(tiles):
                got, meta = _record_bytes(eng, 0, e, t)
                ref, rmeta = ref_mod.encode(raw[t * n:(t + 1) * n])
                assert meta["format"] == rmeta["format"]
                if meta["format"]:
                    assert got == ref
        assert eng.expert_tile_record(0, 0, 0)["format"] == code
        # the device decode path (copy_tiles: staging + decode kernels) on every tile
        import torch
        buf = torch.empty(eng.expert_bytes() // 2, dtype=torch.int16, device="cuda")
        for e in range(3):
            eng.copy_tiles(0, e, 0, tiles, buf.data_ptr())
            torch.cuda.synchronize()
            assert np.array_equal(buf.cpu().numpy().view(np.uint16), raw_eng.expert_read(0, e))


def test_xbh_last_code_straddles_into_a_new_block():
    """The sweep's seed-90427 failure mode, pinned: a tile whose last code runs into a final chunk
    that opens a new decode block without a code start (gap -> end of codes, block base n)."""
    import torch
    from test_xbh_cpu import straddle_tile
    d, f = 256, 160
    n = 3 * f * d
    w, total = straddle_tile(n=n)
    # invert the tile-major packing (one tile): rows (W1 r, W3 r) for r < f, then W2^T rows
    w1 = np.stack([w[r * 2 * d: r * 2 * d + d] for r in range(f)])
    w3 = np.stack([w[r * 2 * d + d: (r + 1) * 2 * d] for r in range(f)])
    w2 = np.ascontiguousarray(w[2 * f * d:].reshape(f, d).T)
    with P.Engine(P.ModelSpec(1, 2, 2, d)) as eng:
        eng.experts_alloc(f, 1, store_format="xbh")
        eng.expert_set(0, 1, w1, w3, w2)
        assert np.array_equal(eng.expert_read(0, 1), w)
        got, meta = _record_bytes(eng, 0, 1, 0)
        ref, rmeta = XH.encode(w)
        assert meta["format"] == 2 and got == ref
        buf = torch.empty(n, dtype=torch.int16, device="cuda")
        eng.copy_tiles(0, 1, 0, 1, buf.data_ptr())
        torch.cuda.synchronize()
        assert np.array_equal(buf.cpu().numpy().view(np.uint16), w)


def test_xbh_largest_tiles_8x22b_single_tile():
    """Mixtral-8x22B expert shape as ONE tile (d 6144, ffn 16384: 302 M values, ~3.3 G code bits —
    near the format's u32 bit-offset limit; ~24k decode blocks): store, host and device decodes exact."""
    import torch
    d, f, tiles = 6144, 16384, 1
    with P.Engine(P.ModelSpec(1, 2, 2, d)) as eng:
        eng.experts_init(f, tiles, seed=21, store_format="xbh")
        r = eng.expert_tile_record(0, 1, 0)
        assert r["format"] == 2 and r["bytes"] < 0.67 * 3 * f * d * 2
        ref = O.expert_init(21, 0, 1, d, f, tiles)
        assert np.array_equal(eng.expert_read(0, 1), ref)
        buf = torch.empty(ref.size, dtype=torch.int16, device="cuda")
        eng.copy_tiles(0, 1, 0, 1, buf.data_ptr())
        torch.cuda.synchronize()
        assert np.array_equal(buf.cpu().numpy().view(np.uint16), ref)


def test_coded_store_pins_only_its_records():
    """A synthetic coded store is encoded into unpinned blocks and pinned over its records only: pinned
    bytes ~ the records (XBH ~0.67 of bf16); reads, copies and a later expert_set (which pins the
    whole block) still work."""
    import torch
    d, f, tiles = 4096, 14336, 4
    with P.Engine(P.ModelSpec(1, 4, 2, d)) as eng:
        eng.experts_init(f, tiles, seed=8, store_format="xbh")
        info = eng.experts_info()
        raw_bytes = 4 * 3 * f * d * 2
        assert info["pinned_bytes"] < 0.69 * raw_bytes, info
        ref = O.expert_init(8, 0, 2, d, f, tiles)
        assert np.array_equal(eng.expert_read(0, 2), ref)
        buf = torch.empty(ref.size, dtype=torch.int16, device="cuda")
        eng.copy_tiles(0, 2, 0, tiles, buf.data_ptr())
        torch.cuda.synchronize()
        assert np.array_equal(buf.cpu().numpy().view(np.uint16), ref)
        # overwrite one expert with real-layout weights: the block is pinned whole again
        rng = np.random.default_rng(3)
        w1 = X_bf16(rng.standard_normal((f, d)) * 0.02)
        w3 = X_bf16(rng.standard_normal((f, d)) * 0.02)
        w2 = X_bf16(rng.standard_normal((d, f)) * 0.02)
        eng.expert_set(0, 1, w1, w3, w2)
        assert eng.experts_info()["pinned_bytes"] > info["pinned_bytes"]
        got = eng.expert_read(0, 1)
        n = 3 * f * d // tiles
        assert np.array_equal(got[:d], w1[0]) and np.array_equal(got[d:2 * d], w3[0])
        eng.copy_tiles(0, 1, 0, tiles, buf.data_ptr())
        torch.cuda.synchronize()
        assert np.array_equal(buf.cpu().numpy().view(np.uint16), got)
        assert n % 16 == 0
