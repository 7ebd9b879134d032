"""Batched decode (BASELINE config 4): B token streams share one expert cache.

The reference is batch-1, so the batched policy is builder-defined (union of the
streams' selections and look-ahead lists, oracle/moe_oracle.c orc_simulate_batch) and pinned to the
reference at B = 1.  Contracts:
  * [cpu] orc_simulate_batch with B = 1 reproduces every golden (metrics, timeline, decisions);
  * [cpu] B identical streams behave like one stream (except per-stream single-decision counts);
  * [cpu] identity activated = cache hits + prefetch hits + on-demand, for any B;
  * [gpu] the batched decode session (K1 over B streams + union policy + grouped tcgen05 FFN)
    returns the oracle's logical metrics and timeline bit-exactly, and every stream's MoE-layer
    output within BF16_TOL relative (bf16 activations into the tensor cores; north star: 2e-2 in
    bf16) of the fp64 oracle SwiGLU.
"""
import numpy as np
import pytest

from conftest import golden_names, load_golden
from helpers import assert_metrics, assert_timeline, oracle_inputs, sim_kwargs
from oracle import oracle as O

BF16_TOL = 2e-2


@pytest.mark.parametrize("name", golden_names())
def test_batch_core_b1_is_reference(name):
    g = load_golden(name)
    w, fg = oracle_inputs(g)
    r = O.simulate_batch([w], g["sim_capacities"], g["tau"], first_gate=fg, **sim_kwargs(g))
    assert_metrics(g, r.metrics, r.latency_per_token, r.od_per_layer)
    assert_timeline(g, r.timeline)
    assert np.array_equal(r.decisions[0], O.simulate(w, g["sim_capacities"], g["tau"], first_gate=fg,
                                                     **sim_kwargs(g)).decisions)


def _streams(B, L=4, N=8, K=2, D=256, T=10, seed0=5000):
    return [O.generate_trace(L, N, K, D, T, 0.6, 0.18, 99, seed0 + b, False, [2.0, 1.2, 0.7, 0.35][:L],
                             [1.8, 1.2, 0.8, 0.45][:L]) for b in range(B)]


def test_identical_streams_equal_one_stream():
    w = _streams(1)[0]
    fg = O.train_first_gate(w, steps=50)
    tau = O.calibrate_threshold(w, 0.24)
    one = O.simulate_batch([w], [3, 2, 2, 1], tau, first_gate=fg)
    many = O.simulate_batch([w] * 5, [3, 2, 2, 1], tau, first_gate=fg)
    for k, v in one.metrics.items():
        assert many.metrics[k] == (5 * v if k == "single_expert_decisions" else v), k
    assert np.array_equal(one.timeline, many.timeline)
    for b in range(5):
        assert np.array_equal(many.decisions[b], one.decisions[0])


@pytest.mark.parametrize("B", [2, 4, 16])
def test_batch_identity_and_per_stream_decisions(B):
    ws = _streams(B)
    tau = O.calibrate_threshold(ws[0], 0.24)
    r = O.simulate_batch(ws, [4, 3, 2, 2], tau)
    m = r.metrics
    assert m["experts_activated_total"] == m["cache_hits"] + m["prefetch_hits"] + m["on_demand_loads"]
    # per-stream decisions are the reference rule on each stream's own scores
    for b in (0, B - 1):
        solo = O.simulate(ws[b], [4, 3, 2, 2], tau)
        assert np.array_equal(r.decisions[b], solo.decisions)
        assert np.array_equal(r.predictions[b], solo.predictions)
    # union bound: each layer-step activates at most min(N, sum of stream selections)
    assert m["experts_activated_total"] <= ws[0].T * ws[0].L * min(8, 2 * B)


# ---------------------------------------------------------------------------------------------- gpu

def _moe_ref(ws, decisions, t, l, b, ffn, tiles, seed, cache):
    w = ws[b]
    sel = [int(e) for e in decisions[b, t, l] if e >= 0]
    sc = w.scores[t, l]
    denom = sum(sc[e] for e in sel)
    x32 = w.acts[t, l].astype(np.float32)
    acc = np.zeros(w.D)
    for e in sel:
        if (l, e) not in cache:
            cache[(l, e)] = O.expert_init(seed, l, e, w.D, ffn, tiles)
        wgt = 1.0 if len(sel) == 1 else sc[e] / denom
        acc += wgt * O.swiglu(cache[(l, e)], w.D, ffn, tiles, x32)
    return acc


def _run_batch(ws, caps, tau, fg, ffn, tiles, seed, calls, store="bf16"):
    import paper_2408_10284_b200 as P
    w0 = ws[0]
    B, T = len(ws), w0.T
    acts = np.ascontiguousarray(np.stack([w.acts for w in ws], axis=1))      # [T][B][L][d]
    scores = np.ascontiguousarray(np.stack([w.scores for w in ws], axis=1))  # [T][B][L][N]
    cfg = P.SimConfig()
    with P.Engine(P.ModelSpec(w0.L, w0.N, w0.K, w0.D)) as eng:
        eng.load_gates(w0.gates, fg)
        eng.experts_init(ffn, tiles, seed=seed, store_format=store)
        eng.decode_begin(caps, w0.fisher, tau, cfg, 0, T, batch=B)
        hid = np.zeros((T, B, w0.L, w0.D), dtype=np.float32)
        for a, b in zip(calls, calls[1:]):
            eng.decode_tokens(acts[a:b], scores[a:b], hid[a:b])
        r = eng.decode_end(cfg, T)
    return r, hid


@pytest.mark.gpu
@pytest.mark.parametrize("store", ["bf16", "xbh"])
@pytest.mark.parametrize("merge", ["0", "1", "2"])
@pytest.mark.parametrize("B,caps", [(4, [3, 2, 2, 1]), (16, [8, 4, 2, 0]), (64, [2, 2, 2, 2])])
def test_batched_decode_tiny(B, caps, merge, store, monkeypatch):
    """merge: ADAPMOE_TILE_MERGE — on-demand tiles (and the resident experts) grouped into fewer
    grouped launches off the critical path, or one launch per landed tile; store: bf16 or the
    Huffman-coded XBH store (tiles decoded on the copy engine's stream before K3 reads them)."""
    monkeypatch.setenv("ADAPMOE_TILE_MERGE", merge)
    ws = _streams(B, T=8)
    fg = O.train_first_gate(ws[0], steps=50)
    tau = O.calibrate_threshold(ws[0], 0.24)
    ffn, tiles, seed = 1024, 4, 7
    ref = O.simulate_batch(ws, caps, tau, first_gate=fg)
    r, hid = _run_batch(ws, caps, tau, fg, ffn, tiles, seed, [0, 3, 8], store=store)
    assert r.metrics == ref.metrics
    assert np.array_equal(r.timeline, ref.timeline)
    assert r.stats["tokens"] == 8 * B
    cache = {}
    for (t, l, b) in [(0, 0, 0), (2, 1, B - 1), (5, 3, B // 2), (7, 2, 1 % B), (3, 0, B - 1)]:
        moe = _moe_ref(ws, ref.decisions, t, l, b, ffn, tiles, seed, cache)
        got = hid[t, b, l].astype(np.float64) - ws[b].acts[t, l].astype(np.float32).astype(np.float64)
        err = np.abs(got - moe).max() / np.abs(moe).max()
        assert err < BF16_TOL, (t, l, b, err)


@pytest.mark.gpu
def test_batched_decode_mixtral_width():
    """Mixtral-8x7B expert shape (d 4096, ffn 14336, 4 tiles of 88 MB) on the grouped tcgen05 path,
    batch 16 over 2 layers with a small cache (on-demand tiles + resident experts)."""
    from paper_2408_10284_b200 import workloads as W
    wl = W.mixtral_8x7b(tokens=3, budget=8)
    L, B = 2, 16
    ws = [O.generate_trace(L, 8, 2, 4096, wl.tokens, wl.concentration, wl.drift, wl.gate_seed, wl.token_seed + b,
                           False, wl.fisher_scales[:L], wl.drift_scales[:L]) for b in range(B)]
    tau = O.calibrate_threshold(ws[0], wl.target_single_ratio)
    caps = [5, 3]
    ref = O.simulate_batch(ws, caps, tau)
    r, hid = _run_batch(ws, caps, tau, None, wl.ffn, 4, 9, [0, wl.tokens])
    assert r.metrics == ref.metrics
    assert np.array_equal(r.timeline, ref.timeline)
    cache = {}
    for (t, l, b) in [(0, 0, 3), (2, 1, 15)]:
        moe = _moe_ref(ws, ref.decisions, t, l, b, wl.ffn, 4, 9, cache)
        got = hid[t, b, l].astype(np.float64) - ws[b].acts[t, l].astype(np.float32).astype(np.float64)
        err = np.abs(got - moe).max() / np.abs(moe).max()
        assert err < BF16_TOL, (t, l, b, err)
