"""BASELINE config 5 shape (Mixtral-8x22B: d 6144, ffn 16384, 4 tiles of 151 MB), the d > 8192 K2
instantiations, batch 64 at Mixtral-8x7B width, and the full 32-layer 8x7B headline decode against
the reference's own golden (tests/golden/mixtral_8x7b_t12.json, written by the unmodified
reference, oracle/_ref/moesim_ref).

Tolerances (north star): 1e-4 relative to max|y| for the batch-1 fp32-activation path (K2), 2e-2
for the batched bf16 path (K3).  Cache/transfer traces are bit-exact.
"""
import numpy as np
import pytest

import paper_2408_10284_b200 as P
from conftest import load_golden
from helpers import assert_metrics, assert_timeline, oracle_inputs, sim_config
from oracle import oracle as O
from paper_2408_10284_b200 import workloads as W

pytestmark = pytest.mark.gpu

REL_TOL = 1e-4
BF16_TOL = 2e-2


def _rel_err(got, ref):
    return float(np.abs(np.asarray(got, np.float64) - ref).max() / max(np.abs(ref).max(), 1e-30))


def _moe_ref(w, decisions, t, l, ffn, tiles, seed, cache):
    sel = [int(e) for e in decisions[t, l] if e >= 0]
    sc = w.scores[t, l]
    denom = sum(sc[e] for e in sel)
    x32 = w.acts[t, l].astype(np.float32)
    acc = np.zeros(w.D)
    for e in sel:
        if (l, e) not in cache:
            cache[(l, e)] = O.expert_init(seed, l, e, w.D, ffn, tiles)
        acc += (1.0 if len(sel) == 1 else sc[e] / denom) * O.swiglu(cache[(l, e)], w.D, ffn, tiles, x32)
    return acc


@pytest.mark.parametrize("kernel", ["ring", "rows"])
@pytest.mark.parametrize("d,f,tiles", [(6144, 16384, 4), (12288, 2048, 2), (16384, 1024, 1), (8192, 4096, 4)])
def test_expert_ffn_large_hidden(d, f, tiles, kernel, monkeypatch):
    """One expert through K2 at the 8x22B shape and at d > 8192 (the DV = 3/4 ring and DC = 4 row
    instantiations), both K2 kernels, against the fp64 oracle SwiGLU."""
    monkeypatch.setenv("ADAPMOE_K2", kernel)
    rng = np.random.default_rng(d ^ f)
    with P.Engine(P.ModelSpec(1, 2, 2, d)) as eng:
        eng.experts_init(f, tiles, seed=21)
        for e in range(2):
            x = rng.standard_normal(d)
            y = eng.expert_ffn(0, e, x)
            ref = O.swiglu(O.expert_init(21, 0, e, d, f, tiles), d, f, tiles, x.astype(np.float32))
            assert _rel_err(y, ref) < REL_TOL, (e, _rel_err(y, ref))


def _x22b_trace(L, tokens, budget, batch=1):
    wl = W.mixtral_8x22b(tokens=tokens, budget=budget)
    ws = [O.generate_trace(L, 8, 2, 6144, tokens, wl.concentration, wl.drift, wl.gate_seed, wl.token_seed + b,
                           False, wl.fisher_scales[:L], wl.drift_scales[:L]) for b in range(batch)]
    return wl, ws


@pytest.mark.parametrize("merge", ["0", "2"])
def test_decode_8x22b_shape_layers(merge, monkeypatch):
    """Config 5 expert shape over 4 layers at batch 1: 151 MB tiles copied tile by tile, prefetch,
    DP-sized cache of 12 experts; trace bit-exact with the oracle, sampled layer outputs within 1e-4.
    merge 0 = one K2 launch per landed tile, 2 = one launch per layer (the default at this size)."""
    monkeypatch.setenv("ADAPMOE_TILE_MERGE", merge)
    L, T = 4, 5
    wl, (w,) = _x22b_trace(L, T, 12)
    tau = O.calibrate_threshold(w, wl.target_single_ratio)
    alpha, beta = O.generate_profiles(w, tau, None)
    caps, _ = O.dp_allocate(O.cost_table(alpha, beta, 8), wl.budget)
    ref = O.simulate(w, caps, tau)
    cfg = P.SimConfig()
    with P.Engine(P.ModelSpec(L, 8, 2, 6144)) as eng:
        eng.load_gates(w.gates)
        eng.experts_init(wl.ffn, 4, seed=17)
        eng.decode_begin(caps, w.fisher, tau, cfg, 0, T)
        hid = np.zeros((T, L, 6144), dtype=np.float32)
        eng.decode_tokens(w.acts, w.scores, hid)
        r = eng.decode_end(cfg, T)
    assert r.metrics == ref.metrics
    assert np.array_equal(r.timeline, ref.timeline)
    cache = {}
    for (t, l) in [(0, 0), (2, 3), (4, 1)]:
        got = hid[t, l].astype(np.float64) - w.acts[t, l].astype(np.float32).astype(np.float64)
        assert _rel_err(got, _moe_ref(w, ref.decisions, t, l, wl.ffn, 4, 17, cache)) < REL_TOL, (t, l)


def _run_batch(ws, caps, tau, ffn, tiles, seed, T):
    w0 = ws[0]
    B = len(ws)
    acts = np.stack([w.acts[:T] for w in ws], axis=1)
    scores = np.stack([w.scores[:T] for w in ws], axis=1)
    cfg = P.SimConfig()
    with P.Engine(P.ModelSpec(w0.L, w0.N, w0.K, w0.D)) as eng:
        eng.load_gates(w0.gates)
        eng.experts_init(ffn, tiles, seed=seed)
        eng.decode_begin(caps, w0.fisher, tau, cfg, 0, T, batch=B)
        hid = np.zeros((T, B, w0.L, w0.D), dtype=np.float32)
        eng.decode_tokens(acts, scores, hid)
        r = eng.decode_end(cfg, T)
    return r, hid


def _batch_outputs_ok(ws, ref, hid, points, ffn, tiles, seed):
    cache = {}
    for (t, l, b) in points:
        moe = _moe_ref(ws[b], ref.decisions[b], t, l, ffn, tiles, seed, cache)
        got = hid[t, b, l].astype(np.float64) - ws[b].acts[t, l].astype(np.float32).astype(np.float64)
        err = np.abs(got - moe).max() / np.abs(moe).max()
        assert err < BF16_TOL, (t, l, b, err)


def test_batched_decode_8x22b_shape():
    """Config 5 shape on the grouped tcgen05 path (K3): batch 16 over 2 layers, small cache."""
    L, B, T = 2, 16, 3
    wl, ws = _x22b_trace(L, T, 8, batch=B)
    tau = O.calibrate_threshold(ws[0], wl.target_single_ratio)
    caps = [5, 3]
    ref = O.simulate_batch(ws, caps, tau)
    r, hid = _run_batch(ws, caps, tau, wl.ffn, 4, 23, T)
    assert r.metrics == ref.metrics
    assert np.array_equal(r.timeline, ref.timeline)
    _batch_outputs_ok(ws, ref, hid, [(0, 0, 3), (2, 1, 15), (1, 0, 8)], wl.ffn, 4, 23)


def test_batched_decode_b64_mixtral_width():
    """BASELINE config 4 at its own size: batch 64 at the Mixtral-8x7B expert shape over 2 layers."""
    wl = W.mixtral_8x7b(tokens=3, budget=8)
    L, B, T = 2, 64, 3
    ws = [O.generate_trace(L, 8, 2, 4096, T, wl.concentration, wl.drift, wl.gate_seed, wl.token_seed + b, False,
                           wl.fisher_scales[:L], wl.drift_scales[:L]) for b in range(B)]
    tau = O.calibrate_threshold(ws[0], wl.target_single_ratio)
    caps = [4, 2]
    ref = O.simulate_batch(ws, caps, tau)
    r, hid = _run_batch(ws, caps, tau, wl.ffn, 4, 29, T)
    assert r.metrics == ref.metrics
    assert np.array_equal(r.timeline, ref.timeline)
    assert r.stats["tokens"] == T * B
    _batch_outputs_ok(ws, ref, hid, [(0, 0, 0), (1, 1, 63), (2, 0, 31), (2, 1, 47)], wl.ffn, 4, 29)


def test_headline_decode_32_layers_budget64_vs_reference_golden():
    """The headline configuration itself: Mixtral-8x7B shape, 32 layers, budget 64 (the reference's
    DP allocation in the golden), 12 tokens of the reference's own trace, physically decoded (all
    256 experts pinned in host memory, 88 MB tile copies, K1 + K2).  Metrics, per-token latency,
    per-layer on-demand loads and the full event timeline equal the unmodified reference's golden;
    layer outputs at sampled (token, layer) points are within 1e-4 of the fp64 oracle."""
    g = load_golden("mixtral_8x7b_t12")
    w, fg = oracle_inputs(g)
    cfg = sim_config(g)
    T, ffn, seed = w.T, 14336, 31
    with P.Engine(P.ModelSpec(w.L, w.N, w.K, w.D)) as eng:
        eng.load_gates(w.gates, fg)
        eng.experts_init(ffn, cfg.tile_count_per_expert, seed=seed)
        eng.decode_begin(g["sim_capacities"], w.fisher, g["tau"], cfg, int(g["workload"]["seed"]), T)
        hid = np.zeros((T, w.L, w.D), dtype=np.float32)
        eng.decode_tokens(w.acts[:5], w.scores[:5], hid[:5])  # two calls: session state carries over
        eng.decode_tokens(w.acts[5:], w.scores[5:], hid[5:])
        r = eng.decode_end(cfg, T)
    assert_metrics(g, r.metrics, r.latency_per_token, r.on_demand_loads_per_layer)
    assert_timeline(g, r.timeline)
    assert r.stats["ffn_bytes"] == r.metrics["experts_activated_total"] * 3 * ffn * w.D * 2
    sim = O.simulate(w, g["sim_capacities"], g["tau"], first_gate=fg)
    cache = {}
    for (t, l) in [(0, 0), (3, 17), (7, 31), (11, 9)]:
        got = hid[t, l].astype(np.float64) - w.acts[t, l].astype(np.float32).astype(np.float64)
        assert _rel_err(got, _moe_ref(w, sim.decisions, t, l, ffn, cfg.tile_count_per_expert, seed, cache)) < REL_TOL


def test_free_running_8x22b_shape():
    """Free-running decode at the config-5 width (d 6144: the RMSNorm / fused-combine kernels need
    > 48 KB of shared memory): layer 1 of every token must equal x1 + sum_e w_e E_e(RMSNorm(x1)) on the
    GPU's own layer-0 output x1 (per-step parity of the hidden state, 1e-4)."""
    import math
    L, T = 2, 3
    wl, (w,) = _x22b_trace(L, T, 6)
    tau = O.calibrate_threshold(w, wl.target_single_ratio)
    caps = [3, 3]
    cfg = P.SimConfig()
    with P.Engine(P.ModelSpec(L, 8, 2, 6144)) as eng:
        eng.load_gates(w.gates)
        eng.experts_init(wl.ffn, 4, seed=19)
        eng.decode_begin(caps, w.fisher, tau, cfg, 0, T, free_running=True, concentration=wl.concentration)
        hid = np.zeros((T, L, 6144), dtype=np.float32)
        eng.decode_tokens(w.acts, w.scores, hid)
        r = eng.decode_end(cfg, T)
    assert np.isfinite(hid).all()
    assert r.stats["router_launches"] == L * T
    cache = {}
    for t in range(T):
        x1 = hid[t, 0].astype(np.float64)
        rms = math.sqrt(float(np.dot(x1, x1)) / 6144 + 1e-5)
        xn = (x1 / rms).astype(np.float32)
        logits = xn.astype(np.float64) @ w.gates[1]
        s = np.exp((logits - logits.max()) / wl.concentration)
        s /= s.sum()
        top = np.argsort(-s, kind="stable")[:2]
        got = hid[t, 1].astype(np.float64) - x1
        # the decision may be one or two experts (adaptive gate); accept the closer of the two readings
        errs = []
        for sel in ([int(top[0])], [int(e) for e in top]):
            moe = np.zeros(6144)
            for e in sel:
                if e not in cache:
                    cache[e] = O.expert_init(19, 1, e, 6144, wl.ffn, 4)
                wgt = 1.0 if len(sel) == 1 else s[e] / s[list(sel)].sum()
                moe += wgt * O.swiglu(cache[e], 6144, wl.ffn, 4, xn)
            errs.append(_rel_err(got, moe))
        assert min(errs) < REL_TOL, (t, errs)
