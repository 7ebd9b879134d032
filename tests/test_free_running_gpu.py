"""Free-running decode (SURVEY §7.2's second mode): the residual stream x_l is the caller's input at
layer 0 and layer l-1's output after that; the router and the experts read RMSNorm(x_l) (Mixtral's
pre-MoE norm, no gain, eps 1e-5) and the layer output is x_l + sum_e w_e E_e(RMSNorm(x_l)), so the
hidden state flows through the offloaded experts; decisions come from the layer's gate
(softmax(logits / concentration), like the reference generator).  The reference has no such
mode (it replays stored scores), so parity is per step: given the hidden states the GPU produced,
the oracle restatement (reference rule on softmax of the exact fp64 logits) must yield the same
decisions and the same cache/transfer trace bit for bit, and every layer output must be within
1e-4 (fp32 activations, batch 1) / 2e-2 (bf16 activations, batched) of the fp64 SwiGLU of its
input."""
import math

import numpy as np
import pytest

import paper_2408_10284_b200 as P
from conftest import load_golden
from helpers import oracle_inputs, sim_config
from oracle import oracle as O

pytestmark = pytest.mark.gpu
CONC = 0.6
EPS = 1e-5


def rmsnorm_like_gpu(x):
    """The kernel's exact order: lane j sums x_i^2 for i = j, j+32, ... (separately rounded), then an
    xor butterfly over the 32 lane sums; rms = sqrt(ss / d + eps); x / rms."""
    d = len(x)
    xs = [float(v) for v in x]
    lanes = [0.0] * 32
    for j in range(32):
        acc = 0.0
        for i in range(j, d, 32):
            acc = acc + xs[i] * xs[i]
        lanes[j] = acc
    for off in (16, 8, 4, 2, 1):
        lanes = [lanes[j] + lanes[j ^ off] for j in range(32)]
    rms = math.sqrt(lanes[0] / d + EPS)
    return np.array([v / rms for v in xs])


def run_and_check(batch, tol, caps=None, T=10, store="bf16"):
    """Free-running decode of the tiny case; asserts per-step parity with the oracle; returns
    (result, hidden, decode stats)."""
    g = load_golden("tiny")
    w0, fg = oracle_inputs(g)
    cfg = sim_config(g)
    caps = g["sim_capacities"] if caps is None else caps
    tau = g["tau"]
    L, N, K, D = w0.L, w0.N, w0.K, w0.D
    ffn, tiles, seed = 1024, cfg.tile_count_per_expert, 3
    ws = [w0] + [O.generate_trace(L, N, K, D, T, 0.6, 0.18, 99, 7000 + b, False, [2.0, 1.2, 0.7, 0.35],
                                  [1.8, 1.2, 0.8, 0.45]) for b in range(1, batch)]
    acts = np.ascontiguousarray(np.stack([w.acts[:T] for w in ws], axis=1))      # [T][B][L][d]
    scores = np.ascontiguousarray(np.stack([w.scores[:T] for w in ws], axis=1))
    with P.Engine(P.ModelSpec(L, N, K, D)) as eng:
        eng.load_gates(w0.gates, fg)
        eng.experts_init(ffn, tiles, seed=seed, store_format=store)
        eng.decode_begin(caps, w0.fisher, tau, cfg, 0, T, batch=batch, free_running=True, concentration=CONC)
        hid = np.zeros((T, batch, L, D), dtype=np.float32)
        if batch == 1:
            eng.decode_tokens(acts[:, 0], scores[:, 0], hid[:, 0])
        else:
            eng.decode_tokens(acts, scores, hid)
        stats = eng.decode_stats()
        r = eng.decode_end(cfg, T)
    # the residual stream and router / expert inputs the GPU used
    res = acts.copy()
    res[:, :, 1:] = hid[:, :, :-1].astype(np.float64)
    xin = np.zeros_like(res)
    for t in range(T):
        for b in range(batch):
            for l in range(L):
                xin[t, b, l] = rmsnorm_like_gpu(res[t, b, l])
    streams = []
    for b in range(batch):
        sb = np.zeros((T, L, N))
        for t in range(T):
            for l in range(L):
                sb[t, l] = O.gate_scores(w0.gates[l], xin[t, b, l], CONC)
        streams.append(O.Workload(L, N, K, D, T, w0.gates, np.ascontiguousarray(xin[:, b]), sb,
                                  np.zeros((T, L, K), np.int32), w0.fisher))
    ref = O.simulate_batch(streams, caps, tau, first_gate=fg)
    assert r.metrics == ref.metrics
    assert np.array_equal(r.timeline, ref.timeline)
    # outputs: x + sum_e w_e SwiGLU_e(x) on the GPU's own inputs
    cache = {}
    worst = 0.0
    for t in range(T):
        for l in range(L):
            for b in range(batch):
                sel = [int(e) for e in ref.decisions[b, t, l] if e >= 0]
                sc = streams[b].scores[t, l]
                x32 = xin[t, b, l].astype(np.float32)
                moe = np.zeros(D)
                for e in sel:
                    if (l, e) not in cache:
                        cache[(l, e)] = O.expert_init(seed, l, e, D, ffn, tiles)
                    wgt = 1.0 if len(sel) == 1 else sc[e] / sum(sc[q] for q in sel)
                    moe += wgt * O.swiglu(cache[(l, e)], D, ffn, tiles, x32)
                got = hid[t, b, l].astype(np.float64) - res[t, b, l].astype(np.float32).astype(np.float64)
                worst = max(worst, np.abs(got - moe).max() / np.abs(moe).max())
    assert worst < tol, worst
    # the hidden state really evolves (layer inputs differ from the replayed trace) and stays bounded
    assert not np.allclose(res[:, :, 1:], acts[:, :, 1:])
    assert np.isfinite(hid).all()
    return r, hid, stats


@pytest.mark.parametrize("store", ["bf16", "xbh"])
@pytest.mark.parametrize("batch,tol", [(1, 1e-4), (4, 2e-2)])
def test_free_running_decode_matches_oracle_per_step(batch, tol, store):
    run_and_check(batch, tol, store=store)


@pytest.mark.parametrize("all_resident", [False, True])
def test_speculative_ffn_on_off(monkeypatch, all_resident):
    """Batch-1 free-running decode speculates the look-ahead's top-1 expert of the next layer (see
    DecodeSession::launch_speculative).  A hit sums that expert's partials from a launch with a
    different CTA split, so outputs are not bit-identical across on / off: both runs must keep
    per-step parity with the oracle, the speculative run must actually hit, and where the two runs
    took the same decisions their outputs agree within the fp32 tolerance."""
    caps = [8, 8, 8, 8] if all_resident else None
    monkeypatch.setenv("ADAPMOE_SPECULATE", "1")
    r_on, hid_on, st_on = run_and_check(1, 1e-4, caps=caps, T=12)
    monkeypatch.setenv("ADAPMOE_SPECULATE", "0")
    r_off, hid_off, st_off = run_and_check(1, 1e-4, caps=caps, T=12)
    assert st_off["spec_launches"] == 0 and st_off["spec_hits"] == 0
    assert st_on["spec_launches"] > 0 and st_on["spec_hits"] > 0, st_on
    assert st_on["spec_hits"] <= st_on["spec_launches"]
    if np.array_equal(r_on.timeline, r_off.timeline):
        err = np.abs(hid_on - hid_off).max() / np.abs(hid_off).max()
        assert err < 1e-4, err
