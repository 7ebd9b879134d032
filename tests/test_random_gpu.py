"""Randomized parity sweep on the GPU (the reference's acceptance criterion 4 analogue,
proj/tests/acceptance/acceptance_main.cpp:169-222): seeded random shapes, ticks and policy flags —
including the edges the reference tests exercise (N up to 64, top-1, d = 1 and odd d, one-token
traces, capacity-0 layers, look-ahead 0..3, gating / prefetch off).  For each case the GPU
generate_trace must reproduce the oracle's synthetic inputs bit for bit, and the GPU simulate_trace
(K1 + host engine) must return the oracle's metrics and full event timeline.  The oracle is pinned
to the reference by tests/test_oracle_golden.py and tests/test_oracle_vs_ref.py."""
import numpy as np
import pytest

import paper_2408_10284_b200 as P
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _case(seed):
    r = np.random.default_rng(1000 + seed)
    N = int(r.choice([2, 3, 4, 8, 16, 33, 64]))
    K = int(r.integers(1, min(4, N) + 1))
    L = int(r.integers(1, 7))
    D = int(r.choice([1, 5, 37, 64, 256, 1000, 4096]))
    T = int(r.choice([1, 2, 7, 20]))
    return dict(L=L, N=N, K=K, D=D, T=T, conc=float(r.choice([0.3, 0.6, 1.5])), drift=float(r.uniform(0.0, 0.5)),
                gate_seed=int(r.integers(0, 1000)), token_seed=int(r.integers(0, 1000)),
                target=float(r.choice([0.0, 0.12, 0.24, 0.5])), budget=int(r.integers(0, L * N + 3)),
                tiles=int(r.integers(1, 5)), transfer=int(r.integers(1, 6)), compute=int(r.integers(1, 4)),
                attention=int(r.integers(0, 9)), gate=int(r.integers(0, 3)), lookahead=int(r.integers(0, 4)),
                gating=bool(r.integers(0, 2)), prefetch=bool(r.integers(0, 2)), train=bool(r.integers(0, 2)),
                seed=int(r.integers(0, 50)))


@pytest.mark.parametrize("seed", range(128))
def test_random_pipeline_bit_exact(seed):
    c = _case(seed)
    L, N, K, D, T = c["L"], c["N"], c["K"], c["D"], c["T"]
    w = O.generate_trace(L, N, K, D, T, c["conc"], c["drift"], c["gate_seed"], c["token_seed"])
    fg = O.train_first_gate(w, steps=20) if (c["train"] and T >= 2) else None
    tau = O.calibrate_threshold(w, c["target"])
    alpha, beta = O.generate_profiles(w, tau, fg)
    caps, _ = O.dp_allocate(O.cost_table(alpha, beta, N), c["budget"])
    kw = dict(tiles=c["tiles"], tile_transfer=c["transfer"], tile_compute=c["compute"], attention=c["attention"],
              gate=c["gate"], lookahead=c["lookahead"], gating=c["gating"], prefetch=c["prefetch"], seed=c["seed"])
    ref = O.simulate(w, caps, tau, first_gate=fg, **kw)
    spec = P.ModelSpec(L, N, K, D)
    cfg = P.SimConfig(c["tiles"], c["transfer"], c["compute"], c["attention"], c["gate"], c["lookahead"],
                      P.PolicyFlags(c["gating"], c["prefetch"], True))
    with P.Engine(spec) as eng:
        g = eng.generate_trace(P.SynthConfig(spec, T, c["conc"], c["drift"], c["gate_seed"], c["token_seed"]))
        assert np.array_equal(g.gates, w.gates) and np.array_equal(g.acts, w.acts)
        assert np.array_equal(g.scores, w.scores) and np.array_equal(g.selected, w.selected)
        eng.load_gates(w.gates, fg)
        r = eng.simulate_trace(w.acts, w.scores, w.fisher, caps, tau, cfg, c["seed"])
    assert r.metrics == ref.metrics, c
    assert np.array_equal(r.timeline, ref.timeline), c


@pytest.mark.parametrize("seed", range(8))
def test_random_batched_decode(seed):
    """Batched decode (grouped tcgen05 FFN) on random ragged batches: the logical trace equals the
    oracle's union policy, every stream's layer output is within 2e-2 of the fp64 oracle."""
    r = np.random.default_rng(77 + seed)
    B = int(r.choice([2, 3, 5, 8, 17]))
    L, N, K, D = int(r.integers(1, 4)), 8, 2, int(r.choice([128, 256]))
    tiles = int(r.choice([1, 2, 4]))
    F = 64 * tiles * int(r.integers(1, 4))
    T = int(r.integers(1, 5))
    ws = [O.generate_trace(L, N, K, D, T, 0.6, 0.2, 5, 100 + b) for b in range(B)]
    tau = O.calibrate_threshold(ws[0], 0.24)
    caps = [int(x) for x in r.integers(0, N + 1, size=L)]
    lookahead = int(r.integers(0, 3))
    ref = O.simulate_batch(ws, caps, tau, tiles=tiles, lookahead=lookahead)
    acts = np.ascontiguousarray(np.stack([w.acts for w in ws], axis=1))
    scores = np.ascontiguousarray(np.stack([w.scores for w in ws], axis=1))
    cfg = P.SimConfig(tiles, 2, 1, 8, 1, lookahead, P.PolicyFlags(True, True, True))
    with P.Engine(P.ModelSpec(L, N, K, D)) as eng:
        eng.load_gates(ws[0].gates)
        eng.experts_init(F, tiles, seed=seed)
        eng.decode_begin(caps, ws[0].fisher, tau, cfg, 0, T, batch=B)
        hid = np.zeros((T, B, L, D), dtype=np.float32)
        eng.decode_tokens(acts, scores, hid)
        res = eng.decode_end(cfg, T)
    assert res.metrics == ref.metrics
    assert np.array_equal(res.timeline, ref.timeline)
    for (t, l, b) in [(0, 0, 0), (T - 1, L - 1, B - 1)]:
        sel = [int(e) for e in ref.decisions[b, t, l] if e >= 0]
        sc = ws[b].scores[t, l]
        x32 = ws[b].acts[t, l].astype(np.float32)
        moe = np.zeros(D)
        for e in sel:
            wgt = 1.0 if len(sel) == 1 else sc[e] / sum(sc[q] for q in sel)
            moe += wgt * O.swiglu(O.expert_init(seed, l, e, D, F, tiles), D, F, tiles, x32)
        got = hid[t, b, l].astype(np.float64) - x32.astype(np.float64)
        assert np.abs(got - moe).max() <= 2e-2 * np.abs(moe).max(), (t, l, b)
