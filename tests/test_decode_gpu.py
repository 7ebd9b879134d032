"""Physical offloaded decode on the B200: K2 SwiGLU expert streaming, HBM slot pool, copy engine.

Contracts checked (tolerances written here, north star: 1e-4 relative in fp32):
  * expert weights in the pinned store are bit-identical to the oracle's counter-based init;
  * single-expert SwiGLU (bf16 weights, fp32 accumulation) within 1e-4 of the fp64 oracle,
    relative to max|y|;
  * decode_trace: the logical metrics and event timeline are bit-exact with the reference goldens
    while the FFN really runs, and every layer's MoE output x + sum_e w_e E_e(x) matches the oracle
    within 1e-4 relative to max|sum_e w_e E_e(x)|.
"""
import numpy as np
import pytest

import paper_2408_10284_b200 as P
from conftest import load_golden
from helpers import assert_metrics, assert_timeline, oracle_inputs, sim_config
from oracle import oracle as O

pytestmark = pytest.mark.gpu

REL_TOL = 1e-4


def _rel_err(got, ref):
    return float(np.abs(np.asarray(got, np.float64) - ref).max() / max(np.abs(ref).max(), 1e-30))


def test_expert_store_matches_oracle_init():
    import ctypes
    spec = P.ModelSpec(2, 4, 2, 256)
    with P.Engine(spec) as eng:
        eng.experts_init(896, 4, seed=11)
        n = 3 * 896 * 256
        for l, e in [(0, 0), (1, 3), (0, 2)]:
            ref = O.expert_init(11, l, e, 256, 896, 4)
            assert np.array_equal(eng.expert_read(l, e), ref)
            # zero-copy view of the pinned block (moe_expert_host_ptr)
            view = np.ctypeslib.as_array((ctypes.c_uint16 * n).from_address(eng.expert_host_ptr(l, e)))
            assert np.array_equal(view, ref)
        with pytest.raises(P.MoeError):
            eng.expert_host_ptr(2, 0)


@pytest.mark.parametrize("d,f,tiles", [(256, 896, 4), (512, 1024, 2), (256, 2048, 1), (4096, 14336, 4)])
def test_expert_ffn_matches_oracle(d, f, tiles):
    spec = P.ModelSpec(1, 2, 2, d)
    rng = np.random.default_rng(d + f)
    with P.Engine(spec) as eng:
        eng.experts_init(f, tiles, seed=3)
        for e in range(2):
            x = rng.standard_normal(d)
            y = eng.expert_ffn(0, e, x)
            ref = O.swiglu(O.expert_init(3, 0, e, d, f, tiles), d, f, tiles, x.astype(np.float32))
            assert _rel_err(y, ref) < REL_TOL


def _moe_reference(w, fg_unused, decisions, T, ffn, tiles, seed, layers_subset=None):
    """Oracle MoE-layer output per (token, layer): x + sum_e (s_e / sum_sel s) * SwiGLU_e(x)."""
    cache = {}
    out = {}
    for t in range(T):
        for l in range(w.L):
            if layers_subset is not None and (t, l) not in layers_subset:
                continue
            sel = [int(e) for e in decisions[t, l] if e >= 0]
            sc = w.scores[t, l]
            denom = sum(sc[e] for e in sel)
            x32 = w.acts[t, l].astype(np.float32)
            acc = np.zeros(w.D)
            for e in sel:
                if (l, e) not in cache:
                    cache[(l, e)] = O.expert_init(seed, l, e, w.D, ffn, tiles)
                wgt = 1.0 if len(sel) == 1 else sc[e] / denom
                acc += wgt * O.swiglu(cache[(l, e)], w.D, ffn, tiles, x32)
            out[(t, l)] = acc
    return out


@pytest.mark.parametrize("name", ["tiny", "tiny_budget0", "tiny_transfer_heavy", "tiny_prefetch_off", "tiny_nogate",
                                  "tiny_compute_heavy", "tiny_budget_full"])
def test_decode_trace_tiny(name):
    g = load_golden(name)
    w, fg = oracle_inputs(g)
    cfg = sim_config(g)
    ffn, seed = 224 * cfg.tile_count_per_expert, 5  # ffn/tiles = 224 (= 896/4 of the tiny config)
    T = w.T
    with P.Engine(P.ModelSpec(w.L, w.N, w.K, w.D)) as eng:
        eng.load_gates(w.gates, fg)
        eng.experts_init(ffn, cfg.tile_count_per_expert, seed=seed)
        eng.decode_begin(g["sim_capacities"], w.fisher, g["tau"], cfg, int(g["workload"]["seed"]), T)
        hid = np.zeros((T, w.L, w.D), dtype=np.float32)
        # split the trace over three calls: session state must carry over
        cuts = [0, 5, 37, T]
        for a, b in zip(cuts, cuts[1:]):
            eng.decode_tokens(w.acts[a:b], w.scores[a:b], hid[a:b])
        r = eng.decode_end(cfg, T)
    assert_metrics(g, r.metrics, r.latency_per_token, r.on_demand_loads_per_layer)
    assert_timeline(g, r.timeline)
    st = r.stats
    assert st["tokens"] == T
    assert st["ffn_bytes"] == r.metrics["experts_activated_total"] * 3 * ffn * w.D * 2
    # copy / stall accounting by request class (bench host_link.prefetch_*): prefetch shares are
    # parts of the totals; no prefetch traffic when the policy prefetches nothing
    eps = 1e-6
    assert 0 <= st["prefetch_used_copy_ms"] <= st["prefetch_copy_ms"] + eps <= st["copy_busy_ms"] + 2 * eps
    assert 0 <= st["prefetch_stall_ms"] <= st["stall_ms"] + eps
    assert 0 <= st["prefetch_tile_copies"] <= st["tile_copies"]
    if not cfg.policy.prefetch or cfg.lookahead_depth == 0:
        assert st["prefetch_tile_copies"] == 0 and st["prefetch_copy_ms"] == 0
    sim = O.simulate(w, g["sim_capacities"], g["tau"], first_gate=fg,
                     **{k: v for k, v in __import__("helpers").sim_kwargs(g).items()})
    subset = {(t, l) for t in range(0, T, 7) for l in range(w.L)}
    ref = _moe_reference(w, fg, sim.decisions, T, ffn, cfg.tile_count_per_expert, seed, subset)
    for (t, l), moe in ref.items():
        got = hid[t, l].astype(np.float64) - w.acts[t, l].astype(np.float32).astype(np.float64)
        assert _rel_err(got, moe) < REL_TOL, (t, l)


def test_decode_device_inputs_match_host_inputs():
    import torch
    g = load_golden("tiny")
    w, fg = oracle_inputs(g)
    cfg = sim_config(g)
    T = 12
    outs = []
    for on_device in (False, True):
        with P.Engine(P.ModelSpec(w.L, w.N, w.K, w.D)) as eng:
            eng.load_gates(w.gates, fg)
            eng.experts_init(896, 4, seed=2)
            eng.decode_begin(g["sim_capacities"], w.fisher, g["tau"], cfg, 0, T)
            if on_device:
                a = torch.from_numpy(np.ascontiguousarray(w.acts[:T])).cuda()
                s = torch.from_numpy(np.ascontiguousarray(w.scores[:T])).cuda()
                h = torch.zeros((T, w.L, w.D), dtype=torch.float32, device="cuda")
                torch.cuda.synchronize()
                eng.decode_tokens(a.data_ptr(), s.data_ptr(), (h.data_ptr(), T), on_device=True)
                outs.append(h.cpu().numpy())
            else:
                h = np.zeros((T, w.L, w.D), dtype=np.float32)
                eng.decode_tokens(w.acts[:T], w.scores[:T], h)
                outs.append(h)
            eng.decode_end(cfg, T)
    assert np.array_equal(outs[0], outs[1])


def test_decode_mixtral_width_layers():
    """Mixtral-8x7B expert shape (d 4096, ffn 14336, 4 tiles) over 4 layers: tile-granular on-demand
    copies of 88 MB tiles, prefetch, DP-sized cache of 8 experts."""
    from paper_2408_10284_b200 import workloads as W
    wl = W.mixtral_8x7b(tokens=6, budget=8)
    L = 4
    w = O.generate_trace(L, 8, 2, 4096, wl.tokens, wl.concentration, wl.drift, wl.gate_seed, wl.token_seed, False,
                         wl.fisher_scales[:L], wl.drift_scales[:L])
    tau = O.calibrate_threshold(w, wl.target_single_ratio)
    alpha, beta = O.generate_profiles(w, tau, None)
    caps, _ = O.dp_allocate(O.cost_table(alpha, beta, 8), wl.budget)
    ref = O.simulate(w, caps, tau)
    cfg = P.SimConfig()
    with P.Engine(P.ModelSpec(L, 8, 2, 4096)) as eng:
        eng.load_gates(w.gates)
        eng.experts_init(wl.ffn, 4, seed=9)
        eng.decode_begin(caps, w.fisher, tau, cfg, 0, wl.tokens)
        hid = np.zeros((wl.tokens, L, 4096), dtype=np.float32)
        eng.decode_tokens(w.acts, w.scores, hid)
        r = eng.decode_end(cfg, wl.tokens)
    assert r.metrics == ref.metrics
    assert np.array_equal(r.timeline, ref.timeline)
    moe = _moe_reference(w, None, ref.decisions, wl.tokens, wl.ffn, 4, 9, {(0, 1), (3, 2), (5, 3)})
    for (t, l), m in moe.items():
        got = hid[t, l].astype(np.float64) - w.acts[t, l].astype(np.float32).astype(np.float64)
        assert _rel_err(got, m) < REL_TOL, (t, l)


@pytest.mark.parametrize("name", ["tiny_budget0", "tiny_transfer_heavy", "tiny"])
def test_slot_reuse_ordering_every_output(name):
    """Slot recycling under host run-ahead, at the tightest feasible staging pool: every on-demand /
    prefetch copy reuses a slot that an earlier, possibly still enqueued, layer read.  Slots return to
    the pool only after that layer's completion event, so every (token, layer) output must equal the
    oracle's.  Smaller pools fail loudly (MOE_E_INFEASIBLE, "slot pool exhausted")."""
    g = load_golden(name)
    w, fg = oracle_inputs(g)
    cfg = sim_config(g)
    ffn, seed, T = 224 * cfg.tile_count_per_expert, 9, 24
    for staging in range(1, 33):
        with P.Engine(P.ModelSpec(w.L, w.N, w.K, w.D)) as eng:
            eng.load_gates(w.gates, fg)
            eng.experts_init(ffn, cfg.tile_count_per_expert, seed=seed)
            eng.decode_begin(g["sim_capacities"], w.fisher, g["tau"], cfg, int(g["workload"]["seed"]), T, staging)
            hid = np.zeros((T, w.L, w.D), dtype=np.float32)
            try:
                eng.decode_tokens(w.acts[:T], w.scores[:T], hid)
            except P.MoeError as e:
                assert e.code == 5 and "exhausted" in str(e), e
                continue
            r = eng.decode_end(cfg, T)
            break
    else:
        pytest.fail("no feasible staging pool up to 32 slots")
    sim = O.simulate(w, g["sim_capacities"], g["tau"], first_gate=fg, T=T,
                     **{k: v for k, v in __import__("helpers").sim_kwargs(g).items()})
    assert r.metrics == sim.metrics
    ref = _moe_reference(w, fg, sim.decisions, T, ffn, cfg.tile_count_per_expert, seed)
    for (t, l), moe in ref.items():
        got = hid[t, l].astype(np.float64) - w.acts[t, l].astype(np.float32).astype(np.float64)
        assert _rel_err(got, moe) < REL_TOL, (t, l, staging)


def _decode_outputs(g, T, cuts, batch=1):
    w, fg = oracle_inputs(g)
    cfg = sim_config(g)
    with P.Engine(P.ModelSpec(w.L, w.N, w.K, w.D)) as eng:
        eng.load_gates(w.gates, fg)
        eng.experts_init(224 * cfg.tile_count_per_expert, cfg.tile_count_per_expert, seed=4)
        eng.decode_begin(g["sim_capacities"], w.fisher, g["tau"], cfg, int(g["workload"]["seed"]), T)
        hid = np.zeros((T, w.L, w.D), dtype=np.float32)
        for a, b in zip(cuts, cuts[1:]):
            eng.decode_tokens(w.acts[a:b], w.scores[a:b], hid[a:b])
        r = eng.decode_end(cfg, T)
    return hid, r


@pytest.mark.parametrize("window", ["1", "3", "7"])
def test_route_windows_bit_identical(window, monkeypatch):
    """Trace replay routes a window of tokens per K1 launch (the whole call at bench sizes).  Forcing
    several windows per call (ADAPMOE_ROUTE_WINDOW) must not change a bit of the outputs or trace."""
    g = load_golden("tiny_transfer_heavy")
    T, cuts = 20, [0, 9, 20]
    ref_hid, ref = _decode_outputs(g, T, cuts)
    monkeypatch.setenv("ADAPMOE_ROUTE_WINDOW", window)
    hid, r = _decode_outputs(g, T, cuts)
    assert r.metrics == ref.metrics and np.array_equal(r.timeline, ref.timeline)
    assert np.array_equal(hid, ref_hid)
    assert r.stats["router_launches"] == sum(-(-(b - a) // int(window)) for a, b in zip(cuts, cuts[1:]))


@pytest.mark.parametrize("merge", ["1", "2"])
@pytest.mark.parametrize("name", ["tiny", "tiny_transfer_heavy", "tiny_budget0", "tiny_prefetch_off"])
def test_tile_merge_every_output(name, merge, monkeypatch):
    """ADAPMOE_TILE_MERGE=1 ("groups"): an on-demand expert's tiles share one K2 launch once landed,
    the layer's last expert keeps its final tile alone, resident experts ride with the first
    on-demand group.  ADAPMOE_TILE_MERGE=2 ("layer", the default for >= 8 MiB tiles): the layer's
    whole FFN in one launch after its last tile lands.  The trace is untouched and every output
    matches the oracle."""
    monkeypatch.setenv("ADAPMOE_TILE_MERGE", merge)
    g = load_golden(name)
    w, fg = oracle_inputs(g)
    cfg = sim_config(g)
    ffn, seed, T = 224 * cfg.tile_count_per_expert, 13, 24
    with P.Engine(P.ModelSpec(w.L, w.N, w.K, w.D)) as eng:
        eng.load_gates(w.gates, fg)
        eng.experts_init(ffn, cfg.tile_count_per_expert, seed=seed)
        eng.decode_begin(g["sim_capacities"], w.fisher, g["tau"], cfg, int(g["workload"]["seed"]), T)
        hid = np.zeros((T, w.L, w.D), dtype=np.float32)
        eng.decode_tokens(w.acts[:T], w.scores[:T], hid)
        r = eng.decode_end(cfg, T)
    sim = O.simulate(w, g["sim_capacities"], g["tau"], first_gate=fg, T=T,
                     **{k: v for k, v in __import__("helpers").sim_kwargs(g).items()})
    assert r.metrics == sim.metrics and np.array_equal(r.timeline, sim.timeline)
    assert r.stats["ffn_bytes"] == r.metrics["experts_activated_total"] * 3 * ffn * w.D * 2
    if merge == "2":  # one K2 launch per (token, layer)
        assert r.stats["ffn_launches"] == T * w.L, r.stats["ffn_launches"]
    ref = _moe_reference(w, fg, sim.decisions, T, ffn, cfg.tile_count_per_expert, seed)
    for (t, l), moe in ref.items():
        got = hid[t, l].astype(np.float64) - w.acts[t, l].astype(np.float32).astype(np.float64)
        assert _rel_err(got, moe) < REL_TOL, (t, l)


def _bf16_bits(a):
    """fp32 -> bf16 bit patterns (round to nearest even) and their exact fp32 values."""
    u = np.ascontiguousarray(a, dtype=np.float32).view(np.uint32)
    b = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)
    return b, (b.astype(np.uint32) << 16).view(np.float32)


def test_expert_set_checkpoint_layout():
    """Real weights (moe_experts_alloc + moe_expert_set): checkpoint-layout W1 / W3 [ffn][d] and
    W2 [d][ffn] land in the tile-major store and the K2 path computes W2 (silu(W1 x) * (W3 x))
    within 1e-4 of fp64 numpy on the same bf16 values; then a decode over them matches too."""
    rng = np.random.default_rng(5)
    L, N, K, D, F, tiles = 2, 4, 2, 256, 512, 2
    spec = P.ModelSpec(L, N, K, D)
    mats = {}
    with P.Engine(spec) as eng:
        eng.experts_alloc(F, tiles)
        for l in range(L):
            for e in range(N):
                w1, f1 = _bf16_bits(rng.standard_normal((F, D)) / np.sqrt(D))
                w3, f3 = _bf16_bits(rng.standard_normal((F, D)) / np.sqrt(D))
                w2, f2 = _bf16_bits(rng.standard_normal((D, F)) / np.sqrt(F))
                eng.expert_set(l, e, w1, w3, w2)
                mats[(l, e)] = (f1.astype(np.float64), f3.astype(np.float64), f2.astype(np.float64))
        # tile-major packing: tile t = rows [t*Ft, (t+1)*Ft) as (W1 row, W3 row) pairs, then W2^T rows
        Ft = F // tiles
        blob = eng.expert_read(1, 2).reshape(tiles, 3 * Ft, D)
        w1, w3, w2 = (_bf16_bits(m.astype(np.float32))[0] for m in mats[(1, 2)])
        for t in range(tiles):
            assert np.array_equal(blob[t, 0:2 * Ft:2], w1[t * Ft:(t + 1) * Ft])
            assert np.array_equal(blob[t, 1:2 * Ft:2], w3[t * Ft:(t + 1) * Ft])
            assert np.array_equal(blob[t, 2 * Ft:], w2[:, t * Ft:(t + 1) * Ft].T)
        for (l, e), (a1, a3, a2) in list(mats.items())[:3]:
            x = rng.standard_normal(D)
            xf = x.astype(np.float32).astype(np.float64)
            g, u = a1 @ xf, a3 @ xf
            ref = a2 @ (g / (1.0 + np.exp(-g)) * u)
            assert _rel_err(eng.expert_ffn(l, e, x), ref) < REL_TOL
        # decode with the set weights (trace replay, every expert resident)
        w = O.generate_trace(L, N, K, D, 6, 0.6, 0.2, 3, 44)
        eng.load_gates(w.gates)
        cfg = P.SimConfig(tile_count_per_expert=tiles)
        tau = O.calibrate_threshold(w, 0.24)
        eng.decode_begin([N] * L, w.fisher, tau, cfg, 0, 6)
        hid = np.zeros((6, L, D), dtype=np.float32)
        eng.decode_tokens(w.acts, w.scores, hid)
        eng.decode_end(cfg, 6)
        with pytest.raises(P.MoeError):
            eng.decode_begin([N] * L, w.fisher, tau, cfg, 0, 6)
            eng.expert_set(0, 0, w1, w3, w2)  # not while a session holds HBM copies
    sim = O.simulate(w, [N] * L, tau, tiles=tiles)
    for t in range(6):
        for l in range(L):
            sel = [int(e) for e in sim.decisions[t, l] if e >= 0]
            sc = w.scores[t, l]
            xf = w.acts[t, l].astype(np.float32).astype(np.float64)
            moe = np.zeros(D)
            for e in sel:
                a1, a3, a2 = mats[(l, e)]
                g, u = a1 @ xf, a3 @ xf
                wgt = 1.0 if len(sel) == 1 else sc[e] / sum(sc[q] for q in sel)
                moe += wgt * (a2 @ (g / (1.0 + np.exp(-g)) * u))
            assert _rel_err(hid[t, l].astype(np.float64) - xf, moe) < REL_TOL, (t, l)


def test_copy_engine_error_surfaces(monkeypatch):
    """A failure inside the copy thread (injected: ADAPMOE_COPY_FAULT_AFTER) surfaces as MOE_E_DEVICE
    from the decode call instead of a hang, a crash or silently stale expert slots."""
    monkeypatch.setenv("ADAPMOE_COPY_FAULT_AFTER", "3")
    g = load_golden("tiny_budget0")
    w, fg = oracle_inputs(g)
    cfg = sim_config(g)
    with P.Engine(P.ModelSpec(w.L, w.N, w.K, w.D)) as eng:
        eng.load_gates(w.gates, fg)
        eng.experts_init(224 * cfg.tile_count_per_expert, cfg.tile_count_per_expert, seed=1)
        eng.decode_begin(g["sim_capacities"], w.fisher, g["tau"], cfg, 0, 8)
        with pytest.raises(P.MoeError) as e:
            eng.decode_tokens(w.acts[:8], w.scores[:8], np.zeros((8, w.L, w.D), dtype=np.float32))
        assert e.value.code == 6 and "injected copy fault" in str(e.value)
