"""K1 (fused router + pre-gate, sm_100a) and the GPU-backed moesim pipeline vs the reference.

Everything here is bit-exact against the golden fixtures made by the unmodified reference:
synthetic workload (host RNG + GPU gate GEMVs), actual decisions, look-ahead predictions, alpha/beta
profiles, and simulate_trace's metrics + event timeline."""
import numpy as np
import pytest

import paper_2408_10284_b200 as P
from conftest import golden_names, load_golden
from helpers import (assert_metrics, assert_timeline, golden_decisions, oracle_inputs, parse_scales, sim_config,
                     sim_kwargs, wl_args)
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _spec(g):
    L, N, K, D = g["spec"]
    return P.ModelSpec(L, N, K, D)


@pytest.mark.parametrize("name", golden_names())
def test_simulate_trace_bit_exact(name):
    g = load_golden(name)
    w, fg = oracle_inputs(g)
    with P.Engine(_spec(g)) as eng:
        eng.load_gates(w.gates, fg)
        cfg = sim_config(g)
        dec, single, pert, preds = eng.route_trace(w.acts, w.scores, w.fisher, g["tau"], cfg)
        gdec, gsingle, gpreds = golden_decisions(g)
        assert np.array_equal(dec, gdec)
        assert np.array_equal(single, gsingle)
        if cfg.policy.adaptive_gating:
            assert pert.ravel().tolist() == g["decision_perturbation"]
        mism = np.argwhere((preds != gpreds).any(axis=-1))
        assert mism.size == 0, f"{len(mism)} prediction flips, first at (tok, layer, slot) {mism[0].tolist()}"
        r = eng.simulate_trace(w.acts, w.scores, w.fisher, g["sim_capacities"], g["tau"], cfg,
                               int(g["workload"]["seed"]))
        assert_metrics(g, r.metrics, r.latency_per_token, r.on_demand_loads_per_layer)
        assert_timeline(g, r.timeline)


@pytest.mark.parametrize("name", ["tiny", "demo8_300", "wide_n16", "top3", "odd_d", "mixtral_8x7b_t12"])
def test_gpu_pipeline_end_to_end(name):
    """generate -> calibrate -> [oracle-trained first gate] -> profile -> allocate -> simulate, with the
    product doing every step it owns."""
    g = load_golden(name)
    a = g["workload"]
    wa = wl_args(g)
    spec = _spec(g)
    with P.Engine(spec) as eng:
        wl = eng.generate_trace(P.SynthConfig(spec, wa["T"], wa["concentration"], wa["drift"], wa["gate_seed"],
                                              wa["token_seed"], False, wa["fisher_scales"], wa["drift_scales"]))
        assert O.fnv1a(wl.gates) == g["hash_gates"]
        assert O.fnv1a(wl.acts) == g["hash_activations"]
        assert O.fnv1a(wl.scores) == g["hash_scores"], "GPU gate GEMV + softmax differs from the reference"
        assert wl.selected.ravel().tolist() == g["generated_selected"]
        tau, _ = P.calibrate_threshold(spec, wl.scores, wl.fisher, float(a["target"]))
        assert tau == g["tau"]
        fg = None
        if int(a["train_gate"]):
            w_or = O.Workload(spec.num_layers, spec.experts_per_layer, spec.top_k, spec.hidden_dim, wa["T"],
                              wl.gates, wl.acts, wl.scores, wl.selected, wl.fisher)
            fg = O.train_first_gate(w_or, lr=float(a["train_lr"]), steps=int(a["train_steps"]),
                                    seed=int(a["train_seed"]))
            eng.load_gates(wl.gates, fg)
        alpha, beta = eng.generate_profiles(wl.acts, wl.scores, wl.fisher, tau)
        assert alpha.tolist() == g["alpha"] and beta.tolist() == g["beta"]
        caps, cost = P.dp_allocate(spec, P.build_cost_table(spec, alpha, beta), g["budget"])
        assert caps.tolist() == g["capacities"] and cost == g["total_cost"]
        r = eng.simulate_trace(wl.acts, wl.scores, wl.fisher, g["sim_capacities"], tau, sim_config(g),
                               int(a["seed"]))
        assert_metrics(g, r.metrics, r.latency_per_token, r.on_demand_loads_per_layer)
        assert_timeline(g, r.timeline)


def test_router_tie_break_and_inclusive_boundary():
    """proj/tests/test_core.cpp:74-80 (ties -> lowest index) and test_gating.cpp:74-81 (p == tau
    is single) evaluated by K1 on crafted stored scores."""
    spec = P.ModelSpec(1, 4, 2, 2)
    cfg_plain = P.SimConfig(policy=P.PolicyFlags(False, False, False))
    cfg_adapt = P.SimConfig(policy=P.PolicyFlags(True, False, False))
    scores = np.array([[[0.25, 0.25, 0.25, 0.25]], [[0.1, 0.4, 0.4, 0.1]], [[0.0, 0.3, 0.0, 0.7]]])
    acts = np.zeros((3, 1, 2))
    with P.Engine(spec) as eng:
        eng.load_gates(np.zeros((1, 2, 4)))
        dec, single, _, _ = eng.route_trace(acts, scores, [1.0], 0.0, cfg_plain)
        assert dec[0, 0].tolist() == [0, 1] and dec[1, 0].tolist() == [1, 2] and dec[2, 0].tolist() == [3, 1]
        # alpha = .9 -> p = (.1)^2 * 5 = 0.05 computed in fp64; tau equal to that value -> single
        s = np.array([[[0.9, 0.1, 0.0, 0.0]]])
        gap = 1.0 - 0.9 / (0.9 + 0.1)
        tau = gap * gap * 5.0
        dec, single, pert, _ = eng.route_trace(np.zeros((1, 1, 2)), s, [5.0], tau, cfg_adapt)
        assert single[0, 0] == 1 and dec[0, 0].tolist() == [0, -1] and pert[0, 0] == tau
        dec, single, _, _ = eng.route_trace(np.zeros((1, 1, 2)), s, [5.0], np.nextafter(tau, 0), cfg_adapt)
        assert single[0, 0] == 0 and dec[0, 0].tolist() == [0, 1]


def test_router_logits_match_reference_order():
    """Predicted lists at d=4096 against the oracle's fp64 sequential GateMatrix::logits, many
    random activations (including exact zeros, which the reference skips)."""
    rng = np.random.default_rng(3)
    L, N, K, D, T = 4, 8, 2, 4096, 24
    gates = rng.standard_normal((L, D, N)) / 64.0
    acts = rng.standard_normal((T, L, D))
    acts[acts < -1.5] = 0.0
    scores = np.full((T, L, N), 1.0 / N)
    spec = P.ModelSpec(L, N, K, D)
    cfg = P.SimConfig(lookahead_depth=3, policy=P.PolicyFlags(False, True, False))
    with P.Engine(spec) as eng:
        eng.load_gates(gates)
        _, _, _, preds = eng.route_trace(acts, scores, np.ones(L), 0.0, cfg)
    for t in range(T):
        for l in range(L - 1):
            for s in range(min(3, L - 1 - l)):
                lg = np.zeros(N)
                O.lib().orc_gate_logits(gates[l + s + 1].ctypes.data_as(O._d), D, N,
                                        np.ascontiguousarray(acts[t, l]).ctypes.data_as(O._d), lg.ctypes.data_as(O._d))
                sc = np.zeros(N)
                O.lib().orc_softmax(lg.ctypes.data_as(O._d), N, sc.ctypes.data_as(O._d))
                top = np.zeros(K, dtype=np.int32)
                O.lib().orc_top_k(sc.ctypes.data_as(O._d), N, K, top.ctypes.data_as(O._i))
                assert preds[t, l, s, 0] == l + s + 1
                assert preds[t, l, s, 2:].tolist() == top.tolist()


@pytest.mark.parametrize("name", ["tiny", "wide_n16", "top3", "mixtral_8x7b_t12"])
@pytest.mark.parametrize("lookahead", [0, 2, 3])
def test_router_forward_matches_route_trace(name, lookahead):
    """moe_router_forward (device rows, caller's stream) decides and predicts exactly like the
    trace router: for every layer, rows = the trace's tokens; decisions from the stored scores equal
    route_trace's, look-ahead item d equals route_trace's prediction slot d-1 (at the last layer:
    the first-layer gate, for tokens that have a successor); deciding from the layer's own gate
    logits equals deciding from the reference softmax of those logits."""
    import torch
    g = load_golden(name)
    w, fg = oracle_inputs(g)
    cfg = sim_config(g)
    cfg.lookahead_depth = lookahead
    L, K, T = w.L, w.K, w.T
    with P.Engine(_spec(g)) as eng:
        eng.load_gates(w.gates, fg)
        dec, single, pert, preds = eng.route_trace(w.acts, w.scores, w.fisher, g["tau"], cfg)
        stream = torch.cuda.Stream()
        for l in range(L):
            x = torch.from_numpy(np.ascontiguousarray(w.acts[:, l])).cuda()
            s = torch.from_numpy(np.ascontiguousarray(w.scores[:, l])).cuda()
            torch.cuda.synchronize()
            with torch.cuda.stream(stream):
                sel, cnt, sgl, prt = eng.router_forward(l, x, w.fisher, g["tau"], lookahead, scores=s, stream=stream)
            stream.synchronize()
            sel, cnt, sgl = sel.cpu().numpy(), cnt.cpu().numpy(), sgl.cpu().numpy()
            assert np.array_equal(sel[:, 0], dec[:, l]) and np.array_equal(sgl[:, 0], single[:, l])
            assert np.array_equal(prt.cpu().numpy()[:, 0], pert[:, l])
            for dep in range(1, lookahead + 1):
                if l + dep < L:
                    rows = range(T)
                elif l == L - 1 and dep == 1 and fg is not None:
                    rows = range(T - 1)  # route_trace predicts the next token's layer 0 only if one exists
                else:
                    assert (cnt[:, dep] == 0).all()
                    continue
                for t in rows:
                    target, count = preds[t, l, dep - 1, 0], preds[t, l, dep - 1, 1]
                    assert target == (l + dep if l + dep < L else 0)
                    assert cnt[t, dep] == count
                    assert list(sel[t, dep, :count]) == list(preds[t, l, dep - 1, 2:2 + count])
            # decide from the gate's logits == decide from the reference softmax of those logits
            ref_scores = torch.from_numpy(np.stack([O.gate_scores(w.gates[l], w.acts[t, l]) for t in range(T)])).cuda()
            a = eng.router_forward(l, x, w.fisher, g["tau"], 0)
            b = eng.router_forward(l, x, w.fisher, g["tau"], 0, scores=ref_scores)
            torch.cuda.synchronize()
            for u, v in zip(a[:3], b[:3]):
                assert torch.equal(u, v)


@pytest.mark.parametrize("name", ["mixtral_8x7b_t12", "tiny", "wide_n16", "top3", "odd_d"])
def test_forced_exact_path_host_decisions_bit_exact(monkeypatch, name):
    """ADAPMOE_ROUTE_FORCE_EXACT=1 sends EVERY gate item down K1's exact path: reference-order fp64
    logits on the device, decision on the host with the reference's libm softmax
    (route_host_decide).  Predictions, decisions and the whole simulate_trace timeline must still
    equal the reference's bit for bit — the path the ~1-in-600 uncertified items take normally."""
    monkeypatch.setenv("ADAPMOE_ROUTE_FORCE_EXACT", "1")
    g = load_golden(name)
    w, fg = oracle_inputs(g)
    cfg = sim_config(g)
    with P.Engine(_spec(g)) as eng:
        eng.load_gates(w.gates, fg)
        dec, single, pert, preds = eng.route_trace(w.acts, w.scores, w.fisher, g["tau"], cfg)
        gdec, gsingle, gpreds = golden_decisions(g)
        assert np.array_equal(dec, gdec) and np.array_equal(single, gsingle)
        mism = np.argwhere((preds != gpreds).any(axis=-1))
        assert mism.size == 0, f"{len(mism)} prediction flips, first at (tok, layer, slot) {mism[0].tolist()}"
        r = eng.simulate_trace(w.acts, w.scores, w.fisher, g["sim_capacities"], g["tau"], cfg,
                               int(g["workload"]["seed"]))
        assert_metrics(g, r.metrics, r.latency_per_token, r.on_demand_loads_per_layer)
        assert_timeline(g, r.timeline)
        if g["spec"][3] <= 256 and cfg.policy.prefetch:  # the physical decode's routing takes the same path
            T = min(8, w.T)
            ffn = 4 * g["spec"][3] if g["spec"][3] % 32 == 0 else None
            if ffn is not None:
                eng.experts_init(ffn, cfg.tile_count_per_expert, seed=5)
                eng.decode_begin(g["sim_capacities"], w.fisher, g["tau"], cfg, int(g["workload"]["seed"]), T)
                hid = np.zeros((T, w.L, w.D), dtype=np.float32)
                eng.decode_tokens(w.acts[:T], w.scores[:T], hid)
                st = eng.decode_stats()
                res = eng.decode_end(cfg, T)
                ref = O.simulate(w, g["sim_capacities"], g["tau"], first_gate=fg, T=T, **sim_kwargs(g))
                assert res.metrics == ref.metrics
                assert np.array_equal(res.timeline, ref.timeline)
                assert st["router_exact_items"] > 0
