"""Host half of the product (C++ engine through the C ABI, no GPU needed): the tick-model
policy engine, tau calibration, cost model and DP allocation, checked against the reference's own
known answers (proj/tests/test_*.cpp) and against the golden fixtures."""
import itertools
import random

import numpy as np
import pytest

import paper_2408_10284_b200 as P
from conftest import golden_names, load_golden
from helpers import assert_metrics, assert_timeline, golden_decisions, oracle_inputs, sim_config
from oracle import oracle as O


# ---- policy engine replay: fed the reference's decisions/predictions, must reproduce its trace ----
@pytest.mark.parametrize("name", golden_names())
def test_replay_matches_reference_trace(name):
    g = load_golden(name)
    L, N, K, D = g["spec"]
    spec = P.ModelSpec(L, N, K, D)
    dec, single, preds = golden_decisions(g)
    r = P.replay_policy(spec, g["sim_capacities"], sim_config(g), int(g["workload"]["seed"]), dec, single, preds)
    assert_metrics(g, r.metrics, r.latency_per_token, r.on_demand_loads_per_layer)
    assert_timeline(g, r.timeline)


def _timeline_checks(tl: np.ndarray, metrics: dict):
    """Engine-independent invariants (proj/tests/support/timeline_checks.hpp:24-102)."""
    ends = {}
    for ev in tl:
        if ev[1] == 4:
            ends.setdefault((ev[5], ev[6], ev[7]), []).append(ev[3])
    for ev in tl:
        if ev[1] == 3:
            assert min(ends[(ev[5], ev[6], ev[7])]) <= ev[2], "tile compute before its transfer"
    for stream in (0, 1):
        evs = sorted((e for e in tl if e[0] == stream), key=lambda e: e[2])
        for a, b in zip(evs, evs[1:]):
            assert a[3] <= b[2], "overlap on a stream"
    whole = int((tl[:, 1] == 2).sum())
    od = len({(e[4], e[5], e[6]) for e in tl if e[1] == 3})
    assert whole + od == metrics["experts_activated_total"]
    assert od == metrics["on_demand_loads"]
    assert metrics["cache_hits"] + metrics["prefetch_hits"] + metrics["on_demand_loads"] == metrics["experts_activated_total"]


@pytest.mark.parametrize("name", ["tiny", "tiny_transfer_heavy", "demo8_300", "top3"])
def test_replay_timeline_invariants(name):
    g = load_golden(name)
    L, N, K, D = g["spec"]
    dec, single, preds = golden_decisions(g)
    r = P.replay_policy(P.ModelSpec(L, N, K, D), g["sim_capacities"], sim_config(g), int(g["workload"]["seed"]),
                        dec, single, preds)
    _timeline_checks(r.timeline, r.metrics)


def _cfg(tiles, transfer, compute, attention, gate, lookahead=2, gating=False, prefetch=False):
    return P.SimConfig(tiles, transfer, compute, attention, gate, lookahead, P.PolicyFlags(gating, prefetch, False))


def test_fully_resident_runs_without_stalls():
    """proj/tests/test_simulator.cpp:104-136: latency 3*(5+1+2*(2*2)) = 42 per token."""
    spec = P.ModelSpec(3, 4, 2, 4)
    T = 10
    rng = np.random.default_rng(0)
    dec = np.stack([np.stack([rng.permutation(4)[:2] for _ in range(3)]) for _ in range(T)]).astype(np.int32)
    r = P.replay_policy(spec, [4, 4, 4], _cfg(2, 3, 2, 5, 1), 7, dec, None, None)
    assert r.metrics["stall_time"] == 0 and r.metrics["on_demand_loads"] == 0
    assert r.metrics["cache_hits"] == r.metrics["experts_activated_total"]
    assert r.latency_per_token.tolist() == [42] * T
    _timeline_checks(r.timeline, r.metrics)


def test_cold_single_expert_serializes():
    """proj/tests/test_simulator.cpp:138-162: latency 3+1+6+2, stall 6."""
    spec = P.ModelSpec(1, 2, 1, 2)
    dec = np.zeros((1, 1, 1), dtype=np.int32)
    r = P.replay_policy(spec, [0], _cfg(1, 6, 2, 3, 1), 1, dec, None, None)
    assert r.latency_per_token[0] == 3 + 1 + 6 + 2
    assert r.metrics["stall_time"] == 6 and r.metrics["on_demand_loads"] == 1


def test_on_demand_completion_matches_pipeline_formula():
    """proj/tests/test_simulator.cpp:164-198 sweep."""
    spec = P.ModelSpec(1, 2, 1, 2)
    dec = np.zeros((1, 1, 1), dtype=np.int32)
    for tiles in range(1, 17, 3):
        for transfer in range(6):
            for compute in range(6):
                r = P.replay_policy(spec, [0], _cfg(tiles, transfer, compute, 2, 1), 3, dec, None, None)
                tl = r.timeline
                start = tl[tl[:, 1] == 4][0, 2]
                end = tl[tl[:, 1] == 3][:, 3].max()
                assert start == 3
                assert end - start == P.tile_pipeline_latency(tiles, transfer, compute)


def test_tile_pipeline_formula():
    """proj/tests/test_simulator.cpp:57-64."""
    assert P.tile_pipeline_latency(1, 3, 2) == 5
    assert P.tile_pipeline_latency(4, 1, 1) == 5
    assert P.tile_pipeline_latency(1, 4, 4) == 8
    for n, t, c in itertools.product(range(1, 6), range(5), range(5)):
        assert P.tile_pipeline_latency(n, t, c) == O.lib().orc_tile_pipeline_latency(n, t, c)


# ---- cost model + DP (proj/tests/test_cache_model.cpp, test_allocator.cpp) ----
def test_expected_cost_known_answers():
    assert abs(P.expected_cost(4, 8, 0.5, 0.5) - 3 / 7) < 1e-15
    assert P.expected_cost(8, 8, 0.3, 0.2) == 0.0
    assert P.expected_cost(0, 8, 1.0, 0.0) == 1.0
    assert P.expected_cost(0, 8, 0.0, 0.0) == 2.0
    for t, a, b in itertools.product(range(9), (0.0, 0.3, 1.0), (0.0, 0.45, 1.0)):
        assert P.expected_cost(t, 8, a, b) == O.lib().orc_expected_cost(t, 8, a, b)


def test_cost_table_monotone_in_capacity():
    spec = P.ModelSpec(3, 8, 2, 1)
    t = P.build_cost_table(spec, [0.1, 0.5, 0.9], [0.2, 0.6, 0.95])
    assert (np.diff(t, axis=1) <= 1e-15).all()


def test_dp_tiny_instance():
    """proj/tests/test_allocator.cpp:26-38: 2 layers, N=2, budget 2 -> {0, 2}."""
    spec = P.ModelSpec(2, 2, 1, 1)
    table = np.array([[1.0, 0.9, 0.8], [1.0, 0.5, 0.0]])
    caps, cost = P.dp_allocate(spec, table, 2)
    assert caps.tolist() == [0, 2] and cost == 1.0


def test_dp_zero_table_and_unconstrained():
    spec = P.ModelSpec(3, 4, 2, 1)
    caps, cost = P.dp_allocate(spec, np.zeros((3, 5)), 7)
    assert caps.tolist() == [0, 0, 0] and cost == 0.0
    table = np.array([[4, 3, 2, 1, 0], [4, 3, 2, 1, 0], [4, 3, 2, 1, 0]], dtype=float)
    caps, _ = P.dp_allocate(spec, table, 100)  # clamped to L*N
    assert caps.tolist() == [4, 4, 4]


def _brute(table, budget):
    L, N1 = table.shape
    best, arg = float("inf"), None
    for caps in itertools.product(range(N1), repeat=L):
        if sum(caps) > budget:
            continue
        c = 0.0
        for i, k in enumerate(caps):
            c += table[i][k]
        if c < best:
            best, arg = c, list(caps)
    return arg, best


@pytest.mark.parametrize("seed", range(25))
def test_dp_equals_brute_force(seed):
    """proj/tests/test_allocator.cpp:63-84 / acceptance criterion 2."""
    rng = random.Random(seed)
    L, N = rng.randint(1, 4), rng.randint(2, 5)
    spec = P.ModelSpec(L, N, min(2, N), 1)
    alpha = [rng.random() for _ in range(L)]
    beta = [rng.random() for _ in range(L)]
    table = P.build_cost_table(spec, alpha, beta)
    assert table.ravel().tolist() == O.cost_table(alpha, beta, N).ravel().tolist()
    budget = rng.randint(0, L * N)
    caps, cost = P.dp_allocate(spec, table, budget)
    bcaps, bcost = _brute(table, budget)
    assert cost == bcost and caps.tolist() == bcaps


def test_uniform_allocation():
    spec = P.ModelSpec(3, 4, 2, 1)
    assert P.uniform_allocation(spec, 7).tolist() == [3, 2, 2]
    assert P.uniform_allocation(spec, 100).tolist() == [4, 4, 4]


# ---- tau calibration (proj/tests/test_gating.cpp:132-154, 191-205) ----
def test_calibrate_matches_oracle_on_goldens():
    for name in ("tiny", "demo8_300", "top3", "wide_n16"):
        g = load_golden(name)
        w, _ = oracle_inputs(g)
        spec = P.ModelSpec(w.L, w.N, w.K, w.D)
        for target in (0.0, 0.12, 0.24, 0.5, 0.9, 1.0):
            tau, realized = P.calibrate_threshold(spec, w.scores, w.fisher, target)
            assert tau == O.calibrate_threshold(w, target)
            assert realized >= target or tau == 0.0


def test_calibrate_known_multiset():
    """Perturbations {.1,.2,.3,.4} (F=1 each, two experts): target .5 -> .2, 1 -> .4, 0 -> 0."""
    ps = [0.1, 0.2, 0.3, 0.4]
    scores = []
    for p in ps:
        g = np.sqrt(p / 4.0)  # 1 - alpha, with F = 4
        scores.append([1.0 - g, g])
    scores = np.array(scores).reshape(4, 1, 2)
    spec = P.ModelSpec(1, 2, 2, 1)

    def pert(s):
        gap = 1.0 - s[0] / (s[0] + s[1])
        return gap * gap * 4.0
    observed = sorted(pert(s[0]) for s in scores)
    assert np.allclose(observed, ps)
    tau, _ = P.calibrate_threshold(spec, scores, [4.0], 0.5)
    assert tau == observed[1]
    tau, _ = P.calibrate_threshold(spec, scores, [4.0], 1.0)
    assert tau == observed[3]
    tau, _ = P.calibrate_threshold(spec, scores, [4.0], 0.0)
    assert tau == 0.0


def test_error_classes():
    spec = P.ModelSpec(2, 4, 2, 1)
    with pytest.raises(P.MoeError) as e:
        P.dp_allocate(spec, np.zeros((2, 5)), -1)
    assert e.value.code == 5  # infeasible budget (CLI exit 5)
    with pytest.raises(P.MoeError) as e:
        P.uniform_allocation(P.ModelSpec(0, 4, 2, 1), 3)
    assert e.value.code == 1
    with pytest.raises(P.MoeError) as e:
        P.calibrate_threshold(spec, np.full((1, 2, 4), 0.25), [1.0, 1.0], 1.5)
    assert e.value.code == 1
