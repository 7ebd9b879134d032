"""Pin the C oracle: every golden case produced by the unmodified reference (tests/golden/, made by
make_goldens.py from oracle/_ref/moesim_ref) must be reproduced bit-exactly by oracle/liboracle.so:
synthetic inputs, tau, trained first-layer gate, alpha/beta, cost table, DP allocation, metrics,
timeline, decisions and look-ahead predictions."""
import numpy as np
import pytest

from conftest import golden_names, load_golden
from helpers import assert_metrics, assert_timeline, oracle_inputs, sim_kwargs
from oracle import oracle as O


@pytest.mark.parametrize("name", golden_names())
def test_oracle_reproduces_reference(name):
    g = load_golden(name)
    w, fg = oracle_inputs(g)
    assert O.fnv1a(w.gates) == g["hash_gates"]
    assert O.fnv1a(w.acts) == g["hash_activations"]
    assert O.fnv1a(w.scores) == g["hash_scores"]
    assert w.selected.ravel().tolist() == g["generated_selected"]
    assert w.fisher.tolist() == g["fisher"]
    if fg is not None:
        assert O.fnv1a(fg) == g["hash_first_gate"]
    else:
        assert g["hash_first_gate"] is None
    a = g["workload"]
    tau = float(a["tau"]) if "tau" in a else O.calibrate_threshold(w, float(a["target"]))
    assert tau == g["tau"]
    alpha, beta = O.generate_profiles(w, tau, fg)
    assert alpha.tolist() == g["alpha"] and beta.tolist() == g["beta"]
    table = O.cost_table(alpha, beta, w.N)
    assert table.ravel().tolist() == g["cost_table"]
    caps, cost = O.dp_allocate(table, g["budget"])
    assert caps.tolist() == g["capacities"] and cost == g["total_cost"]
    assert O.uniform_allocation(g["budget"], w.L, w.N).tolist() == g["uniform_capacities"]
    so = O.simulate(w, g["sim_capacities"], tau, first_gate=fg, **sim_kwargs(g))
    assert_metrics(g, so.metrics, so.latency_per_token, so.od_per_layer)
    assert_timeline(g, so.timeline)
    assert so.decisions.ravel().tolist() == g["decision_selected"]
    assert so.predictions.ravel().tolist() == g["predictions"]


def test_golden_anchor_values():
    """SURVEY.md Appendix B anchors (reference run on the tiny config)."""
    g = load_golden("tiny")
    assert g["tau"] == 0.026507221949201038
    assert g["capacities"] == [5, 4, 4, 3]
    m = g["metrics"]
    assert (m["cache_hits"], m["prefetch_hits"], m["on_demand_loads"]) == (179, 213, 58)
    assert (m["stall_time"], m["total_latency"], g["timeline_events"]) == (89, 4193, 2384)
    # token 0 generated top-2 selections: L0 [2,0], L1 [4,2], L2 [0,4], L3 [5,4]
    assert g["generated_selected"][:8] == [2, 0, 4, 2, 0, 4, 5, 4]
