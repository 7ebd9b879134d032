"""Randomized differential test: C oracle vs the unmodified reference (oracle/_ref/moesim_ref) on
many small configurations (topologies, ticks, budgets, policies, seeds).  Skipped where the
reference could not be compiled (e.g. on the GPU box, which has no /root/reference)."""
import random

import numpy as np
import pytest

from oracle import oracle as O

pytestmark = pytest.mark.skipif(not O.have_ref(), reason="oracle/_ref/moesim_ref not built (no /root/reference)")


def random_case(rng: random.Random):
    L = rng.randint(1, 6)
    N = rng.choice([2, 3, 4, 6, 8, 12])
    K = rng.randint(1, min(3, N))
    D = rng.choice([1, 2, 3, 5, 8, 16, 33])
    T = rng.randint(2, 40)
    a = dict(layers=L, experts=N, top_k=K, hidden=D, tokens=T,
             concentration=repr(rng.choice([0.3, 0.6, 1.0, 2.5])), drift=repr(rng.choice([0.0, 0.1, 0.4, 1.0])),
             gate_seed=rng.randint(0, 1000), token_seed=rng.randint(0, 1000),
             target=repr(rng.choice([0.0, 0.12, 0.24, 0.5, 1.0])), train_gate=rng.randint(0, 1),
             train_steps=rng.choice([1, 10, 30]), budget=rng.randint(0, L * N + 3),
             tiles=rng.randint(1, 5), tile_transfer=rng.randint(0, 6), tile_compute=rng.randint(0, 4),
             attention=rng.randint(0, 9), gate_time=rng.randint(0, 2), lookahead=rng.randint(0, 3),
             gating=rng.randint(0, 1), prefetch=rng.randint(0, 1), seed=rng.randint(0, 99),
             shared_gates=int(rng.random() < 0.2), uniform=int(rng.random() < 0.3))
    if rng.random() < 0.6:
        a["fisher_scales"] = ",".join(repr(round(rng.uniform(0.0, 3.0), 3)) for _ in range(L))
    if rng.random() < 0.6:
        a["drift_scales"] = ",".join(repr(round(rng.uniform(0.0, 2.0), 3)) for _ in range(L))
    return a


@pytest.mark.parametrize("case_seed", range(40))
def test_random_config(case_seed):
    a = random_case(random.Random(1234 + case_seed))
    r = O.run_ref(**a)
    L, N, K, D, T = a["layers"], a["experts"], a["top_k"], a["hidden"], a["tokens"]
    fs = [float(v) for v in a["fisher_scales"].split(",")] if "fisher_scales" in a else None
    ds = [float(v) for v in a["drift_scales"].split(",")] if "drift_scales" in a else None
    w = O.generate_trace(L, N, K, D, T, float(a["concentration"]), float(a["drift"]), a["gate_seed"], a["token_seed"],
                         bool(a["shared_gates"]), fs, ds)
    assert O.fnv1a(w.acts) == r["hash_activations"] and O.fnv1a(w.scores) == r["hash_scores"]
    assert O.fnv1a(w.gates) == r["hash_gates"]
    tau = O.calibrate_threshold(w, float(a["target"]))
    assert tau == r["tau"]
    fg = O.train_first_gate(w, steps=a["train_steps"]) if a["train_gate"] else None
    if fg is not None:
        assert O.fnv1a(fg) == r["hash_first_gate"]
    alpha, beta = O.generate_profiles(w, tau, fg)
    assert alpha.tolist() == r["alpha"] and beta.tolist() == r["beta"]
    caps, cost = O.dp_allocate(O.cost_table(alpha, beta, N), r["budget"])
    assert caps.tolist() == r["capacities"] and cost == r["total_cost"]
    so = O.simulate(w, r["sim_capacities"], tau, first_gate=fg, tiles=a["tiles"], tile_transfer=a["tile_transfer"],
                    tile_compute=a["tile_compute"], attention=a["attention"], gate=a["gate_time"],
                    lookahead=a["lookahead"], gating=bool(a["gating"]), prefetch=bool(a["prefetch"]), seed=a["seed"])
    for k, v in r["metrics"].items():
        if k == "latency_per_token":
            assert so.latency_per_token.tolist() == v
        elif k == "on_demand_loads_per_layer":
            assert so.od_per_layer.tolist() == v
        else:
            assert so.metrics[k] == v, k
    assert so.timeline.ravel().tolist() == r["timeline"]
    assert so.predictions.ravel().tolist() == r["predictions"]
    assert so.decisions.ravel().tolist() == r["decision_selected"]
