"""Ablation grid (compare_policies, inc/simulator.hpp:476-550) on the GPU engine:
every row's flags, allocation, metrics (per-token latency, per-layer on-demand loads) and
speedup_vs_baseline must equal the unmodified reference's (tests/golden/compare/, made by
make_compare_goldens.py)."""
import json
import os

import pytest

import paper_2408_10284_b200 as P
from helpers import oracle_inputs
from oracle import oracle as O

pytestmark = pytest.mark.gpu
DIR = os.path.join(os.path.dirname(__file__), "golden", "compare")


def _cases():
    return sorted(n[:-5] for n in os.listdir(DIR) if n.endswith(".json"))


@pytest.mark.parametrize("name", _cases())
def test_compare_policies_matches_reference(name):
    g = json.load(open(os.path.join(DIR, f"{name}.json")))
    a = g["workload"]
    w, fg = oracle_inputs(g)
    tau = O.calibrate_threshold(w, float(a["target"]))
    assert tau == g["tau"]
    alpha, beta = O.generate_profiles(w, tau, fg)
    cfg = P.SimConfig(int(a["tiles"]), int(a["tile_transfer"]), int(a["tile_compute"]), int(a["attention"]),
                      int(a["gate_time"]), int(a["lookahead"]), P.PolicyFlags(True, True, True))
    with P.Engine(P.ModelSpec(w.L, w.N, w.K, w.D)) as eng:
        eng.load_gates(w.gates, fg)
        rows = eng.compare_policies(w.acts, w.scores, w.fisher, alpha, beta, tau, cfg, int(a["budget"]),
                                    int(a["seed"]))
    assert len(rows) == len(g["rows"]) == 7
    for got, ref in zip(rows, g["rows"]):
        assert got["name"] == ref["name"]
        assert got["flags"] == ref["flags"]
        assert got["capacities"] == ref["capacities"], ref["name"]
        assert got["metrics"] == ref["metrics"], ref["name"]
        assert got["speedup_vs_baseline"] == ref["speedup_vs_baseline"], ref["name"]
