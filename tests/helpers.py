"""Test helpers: rebuild a golden case's inputs with the C oracle, compare structures."""
from __future__ import annotations

import numpy as np

from oracle import oracle as O


def parse_scales(v):
    if v is None:
        return None
    return [float(x) for x in str(v).split(",")]


def wl_args(g):
    a = g["workload"]
    return dict(L=int(a["layers"]), N=int(a["experts"]), K=int(a["top_k"]), D=int(a["hidden"]), T=int(a["tokens"]),
                concentration=float(a["concentration"]), drift=float(a["drift"]), gate_seed=int(a["gate_seed"]),
                token_seed=int(a["token_seed"]), fisher_scales=parse_scales(a.get("fisher_scales")),
                drift_scales=parse_scales(a.get("drift_scales")))


def sim_kwargs(g):
    a = g["workload"]
    return dict(tiles=int(a["tiles"]), tile_transfer=int(a["tile_transfer"]), tile_compute=int(a["tile_compute"]),
                attention=int(a["attention"]), gate=int(a["gate_time"]), lookahead=int(a["lookahead"]),
                gating=bool(int(a["gating"])), prefetch=bool(int(a["prefetch"])), seed=int(a["seed"]))


def oracle_inputs(g):
    """Workload + trained first gate (if the case trains one) from the oracle."""
    a = g["workload"]
    w = O.generate_trace(**wl_args(g))
    fg = None
    if int(a["train_gate"]) and w.T >= 2:
        fg = O.train_first_gate(w, lr=float(a["train_lr"]), steps=int(a["train_steps"]), seed=int(a["train_seed"]))
    return w, fg


def sim_config(g):
    """paper_2408_10284_b200.SimConfig for the case."""
    from paper_2408_10284_b200 import PolicyFlags, SimConfig
    k = sim_kwargs(g)
    return SimConfig(k["tiles"], k["tile_transfer"], k["tile_compute"], k["attention"], k["gate"], k["lookahead"],
                     PolicyFlags(k["gating"], k["prefetch"], True))


def golden_decisions(g):
    L, K = g["spec"][0], g["spec"][2]
    T = g["tokens"]
    dec = np.asarray(g["decision_selected"], dtype=np.int32).reshape(T, L, K)
    single = np.asarray(g["decision_single"], dtype=np.int32).reshape(T, L)
    preds = np.asarray(g["predictions"], dtype=np.int32).reshape(T, L, 3, 2 + K)
    return dec, single, preds


def assert_timeline(g, timeline: np.ndarray):
    assert timeline.shape[0] == g["timeline_events"], (timeline.shape, g["timeline_events"])
    if "timeline" in g:
        exp = np.asarray(g["timeline"], dtype=np.int64).reshape(-1, 8)
        bad = np.nonzero((exp != timeline).any(axis=1))[0]
        assert bad.size == 0, f"first differing event {bad[0]}: ref {exp[bad[0]].tolist()} got {timeline[bad[0]].tolist()}"
    assert O.fnv1a(np.ascontiguousarray(timeline, dtype=np.int64)) == g["hash_timeline"]


def assert_metrics(g, metrics: dict, latency_per_token, od_per_layer):
    m = g["metrics"]
    for k, v in m.items():
        if k in ("latency_per_token", "on_demand_loads_per_layer"):
            continue
        assert metrics[k] == v, (k, metrics[k], v)
    assert list(map(int, latency_per_token)) == m["latency_per_token"]
    assert list(map(int, od_per_layer)) == m["on_demand_loads_per_layer"]
