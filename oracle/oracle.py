"""TEST INFRASTRUCTURE ONLY — ctypes front-end for the C oracle (oracle/liboracle.so) and the
compiled reference driver (oracle/_ref/moesim_ref).

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference arm import this
module.  The product path (paper_2408_10284_b200) never does.
"""
from __future__ import annotations

import ctypes as C
import json
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")
REF_BIN = os.path.join(HERE, "_ref", "moesim_ref")

_lib = None


def build() -> None:
    subprocess.run(["make", "-s", "-C", HERE, "liboracle.so"], check=True)


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        _lib = C.CDLL(LIB_PATH)
        _declare(_lib)
    return _lib


def have_ref() -> bool:
    return os.path.exists(REF_BIN)


_d = C.POINTER(C.c_double)
_i = C.POINTER(C.c_int)
_i64 = C.POINTER(C.c_int64)
_u16 = C.POINTER(C.c_uint16)
_f = C.POINTER(C.c_float)


class SimCfg(C.Structure):
    _fields_ = [("tiles", C.c_int), ("tile_transfer", C.c_int64), ("tile_compute", C.c_int64),
                ("attention", C.c_int64), ("gate", C.c_int64), ("lookahead", C.c_int),
                ("gating", C.c_int), ("prefetch", C.c_int)]


class Metrics(C.Structure):
    _fields_ = [("total_latency", C.c_int64), ("stall_time", C.c_int64), ("on_demand_loads", C.c_int64),
                ("cache_hits", C.c_int64), ("prefetch_hits", C.c_int64),
                ("single_expert_decisions", C.c_int64), ("experts_activated_total", C.c_int64)]


def _declare(L):
    L.orc_generate_trace.argtypes = [C.c_int] * 5 + [C.c_double, C.c_double, C.c_uint64, C.c_uint64, C.c_int,
                                                     _d, _d, _d, _d, _d, _i, _d]
    L.orc_calibrate_threshold.argtypes = [_d, C.c_int, C.c_int, C.c_int, _d, C.c_double]
    L.orc_calibrate_threshold.restype = C.c_double
    L.orc_train_first_gate.argtypes = [_d, _d, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, C.c_int,
                                       C.c_uint64, _d]
    L.orc_generate_profiles.argtypes = [_d, _d, _d, _d] + [C.c_int] * 5 + [C.c_double, _d, _d, _d]
    L.orc_cost_table.argtypes = [_d, _d, C.c_int, C.c_int, _d]
    L.orc_dp_allocate.argtypes = [_d, C.c_int, C.c_int, C.c_int, _i, _d]
    L.orc_uniform_allocation.argtypes = [C.c_int, C.c_int, C.c_int, _i]
    L.orc_expected_cost.argtypes = [C.c_int, C.c_int, C.c_double, C.c_double]
    L.orc_expected_cost.restype = C.c_double
    L.orc_simulate.argtypes = [_d, _d, _d, _d] + [C.c_int] * 5 + [_d, _i, C.c_double, SimCfg, C.c_uint64,
                                                                  C.POINTER(Metrics), _i64, _i64, _i64, C.c_int64,
                                                                  _i64, _i, _i]
    L.orc_simulate_batch.argtypes = [_d, _d, _d, _d] + [C.c_int] * 6 + [_d, _i, C.c_double, SimCfg, C.c_uint64,
                                                                        C.POINTER(Metrics), _i64, _i64, _i64,
                                                                        C.c_int64, _i64, _i, _i]
    L.orc_top_k.argtypes = [_d, C.c_int, C.c_int, _i]
    L.orc_softmax.argtypes = [_d, C.c_int, _d]
    L.orc_top1_share.argtypes = [_d, C.c_int]
    L.orc_top1_share.restype = C.c_double
    L.orc_gate_decide.argtypes = [_d, C.c_int, C.c_int, C.c_double, C.c_double, _i, _i, _d]
    L.orc_gate_logits.argtypes = [_d, C.c_int, C.c_int, _d, _d]
    L.orc_tile_pipeline_latency.argtypes = [C.c_int, C.c_int64, C.c_int64]
    L.orc_tile_pipeline_latency.restype = C.c_int64
    L.orc_expert_init.argtypes = [C.c_uint64, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _u16]
    L.orc_swiglu.argtypes = [_u16, C.c_int, C.c_int, C.c_int, _f, _d]
    L.orc_init_scale.argtypes = [C.c_int]
    L.orc_init_scale.restype = C.c_float
    L.orc_fnv1a.argtypes = [C.c_void_p, C.c_size_t, C.c_uint64]
    L.orc_fnv1a.restype = C.c_uint64


def _p(a, t):
    return a.ctypes.data_as(t)


def fnv1a(arr: np.ndarray, h: int = 0xcbf29ce484222325) -> str:
    """FNV-1a over the raw little-endian bytes (same hash the reference driver prints)."""
    data = np.ascontiguousarray(arr)
    return f"{lib().orc_fnv1a(data.ctypes.data, data.nbytes, h):016x}"


@dataclass
class Workload:
    L: int
    N: int
    K: int
    D: int
    T: int
    gates: np.ndarray
    acts: np.ndarray
    scores: np.ndarray
    selected: np.ndarray
    fisher: np.ndarray
    first_gate: np.ndarray | None = None


def generate_trace(L, N, K, D, T, concentration=0.6, drift=0.18, gate_seed=99, token_seed=5000,
                   shared_gates=False, fisher_scales=None, drift_scales=None) -> Workload:
    gates = np.zeros((L, D, N))
    acts = np.zeros((T, L, D))
    scores = np.zeros((T, L, N))
    sel = np.zeros((T, L, K), dtype=np.int32)
    fisher = np.zeros(L)
    fs = None if fisher_scales is None else np.ascontiguousarray(fisher_scales, dtype=np.float64)
    ds = None if drift_scales is None else np.ascontiguousarray(drift_scales, dtype=np.float64)
    rc = lib().orc_generate_trace(L, N, K, D, T, concentration, drift, gate_seed, token_seed, int(shared_gates),
                                  None if fs is None else _p(fs, _d), None if ds is None else _p(ds, _d),
                                  _p(gates, _d), _p(acts, _d), _p(scores, _d), _p(sel, _i), _p(fisher, _d))
    assert rc == 0, rc
    return Workload(L, N, K, D, T, gates, acts, scores, sel, fisher)


def calibrate_threshold(w: Workload, target: float) -> float:
    return lib().orc_calibrate_threshold(_p(w.scores, _d), w.T, w.L, w.N, _p(w.fisher, _d), target)


def train_first_gate(w: Workload, lr=0.1, steps=500, seed=0) -> np.ndarray:
    W = np.zeros((w.D, w.N))
    rc = lib().orc_train_first_gate(_p(w.acts, _d), _p(w.scores, _d), w.T, w.L, w.D, w.N, lr, steps, seed, _p(W, _d))
    assert rc == 0
    return W


def generate_profiles(w: Workload, tau: float, first_gate=None):
    a = np.zeros(w.L)
    b = np.zeros(w.L)
    fg = None if first_gate is None else np.ascontiguousarray(first_gate)
    rc = lib().orc_generate_profiles(_p(w.acts, _d), _p(w.scores, _d), _p(w.gates, _d),
                                     None if fg is None else _p(fg, _d), w.T, w.L, w.N, w.K, w.D, tau,
                                     _p(w.fisher, _d), _p(a, _d), _p(b, _d))
    assert rc == 0
    return a, b


def cost_table(alpha, beta, N):
    L = len(alpha)
    t = np.zeros((L, N + 1))
    lib().orc_cost_table(_p(np.ascontiguousarray(alpha, np.float64), _d),
                         _p(np.ascontiguousarray(beta, np.float64), _d), L, N, _p(t, _d))
    return t


def dp_allocate(table: np.ndarray, budget: int):
    L, N1 = table.shape
    caps = np.zeros(L, dtype=np.int32)
    cost = C.c_double()
    t = np.ascontiguousarray(table, np.float64)
    lib().orc_dp_allocate(_p(t, _d), L, N1 - 1, budget, _p(caps, _i), C.byref(cost))
    return caps, cost.value


def uniform_allocation(budget, L, N):
    caps = np.zeros(L, dtype=np.int32)
    lib().orc_uniform_allocation(budget, L, N, _p(caps, _i))
    return caps


@dataclass
class SimOut:
    metrics: dict
    latency_per_token: np.ndarray
    od_per_layer: np.ndarray
    timeline: np.ndarray
    predictions: np.ndarray
    decisions: np.ndarray = field(default=None)


def simulate(w: Workload, caps, tau, fisher=None, first_gate=None, tiles=4, tile_transfer=2, tile_compute=1,
             attention=8, gate=1, lookahead=2, gating=True, prefetch=True, seed=0, T=None) -> SimOut:
    T = w.T if T is None else T
    fisher = w.fisher if fisher is None else np.ascontiguousarray(fisher, np.float64)
    caps = np.ascontiguousarray(caps, dtype=np.int32)
    cfg = SimCfg(tiles, tile_transfer, tile_compute, attention, gate, lookahead, int(gating), int(prefetch))
    m = Metrics()
    lat = np.zeros(T, dtype=np.int64)
    odl = np.zeros(w.L, dtype=np.int64)
    cap = T * w.L * (4 + 4 * w.K * tiles + 8 * tiles) + 64
    tl = np.zeros((cap, 8), dtype=np.int64)
    n = C.c_int64()
    pw = 2 + w.K
    preds = np.zeros((T, w.L, 3, pw), dtype=np.int32)
    dec = np.zeros((T, w.L, w.K), dtype=np.int32)
    fg = None if first_gate is None else np.ascontiguousarray(first_gate)
    rc = lib().orc_simulate(_p(w.acts, _d), _p(w.scores, _d), _p(w.gates, _d), None if fg is None else _p(fg, _d),
                            T, w.L, w.N, w.K, w.D, _p(fisher, _d), _p(caps, _i), tau, cfg, seed, C.byref(m),
                            _p(lat, _i64), _p(odl, _i64), _p(tl, _i64), cap, C.byref(n), _p(preds, _i), _p(dec, _i))
    assert rc == 0, rc
    metrics = {k: getattr(m, k) for k, _ in Metrics._fields_}
    return SimOut(metrics, lat, odl, tl[: n.value].copy(), preds, dec)


def simulate_batch(streams: list, caps, tau, fisher=None, first_gate=None, tiles=4, tile_transfer=2, tile_compute=1,
                   attention=8, gate=1, lookahead=2, gating=True, prefetch=True, seed=0, T=None) -> SimOut:
    """B token streams sharing one expert cache (builder-defined union policy, see
    orc_simulate_batch).  All streams must share the gates (same gate_seed) and fisher.
    Returns decisions [B][T][L][K] and predictions [B][T][L][3][2+K]."""
    w0 = streams[0]
    B = len(streams)
    T = w0.T if T is None else T
    fisher = w0.fisher if fisher is None else np.ascontiguousarray(fisher, np.float64)
    for w in streams[1:]:
        assert np.array_equal(w.gates, w0.gates) and np.array_equal(w.fisher, w0.fisher)
    acts = np.ascontiguousarray(np.stack([w.acts[:T] for w in streams]))
    scores = np.ascontiguousarray(np.stack([w.scores[:T] for w in streams]))
    caps = np.ascontiguousarray(caps, dtype=np.int32)
    cfg = SimCfg(tiles, tile_transfer, tile_compute, attention, gate, lookahead, int(gating), int(prefetch))
    m = Metrics()
    lat = np.zeros(T, dtype=np.int64)
    odl = np.zeros(w0.L, dtype=np.int64)
    cap = T * w0.L * (4 + 4 * min(w0.N, B * w0.K) * tiles + 8 * tiles * w0.N) + 64
    tl = np.zeros((cap, 8), dtype=np.int64)
    n = C.c_int64()
    pw = 2 + w0.K
    preds = np.zeros((B, T, w0.L, 3, pw), dtype=np.int32)
    dec = np.zeros((B, T, w0.L, w0.K), dtype=np.int32)
    fg = None if first_gate is None else np.ascontiguousarray(first_gate)
    rc = lib().orc_simulate_batch(_p(acts, _d), _p(scores, _d), _p(w0.gates, _d), None if fg is None else _p(fg, _d),
                                  B, T, w0.L, w0.N, w0.K, w0.D, _p(fisher, _d), _p(caps, _i), tau, cfg, seed,
                                  C.byref(m), _p(lat, _i64), _p(odl, _i64), _p(tl, _i64), cap, C.byref(n),
                                  _p(preds, _i), _p(dec, _i))
    assert rc == 0, rc
    metrics = {k: getattr(m, k) for k, _ in Metrics._fields_}
    return SimOut(metrics, lat, odl, tl[: n.value].copy(), preds, dec)


def gate_scores(gate: np.ndarray, x: np.ndarray, concentration: float = 1.0) -> np.ndarray:
    """softmax(GateMatrix::logits(x) / concentration) exactly as the reference generator forms the
    stored scores (inc/prefetch.hpp:24-35, inc/workload.hpp:93-98, inc/core.hpp:205-216)."""
    D, N = gate.shape
    lg = np.zeros(N)
    xx = np.ascontiguousarray(x, dtype=np.float64)
    g = np.ascontiguousarray(gate, dtype=np.float64)
    lib().orc_gate_logits(_p(g, _d), D, N, _p(xx, _d), _p(lg, _d))
    lg = np.array([v / concentration for v in lg])
    out = np.zeros(N)
    lib().orc_softmax(_p(lg, _d), N, _p(out, _d))
    return out


def expert_init(seed, layer, expert, D, F, tiles) -> np.ndarray:
    out = np.zeros(3 * F * D, dtype=np.uint16)
    rc = lib().orc_expert_init(seed, layer, expert, D, F, tiles, _p(out, _u16))
    assert rc == 0
    return out


def swiglu(w_u16: np.ndarray, D, F, tiles, x: np.ndarray) -> np.ndarray:
    y = np.zeros(D)
    xf = np.ascontiguousarray(x, dtype=np.float32)
    rc = lib().orc_swiglu(_p(np.ascontiguousarray(w_u16), _u16), D, F, tiles, _p(xf, _f), _p(y, _d))
    assert rc == 0
    return y


# ------------------------------------------------------------------------------------------
# reference driver (oracle/_ref/moesim_ref), available where /root/reference compiled
# ------------------------------------------------------------------------------------------

def run_ref(blob: str | None = None, **kw) -> dict:
    args = [REF_BIN] + [f"{k}={','.join(map(str, v)) if isinstance(v, (list, tuple)) else v}"
                        for k, v in kw.items()]
    if blob:
        args.append(f"blob={blob}")
    out = subprocess.run(args, check=True, capture_output=True, text=True).stdout
    return json.loads(out)


def read_blob(path, L, N, D, T, first_gate: bool):
    raw = np.fromfile(path, dtype=np.float64)
    o = 0
    gates = raw[o:o + L * D * N].reshape(L, D, N); o += L * D * N
    fg = None
    if first_gate:
        fg = raw[o:o + D * N].reshape(D, N); o += D * N
    acts = raw[o:o + T * L * D].reshape(T, L, D); o += T * L * D
    scores = raw[o:o + T * L * N].reshape(T, L, N); o += T * L * N
    assert o == raw.size
    return gates, fg, acts, scores
