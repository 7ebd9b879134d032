"""Artifact files of the reference (inc/io.hpp) through the C ABI (include/adapmoe.h, [host] calls).

Same names and meaning as the reference: load_trace / save_trace (JSON Lines; the binary container
with binary=True), load_gates / save_gates, load_profiles / save_profiles (+ profile_hash),
load_threshold / save_threshold, load_allocation / save_allocation, load_cost_table /
save_cost_table, validate_trace.  Files written here are byte-identical to the reference's; errors
raise MoeError with the reference CLI's exit classes (2 io_error, 3 parse/schema/version error,
4 validation).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _capi
from ._capi import check, load
from .moesim import ModelSpec, _f64, _i32, _p


def _spec_py(s) -> ModelSpec:
    return ModelSpec(s.num_layers, s.experts_per_layer, s.top_k, s.hidden_dim)


@dataclass
class TraceFile:                      # inc/io.hpp:141 TraceFile, in array form
    spec: ModelSpec
    acts: np.ndarray                  # [T][L][d]
    scores: np.ndarray                # [T][L][N]
    selected: np.ndarray              # [T][L][K] (-1 padded)
    violations: list


def load_trace(path: str) -> TraceFile:
    h = C.c_void_p()
    check(load().moe_trace_load(path.encode(), C.byref(h)))
    try:
        s = _capi.ModelSpecC()
        T = C.c_int32()
        check(load().moe_trace_info(h, C.byref(s), C.byref(T)))
        L, N, K, D = s.num_layers, s.experts_per_layer, s.top_k, s.hidden_dim
        acts = np.zeros((T.value, L, D))
        scores = np.zeros((T.value, L, N))
        sel = np.zeros((T.value, L, K), dtype=np.int32)
        check(load().moe_trace_read(h, _p(acts, _capi._d), _p(scores, _capi._d), _p(sel, _capi._i32)))
        n = C.c_int64()
        msg = C.create_string_buffer(512)
        check(load().moe_trace_validate(h, C.byref(n), msg, 512))
        violations = [msg.value.decode()] if n.value else []
        if n.value > 1:
            violations.append(f"... {n.value - 1} more")
        return TraceFile(_spec_py(s), acts, scores, sel, violations)
    finally:
        load().moe_trace_free(h)


def save_trace(path: str, spec: ModelSpec, acts, scores, selected, binary: bool = False) -> None:
    acts, scores, sel = _f64(acts), _f64(scores), _i32(selected)
    check(load().moe_trace_save(path.encode(), C.byref(spec.c()), acts.shape[0], _p(acts, _capi._d),
                                _p(scores, _capi._d), _p(sel, _capi._i32), int(binary)))


def load_gates(path: str):
    """-> (spec, gates [L][d][N], first_gate [d][N] or None, (learning_rate, steps, seed) or None)"""
    s = _capi.ModelSpecC()
    has = C.c_int32()
    check(load().moe_gates_load(path.encode(), C.byref(s), None, None, C.byref(has), None, None, None))
    gates = np.zeros((s.num_layers, s.hidden_dim, s.experts_per_layer))
    fg = np.zeros((s.hidden_dim, s.experts_per_layer)) if has.value else None
    lr, steps, seed = C.c_double(), C.c_int32(), C.c_uint64()
    check(load().moe_gates_load(path.encode(), C.byref(s), _p(gates, _capi._d), None if fg is None else _p(fg, _capi._d),
                                C.byref(has), C.byref(lr), C.byref(steps), C.byref(seed)))
    return _spec_py(s), gates, fg, ((lr.value, steps.value, seed.value) if has.value else None)


def save_gates(path: str, spec: ModelSpec, gates, first_gate=None, learning_rate=0.1, steps=500, seed=0) -> None:
    g = _f64(gates)
    fg = None if first_gate is None else _f64(first_gate)
    check(load().moe_gates_save(path.encode(), C.byref(spec.c()), _p(g, _capi._d),
                                None if fg is None else _p(fg, _capi._d), float(learning_rate), int(steps), int(seed)))


def load_profiles(path: str):
    """-> (spec, alpha, beta, fisher) = single_expert_prob, prefetch_accuracy, fisher_diag_sum"""
    s = _capi.ModelSpecC()
    check(load().moe_profiles_load(path.encode(), C.byref(s), None, None, None))
    a, b, f = (np.zeros(s.num_layers) for _ in range(3))
    check(load().moe_profiles_load(path.encode(), C.byref(s), _p(a, _capi._d), _p(b, _capi._d), _p(f, _capi._d)))
    return _spec_py(s), a, b, f


def save_profiles(path: str | None, spec: ModelSpec, alpha, beta, fisher) -> str:
    """Writes the profiles file (if path) and returns profile_hash (inc/io.hpp:290)."""
    h = C.create_string_buffer(17)
    check(load().moe_profiles_save(path.encode() if path else None, C.byref(spec.c()), _p(_f64(alpha), _capi._d),
                                   _p(_f64(beta), _capi._d), _p(_f64(fisher), _capi._d), h))
    return h.value.decode()


def profile_hash(spec: ModelSpec, alpha, beta, fisher) -> str:
    return save_profiles(None, spec, alpha, beta, fisher)


def load_threshold(path: str):
    """-> (tau, target_single_ratio, realized_single_ratio)"""
    t, a, r = C.c_double(), C.c_double(), C.c_double()
    check(load().moe_threshold_load(path.encode(), C.byref(t), C.byref(a), C.byref(r)))
    return t.value, a.value, r.value


def save_threshold(path: str, tau: float, target_single_ratio: float, realized_single_ratio: float) -> None:
    check(load().moe_threshold_save(path.encode(), float(tau), float(target_single_ratio),
                                    float(realized_single_ratio)))


def load_allocation(path: str):
    """-> (capacities, budget, total_cost, profile_hash)"""
    b, n, cost = C.c_int32(), C.c_int32(), C.c_double()
    check(load().moe_allocation_load(path.encode(), C.byref(b), C.byref(n), None, None, None))
    caps = np.zeros(n.value, dtype=np.int32)
    h = C.create_string_buffer(17)
    check(load().moe_allocation_load(path.encode(), C.byref(b), C.byref(n), _p(caps, _capi._i32), C.byref(cost), h))
    return caps, b.value, cost.value, h.value.decode()


def save_allocation(path: str, capacities, budget: int, total_cost: float, profile_hash: str) -> None:
    caps = _i32(capacities)
    check(load().moe_allocation_save(path.encode(), int(budget), caps.shape[0], _p(caps, _capi._i32),
                                     float(total_cost), profile_hash.encode()))


def load_cost_table(path: str) -> np.ndarray:
    n, L = C.c_int32(), C.c_int32()
    check(load().moe_cost_table_load(path.encode(), C.byref(n), C.byref(L), None))
    t = np.zeros((L.value, n.value + 1))
    check(load().moe_cost_table_load(path.encode(), C.byref(n), C.byref(L), _p(t, _capi._d)))
    return t


def save_cost_table(path: str, table) -> None:
    t = _f64(table)
    check(load().moe_cost_table_save(path.encode(), t.shape[1] - 1, t.shape[0], _p(t, _capi._d)))
