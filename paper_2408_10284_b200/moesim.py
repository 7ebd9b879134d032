"""Python mirror of the reference moesim API (``inc/`` = /root/reference/proj/include/moesim) over
the B200 engine's C ABI.  Names and argument meanings follow the reference so call sites read the
same: ``calibrate_threshold``, ``build_cost_table``, ``dp_allocate``, ``uniform_allocation``,
``simulate_trace``, ``generate_trace``, ``generate_profiles`` ...  Errors surface as
:class:`MoeError` carrying the reference CLI exit-code class (proj/tools/moesim_main.cpp:26-40).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from . import _capi
from ._capi import check, load, MoeError  # noqa: F401

EVENT_KINDS = ("attention", "gate", "expert_compute", "tile_compute", "tile_transfer")


@dataclass(frozen=True)
class ModelSpec:                      # inc/core.hpp:22
    num_layers: int = 1
    experts_per_layer: int = 8
    top_k: int = 2
    hidden_dim: int = 1

    def c(self):
        return _capi.ModelSpecC(self.num_layers, self.experts_per_layer, self.top_k, self.hidden_dim)


@dataclass
class PolicyFlags:                    # inc/simulator.hpp:26
    adaptive_gating: bool = False
    prefetch: bool = False
    adaptive_cache: bool = False


@dataclass
class SimConfig:                      # inc/simulator.hpp:34 (defaults = CLI defaults, moesim_main.cpp:259-267)
    tile_count_per_expert: int = 4
    tile_transfer_time: int = 2
    tile_compute_time: int = 1
    attention_compute_time: int = 8
    gate_compute_time: int = 1
    lookahead_depth: int = 2
    policy: PolicyFlags = field(default_factory=lambda: PolicyFlags(True, True, True))

    def c(self):
        p = self.policy
        return _capi.SimConfigC(self.tile_count_per_expert, self.tile_transfer_time, self.tile_compute_time,
                                self.attention_compute_time, self.gate_compute_time, self.lookahead_depth,
                                int(p.adaptive_gating), int(p.prefetch), int(p.adaptive_cache))


@dataclass
class SynthConfig:                    # inc/workload.hpp:19
    spec: ModelSpec
    tokens: int = 1000
    dirichlet_concentration: float = 1.0
    residual_drift: float = 0.1
    gate_seed: int = 1
    token_seed: int = 2
    shared_gates: bool = False
    fisher_scales: list | None = None
    drift_scales: list | None = None


@dataclass
class Workload:                       # GeneratedWorkload (inc/workload.hpp:51) in array form
    spec: ModelSpec
    gates: np.ndarray                 # [L][d][N] fp64
    acts: np.ndarray                  # [T][L][d] fp64
    scores: np.ndarray                # [T][L][N] fp64
    selected: np.ndarray              # [T][L][K] int32
    fisher: np.ndarray                # [L]

    @property
    def tokens(self) -> int:
        return self.acts.shape[0]


@dataclass
class SimResult:                      # SimResult (inc/simulator.hpp:168)
    metrics: dict
    latency_per_token: np.ndarray
    on_demand_loads_per_layer: np.ndarray
    timeline: np.ndarray | None       # [n_events][8] int64: stream, kind, start, end, token, layer, expert, tile
    n_events: int = 0
    stats: dict | None = None


def _p(a, t):
    return a.ctypes.data_as(t)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def _i32(a):
    return np.ascontiguousarray(a, dtype=np.int32)


# ------------------------------- host tools -------------------------------------------------

def calibrate_threshold(spec: ModelSpec, scores, fisher, target_single_ratio: float):
    """inc/gating.hpp:85 — returns (tau, realized single ratio)."""
    scores = _f64(scores)
    fisher = _f64(fisher)
    tau = C.c_double()
    real = C.c_double()
    T = scores.shape[0] if scores.ndim == 3 else scores.size // (spec.num_layers * spec.experts_per_layer)
    check(load().moe_calibrate_threshold(C.byref(spec.c()), _p(scores, _capi._d), T, _p(fisher, _capi._d),
                                         float(target_single_ratio), C.byref(tau), C.byref(real)))
    return tau.value, real.value


def build_cost_table(spec: ModelSpec, alpha, beta) -> np.ndarray:
    """inc/cache_model.hpp:189 — [L][N+1] expected on-demand loads."""
    t = np.zeros((spec.num_layers, spec.experts_per_layer + 1))
    check(load().moe_build_cost_table(C.byref(spec.c()), _p(_f64(alpha), _capi._d), _p(_f64(beta), _capi._d),
                                      _p(t, _capi._d)))
    return t


def dp_allocate(spec: ModelSpec, table, budget: int):
    """inc/allocator.hpp:66 — (capacities, total_cost)."""
    caps = np.zeros(spec.num_layers, dtype=np.int32)
    cost = C.c_double()
    check(load().moe_dp_allocate(C.byref(spec.c()), _p(_f64(table), _capi._d), int(budget), _p(caps, _capi._i32),
                                 C.byref(cost)))
    return caps, cost.value


def uniform_allocation(spec: ModelSpec, budget: int) -> np.ndarray:
    caps = np.zeros(spec.num_layers, dtype=np.int32)
    check(load().moe_uniform_allocation(C.byref(spec.c()), int(budget), _p(caps, _capi._i32)))
    return caps


def expected_cost(t: int, n: int, alpha: float, beta: float) -> float:
    out = C.c_double()
    check(load().moe_expected_cost(t, n, alpha, beta, C.byref(out)))
    return out.value


def tile_pipeline_latency(tiles: int, transfer: int, compute: int) -> int:
    out = C.c_int64()
    check(load().moe_tile_pipeline_latency(tiles, transfer, compute, C.byref(out)))
    return out.value


def _events_buf(spec: ModelSpec, T: int, cfg: SimConfig, batch: int = 1):
    """Uninitialised [cap][8] int64 event buffer (moe_event layout) and its capacity."""
    k = min(spec.experts_per_layer, spec.top_k * batch)  # experts a layer can activate
    per_layer = 2 + k * (1 + 2 * cfg.tile_count_per_expert) + 3 * k * cfg.tile_count_per_expert
    cap = T * spec.num_layers * per_layer + 64
    return np.empty((cap, 8), dtype=np.int64), cap


def _evp(buf):
    return None if buf is None else buf.ctypes.data_as(C.POINTER(_capi.EventC))


def _events_np(buf, n):
    return buf[:n].copy()


def replay_policy(spec: ModelSpec, caps, cfg: SimConfig, seed: int, decisions, single, predictions,
                  timeline: bool = True) -> SimResult:
    """Host tick-model engine (simulate_trace's cache/transfer half) over router outputs."""
    decisions = _i32(decisions)
    T = decisions.shape[0]
    single = None if single is None else _i32(single)
    predictions = None if predictions is None else _i32(predictions)
    m = _capi.MetricsC()
    lat = np.zeros(T, dtype=np.int64)
    odl = np.zeros(spec.num_layers, dtype=np.int64)
    n = C.c_int64()
    buf, cap = _events_buf(spec, T, cfg) if timeline else (None, 0)
    check(load().moe_replay_policy(C.byref(spec.c()), T, _p(_i32(caps), _capi._i32), C.byref(cfg.c()), seed,
                                   _p(decisions, _capi._i32), None if single is None else _p(single, _capi._i32),
                                   None if predictions is None else _p(predictions, _capi._i32), C.byref(m),
                                   _p(lat, _capi._i64), _p(odl, _capi._i64), _evp(buf), cap, C.byref(n)))
    return SimResult({k: getattr(m, k) for k, _ in _capi.MetricsC._fields_}, lat, odl,
                     _events_np(buf, n.value) if timeline else None, n.value)


# ------------------------------- device engine ----------------------------------------------

class Engine:
    """One B200 engine (one process per GPU).  Wraps moe_engine_t."""

    def __init__(self, spec: ModelSpec, device: int = 0):
        self.spec = spec
        self._h = C.c_void_p()
        check(load().moe_engine_create(C.byref(spec.c()), device, C.byref(self._h)))

    def close(self):
        if self._h:
            load().moe_engine_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()

    # -- routing / simulation ------------------------------------------------------------------
    def load_gates(self, gates, first_gate=None):
        g = _f64(gates)
        fg = None if first_gate is None else _f64(first_gate)
        check(load().moe_load_gates(self._h, _p(g, _capi._d), None if fg is None else _p(fg, _capi._d)))

    def route_trace(self, acts, scores, fisher, tau, cfg: SimConfig):
        acts, scores, fisher = _f64(acts), _f64(scores), _f64(fisher)
        T, L, K = acts.shape[0], self.spec.num_layers, self.spec.top_k
        dec = np.zeros((T, L, K), dtype=np.int32)
        single = np.zeros((T, L), dtype=np.int32)
        pert = np.zeros((T, L))
        preds = np.zeros((T, L, 3, 2 + K), dtype=np.int32)
        check(load().moe_route_trace(self._h, _p(acts, _capi._d), _p(scores, _capi._d), T, _p(fisher, _capi._d),
                                     float(tau), C.byref(cfg.c()), _p(dec, _capi._i32), _p(single, _capi._i32),
                                     _p(pert, _capi._d), _p(preds, _capi._i32)))
        return dec, single, pert, preds

    def router_forward(self, layer: int, x, fisher, tau: float, lookahead: int = 2, scores=None,
                       adaptive: bool = True, stream=None):
        """K1 for one layer on device rows (moe_router_forward).  x: CUDA fp64 tensor [B][d]; scores:
        optional CUDA fp64 [B][N] stored scores to decide from.  Returns CUDA tensors selected
        [B][1+lookahead][K], count / single [B][1+lookahead], perturbation [B][1+lookahead],
        enqueued on `stream` (a torch.cuda.Stream; default: the current stream)."""
        import torch
        B, K = x.shape[0], self.spec.top_k
        rows = B * (1 + lookahead)
        dev = x.device
        sel = torch.empty((B, 1 + lookahead, K), dtype=torch.int32, device=dev)
        cnt = torch.empty((B, 1 + lookahead), dtype=torch.int32, device=dev)
        sgl = torch.empty((B, 1 + lookahead), dtype=torch.int32, device=dev)
        pert = torch.empty((B, 1 + lookahead), dtype=torch.float64, device=dev)
        if rows:
            s = stream if stream is not None else torch.cuda.current_stream(dev)
            out = _capi.RouteOutC(sel.data_ptr(), cnt.data_ptr(), sgl.data_ptr(), pert.data_ptr())
            check(load().moe_router_forward(self._h, layer, x.data_ptr(), B,
                                            None if scores is None else scores.data_ptr(), float(tau),
                                            _p(_f64(fisher), _capi._d), lookahead, 1 if adaptive else 0,
                                            C.byref(out), s.cuda_stream))
        return sel, cnt, sgl, pert

    def simulate_trace(self, acts, scores, fisher, caps, tau, cfg: SimConfig, seed: int = 0,
                       timeline: bool = True) -> SimResult:
        """inc/simulator.hpp:329 with K1 on the GPU."""
        acts, scores, fisher = _f64(acts), _f64(scores), _f64(fisher)
        T = acts.shape[0]
        m = _capi.MetricsC()
        lat = np.zeros(T, dtype=np.int64)
        odl = np.zeros(self.spec.num_layers, dtype=np.int64)
        n = C.c_int64()
        buf, cap = _events_buf(self.spec, T, cfg) if timeline else (None, 0)
        check(load().moe_simulate_trace(self._h, _p(acts, _capi._d), _p(scores, _capi._d), T, _p(fisher, _capi._d),
                                        _p(_i32(caps), _capi._i32), float(tau), C.byref(cfg.c()), seed, C.byref(m),
                                        _p(lat, _capi._i64), _p(odl, _capi._i64), _evp(buf), cap, C.byref(n)))
        return SimResult({k: getattr(m, k) for k, _ in _capi.MetricsC._fields_}, lat, odl,
                         _events_np(buf, n.value) if timeline else None, n.value)

    def generate_trace(self, cfg: SynthConfig) -> Workload:
        """inc/workload.hpp:60 — host RNG stream + GPU gate GEMVs; also loads the gates."""
        s = cfg.spec
        assert s == self.spec
        L, N, K, D, T = s.num_layers, s.experts_per_layer, s.top_k, s.hidden_dim, cfg.tokens
        gates = np.zeros((L, D, N))
        acts = np.zeros((T, L, D))
        scores = np.zeros((T, L, N))
        sel = np.zeros((T, L, K), dtype=np.int32)
        fisher = np.zeros(L)
        fs = None if cfg.fisher_scales is None else _f64(cfg.fisher_scales)
        ds = None if cfg.drift_scales is None else _f64(cfg.drift_scales)
        c = _capi.SynthConfigC(s.c(), T, cfg.dirichlet_concentration, cfg.residual_drift, cfg.gate_seed,
                               cfg.token_seed, int(cfg.shared_gates),
                               None if fs is None else _p(fs, _capi._d), None if ds is None else _p(ds, _capi._d))
        check(load().moe_generate_trace(self._h, C.byref(c), _p(gates, _capi._d), _p(acts, _capi._d),
                                        _p(scores, _capi._d), _p(sel, _capi._i32), _p(fisher, _capi._d)))
        return Workload(s, gates, acts, scores, sel, fisher)

    def generate_profiles(self, acts, scores, fisher, tau):
        """inc/workload.hpp:133 — (alpha, beta) per layer."""
        acts, scores, fisher = _f64(acts), _f64(scores), _f64(fisher)
        a = np.zeros(self.spec.num_layers)
        b = np.zeros(self.spec.num_layers)
        check(load().moe_generate_profiles(self._h, _p(acts, _capi._d), _p(scores, _capi._d), acts.shape[0],
                                           _p(fisher, _capi._d), float(tau), _p(a, _capi._d), _p(b, _capi._d)))
        return a, b

    def compare_policies(self, acts, scores, fisher, alpha, beta, tau, cfg: SimConfig, budget: int,
                         seed: int = 0) -> list[dict]:
        """compare_policies (inc/simulator.hpp:504): the 7-row ablation grid with K1 on the GPU."""
        acts, scores = _f64(acts), _f64(scores)
        T, L = acts.shape[0], self.spec.num_layers
        rows = (_capi.CompareRowC * 7)()
        caps = np.zeros((7, L), dtype=np.int32)
        lat = np.zeros((7, T), dtype=np.int64)
        odl = np.zeros((7, L), dtype=np.int64)
        check(load().moe_compare_policies(self._h, _p(acts, _capi._d), _p(scores, _capi._d), T, _p(_f64(fisher), _capi._d),
                                          _p(_f64(alpha), _capi._d), _p(_f64(beta), _capi._d), float(tau),
                                          C.byref(cfg.c()), int(budget), int(seed), rows, _p(caps, _capi._i32),
                                          _p(lat, _capi._i64), _p(odl, _capi._i64)))
        out = []
        for i, r in enumerate(rows):
            m = {k: getattr(r.metrics, k) for k, _ in _capi.MetricsC._fields_}
            m["latency_per_token"] = lat[i].tolist()
            m["on_demand_loads_per_layer"] = odl[i].tolist()
            out.append({"name": r.name.decode(), "flags": [r.adaptive_gating, r.prefetch, r.adaptive_cache],
                        "capacities": caps[i].tolist(), "speedup_vs_baseline": r.speedup_vs_baseline, "metrics": m})
        return out

    def train_first_gate(self, acts, scores, learning_rate: float = 0.1, steps: int = 500, seed: int = 0) -> np.ndarray:
        """first_layer_training_pairs + train_predictive_gate (inc/prefetch.hpp:194) on the GPU,
        bit-exact with the reference; returns the [d][N] first-layer predictive gate."""
        acts, scores = _f64(acts), _f64(scores)
        w = np.zeros((self.spec.hidden_dim, self.spec.experts_per_layer))
        check(load().moe_train_first_gate(self._h, _p(acts, _capi._d), _p(scores, _capi._d), acts.shape[0],
                                          float(learning_rate), int(steps), int(seed), _p(w, _capi._d)))
        return w

    # -- physical decode -----------------------------------------------------------------------
    STORE_FORMATS = {"bf16": 0, "xb12": 1, "xbh": 2}

    def experts_init(self, ffn_dim: int, tiles: int, seed: int = 0, host_alias: int = 0, expert_owner=None,
                     rank: int = 0, store_format: str = "bf16"):
        """Pinned host expert store with the deterministic init.  expert_owner ([L][N] shard table) +
        rank: an expert-parallel shard's store, holding only the experts it owns.  store_format
        "xb12" / "xbh": lossless exponent-coded tiles (4-bit window codes / per-tile Huffman codes;
        moe_experts_set_format)."""
        check(load().moe_experts_set_format(self._h, self.STORE_FORMATS[store_format]))
        if expert_owner is None:
            check(load().moe_experts_init(self._h, ffn_dim, tiles, seed, host_alias))
        else:
            own = np.ascontiguousarray(expert_owner, dtype=np.int32).reshape(-1)
            check(load().moe_experts_init_shard(self._h, ffn_dim, tiles, seed, host_alias, _p(own, _capi._i32), rank))

    def experts_format(self) -> tuple[str, int]:
        """(store format, bytes a copy of every stored record moves over the host link)."""
        f, b = C.c_int32(), C.c_int64()
        check(load().moe_experts_format(self._h, C.byref(f), C.byref(b)))
        return {v: k for k, v in self.STORE_FORMATS.items()}[f.value], b.value

    def expert_tile_record(self, layer: int, expert: int, tile: int) -> dict:
        """Host address and XB12 / XBH metadata of one stored tile record (moe_expert_tile_record)."""
        r, b, f, base, m, nib, esc = (C.c_void_p(), C.c_int64(), C.c_int32(), C.c_uint32(), C.c_int64(), C.c_int64(),
                                      C.c_int64())
        check(load().moe_expert_tile_record(self._h, layer, expert, tile, C.byref(r), C.byref(b), C.byref(f),
                                            C.byref(base), C.byref(m), C.byref(nib), C.byref(esc)))
        return {"ptr": int(r.value), "bytes": b.value, "format": f.value, "base": base.value, "n_escapes": m.value,
                "nib_offset": nib.value, "esc_offset": esc.value}

    def experts_alloc(self, ffn_dim: int, tiles: int, expert_owner=None, rank: int = 0, store_format: str = "bf16"):
        """Pinned store for real weights (moe_experts_alloc); fill it with expert_set."""
        check(load().moe_experts_set_format(self._h, self.STORE_FORMATS[store_format]))
        if expert_owner is None:
            check(load().moe_experts_alloc(self._h, ffn_dim, tiles))
        else:
            own = np.ascontiguousarray(expert_owner, dtype=np.int32).reshape(-1)
            check(load().moe_experts_alloc_shard(self._h, ffn_dim, tiles, _p(own, _capi._i32), rank))

    def experts_info(self) -> dict:
        """Pinned bytes, distinct stored experts and host NUMA node of the store."""
        b, n, node = C.c_int64(), C.c_int32(), C.c_int32()
        check(load().moe_experts_info(self._h, C.byref(b), C.byref(n), C.byref(node)))
        return {"pinned_bytes": b.value, "stored_experts": n.value, "numa_node": node.value}

    def expert_set(self, layer: int, expert: int, w1, w3, w2):
        """One expert's weights in checkpoint layout: w1 = gate_proj [ffn][d], w3 = up_proj [ffn][d],
        w2 = down_proj [d][ffn]; bf16 (torch.bfloat16 tensors or uint16 bit patterns)."""
        def bits(w):
            if hasattr(w, "detach"):  # torch tensor
                import torch
                w = w.detach().contiguous().cpu()
                if w.dtype == torch.bfloat16:
                    w = w.view(torch.int16)
                w = w.numpy()
            return np.ascontiguousarray(w).view(np.uint16)
        w1, w3, w2 = bits(w1), bits(w3), bits(w2)
        d, F = self.spec.hidden_dim, w1.shape[0]
        if w1.shape != (F, d) or w3.shape != (F, d) or w2.shape != (d, F):
            raise ValueError(f"expert_set: want w1/w3 [{F}][{d}] and w2 [{d}][{F}], got {w1.shape} {w3.shape} {w2.shape}")
        if self.expert_bytes() != 3 * F * d * 2:
            raise ValueError("expert_set: ffn does not match the allocated store")
        check(load().moe_expert_set(self._h, layer, expert, _p(w1, _capi._u16), _p(w3, _capi._u16),
                                    _p(w2, _capi._u16)))

    def expert_bytes(self) -> int:
        b = C.c_int64()
        check(load().moe_expert_bytes(self._h, C.byref(b)))
        return b.value

    def copy_tiles(self, layer: int, expert: int, tile0: int, n_tiles: int, dst_ptr: int, stream: int | None = None,
                   tile_events=None) -> None:
        """Stream-ordered copy of expert tiles from the pinned store into device memory (moe_copy_tiles);
        tile_events: optional list of cudaEvent_t handles (ints) recorded after each tile."""
        ev = None if tile_events is None else (C.c_void_p * len(tile_events))(*[C.c_void_p(int(e)) for e in tile_events])
        check(load().moe_copy_tiles(self._h, layer, expert, tile0, n_tiles, C.c_void_p(dst_ptr),
                                    C.c_void_p(stream) if stream else None, ev))

    def expert_ffn_async(self, expert_ptr: int, x_ptr: int, y_ptr: int, rows: int, weights=None,
                         accumulate: bool = False, tile_events=None, stream: int | None = None) -> None:
        """y[b] (+)= w[b] * SwiGLU(x[b]) on device buffers, stream-ordered (moe_expert_ffn_async)."""
        w = None if weights is None else _f64(weights)
        ev = None if tile_events is None else (C.c_void_p * len(tile_events))(*[C.c_void_p(int(e)) for e in tile_events])
        check(load().moe_expert_ffn_async(self._h, C.c_void_p(expert_ptr), C.c_void_p(x_ptr), C.c_void_p(y_ptr), rows,
                                          None if w is None else _p(w, _capi._d), int(accumulate), ev,
                                          C.c_void_p(stream) if stream else None))

    def expert_host_ptr(self, layer: int, expert: int) -> int:
        """Address of the expert's tile-major block in the pinned host store (moe_expert_host_ptr)."""
        p = C.c_void_p()
        check(load().moe_expert_host_ptr(self._h, layer, expert, C.byref(p)))
        return int(p.value)

    def expert_read(self, layer: int, expert: int) -> np.ndarray:
        out = np.zeros(self.expert_bytes() // 2, dtype=np.uint16)
        check(load().moe_expert_read(self._h, layer, expert, _p(out, _capi._u16)))
        return out

    def decode_begin(self, caps, fisher, tau, cfg: SimConfig, seed: int, total_tokens: int, staging_slots: int = 0,
                     batch: int = 1, ep_rank: int = 0, ep_world: int = 1, free_running: bool = False,
                     concentration: float = 1.0, expert_owner=None):
        """Start a decode session (moe_decode_begin_ex).  batch > 1: B token streams share the
        cache; decode_tokens then takes acts [n][B][L][d] and scores [n][B][L][N].  ep_world > 1:
        this engine is expert-parallel shard ep_rank (experts e % ep_world == ep_rank) and
        decode_tokens returns its partial layer outputs (see paper_2408_10284_b200/ep.py).
        free_running: layer l > 0 routes and computes on layer l-1's output (decisions from the
        layer's gate, softmax(logits / concentration)); layer 0 takes acts[:, ..., 0, :]."""
        owner = None if expert_owner is None else _i32(np.asarray(expert_owner).reshape(-1))
        opts = _capi.DecodeOptsC(batch, ep_rank, ep_world, int(free_running), float(concentration),
                                 None if owner is None else owner.ctypes.data)
        check(load().moe_decode_begin_ex(self._h, _p(_i32(caps), _capi._i32), staging_slots,
                                         _p(_f64(fisher), _capi._d), float(tau), C.byref(cfg.c()), seed,
                                         total_tokens, C.byref(opts)))
        self._batch = batch

    def decode_ep_export(self, max_tokens_per_call: int) -> tuple[int, bytes]:
        """Expert-parallel exchange region of this shard: (device pointer, 64-byte CUDA IPC handle)."""
        ptr = C.c_uint64()
        h = C.create_string_buffer(64)
        check(load().moe_decode_ep_export(self._h, int(max_tokens_per_call), C.byref(ptr), h))
        return ptr.value, h.raw

    def decode_ep_connect(self, peer_ptrs=None, peer_ipc=None):
        """peer_ptrs[g]: region pointers of same-process shards (0 = use peer_ipc[g], 64 bytes each)."""
        ptrs = None if peer_ptrs is None else (C.c_uint64 * len(peer_ptrs))(*[int(p) for p in peer_ptrs])
        ipc = None if peer_ipc is None else b"".join(bytes(b).ljust(64, b"\0")[:64] for b in peer_ipc)
        check(load().moe_decode_ep_connect(self._h, ptrs, ipc))

    def decode_layer(self, layer: int, x_ptr: int, scores_ptr: int | None, out_ptr: int, add_input: bool = True,
                     stream: int | None = None) -> None:
        """One MoE layer on device buffers, ordered with the caller's CUDA stream (moe_decode_layer):
        x [B][d] fp64, scores [B][N] fp64 or None (decide from the gate), out [B][d] fp32."""
        check(load().moe_decode_layer(self._h, layer, C.c_void_p(x_ptr), C.c_void_p(scores_ptr or 0) if scores_ptr else None,
                                      C.c_void_p(out_ptr), int(add_input), C.c_void_p(stream) if stream else None))

    def decode_record_timeline(self, enable: bool = True) -> None:
        """Start / stop recording the physical timeline (moe_decode_record_timeline)."""
        check(load().moe_decode_record_timeline(self._h, int(enable)))

    def decode_timeline_write(self, path: str) -> int:
        """Write the physical timeline recorded so far as JSONL (moe_decode_timeline_write)."""
        n = C.c_int64()
        check(load().moe_decode_timeline_write(self._h, str(path).encode(), C.byref(n)))
        return n.value

    def decode_tokens(self, acts, scores, hidden_out=None, on_device: bool = False) -> float:
        """acts [n][L][d], scores [n][L][N] host numpy arrays (or device pointers via on_device)."""
        ms = C.c_double()
        if on_device:
            a_ptr, s_ptr, n = acts, scores, hidden_out[1]
            check(load().moe_decode_tokens(self._h, C.cast(a_ptr, _capi._d), C.cast(s_ptr, _capi._d), n, 1,
                                           C.cast(hidden_out[0], _capi._f) if hidden_out[0] else None, C.byref(ms)))
            return ms.value
        acts, scores = _f64(acts), _f64(scores)
        out = None
        if hidden_out is not None:
            assert hidden_out.dtype == np.float32 and hidden_out.flags.c_contiguous
            out = _p(hidden_out, _capi._f)
        check(load().moe_decode_tokens(self._h, _p(acts, _capi._d), _p(scores, _capi._d), acts.shape[0], 0, out,
                                       C.byref(ms)))
        return ms.value

    def decode_end(self, cfg: SimConfig | None = None, tokens: int | None = None, timeline: bool = True) -> SimResult:
        m = _capi.MetricsC()
        st = _capi.DecodeStatsC()
        n = C.c_int64()
        T = tokens or 0
        lat = np.zeros(max(T, 1), dtype=np.int64)
        odl = np.zeros(self.spec.num_layers, dtype=np.int64)
        buf, cap = (_events_buf(self.spec, T, cfg, getattr(self, "_batch", 1)) if (timeline and cfg is not None and T)
                    else (None, 0))
        check(load().moe_decode_end(self._h, C.byref(m), _p(lat, _capi._i64) if T else None, _p(odl, _capi._i64),
                                    _evp(buf), cap, C.byref(n), C.byref(st)))
        return SimResult({k: getattr(m, k) for k, _ in _capi.MetricsC._fields_}, lat[:T], odl,
                         _events_np(buf, n.value) if buf is not None else None, n.value,
                         {k: getattr(st, k) for k, _ in _capi.DecodeStatsC._fields_})

    def decode_stats(self) -> dict:
        st = _capi.DecodeStatsC()
        check(load().moe_decode_stats_snapshot(self._h, C.byref(st)))
        return {k: getattr(st, k) for k, _ in _capi.DecodeStatsC._fields_}

    def expert_ffn(self, layer: int, expert: int, x) -> np.ndarray:
        """y = W2 (silu(W1 x) * (W3 x)) for one stored expert, through the decode path's kernels."""
        x = _f64(x)
        y = np.zeros(self.spec.hidden_dim, dtype=np.float32)
        check(load().moe_expert_ffn(self._h, layer, expert, _p(x, _capi._d), _p(y, _capi._f)))
        return y
