"""ctypes declarations for include/adapmoe.h (the C ABI of libadapmoe.so).

The library is built in-tree (``paper_2408_10284_b200/libadapmoe.so``) by
``__graft_entry__.build()`` / ``make -C paper_2408_10284_b200/csrc``.  There is no fallback: if the
library is missing, importing this module raises.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "libadapmoe.so")

MOE_OK = 0
MOE_E_USAGE = 1
MOE_E_IO = 2
MOE_E_FORMAT = 3
MOE_E_VALIDATION = 4
MOE_E_INFEASIBLE = 5
MOE_E_DEVICE = 6
MOE_E_INTERNAL = 7


class ModelSpecC(C.Structure):
    _fields_ = [("num_layers", C.c_int32), ("experts_per_layer", C.c_int32), ("top_k", C.c_int32),
                ("hidden_dim", C.c_int32)]


class SimConfigC(C.Structure):
    _fields_ = [("tile_count_per_expert", C.c_int32), ("tile_transfer_time", C.c_int64),
                ("tile_compute_time", C.c_int64), ("attention_compute_time", C.c_int64),
                ("gate_compute_time", C.c_int64), ("lookahead_depth", C.c_int32), ("adaptive_gating", C.c_int32),
                ("prefetch", C.c_int32), ("adaptive_cache", C.c_int32)]


class MetricsC(C.Structure):
    _fields_ = [("total_latency", C.c_int64), ("stall_time", C.c_int64), ("on_demand_loads", C.c_int64),
                ("cache_hits", C.c_int64), ("prefetch_hits", C.c_int64), ("single_expert_decisions", C.c_int64),
                ("experts_activated_total", C.c_int64)]


class EventC(C.Structure):
    _fields_ = [(n, C.c_int64) for n in ("stream", "kind", "start", "end", "token", "layer", "expert", "tile")]


class SynthConfigC(C.Structure):
    _fields_ = [("spec", ModelSpecC), ("tokens", C.c_int32), ("dirichlet_concentration", C.c_double),
                ("residual_drift", C.c_double), ("gate_seed", C.c_uint64), ("token_seed", C.c_uint64),
                ("shared_gates", C.c_int32), ("fisher_scales", C.POINTER(C.c_double)),
                ("drift_scales", C.POINTER(C.c_double))]


class CompareRowC(C.Structure):
    _fields_ = [("name", C.c_char * 24), ("adaptive_gating", C.c_int32), ("prefetch", C.c_int32),
                ("adaptive_cache", C.c_int32), ("metrics", MetricsC), ("speedup_vs_baseline", C.c_double)]


class DecodeOptsC(C.Structure):
    _fields_ = [("batch", C.c_int32), ("ep_rank", C.c_int32), ("ep_world", C.c_int32), ("free_running", C.c_int32),
                ("dirichlet_concentration", C.c_double), ("expert_owner", C.c_void_p)]


class RouteOutC(C.Structure):
    _fields_ = [("selected", C.c_void_p), ("count", C.c_void_p), ("single", C.c_void_p), ("perturbation", C.c_void_p)]


class DecodeStatsC(C.Structure):
    _fields_ = [("tokens", C.c_int64), ("kernels_launched", C.c_int64), ("ffn_launches", C.c_int64),
                ("tile_copies", C.c_int64), ("copy_bytes", C.c_int64), ("input_bytes", C.c_int64),
                ("ffn_bytes", C.c_int64), ("copy_busy_ms", C.c_double), ("ffn_ms", C.c_double),
                ("ffn_gate_up_ms", C.c_double), ("ffn_down_ms", C.c_double), ("ffn_gate_up_bytes", C.c_double),
                ("ffn_down_bytes", C.c_double), ("router_ms", C.c_double), ("stall_ms", C.c_double),
                ("router_exact_items", C.c_int64), ("host_sync_ms", C.c_double), ("host_step_ms", C.c_double), ("slots_total", C.c_int32), ("staging_high_water", C.c_int32),
                ("prefetch_copy_ms", C.c_double), ("prefetch_stall_ms", C.c_double),
                ("prefetch_tile_copies", C.c_int64), ("prefetch_used_copy_ms", C.c_double),
                ("router_launches", C.c_int64), ("spec_launches", C.c_int64), ("spec_hits", C.c_int64),
                ("record_decode_ms", C.c_double), ("record_decodes", C.c_int64), ("record_decode_bytes", C.c_double)]


_d = C.POINTER(C.c_double)
_f = C.POINTER(C.c_float)
_i32 = C.POINTER(C.c_int32)
_i64 = C.POINTER(C.c_int64)
_u16 = C.POINTER(C.c_uint16)
_spec = C.POINTER(ModelSpecC)
_cfg = C.POINTER(SimConfigC)
_eng = C.c_void_p

# name -> (restype, argtypes); every symbol declared in include/adapmoe.h
SIGNATURES = {
    "moe_last_error": (C.c_char_p, []),
    "moe_version": (C.c_char_p, []),
    "moe_calibrate_threshold": (C.c_int, [_spec, _d, C.c_int32, _d, C.c_double, _d, _d]),
    "moe_build_cost_table": (C.c_int, [_spec, _d, _d, _d]),
    "moe_dp_allocate": (C.c_int, [_spec, _d, C.c_int32, _i32, _d]),
    "moe_uniform_allocation": (C.c_int, [_spec, C.c_int32, _i32]),
    "moe_expected_cost": (C.c_int, [C.c_int32, C.c_int32, C.c_double, C.c_double, _d]),
    "moe_tile_pipeline_latency": (C.c_int, [C.c_int32, C.c_int64, C.c_int64, _i64]),
    "moe_replay_policy": (C.c_int, [_spec, C.c_int32, _i32, _cfg, C.c_uint64, _i32, _i32, _i32,
                                    C.POINTER(MetricsC), _i64, _i64, C.POINTER(EventC), C.c_int64, _i64]),
    "moe_engine_create": (C.c_int, [_spec, C.c_int32, C.POINTER(_eng)]),
    "moe_engine_destroy": (C.c_int, [_eng]),
    "moe_load_gates": (C.c_int, [_eng, _d, _d]),
    "moe_route_trace": (C.c_int, [_eng, _d, _d, C.c_int32, _d, C.c_double, _cfg, _i32, _i32, _d, _i32]),
    "moe_simulate_trace": (C.c_int, [_eng, _d, _d, C.c_int32, _d, _i32, C.c_double, _cfg, C.c_uint64,
                                     C.POINTER(MetricsC), _i64, _i64, C.POINTER(EventC), C.c_int64, _i64]),
    "moe_generate_trace": (C.c_int, [_eng, C.POINTER(SynthConfigC), _d, _d, _d, _i32, _d]),
    "moe_generate_profiles": (C.c_int, [_eng, _d, _d, C.c_int32, _d, C.c_double, _d, _d]),
    "moe_experts_init": (C.c_int, [_eng, C.c_int32, C.c_int32, C.c_uint64, C.c_int32]),
    "moe_expert_bytes": (C.c_int, [_eng, _i64]),
    "moe_expert_read": (C.c_int, [_eng, C.c_int32, C.c_int32, _u16]),
    "moe_expert_host_ptr": (C.c_int, [_eng, C.c_int32, C.c_int32, C.POINTER(C.c_void_p)]),
    "moe_experts_set_format": (C.c_int, [_eng, C.c_int32]),
    "moe_experts_format": (C.c_int, [_eng, C.POINTER(C.c_int32), C.POINTER(C.c_int64)]),
    "moe_expert_tile_record": (C.c_int, [_eng, C.c_int32, C.c_int32, C.c_int32, C.POINTER(C.c_void_p),
                                         C.POINTER(C.c_int64), C.POINTER(C.c_int32), C.POINTER(C.c_uint32),
                                         C.POINTER(C.c_int64), C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    "moe_copy_tiles": (C.c_int, [_eng, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_void_p, C.c_void_p,
                                 C.POINTER(C.c_void_p)]),
    "moe_expert_ffn_async": (C.c_int, [_eng, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, _d, C.c_int32,
                                       C.POINTER(C.c_void_p), C.c_void_p]),
    "moe_experts_alloc": (C.c_int, [_eng, C.c_int32, C.c_int32]),
    "moe_experts_init_shard": (C.c_int, [_eng, C.c_int32, C.c_int32, C.c_uint64, C.c_int32, _i32, C.c_int32]),
    "moe_experts_alloc_shard": (C.c_int, [_eng, C.c_int32, C.c_int32, _i32, C.c_int32]),
    "moe_experts_info": (C.c_int, [_eng, C.POINTER(C.c_int64), C.POINTER(C.c_int32), C.POINTER(C.c_int32)]),
    "moe_router_forward": (C.c_int, [_eng, C.c_int32, C.c_void_p, C.c_int32, C.c_void_p, C.c_double, _d, C.c_int32,
                                     C.c_int32, C.c_void_p, C.c_void_p]),
    "moe_expert_set": (C.c_int, [_eng, C.c_int32, C.c_int32, _u16, _u16, _u16]),
    "moe_trace_load": (C.c_int, [C.c_char_p, C.POINTER(C.c_void_p)]),
    "moe_trace_info": (C.c_int, [C.c_void_p, C.POINTER(ModelSpecC), _i32]),
    "moe_trace_read": (C.c_int, [C.c_void_p, _d, _d, _i32]),
    "moe_trace_validate": (C.c_int, [C.c_void_p, _i64, C.c_char_p, C.c_int64]),
    "moe_trace_free": (C.c_int, [C.c_void_p]),
    "moe_trace_save": (C.c_int, [C.c_char_p, C.POINTER(ModelSpecC), C.c_int32, _d, _d, _i32, C.c_int32]),
    "moe_gates_load": (C.c_int, [C.c_char_p, C.POINTER(ModelSpecC), _d, _d, _i32, _d, _i32, C.POINTER(C.c_uint64)]),
    "moe_gates_save": (C.c_int, [C.c_char_p, C.POINTER(ModelSpecC), _d, _d, C.c_double, C.c_int32, C.c_uint64]),
    "moe_profiles_load": (C.c_int, [C.c_char_p, C.POINTER(ModelSpecC), _d, _d, _d]),
    "moe_profiles_save": (C.c_int, [C.c_char_p, C.POINTER(ModelSpecC), _d, _d, _d, C.c_char_p]),
    "moe_threshold_load": (C.c_int, [C.c_char_p, _d, _d, _d]),
    "moe_threshold_save": (C.c_int, [C.c_char_p, C.c_double, C.c_double, C.c_double]),
    "moe_allocation_load": (C.c_int, [C.c_char_p, _i32, _i32, _i32, _d, C.c_char_p]),
    "moe_allocation_save": (C.c_int, [C.c_char_p, C.c_int32, C.c_int32, _i32, C.c_double, C.c_char_p]),
    "moe_cost_table_load": (C.c_int, [C.c_char_p, _i32, _i32, _d]),
    "moe_cost_table_save": (C.c_int, [C.c_char_p, C.c_int32, C.c_int32, _d]),
    "moe_compare_policies": (C.c_int, [_eng, _d, _d, C.c_int32, _d, _d, _d, C.c_double, _cfg, C.c_int32, C.c_uint64,
                                       C.POINTER(CompareRowC), _i32, _i64, _i64]),
    "moe_train_first_gate": (C.c_int, [_eng, _d, _d, C.c_int32, C.c_double, C.c_int32, C.c_uint64, _d]),
    "moe_decode_begin": (C.c_int, [_eng, _i32, C.c_int32, _d, C.c_double, _cfg, C.c_uint64, C.c_int32]),
    "moe_decode_begin_ex": (C.c_int, [_eng, _i32, C.c_int32, _d, C.c_double, _cfg, C.c_uint64, C.c_int32,
                                      C.POINTER(DecodeOptsC)]),
    "moe_decode_ep_export": (C.c_int, [_eng, C.c_int32, C.POINTER(C.c_uint64), C.c_char_p]),
    "moe_decode_ep_connect": (C.c_int, [_eng, C.POINTER(C.c_uint64), C.c_char_p]),
    "moe_decode_tokens": (C.c_int, [_eng, _d, _d, C.c_int32, C.c_int32, _f, _d]),
    "moe_decode_end": (C.c_int, [_eng, C.POINTER(MetricsC), _i64, _i64, C.POINTER(EventC), C.c_int64, _i64,
                                 C.POINTER(DecodeStatsC)]),
    "moe_expert_ffn": (C.c_int, [_eng, C.c_int32, C.c_int32, _d, _f]),
    "moe_decode_stats_snapshot": (C.c_int, [_eng, C.POINTER(DecodeStatsC)]),
    "moe_decode_layer": (C.c_int, [_eng, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p]),
    "moe_decode_record_timeline": (C.c_int, [_eng, C.c_int32]),
    "moe_decode_timeline_write": (C.c_int, [_eng, C.c_char_p, C.POINTER(C.c_int64)]),
}


class MoeError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


_lib = None


def load():
    """Load libadapmoe.so; raises if it has not been built (no CPU fallback exists)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'`")
        lib = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def check(rc: int) -> None:
    if rc != MOE_OK:
        raise MoeError(rc, load().moe_last_error().decode())
