"""B200-native AdapMoE offloaded-MoE decode path (arXiv 2408.10284).

Hand-written sm_100a CUDA (K1 router + pre-gate, K2 batch-1 SwiGLU expert streaming, K3 grouped
tcgen05/TMEM SwiGLU for batched decode) behind the C ABI in ``include/adapmoe.h``, a C++ host engine
(tick-model policy engine, DP cache allocation, HBM slot pool, copy engine, artifact files), and
this thin Python mirror of the reference moesim API (``moesim``, ``io``, ``ep``).
"""
from ._capi import MoeError, load  # noqa: F401
from .moesim import (  # noqa: F401
    Engine,
    ModelSpec,
    PolicyFlags,
    SimConfig,
    SimResult,
    SynthConfig,
    Workload,
    build_cost_table,
    calibrate_threshold,
    dp_allocate,
    expected_cost,
    replay_policy,
    tile_pipeline_latency,
    uniform_allocation,
)

__all__ = [
    "Engine", "ModelSpec", "PolicyFlags", "SimConfig", "SimResult", "SynthConfig", "Workload", "MoeError",
    "build_cost_table", "calibrate_threshold", "dp_allocate", "expected_cost", "replay_policy",
    "tile_pipeline_latency", "uniform_allocation", "load",
]
