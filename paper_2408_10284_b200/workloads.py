"""BASELINE.json workloads as concrete synthetic configurations.

Generator settings follow the reference demo config (proj/configs/demo8.json: concentration 0.6,
drift 0.18, gate_seed 99, token_seed 5000).  Builder choices are marked.  The simulation ticks are
the reference CLI defaults (proj/tools/moesim_main.cpp:259-267: tiles 4, transfer 2, compute 1,
attention 8, gate 1, lookahead 2, seed 0).
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

DEMO8_FISHER = [2.0, 1.6, 1.2, 0.9, 0.7, 0.5, 0.35, 0.25]   # proj/configs/demo8.json:10
DEMO8_DRIFT = [1.8, 1.5, 1.2, 1.0, 0.8, 0.6, 0.45, 0.35]    # proj/configs/demo8.json:11


def interp_scales(values, layers: int) -> list[float]:
    """Builder choice: stretch demo8's 8 per-layer scales linearly over `layers` layers."""
    if layers == len(values):
        return list(values)
    xs = np.linspace(0.0, len(values) - 1.0, layers)
    return [float(v) for v in np.interp(xs, np.arange(len(values)), values)]


@dataclass
class Workload:
    name: str
    layers: int
    experts: int
    top_k: int
    hidden: int
    tokens: int
    ffn: int = 0                      # expert FFN width (0 = no FFN, policy-only)
    concentration: float = 0.6
    drift: float = 0.18
    gate_seed: int = 99
    token_seed: int = 5000
    fisher_scales: list | None = None
    drift_scales: list | None = None
    target_single_ratio: float = 0.24
    train_first_gate: bool = True
    train_steps: int = 500
    train_lr: float = 0.1
    train_seed: int = 0
    budget: int = 16
    # SimConfig (CLI defaults)
    tiles: int = 4
    tile_transfer: int = 2
    tile_compute: int = 1
    attention: int = 8
    gate_time: int = 1
    lookahead: int = 2
    gating: bool = True
    prefetch: bool = True
    seed: int = 0
    extra: dict = field(default_factory=dict)

    def ref_args(self) -> dict:
        """Arguments for oracle/_ref/moesim_ref (test infrastructure)."""
        a = dict(layers=self.layers, experts=self.experts, top_k=self.top_k, hidden=self.hidden, tokens=self.tokens,
                 concentration=repr(self.concentration), drift=repr(self.drift), gate_seed=self.gate_seed,
                 token_seed=self.token_seed, target=repr(self.target_single_ratio),
                 train_gate=int(self.train_first_gate), train_steps=self.train_steps, train_lr=repr(self.train_lr),
                 train_seed=self.train_seed, budget=self.budget, tiles=self.tiles, tile_transfer=self.tile_transfer,
                 tile_compute=self.tile_compute, attention=self.attention, gate_time=self.gate_time,
                 lookahead=self.lookahead, gating=int(self.gating), prefetch=int(self.prefetch), seed=self.seed)
        if self.fisher_scales is not None:
            a["fisher_scales"] = ",".join(repr(float(v)) for v in self.fisher_scales)
        if self.drift_scales is not None:
            a["drift_scales"] = ",".join(repr(float(v)) for v in self.drift_scales)
        a.update(self.extra)
        return a


def tiny(**kw) -> Workload:
    """BASELINE config 1: tiny Mixtral-style MoE {4, 8, 2, 256}; builder-chosen scales = every
    other demo8 entry; ffn 896 = 3.5 d (Mixtral's ratio)."""
    base = dict(name="tiny", layers=4, experts=8, top_k=2, hidden=256, tokens=64, ffn=896,
                fisher_scales=[2.0, 1.2, 0.7, 0.35], drift_scales=[1.8, 1.2, 0.8, 0.45], budget=16)
    base.update(kw)
    return Workload(**base)


def mixtral_8x7b(tokens: int = 64, budget: int = 64, **kw) -> Workload:
    """BASELINE config 2: Mixtral-8x7B shape {32, 8, 2, 4096}, ffn 14336, bf16, budget 64 of 256.
    No trained first-layer gate (SURVEY App. B anchor); demo8 scales stretched over 32 layers."""
    base = dict(name="mixtral-8x7b", layers=32, experts=8, top_k=2, hidden=4096, tokens=tokens, ffn=14336,
                fisher_scales=interp_scales(DEMO8_FISHER, 32), drift_scales=interp_scales(DEMO8_DRIFT, 32),
                budget=budget, train_first_gate=False)
    base.update(kw)
    return Workload(**base)


def mixtral_8x22b(tokens: int = 64, budget: int = 112, **kw) -> Workload:
    """BASELINE config 5 shape {56, 8, 2, 6144}, ffn 16384 (public Mixtral-8x22B value)."""
    base = dict(name="mixtral-8x22b", layers=56, experts=8, top_k=2, hidden=6144, tokens=tokens, ffn=16384,
                fisher_scales=interp_scales(DEMO8_FISHER, 56), drift_scales=interp_scales(DEMO8_DRIFT, 56),
                budget=budget, train_first_gate=False)
    base.update(kw)
    return Workload(**base)


def demo8(tokens: int = 2000, budget: int = 32, train_steps: int = 100, **kw) -> Workload:
    """proj/configs/demo8.json."""
    base = dict(name="demo8", layers=8, experts=8, top_k=2, hidden=16, tokens=tokens, fisher_scales=DEMO8_FISHER,
                drift_scales=DEMO8_DRIFT, budget=budget, train_steps=train_steps)
    base.update(kw)
    return Workload(**base)
