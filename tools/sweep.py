#!/usr/bin/env python
"""BASELINE config 3: Mixtral-8x7B-shape batch-1 decode sweeping the HBM expert-cache budget
(32..256 experts) and the gating threshold (tau calibrated to a target single-expert ratio).

Per point: reference pipeline on the GPU engine (generate -> calibrate(target) -> profile ->
DP allocate(budget)), then the physical offloaded decode (one shared 90 GB pinned expert store).
Reports on-demand loads/token, prefetch-hit and cache-hit rates, prefetch accuracy (mean beta),
tok/s (CUDA events), host-link utilisation and K2 bandwidth; cross-checks the logical on-demand
count against the unmodified reference (oracle/_ref, where built).  One JSON line per point.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--budgets", default="32,64,96,128,160,192,224,256")
    ap.add_argument("--targets", default="0,0.12,0.24,0.36,0.48")
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--steps", type=int, default=4)
    ap.add_argument("--out", default="gpurun_out/sweep_r2.jsonl")
    ap.add_argument("--store-format", default="xbh", choices=["bf16", "xb12", "xbh"])
    args = ap.parse_args()

    import numpy as np
    import torch

    import paper_2408_10284_b200 as P
    from paper_2408_10284_b200 import workloads as W
    import bench

    wl0 = W.mixtral_8x7b(tokens=64)
    spec = P.ModelSpec(wl0.layers, wl0.experts, wl0.top_k, wl0.hidden)
    eng = P.Engine(spec, 0)
    trace = eng.generate_trace(P.SynthConfig(spec, wl0.tokens, wl0.concentration, wl0.drift, wl0.gate_seed,
                                             wl0.token_seed, False, wl0.fisher_scales, wl0.drift_scales))
    t0 = time.time()
    eng.experts_init(wl0.ffn, wl0.tiles, seed=1234, store_format=args.store_format)
    store_s = time.time() - t0
    W_, K = args.warmup, args.steps
    n = W_ + K
    d_acts = torch.from_numpy(np.ascontiguousarray(trace.acts[:n])).cuda()
    d_scores = torch.from_numpy(np.ascontiguousarray(trace.scores[:n])).cuda()
    d_hidden = torch.zeros((n, wl0.layers, wl0.hidden), dtype=torch.float32, device="cuda")
    cfg = P.SimConfig()
    os.makedirs(os.path.dirname(args.out) or ".", exist_ok=True)
    out = open(args.out, "w")
    for target in [float(v) for v in args.targets.split(",")]:
        tau, realized = P.calibrate_threshold(spec, trace.scores, trace.fisher, target)
        alpha, beta = eng.generate_profiles(trace.acts, trace.scores, trace.fisher, tau)
        table = P.build_cost_table(spec, alpha, beta)
        for budget in [int(v) for v in args.budgets.split(",")]:
            caps, exp_loads = P.dp_allocate(spec, table, budget)
            eng.decode_begin(caps, trace.fisher, tau, cfg, 0, wl0.tokens)
            step = wl0.layers * wl0.hidden

            def call(a, b):
                return eng.decode_tokens(d_acts.data_ptr() + a * step * 8,
                                         d_scores.data_ptr() + a * wl0.layers * wl0.experts * 8,
                                         (d_hidden.data_ptr() + a * step * 4, b - a), on_device=True)
            call(0, W_)
            s0 = eng.decode_stats()
            torch.cuda.synchronize()
            ms = call(W_, n)
            s1 = eng.decode_stats()
            res = eng.decode_end(cfg, wl0.tokens)
            tl = res.timeline
            tok = tl[:, 4]
            win = (tok >= W_) & (tok < n)
            od = int(((tl[:, 1] == 3) & (tl[:, 7] == 0) & win).sum())
            m = res.metrics
            dd = {k: s1[k] - s0[k] for k in s0}
            line = {"store_format": args.store_format, "target_single_ratio": target, "tau": tau, "realized_single_ratio": realized, "budget": budget,
                    "capacities": [int(c) for c in caps], "dp_expected_loads_per_token": exp_loads,
                    "mean_beta": float(np.mean(beta)), "mean_alpha": float(np.mean(alpha)),
                    "tok_s": K / (ms * 1e-3), "ms_per_token": ms / K,
                    "on_demand_loads_per_token": od / K,
                    "trace_on_demand": m["on_demand_loads"], "trace_cache_hits": m["cache_hits"],
                    "trace_prefetch_hits": m["prefetch_hits"], "trace_activated": m["experts_activated_total"],
                    "prefetch_hit_rate": m["prefetch_hits"] / max(1, m["experts_activated_total"]),
                    "link_busy_frac": dd["copy_busy_ms"] / ms if ms else None,
                    "copy_hidden_frac": 1.0 - dd["stall_ms"] / dd["copy_busy_ms"] if dd["copy_busy_ms"] > 0 else None,
                    "prefetch_copy_ms": dd["prefetch_copy_ms"], "prefetch_stall_ms": dd["prefetch_stall_ms"],
                    "prefetch_used_copy_ms": dd["prefetch_used_copy_ms"],
                    "prefetch_hidden_frac": (1.0 - dd["prefetch_stall_ms"] / dd["prefetch_used_copy_ms"]
                                             if dd["prefetch_used_copy_ms"] > 0 else None),
                    "prefetch_wasted_frac": (1.0 - dd["prefetch_used_copy_ms"] / dd["prefetch_copy_ms"]
                                             if dd["prefetch_copy_ms"] > 0 else None),
                    "ffn_ms_per_token": dd["ffn_ms"] / K, "stall_ms_per_token": dd["stall_ms"] / K,
                    "k2_gbs": (dd["ffn_gate_up_bytes"] + dd["ffn_down_bytes"]) / max(1e-9, dd["ffn_ms"] * 1e-3) / 1e9}
            r = bench.run_reference_driver(W.mixtral_8x7b(tokens=64, budget=budget, target_single_ratio=target), n, 1)
            if r is not None:
                # the whole SimMetrics struct and the event timeline's FNV-1a hash vs the unmodified
                # reference over the same tokens (as bench.py's parity object)
                rm = r["metrics"]
                ours = dict(m)
                ours["on_demand_loads_per_layer"] = [int(v) for v in res.on_demand_loads_per_layer]
                ours["latency_per_token"] = [int(v) for v in res.latency_per_token[:n]]
                line["reference_on_demand"] = r["on_demand_loads"]
                line["metrics_differ"] = sorted(k for k in rm if rm[k] != ours.get(k))
                line["parity"] = (not line["metrics_differ"] and r.get("hash_timeline") == bench.fnv1a_i64(res.timeline))
            out.write(json.dumps(line) + "\n")
            out.flush()
            print(json.dumps({k: line[k] for k in ("target_single_ratio", "budget", "tok_s", "on_demand_loads_per_token",
                                                   "prefetch_hit_rate", "link_busy_frac", "prefetch_hidden_frac", "k2_gbs",
                                                   "parity")
                              if k in line}))
    print(json.dumps({"expert_store_s": store_s, "store_format": args.store_format}))


if __name__ == "__main__":
    main()
