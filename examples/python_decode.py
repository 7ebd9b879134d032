"""Offloaded-MoE decode with real (checkpoint-layout) expert weights, through the Python mirror of
the C ABI.  A small random model stands in for a checkpoint: replace `checkpoint()` with tensors read
from safetensors (gate_proj / up_proj / down_proj per expert, the router weight per layer).

  python examples/python_decode.py            # needs a B200 (sm_100a)

Steps: size the HBM expert cache with the reference's DP (profiles from a short calibration trace),
upload the gates, hand over the expert weights, then decode free-running (every layer routes on
the previous layer's output) and route one layer on device rows with the stream-level router.
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2408_10284_b200 as P  # noqa: E402

L, N, K, D, F, TILES = 4, 8, 2, 256, 512, 2


def to_bf16_bits(a):
    u = np.ascontiguousarray(a, dtype=np.float32).view(np.uint32)
    return ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)


def checkpoint(rng):
    """router [L][d][N] (fp64, the reference's GateMatrix layout) and per-expert gate/up [F][d],
    down [d][F] (bf16)."""
    router = rng.standard_normal((L, D, N)) / np.sqrt(D)
    experts = {(l, e): (to_bf16_bits(rng.standard_normal((F, D)) / np.sqrt(D)),
                        to_bf16_bits(rng.standard_normal((F, D)) / np.sqrt(D)),
                        to_bf16_bits(rng.standard_normal((D, F)) / np.sqrt(F)))
               for l in range(L) for e in range(N)}
    return router, experts


def main():
    rng = np.random.default_rng(0)
    router, experts = checkpoint(rng)
    spec = P.ModelSpec(L, N, K, D)
    with P.Engine(spec) as eng:
        # calibration: a synthetic trace with this model's router gives scores to calibrate tau and to
        # profile alpha / beta for the DP (a real deployment records a trace of the model instead)
        trace = eng.generate_trace(P.SynthConfig(spec, 32, 0.6, 0.18, 99, 5000))
        eng.load_gates(router)
        tau, realized = P.calibrate_threshold(spec, trace.scores, trace.fisher, 0.24)
        alpha, beta = eng.generate_profiles(trace.acts, trace.scores, trace.fisher, tau)
        caps, expected_loads = P.dp_allocate(spec, P.build_cost_table(spec, alpha, beta), 12)
        print(f"tau {tau:.4g} (single-expert ratio {realized:.2f}); cache capacities {[int(c) for c in caps]}; "
              f"expected on-demand loads / token {expected_loads:.2f}")

        # lossless Huffman-coded exponents in the pinned store: ~2/3 of the bytes over the host link,
        # decoded on the GPU as tiles land (outputs identical to store_format="bf16")
        eng.experts_alloc(F, TILES, store_format="xbh")
        for (l, e), (w1, w3, w2) in experts.items():
            eng.expert_set(l, e, w1, w3, w2)
        fmt, link_bytes = eng.experts_format()
        print(f"expert store: {fmt}, {link_bytes / (L * N * 3 * F * D * 2):.2f} of the bf16 bytes")

        cfg = P.SimConfig(tile_count_per_expert=TILES)
        T = 8
        x0 = rng.standard_normal((T, L, D))  # layer-0 inputs; layers > 0 come from the decode itself
        eng.decode_begin(caps, trace.fisher, tau, cfg, 0, T, free_running=True)
        hidden = np.zeros((T, L, D), dtype=np.float32)
        eng.decode_tokens(x0, np.zeros((T, L, N)), hidden)
        res = eng.decode_end(cfg, T)
        m = res.metrics
        print(f"decoded {T} tokens: {m['experts_activated_total']} experts activated, {m['cache_hits']} cache hits, "
              f"{m['prefetch_hits']} prefetch hits, {m['on_demand_loads']} on-demand loads; "
              f"|h| of the last layer {np.abs(hidden[-1, -1]).max():.3f}")

        import torch
        x = torch.from_numpy(np.ascontiguousarray(x0[:, 1])).cuda()
        sel, cnt, single, pert = eng.router_forward(1, x, trace.fisher, tau, lookahead=2)
        torch.cuda.synchronize()
        print("layer-1 routing of the 8 rows on the device:", sel[:, 0].cpu().tolist())
        print("OK")


if __name__ == "__main__":
    main()
