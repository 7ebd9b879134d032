"""Expert-parallel offloaded decode across GPUs (BASELINE config 5).

The reference has no parallelism; this is the B200 extension.  Layout:
  * shard r of G owns experts e with e % G == r in every layer (4 / 2 / 1 experts per GPU per layer
    at G = 2 / 4 / 8 for N = 8); its HBM slot pool holds only its own resident experts
    (sum_l min(t_l, N/G) slots plus staging) and its own host link moves only its own experts;
  * the router (K1) and the logical cache / transfer engine are replicated: every shard routes the
    same inputs and replays the same tick-model trace, so the event trace stays the reference's
    (global logical per-layer LRU with the DP capacities);
  * dispatch: in trace-replay decode every shard already holds the layer inputs (the reference never
    evolves a hidden state, inc/simulator.hpp:392), so no activations move;
  * combine: each shard forms its partial layer output  P_r = [r == 0] x + sum_{e owned} w_e E_e(x)
    (combine weights from the full selection); the layer output is
    P_0 + P_1 + ... + P_{G-1} summed in shard order — the same bits on every shard.  Default
    ("p2p"): the combine kernels store P_r straight into every shard's exchange region over peer
    memory (CUDA IPC, NVLink), a release flag per call publishes it and each shard reduces the slots
    on the device (kernels/ep_exchange.hpp); "allgather": one torch.distributed all_gather per call.
`torch.distributed` swaps the IPC handles / carries the all_gather (NCCL on B200s, gloo in tests).
"""
from __future__ import annotations

import numpy as np


def owned_experts(num_experts: int, world: int, rank: int) -> list[int]:
    """Experts of every layer owned by shard `rank` (e % world == rank)."""
    return [e for e in range(num_experts) if e % world == rank]


def balanced_owners(timeline, num_layers: int, num_experts: int, world: int) -> np.ndarray:
    """[L][N] shard table that balances the host-link traffic: the weight of (layer, expert) is its
    tile transfers in a calibration run's event timeline (simulate_trace / decode_end on a trace of
    the same model; activations break ties, spreading the FFN work too), assigned longest-first to
    the least-loaded shard (ties -> lowest (layer, expert), lowest rank).  Deterministic, so every
    shard computes the same table; the logical trace does not depend on it."""
    tl = np.asarray(timeline)
    w = np.zeros((num_layers, num_experts))
    if tl.size:
        kind, layer, expert = tl[:, 1], tl[:, 5], tl[:, 6]
        np.add.at(w, (layer[kind == 4], expert[kind == 4]), 1000.0)  # TileTransfer
        np.add.at(w, (layer[kind == 3], expert[kind == 3]), 1.0)     # TileCompute
    order = sorted(((-w[l, e], l, e) for l in range(num_layers) for e in range(num_experts)))
    load = [0.0] * world
    owner = np.zeros((num_layers, num_experts), dtype=np.int32)
    for negw, l, e in order:
        r = min(range(world), key=lambda g: (load[g], g))
        owner[l, e] = r
        load[r] += -negw
    return owner


def shard_resident_slots(capacities, num_experts: int, world: int, rank: int) -> int:
    """HBM slots shard `rank` needs for its resident experts: sum_l min(t_l, owned per layer)."""
    owned = len(owned_experts(num_experts, world, rank))
    return int(sum(min(int(c), owned) for c in capacities))


def combine_partials(partial, group=None):
    """Sum the shards' partial layer outputs in shard order (fixed), identical on every shard.

    `partial` is this shard's torch tensor (any shape; CUDA with NCCL, CPU with gloo)."""
    import torch
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized() or dist.get_world_size(group) == 1:
        return partial
    src = partial
    if partial.is_cuda and dist.get_backend(group) == "gloo":  # gloo exchanges through host memory
        src = partial.cpu()
    parts = [torch.empty_like(src) for _ in range(dist.get_world_size(group))]
    dist.all_gather(parts, src.contiguous(), group=group)
    out = parts[0].clone()
    for p in parts[1:]:
        out += p
    return out.to(partial.device)


class ExpertParallelDecoder:
    """One shard of an expert-parallel decode session on this process's GPU.

    decode(acts, scores) returns the full layer outputs (after the cross-shard combine), the same on
    every shard.  acts [n][B][L][d] (or [n][L][d] at batch 1) host numpy arrays."""

    def __init__(self, engine, caps, fisher, tau, cfg, seed: int, total_tokens: int, rank: int, world: int,
                 batch: int = 1, staging_slots: int = 0, group=None, exchange: str = "p2p",
                 max_tokens_per_call: int = 64, expert_owner=None):
        """exchange="p2p": the shards swap exchange regions (CUDA IPC handles) and the combine kernels
        store partials straight into peer memory (NVLink); "allgather": torch.distributed after each
        call."""
        import torch.distributed as dist
        self.engine, self.rank, self.world, self.batch, self.group = engine, rank, world, batch, group
        engine.decode_begin(caps, fisher, tau, cfg, seed, total_tokens, staging_slots, batch=batch, ep_rank=rank,
                            ep_world=world, expert_owner=expert_owner)
        self.p2p = exchange == "p2p" and world > 1
        if self.p2p:
            _, handle = engine.decode_ep_export(max_tokens_per_call)
            handles = [None] * world
            dist.all_gather_object(handles, handle, group=group)
            engine.decode_ep_connect(peer_ptrs=[0] * world, peer_ipc=handles)

    def decode(self, acts, scores):
        import torch
        spec = self.engine.spec
        n = acts.shape[0]
        shape = (n, self.batch, spec.num_layers, spec.hidden_dim) if self.batch > 1 else \
            (n, spec.num_layers, spec.hidden_dim)
        part = np.zeros(shape, dtype=np.float32)
        gpu_ms = self.engine.decode_tokens(acts, scores, part)
        if self.p2p:  # already summed on the device
            return part, gpu_ms
        t = torch.from_numpy(part)
        if torch.cuda.is_available():
            t = t.cuda()
        return combine_partials(t, self.group).cpu().numpy(), gpu_ms

    def end(self, cfg=None, tokens=None, timeline=True):
        return self.engine.decode_end(cfg, tokens, timeline)
