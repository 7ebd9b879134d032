"""Expert parallelism (BASELINE config 5): shard r of G owns experts e % G == r.

  * [cpu] ownership partitions every layer's experts; per-shard slot pools cover the DP capacities;
  * [cpu, gloo world 2] the shard partials (computed here by the fp64 oracle) combined by
    ep.combine_partials equal the full MoE layer output and are bit-identical on both shards;
  * [gpu] shards 0 and 1 of a world-2 session run one after the other on one B200 (the driver's GPU
    tier has one GPU): each replays the reference trace bit-exactly, and their partials summed in
    shard order match the single-GPU decode within 1e-5 relative (only the fp32 summation order
    differs), for batch 1 and batch 4.
"""
import os
import socket

import numpy as np
import pytest

from conftest import load_golden
from helpers import oracle_inputs, sim_config, sim_kwargs
from oracle import oracle as O
from paper_2408_10284_b200 import ep


@pytest.mark.parametrize("N,G", [(8, 1), (8, 2), (8, 4), (8, 8), (6, 4)])
def test_ownership_partitions_experts(N, G):
    shards = [ep.owned_experts(N, G, r) for r in range(G)]
    assert sorted(sum(shards, [])) == list(range(N))
    caps = [N, 3, 0, 1, 2]
    slots = [ep.shard_resident_slots(caps, N, G, r) for r in range(G)]
    assert sum(slots) >= sum(caps)  # every resident expert has a home on its owner
    assert all(s <= sum(min(c, len(sh)) for c in caps) for s, sh in zip(slots, shards))


def _partials_oracle(w, decisions, t, l, ffn, tiles, seed, world, rank):
    sel = [int(e) for e in decisions[t, l] if e >= 0]
    sc = w.scores[t, l]
    denom = sum(sc[e] for e in sel)
    x32 = w.acts[t, l].astype(np.float32).astype(np.float64)
    acc = x32.copy() if rank == 0 else np.zeros(w.D)
    for e in sel:
        if e % world != rank:
            continue
        wgt = 1.0 if len(sel) == 1 else sc[e] / denom
        acc += wgt * O.swiglu(O.expert_init(seed, l, e, w.D, ffn, tiles), w.D, ffn, tiles, x32.astype(np.float32))
    return acc


def _gloo_worker(rank, world, port, out_dir):
    import torch
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = load_golden("tiny")
        w, fg = oracle_inputs(g)
        sim = O.simulate(w, g["sim_capacities"], g["tau"], first_gate=fg, **sim_kwargs(g))
        pts = [(0, 0), (3, 2), (9, 3)]
        part = np.stack([_partials_oracle(w, sim.decisions, t, l, 896, 4, 5, world, rank) for t, l in pts])
        full = ep.combine_partials(torch.from_numpy(part)).numpy()
        np.save(os.path.join(out_dir, f"ep_{rank}.npy"), full)
    finally:
        dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_combine_partials_gloo_world2(tmp_path):
    import torch.multiprocessing as mp
    mp.spawn(_gloo_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)
    r0, r1 = np.load(tmp_path / "ep_0.npy"), np.load(tmp_path / "ep_1.npy")
    assert np.array_equal(r0, r1)  # same bits on every shard
    g = load_golden("tiny")
    w, fg = oracle_inputs(g)
    sim = O.simulate(w, g["sim_capacities"], g["tau"], first_gate=fg, **sim_kwargs(g))
    for i, (t, l) in enumerate([(0, 0), (3, 2), (9, 3)]):
        full = _partials_oracle(w, sim.decisions, t, l, 896, 4, 5, 1, 0)
        assert np.abs(r0[i] - full).max() <= 1e-12 * np.abs(full).max()


@pytest.mark.gpu
@pytest.mark.parametrize("batch", [1, 4])
def test_ep_shards_match_single_gpu(batch):
    import paper_2408_10284_b200 as P
    g = load_golden("tiny")
    w0, fg = oracle_inputs(g)
    cfg = sim_config(g)
    caps, tau, T = g["sim_capacities"], g["tau"], 12
    ws = [w0] + [O.generate_trace(w0.L, w0.N, w0.K, w0.D, T, 0.6, 0.18, 99, 6000 + b, False,
                                  [2.0, 1.2, 0.7, 0.35], [1.8, 1.2, 0.8, 0.45]) for b in range(1, batch)]
    if batch == 1:
        acts, scores, shape = w0.acts[:T], w0.scores[:T], (T, w0.L, w0.D)
    else:
        acts = np.ascontiguousarray(np.stack([w.acts[:T] for w in ws], axis=1))
        scores = np.ascontiguousarray(np.stack([w.scores[:T] for w in ws], axis=1))
        shape = (T, batch, w0.L, w0.D)
    ffn = 1024  # (ffn / tiles) % 64 == 0 for the grouped path
    outs, results = [], []
    for rank, world in [(0, 1), (0, 2), (1, 2)]:
        with P.Engine(P.ModelSpec(w0.L, w0.N, w0.K, w0.D)) as eng:
            eng.load_gates(w0.gates, fg)
            eng.experts_init(ffn, cfg.tile_count_per_expert, seed=5)
            eng.decode_begin(caps, w0.fisher, tau, cfg, 0, T, batch=batch, ep_rank=rank, ep_world=world)
            h = np.zeros(shape, dtype=np.float32)
            eng.decode_tokens(acts, scores, h)
            results.append(eng.decode_end(cfg, T))
            outs.append(h)
    for r in results[1:]:
        assert r.metrics == results[0].metrics
        assert np.array_equal(r.timeline, results[0].timeline)
    if batch == 1:
        ref = O.simulate(w0, caps, tau, first_gate=fg, T=T, **sim_kwargs(g))
        assert results[0].metrics == ref.metrics
    full = outs[0].astype(np.float64)
    sharded = outs[1].astype(np.float64) + outs[2].astype(np.float64)
    x = (acts.astype(np.float32).astype(np.float64))
    moe = full - x
    assert np.abs(sharded - full).max() <= 1e-5 * np.abs(moe).max()
    # each shard only moved / computed its own experts
    b0, b1 = results[1].stats["ffn_bytes"], results[2].stats["ffn_bytes"]
    assert b0 + b1 == results[0].stats["ffn_bytes"]


def _p2p_inputs(batch):
    g = load_golden("tiny")
    w0, fg = oracle_inputs(g)
    T = 12
    ws = [w0] + [O.generate_trace(w0.L, w0.N, w0.K, w0.D, T, 0.6, 0.18, 99, 6000 + b, False,
                                  [2.0, 1.2, 0.7, 0.35], [1.8, 1.2, 0.8, 0.45]) for b in range(1, batch)]
    if batch == 1:
        acts, scores, shape = w0.acts[:T], w0.scores[:T], (T, w0.L, w0.D)
    else:
        acts = np.ascontiguousarray(np.stack([w.acts[:T] for w in ws], axis=1))
        scores = np.ascontiguousarray(np.stack([w.scores[:T] for w in ws], axis=1))
        shape = (T, batch, w0.L, w0.D)
    return g, w0, fg, acts, scores, shape, T


_P2P_CALLS = [0, 5, 6, 12]


def _p2p_decode(rank, world, batch, connect_fn=None, free_running=False):
    import paper_2408_10284_b200 as P
    g, w0, fg, acts, scores, shape, T = _p2p_inputs(batch)
    cfg = sim_config(g)
    eng = P.Engine(P.ModelSpec(w0.L, w0.N, w0.K, w0.D))
    eng.load_gates(w0.gates, fg)
    eng.experts_init(1024, cfg.tile_count_per_expert, seed=5)
    eng.decode_begin(g["sim_capacities"], w0.fisher, g["tau"], cfg, 0, T, batch=batch, ep_rank=rank,
                     ep_world=world, free_running=free_running, concentration=0.6)
    if connect_fn:
        connect_fn(eng)
    out = np.zeros(shape, dtype=np.float32)
    for a, b in zip(_P2P_CALLS, _P2P_CALLS[1:]):
        eng.decode_tokens(acts[a:b], scores[a:b], out[a:b])
    res = eng.decode_end(cfg, T)
    eng.close()
    return out, res


def _p2p_worker(rank, world, port, batch, out_dir, free_running=False):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        def connect(eng):
            ptr, handle = eng.decode_ep_export(max(b - a for a, b in zip(_P2P_CALLS, _P2P_CALLS[1:])))
            handles = [None] * world
            dist.all_gather_object(handles, handle)
            eng.decode_ep_connect(peer_ptrs=[0] * world, peer_ipc=handles)  # other processes: IPC handles

        out, res = _p2p_decode(rank, world, batch, connect, free_running)
        np.save(os.path.join(out_dir, f"p2p_{rank}.npy"), out)
        np.save(os.path.join(out_dir, f"p2p_metrics_{rank}.npy"), np.array(list(res.metrics.values())))
        np.save(os.path.join(out_dir, f"p2p_timeline_{rank}.npy"), res.timeline)
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("batch", [1, 4])
def test_ep_p2p_exchange_two_processes(batch, tmp_path):
    """The device-side exchange through CUDA IPC: two shard processes (sharing this GPU; on a node
    each would own a GPU and the stores would cross NVLink) store their partials into each other's
    exchange regions from the combine epilogue, signal with system-scope release flags and reduce in
    shard order.  Both return identical full outputs equal to the single-GPU decode, over several
    calls (slots double-buffered by call parity)."""
    import torch.multiprocessing as mp
    full, ref = _p2p_decode(0, 1, batch)
    mp.spawn(_p2p_worker, args=(2, _free_port(), batch, str(tmp_path)), nprocs=2, join=True)
    o0, o1 = np.load(tmp_path / "p2p_0.npy"), np.load(tmp_path / "p2p_1.npy")
    assert np.array_equal(o0, o1)  # same bits on every shard
    for r in range(2):
        assert np.load(tmp_path / f"p2p_metrics_{r}.npy").tolist() == list(ref.metrics.values())
    _, _, _, acts, _, _, _ = _p2p_inputs(batch)
    moe = full.astype(np.float64) - acts.astype(np.float32).astype(np.float64)
    assert np.abs(o0.astype(np.float64) - full).max() <= 1e-5 * np.abs(moe).max()


def test_balanced_owners_balances_transfers():
    """LPT placement by a timeline's transfers: every (layer, expert) gets one shard, the busiest
    shard carries at most the lightest plus the heaviest single item, and the table is deterministic."""
    rng = np.random.default_rng(3)
    L, N, G = 6, 8, 4
    rows = []
    for l in range(L):
        for e in range(N):
            for _ in range(int(rng.integers(0, 9))):
                rows.append([1, 4, 0, 1, 0, l, e, 0])  # TileTransfer
            rows.append([0, 3, 0, 1, 0, l, e, 0])      # TileCompute
    tl = np.array(rows, dtype=np.int64)
    own = ep.balanced_owners(tl, L, N, G)
    assert own.shape == (L, N) and own.min() >= 0 and own.max() < G
    w = np.zeros((L, N))
    np.add.at(w, (tl[tl[:, 1] == 4, 5], tl[tl[:, 1] == 4, 6]), 1.0)
    load = [w[own == g].sum() for g in range(G)]
    assert max(load) - min(load) <= w.max()
    assert np.array_equal(own, ep.balanced_owners(tl, L, N, G))
    # modulo placement of the same weights is no better balanced
    mod = np.array([[e % G for e in range(N)] for _ in range(L)])
    assert max(load) <= max(w[mod == g].sum() for g in range(G))


@pytest.mark.gpu
def test_ep_custom_owner_table():
    """A non-modulo owner table (ep.balanced_owners of a calibration run): shards keep the reference
    trace bit for bit, each moves / computes only its own (layer, expert)s, and the partials sum to
    the single-GPU decode."""
    import paper_2408_10284_b200 as P
    g = load_golden("tiny")
    w0, fg = oracle_inputs(g)
    cfg = sim_config(g)
    caps, tau, T = g["sim_capacities"], g["tau"], 12
    ffn = 1024
    with P.Engine(P.ModelSpec(w0.L, w0.N, w0.K, w0.D)) as eng:
        eng.load_gates(w0.gates, fg)
        calib = eng.simulate_trace(w0.acts[T:], w0.scores[T:], w0.fisher, caps, tau, cfg, 0)
    owners = ep.balanced_owners(calib.timeline, w0.L, w0.N, 2)
    assert not np.array_equal(owners, np.array([[e % 2 for e in range(w0.N)]] * w0.L))
    outs, results = [], []
    for rank, world in [(0, 1), (0, 2), (1, 2)]:
        with P.Engine(P.ModelSpec(w0.L, w0.N, w0.K, w0.D)) as eng:
            eng.load_gates(w0.gates, fg)
            eng.experts_init(ffn, cfg.tile_count_per_expert, seed=5)
            eng.decode_begin(caps, w0.fisher, tau, cfg, 0, T, ep_rank=rank, ep_world=world,
                             expert_owner=owners if world > 1 else None)
            h = np.zeros((T, w0.L, w0.D), dtype=np.float32)
            eng.decode_tokens(w0.acts[:T], w0.scores[:T], h)
            results.append(eng.decode_end(cfg, T))
            outs.append(h)
    for r in results[1:]:
        assert r.metrics == results[0].metrics and np.array_equal(r.timeline, results[0].timeline)
    assert results[1].stats["ffn_bytes"] + results[2].stats["ffn_bytes"] == results[0].stats["ffn_bytes"]
    full = outs[0].astype(np.float64)
    moe = full - w0.acts[:T].astype(np.float32).astype(np.float64)
    assert np.abs(outs[1].astype(np.float64) + outs[2].astype(np.float64) - full).max() <= 1e-5 * np.abs(moe).max()


@pytest.mark.gpu
@pytest.mark.parametrize("batch", [1, 4])
def test_ep_p2p_free_running_two_processes(batch, tmp_path):
    """Free-running decode across two shard processes: every layer's partial outputs are exchanged
    over peer memory and summed before the next layer routes on them (one exchange step per layer).
    Both shards hold the same bits, replay the single-GPU free-running trace, and their outputs match
    it within the summation-order / bf16 tolerance."""
    import torch.multiprocessing as mp
    full, ref = _p2p_decode(0, 1, batch, free_running=True)
    mp.spawn(_p2p_worker, args=(2, _free_port(), batch, str(tmp_path), True), nprocs=2, join=True)
    o0, o1 = np.load(tmp_path / "p2p_0.npy"), np.load(tmp_path / "p2p_1.npy")
    assert np.array_equal(o0, o1)
    for r in range(2):
        assert np.load(tmp_path / f"p2p_metrics_{r}.npy").tolist() == list(ref.metrics.values())
        assert np.array_equal(np.load(tmp_path / f"p2p_timeline_{r}.npy"), ref.timeline)
    tol = 1e-4 if batch == 1 else 2e-2
    scale = np.abs(full).max()
    assert np.abs(o0.astype(np.float64) - full.astype(np.float64)).max() <= tol * scale


@pytest.mark.gpu
def test_free_running_ep_requires_exchange():
    import paper_2408_10284_b200 as P
    g, w0, fg, acts, scores, shape, T = _p2p_inputs(1)
    cfg = sim_config(g)
    with P.Engine(P.ModelSpec(w0.L, w0.N, w0.K, w0.D)) as eng:
        eng.load_gates(w0.gates, fg)
        eng.experts_init(1024, cfg.tile_count_per_expert, seed=5)
        eng.decode_begin(g["sim_capacities"], w0.fisher, g["tau"], cfg, 0, T, ep_rank=0, ep_world=2,
                         free_running=True)
        with pytest.raises(P.MoeError, match="connect the shards"):
            eng.decode_tokens(acts[:2], scores[:2], np.zeros((2,) + shape[1:], dtype=np.float32))


def _owners_worker(rank, world, port, out_dir):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = load_golden("tiny")
        w, fg = oracle_inputs(g)
        sim = O.simulate(w, g["sim_capacities"], g["tau"], first_gate=fg, **sim_kwargs(g))
        own = ep.balanced_owners(sim.timeline, w.L, w.N, world)
        tables = [None] * world
        dist.all_gather_object(tables, own.tolist())
        np.save(os.path.join(out_dir, f"owners_{rank}.npy"), np.array(tables))
    finally:
        dist.destroy_process_group()


def test_balanced_owners_identical_on_every_rank_gloo(tmp_path):
    """Every rank derives the placement table from the same calibration run independently; the
    tables must agree (the decode sessions rely on it — no table is broadcast)."""
    import torch.multiprocessing as mp
    mp.spawn(_owners_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)
    t0, t1 = np.load(tmp_path / "owners_0.npy"), np.load(tmp_path / "owners_1.npy")
    assert np.array_equal(t0, t1) and np.array_equal(t0[0], t0[1])
    assert set(np.unique(t0[0])) <= {0, 1}
