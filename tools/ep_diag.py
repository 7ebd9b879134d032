"""Diagnostic (tools/, not product): two expert-parallel shards on one GPU in two host threads,
without and with the peer-memory exchange; prints per-call progress with timestamps."""
import sys
import threading
import time

import numpy as np

sys.path.insert(0, '.')
sys.path.insert(0, 'tests')
import paper_2408_10284_b200 as P  # noqa: E402
from conftest import load_golden  # noqa: E402
from helpers import oracle_inputs, sim_config  # noqa: E402

g = load_golden("tiny")
w0, fg = oracle_inputs(g)
cfg = sim_config(g)
caps, tau, T = g["sim_capacities"], g["tau"], 12
calls = [0, 5, 6, 12]
t0 = time.time()


def make(rank, world):
    eng = P.Engine(P.ModelSpec(w0.L, w0.N, w0.K, w0.D))
    eng.load_gates(w0.gates, fg)
    eng.experts_init(1024, cfg.tile_count_per_expert, seed=5)
    eng.decode_begin(caps, w0.fisher, tau, cfg, 0, T, ep_rank=rank, ep_world=world)
    return eng


for connect in (False, True):
    shards = [make(r, 2) for r in range(2)]
    if connect:
        regions = [s.decode_ep_export(6) for s in shards]
        print("regions", [hex(p) for p, _ in regions], flush=True)
        for s in shards:
            s.decode_ep_connect(peer_ptrs=[p for p, _ in regions])
    outs = [np.zeros((T, w0.L, w0.D), dtype=np.float32) for _ in shards]

    def run(i):
        for a, b in zip(calls, calls[1:]):
            print(f"{time.time() - t0:7.2f} connect={connect} shard {i} call {a}:{b} start", flush=True)
            try:
                shards[i].decode_tokens(w0.acts[a:b], w0.scores[a:b], outs[i][a:b])
            except Exception as e:  # noqa: BLE001
                print("  shard", i, "error", e, flush=True)
                return
            print(f"{time.time() - t0:7.2f} connect={connect} shard {i} call {a}:{b} done", flush=True)

    th = [threading.Thread(target=run, args=(i,), daemon=True) for i in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=40)
    print("alive", [t.is_alive() for t in th], flush=True)
    if any(t.is_alive() for t in th):
        print("stuck; exiting", flush=True)
        import os
        os._exit(3)
    for s in shards:
        s.decode_end(cfg, T)
        s.close()
print("done", flush=True)
