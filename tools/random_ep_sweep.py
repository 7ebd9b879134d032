"""Randomized expert-parallel parity sweep (tools/, evidence run): random shapes / capacities /
batch, random world size and random placement tables; the G shard sessions (run one after another
on one GPU) must replay the single-GPU trace bit for bit, move / compute disjoint expert sets, and
their partial outputs must sum to the single-GPU output (fp32: 1e-5; bf16 batched: 2e-3).  The
expert store is drawn from bf16 / XB12 / XBH per case (ADAPMOE_SWEEP_STORE fixes it)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_2408_10284_b200 as P  # noqa: E402
from oracle import oracle as O  # noqa: E402


def run(seed):
    r = np.random.default_rng(9000 + seed)
    B = int(r.choice([1, 1, 3, 8]))
    L, N, K = int(r.integers(1, 5)), 8, 2
    D = int(r.choice([128, 256]))
    tiles = int(r.choice([1, 2, 4]))
    F = 64 * tiles * int(r.integers(1, 3))
    T = int(r.integers(1, 5))
    G = int(r.choice([2, 3, 4, 8]))
    store = os.environ.get("ADAPMOE_SWEEP_STORE", "all")
    if store == "all":
        store = str(r.choice(["bf16", "xb12", "xbh"]))
    owners = r.integers(0, G, size=(L, N)).astype(np.int32) if r.integers(0, 2) else None
    ws = [O.generate_trace(L, N, K, D, T, 0.6, 0.2, 5, 100 + b) for b in range(B)]
    tau = O.calibrate_threshold(ws[0], 0.24)
    caps = [int(x) for x in r.integers(0, N + 1, size=L)]
    cfg = P.SimConfig(tiles, 2, 1, 8, 1, int(r.integers(0, 3)), P.PolicyFlags(True, True, True))
    if B == 1:
        acts, scores, shape = ws[0].acts, ws[0].scores, (T, L, D)
    else:
        acts = np.ascontiguousarray(np.stack([w.acts for w in ws], axis=1))
        scores = np.ascontiguousarray(np.stack([w.scores for w in ws], axis=1))
        shape = (T, B, L, D)
    outs, res = [], []
    for rank, world in [(0, 1)] + [(g, G) for g in range(G)]:
        with P.Engine(P.ModelSpec(L, N, K, D)) as eng:
            eng.load_gates(ws[0].gates)
            eng.experts_init(F, tiles, seed=seed, store_format=store)
            eng.decode_begin(caps, ws[0].fisher, tau, cfg, 0, T, batch=B, ep_rank=rank, ep_world=world,
                             expert_owner=owners if world > 1 else None)
            h = np.zeros(shape, dtype=np.float32)
            eng.decode_tokens(acts, scores, h)
            res.append(eng.decode_end(cfg, T))
            outs.append(h.astype(np.float64))
    for x in res[1:]:
        if x.metrics != res[0].metrics or not np.array_equal(x.timeline, res[0].timeline):
            return False, "trace"
    if sum(x.stats["ffn_bytes"] for x in res[1:]) != res[0].stats["ffn_bytes"]:
        return False, "ffn bytes"
    full = outs[0]
    moe = full - acts.astype(np.float32).astype(np.float64)
    err = np.abs(sum(outs[1:]) - full).max() / max(np.abs(moe).max(), 1e-30)
    tol = 1e-5 if B == 1 else 2e-3
    return err <= tol, f"rel err {err:.2e} (tol {tol}), G={G}, B={B}"


def main():
    lo, hi = int(sys.argv[1]), int(sys.argv[2])
    t0, bad = time.time(), []
    for s in range(lo, hi):
        try:
            ok, why = run(s)
        except Exception as e:  # noqa: BLE001  (a device error poisons the process: report the seed, stop)
            print("ERROR", s, repr(e)[:300], flush=True)
            raise
        if (s - lo + 1) % 1000 == 0:  # progress: a run cut short by a timeout still counts
            print(f"progress seeds {lo}..{s}: {s - lo + 1 - len(bad)} / {s - lo + 1} pass", flush=True)
        if not ok:
            bad.append(s)
            print("MISMATCH", s, why, flush=True)
    print(f"random EP sweep seeds {lo}..{hi - 1}: {hi - lo - len(bad)} / {hi - lo} pass (shards replay the trace, "
          f"disjoint experts, partials sum to the single-GPU output), {time.time() - t0:.0f} s", flush=True)


if __name__ == "__main__":
    main()
