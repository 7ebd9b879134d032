"""Randomized physical-decode parity sweep (tools/, evidence run): random shapes, capacities,
look-ahead, batch 1 (K2, tolerance 1e-4) and batched (K3, 2e-2), tile grouping forced on or off,
expert store bf16 / XB12 / XBH (ADAPMOE_SWEEP_STORE=all, the default, picks one at random per case;
or a fixed format); the decode's trace must equal the oracle's and every sampled layer output must
match the fp64 oracle SwiGLU within tolerance."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402

import paper_2408_10284_b200 as P  # noqa: E402
from oracle import oracle as O  # noqa: E402


def run(seed):
    r = np.random.default_rng(5000 + seed)
    B = int(r.choice([1, 1, 2, 3, 8]))
    L, N, K = int(r.integers(1, 5)), int(r.choice([4, 8])), 2
    D = int(r.choice([128, 256])) if B > 1 else int(r.choice([64, 96, 256, 512]))
    tiles = int(r.choice([1, 2, 4]))
    F = 64 * tiles * int(r.integers(1, 4))
    T = int(r.integers(1, 6))
    os.environ["ADAPMOE_TILE_MERGE"] = str(int(r.integers(0, 3)))
    store = os.environ.get("ADAPMOE_SWEEP_STORE", "all")
    if store == "all":
        store = str(r.choice(["bf16", "xb12", "xbh"]))
    ws = [O.generate_trace(L, N, K, D, T, 0.6, 0.2, 5, 100 + b) for b in range(B)]
    tau = O.calibrate_threshold(ws[0], 0.24)
    caps = [int(x) for x in r.integers(0, N + 1, size=L)]
    lookahead = int(r.integers(0, 3))
    ref = O.simulate_batch(ws, caps, tau, tiles=tiles, lookahead=lookahead)
    cfg = P.SimConfig(tiles, 2, 1, 8, 1, lookahead, P.PolicyFlags(True, True, True))
    with P.Engine(P.ModelSpec(L, N, K, D)) as eng:
        eng.load_gates(ws[0].gates)
        eng.experts_init(F, tiles, seed=seed, store_format=store)
        eng.decode_begin(caps, ws[0].fisher, tau, cfg, 0, T, batch=B)
        if B == 1:
            hid = np.zeros((T, L, D), dtype=np.float32)
            eng.decode_tokens(ws[0].acts, ws[0].scores, hid)
            hid = hid[:, None]
        else:
            acts = np.ascontiguousarray(np.stack([w.acts for w in ws], axis=1))
            scores = np.ascontiguousarray(np.stack([w.scores for w in ws], axis=1))
            hid = np.zeros((T, B, L, D), dtype=np.float32)
            eng.decode_tokens(acts, scores, hid)
        res = eng.decode_end(cfg, T)
    if res.metrics != ref.metrics or not np.array_equal(res.timeline, ref.timeline):
        return False, f"trace ({store} store)"
    tol = 1e-4 if B == 1 else 2e-2
    worst = 0.0
    for t in range(T):
        for l in range(L):
            for b in range(B):
                sel = [int(e) for e in ref.decisions[b, t, l] if e >= 0]
                sc = ws[b].scores[t, l]
                x32 = ws[b].acts[t, l].astype(np.float32)
                moe = np.zeros(D)
                for e in sel:
                    wgt = 1.0 if len(sel) == 1 else sc[e] / sum(sc[q] for q in sel)
                    moe += wgt * O.swiglu(O.expert_init(seed, l, e, D, F, tiles), D, F, tiles, x32)
                got = hid[t, b, l].astype(np.float64) - x32.astype(np.float64)
                worst = max(worst, np.abs(got - moe).max() / max(np.abs(moe).max(), 1e-30))
    return worst <= tol, f"{store} store: worst rel err {worst:.2e} (tol {tol})"


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
    print(f"random decode sweep seeds {lo}..{hi - 1}: {hi - lo - len(bad)} / {hi - lo} pass (trace bit-exact, "
          f"outputs within 1e-4 fp32 / 2e-2 bf16), {time.time() - t0:.0f} s", flush=True)


if __name__ == "__main__":
    main()
