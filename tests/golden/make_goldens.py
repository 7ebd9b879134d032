"""Generate the committed golden fixtures from the UNMODIFIED reference.

Runs oracle/_ref/moesim_ref (the reference headers under /root/reference/proj/include compiled by
oracle/Makefile with the reference's flags) on each case and stores what it printed.  Large arrays
(activations, scores, gates, long timelines) are stored as FNV-1a hashes of their raw bytes; the
GPU-side tests regenerate them and compare hashes.  Run here (needs /root/reference):

    make -C oracle && python tests/golden/make_goldens.py
"""
from __future__ import annotations

import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from paper_2408_10284_b200 import workloads as W  # noqa: E402

FULL_TIMELINE_MAX = 6000


def cases():
    t = W.tiny()
    out = [("tiny", t)]
    out += [
        ("tiny_nogate", W.tiny(train_first_gate=False)),
        ("tiny_gating_off", W.tiny(gating=False)),
        ("tiny_prefetch_off", W.tiny(prefetch=False)),
        ("tiny_lookahead1", W.tiny(lookahead=1)),
        ("tiny_lookahead3", W.tiny(lookahead=3)),
        ("tiny_uniform", W.tiny(extra={"uniform": 1})),
        ("tiny_transfer_heavy", W.tiny(tile_transfer=5, tile_compute=1, attention=2, tiles=3, seed=7)),
        ("tiny_compute_heavy", W.tiny(tile_transfer=1, tile_compute=3, attention=1, tiles=2, budget=6)),
        ("tiny_budget0", W.tiny(budget=0)),
        ("tiny_budget_full", W.tiny(budget=32)),
        ("demo8_300", W.demo8(tokens=300)),
        ("wide_n16", W.Workload(name="wide", layers=6, experts=16, top_k=2, hidden=128, tokens=40, budget=40,
                                train_steps=50)),
        ("top3", W.Workload(name="top3", layers=4, experts=8, top_k=3, hidden=64, tokens=50, budget=12,
                            train_steps=50, target_single_ratio=0.3)),
        ("odd_d", W.Workload(name="odd", layers=3, experts=8, top_k=2, hidden=37, tokens=30, budget=8,
                             train_steps=50)),
        ("mixtral_8x7b_t12", W.mixtral_8x7b(tokens=12)),
    ]
    return out


def main():
    if not O.have_ref():
        raise SystemExit("oracle/_ref/moesim_ref missing: run `make -C oracle` where /root/reference exists")
    os.makedirs(HERE, exist_ok=True)
    manifest = {}
    for name, wl in cases():
        r = O.run_ref(**wl.ref_args())
        tl = r.pop("timeline")
        r["timeline_events"] = len(tl) // 8
        import numpy as np
        arr = np.asarray(tl, dtype=np.int64)
        r["hash_timeline"] = O.fnv1a(arr)
        if len(tl) // 8 <= FULL_TIMELINE_MAX:
            r["timeline"] = tl
        r["workload"] = wl.ref_args()
        r["ref_flags"] = "g++ -std=c++20 -O2 -pthread (no -march)"
        path = os.path.join(HERE, f"{name}.json")
        with open(path, "w") as f:
            json.dump(r, f, separators=(",", ":"))
        manifest[name] = {"bytes": os.path.getsize(path), "events": r["timeline_events"], "tau": r["tau"],
                          "metrics": {k: v for k, v in r["metrics"].items() if k != "latency_per_token"}}
        print(name, manifest[name]["bytes"], manifest[name]["metrics"])
    with open(os.path.join(HERE, "MANIFEST.json"), "w") as f:
        json.dump(manifest, f, indent=1)


if __name__ == "__main__":
    main()
