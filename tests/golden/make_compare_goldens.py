"""Golden fixtures for the ablation grid (compare_policies, inc/simulator.hpp:476-550) from the
UNMODIFIED reference: oracle/_ref/moesim_ref mode=compare (reference headers compiled by
oracle/Makefile).  Run here (needs /root/reference):

    make -C oracle && python tests/golden/make_compare_goldens.py
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


def cases():
    return [
        ("tiny", W.tiny()),
        ("tiny_budget8_seed3", W.tiny(budget=8, seed=3)),
        ("tiny_nogate_lookahead1", W.tiny(train_first_gate=False, lookahead=1, budget=20)),
        ("mixtral_8x7b_t8", W.mixtral_8x7b(tokens=8)),
    ]


def main():
    if not O.have_ref():
        raise SystemExit("oracle/_ref/moesim_ref missing: run `make -C oracle` where /root/reference exists")
    out_dir = os.path.join(HERE, "compare")
    os.makedirs(out_dir, exist_ok=True)
    for name, wl in cases():
        r = O.run_ref(mode="compare", **wl.ref_args())
        r = {k: v for k, v in r.items() if k not in ("compare_s", "jobs")}  # timing, not a golden
        r["workload"] = wl.ref_args()
        with open(os.path.join(out_dir, f"{name}.json"), "w") as f:
            json.dump(r, f, indent=0)
        print(name, [row["speedup_vs_baseline"] for row in r["rows"]])


if __name__ == "__main__":
    main()
