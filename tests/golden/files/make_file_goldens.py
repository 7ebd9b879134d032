"""Artifact-file fixtures written by the UNMODIFIED reference's own io (inc/io.hpp, nlohmann/json):
oracle/_ref/moesim_ref mode=save writes trace.jsonl, gates.json, profiles.json, threshold.json,
allocation.json and cost_table.json for each case into tests/golden/files/<case>/, and mode=load
reads them back and records the reference's view (array hashes, scalars) in expected.json.
Run here (needs /root/reference):

    make -C oracle && python tests/golden/files/make_file_goldens.py
"""
from __future__ import annotations

import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(HERE)))
sys.path.insert(0, ROOT)

from oracle import oracle as O  # noqa: E402
from paper_2408_10284_b200 import workloads as W  # noqa: E402


def cases():
    return [
        ("tiny_t8", W.tiny(tokens=8, train_steps=60)),
        ("odd_d37", W.Workload(name="odd", layers=3, experts=8, top_k=2, hidden=37, tokens=6, budget=8,
                               train_steps=20)),
        ("top3_nogate", W.Workload(name="top3", layers=2, experts=6, top_k=3, hidden=16, tokens=5, budget=5,
                                   train_first_gate=False, target_single_ratio=0.3)),
    ]


def main():
    if not O.have_ref():
        raise SystemExit("oracle/_ref/moesim_ref missing: run `make -C oracle` where /root/reference exists")
    for name, wl in cases():
        d = os.path.join(HERE, name)
        os.makedirs(d, exist_ok=True)
        saved = O.run_ref(mode="save", dir=d, **wl.ref_args())
        view = O.run_ref(mode="load", dir=d, **wl.ref_args())
        view = {k: v for k, v in view.items() if not k.endswith("_s")}  # drop timings
        view["workload"] = wl.ref_args()
        view["saved_profile_hash"] = saved["profile_hash"]
        with open(os.path.join(d, "expected.json"), "w") as f:
            json.dump(view, f, indent=1)
        print(name, sorted(os.listdir(d)))


if __name__ == "__main__":
    main()
