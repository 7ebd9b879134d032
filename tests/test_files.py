"""Artifact files (inc/io.hpp): the reference's JSON / JSON Lines formats.

Pinned against fixtures written by the unmodified reference's own io (tests/golden/files/, made by
make_file_goldens.py):
  * our loaders return exactly the arrays / scalars the reference wrote (and the oracle regenerates);
  * our writers reproduce the reference's files: the compact JSON Lines trace and profile_hash byte
    for byte; the dump(2) files byte for byte up to whitespace (the only nlohmann/json in this image,
    cudnn_frontend's copy, prints integer arrays compactly even under dump(2) — a local patch; we
    print them like stock nlohmann 3.x, one element per line);
  * the binary trace container round-trips exactly;
  * error classes: io_error -> 2, parse / schema / version error -> 3 (inc/io.hpp:23-37);
  * where the reference compiled here, it reads our files back to the same view.
"""
import json
import os
import re

import numpy as np
import pytest

import paper_2408_10284_b200 as P
from helpers import parse_scales
from oracle import oracle as O
from paper_2408_10284_b200 import io as IO

DIR = os.path.join(os.path.dirname(__file__), "golden", "files")
CASES = sorted(n for n in os.listdir(DIR) if os.path.isdir(os.path.join(DIR, n)))
KINDS = ["trace.jsonl", "gates.json", "profiles.json", "threshold.json", "allocation.json", "cost_table.json"]


def _case(name):
    exp = json.load(open(os.path.join(DIR, name, "expected.json")))
    a = exp["workload"]
    w = O.generate_trace(int(a["layers"]), int(a["experts"]), int(a["top_k"]), int(a["hidden"]), int(a["tokens"]),
                         float(a["concentration"]), float(a["drift"]), int(a["gate_seed"]), int(a["token_seed"]),
                         False, parse_scales(a.get("fisher_scales")), parse_scales(a.get("drift_scales")))
    return exp, a, w


@pytest.mark.parametrize("name", CASES)
def test_loaders_read_reference_files(name):
    exp, a, w = _case(name)
    d = os.path.join(DIR, name)
    tr = IO.load_trace(os.path.join(d, "trace.jsonl"))
    assert tr.violations == []
    assert np.array_equal(tr.acts, w.acts) and np.array_equal(tr.scores, w.scores)
    assert np.array_equal(tr.selected, w.selected)
    assert O.fnv1a(tr.acts) == exp["hash_activations"] and O.fnv1a(tr.scores) == exp["hash_scores"]
    spec, gates, fg, cfg = IO.load_gates(os.path.join(d, "gates.json"))
    assert (spec.num_layers, spec.experts_per_layer, spec.top_k, spec.hidden_dim) == \
        (int(a["layers"]), int(a["experts"]), int(a["top_k"]), int(a["hidden"]))
    assert np.array_equal(gates, w.gates) and O.fnv1a(gates) == exp["hash_gates"]
    if int(a["train_gate"]):
        assert np.array_equal(fg, O.train_first_gate(w, lr=float(a["train_lr"]), steps=int(a["train_steps"]),
                                                     seed=int(a["train_seed"])))
        assert cfg[1] == exp["first_gate_steps"]
    else:
        assert fg is None and exp["first_gate_steps"] == -1
    _, alpha, beta, fisher = IO.load_profiles(os.path.join(d, "profiles.json"))
    assert alpha.tolist() == exp["alpha"] and beta.tolist() == exp["beta"] and fisher.tolist() == exp["fisher"]
    tau, _, _ = IO.load_threshold(os.path.join(d, "threshold.json"))
    assert tau == float(exp["tau"]) == O.calibrate_threshold(w, float(a["target"]))
    caps, budget, cost, h = IO.load_allocation(os.path.join(d, "allocation.json"))
    assert caps.tolist() == exp["capacities"] and budget == exp["budget"] and h == exp["alloc_profile_hash"]
    table = IO.load_cost_table(os.path.join(d, "cost_table.json"))
    assert O.fnv1a(table) == exp["hash_cost_table"]
    assert np.array_equal(table, O.cost_table(alpha, beta, spec.experts_per_layer))


@pytest.mark.parametrize("name", CASES)
def test_writers_reproduce_reference_bytes(name, tmp_path):
    exp, a, w = _case(name)
    d = os.path.join(DIR, name)
    tr = IO.load_trace(os.path.join(d, "trace.jsonl"))
    spec, gates, fg, cfg = IO.load_gates(os.path.join(d, "gates.json"))
    _, alpha, beta, fisher = IO.load_profiles(os.path.join(d, "profiles.json"))
    tau, target, realized = IO.load_threshold(os.path.join(d, "threshold.json"))
    caps, budget, cost, h = IO.load_allocation(os.path.join(d, "allocation.json"))
    table = IO.load_cost_table(os.path.join(d, "cost_table.json"))
    out = str(tmp_path)
    IO.save_trace(os.path.join(out, "trace.jsonl"), spec, tr.acts, tr.scores, tr.selected)
    if fg is None:
        IO.save_gates(os.path.join(out, "gates.json"), spec, gates)
    else:
        IO.save_gates(os.path.join(out, "gates.json"), spec, gates, fg, *cfg)
    ph = IO.save_profiles(os.path.join(out, "profiles.json"), spec, alpha, beta, fisher)
    assert ph == exp["profile_hash"] == exp["saved_profile_hash"]
    IO.save_threshold(os.path.join(out, "threshold.json"), tau, target, realized)
    IO.save_allocation(os.path.join(out, "allocation.json"), caps, budget, cost, h)
    IO.save_cost_table(os.path.join(out, "cost_table.json"), table)
    for k in KINDS:
        ours, ref = open(os.path.join(out, k)).read(), open(os.path.join(d, k)).read()
        if k.endswith(".jsonl"):
            assert ours == ref, k
        else:
            assert re.sub(r"\s", "", ours) == re.sub(r"\s", "", ref), k
    if O.have_ref():  # the reference reads our files back to the same view
        import shutil
        shutil.copy(os.path.join(d, "expected.json"), out)
        view = O.run_ref(mode="load", dir=out, **a)
        for k, v in view.items():
            if k.endswith("_s"):  # timings
                continue
            assert exp[k] == v, k


def test_binary_trace_round_trip(tmp_path):
    w = O.generate_trace(3, 8, 2, 64, 5)
    spec = P.ModelSpec(3, 8, 2, 64)
    p = str(tmp_path / "t.bin")
    IO.save_trace(p, spec, w.acts, w.scores, w.selected, binary=True)
    tr = IO.load_trace(p)
    assert tr.violations == []
    assert np.array_equal(tr.acts, w.acts) and np.array_equal(tr.scores, w.scores)
    assert np.array_equal(tr.selected, w.selected)
    assert os.path.getsize(p) < 8 * w.acts.size + 8 * w.scores.size + 4 * w.selected.size + 4 * 3 * 5 + 128


def test_validate_trace_reports_violations(tmp_path):
    w = O.generate_trace(2, 4, 2, 16, 3)
    bad = w.scores.copy()
    bad[1, 0, 0] += 0.5  # breaks normalisation
    sel = w.selected.copy()
    sel[2, 1, 1] = sel[2, 1, 0]  # duplicate expert
    p = str(tmp_path / "bad.jsonl")
    IO.save_trace(p, P.ModelSpec(2, 4, 2, 16), w.acts, bad, sel)
    v = IO.load_trace(p).violations
    assert v and v[0].startswith("token 1 layer 0: score normalization")


@pytest.mark.parametrize("text,code", [
    (None, 2),                                                                 # io_error
    ("{not json", 3),                                                          # parse_error
    ('{"format_version": 2, "kind": "threshold"}', 3),                         # version_error
    ('{"format_version": 1, "kind": "profiles"}', 3),                          # schema: wrong kind
    ('{"format_version": 1, "kind": "threshold", "tau": "x"}', 3),             # schema: wrong type
])
def test_error_classes(tmp_path, text, code):
    p = str(tmp_path / "f.json")
    if text is not None:
        open(p, "w").write(text)
    with pytest.raises(P.MoeError) as e:
        IO.load_threshold(p)
    assert e.value.code == code
