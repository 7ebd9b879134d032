"""The C++ drop-in example (examples/simulate_files.cpp): host code that links only the C ABI
(include/adapmoe.h), reads the reference's artifact files and runs simulate_trace on the B200 —
what the reference's `moesim simulate` (proj/tools/moesim_main.cpp:291-347) becomes when it binds
this library.

  * [cpu] usage and the reference's exit-code classes (io_error -> 2, missing device -> 6);
  * [gpu] on every reference-written fixture (tests/golden/files/) and several tick / flag settings
    the metrics it prints equal the oracle's simulate() on the same files' contents.
"""
import json
import os
import subprocess

import numpy as np
import pytest

from oracle import oracle as O
from paper_2408_10284_b200 import io as IO

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
EXE = os.path.join(ROOT, "examples", "simulate_files")
DIR = os.path.join(ROOT, "tests", "golden", "files")
CASES = sorted(n for n in os.listdir(DIR) if os.path.isdir(os.path.join(DIR, n)))


@pytest.fixture(scope="module")
def exe():
    if not os.path.exists(EXE):
        subprocess.run(["make", "-C", os.path.join(ROOT, "examples")], check=True, capture_output=True)
    return EXE


def test_usage_and_io_error(exe, tmp_path):
    r = subprocess.run([exe], capture_output=True, text=True)
    assert r.returncode == 1 and "usage" in r.stderr
    r = subprocess.run([exe, str(tmp_path)], capture_output=True, text=True)
    assert r.returncode == 2 and "cannot open" in r.stderr  # io_error class (inc/io.hpp:23)


def test_bad_trace_is_schema_error(exe, tmp_path):
    (tmp_path / "trace.jsonl").write_text('{"format_version": 99}\n')
    r = subprocess.run([exe, str(tmp_path)], capture_output=True, text=True)
    assert r.returncode == 3, r.stderr  # parse / schema / version error class (inc/io.hpp:30-37)


# (tiles, transfer, compute, attention, gate, lookahead, gating, prefetch, seed)
_TICKS = [(4, 2, 1, 8, 1, 2, 1, 1, 0), (2, 3, 1, 4, 0, 1, 0, 1, 7), (1, 1, 2, 0, 2, 3, 1, 0, 3)]


@pytest.mark.gpu
@pytest.mark.parametrize("ticks", _TICKS)
@pytest.mark.parametrize("name", CASES)
def test_example_matches_oracle(exe, name, ticks):
    d = os.path.join(DIR, name)
    r = subprocess.run([exe, d] + [str(v) for v in ticks], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stderr
    got = json.loads(r.stdout)
    tr = IO.load_trace(os.path.join(d, "trace.jsonl"))
    spec, gates, fg, _ = IO.load_gates(os.path.join(d, "gates.json"))
    _, _, _, fisher = IO.load_profiles(os.path.join(d, "profiles.json"))
    tau, _, _ = IO.load_threshold(os.path.join(d, "threshold.json"))
    caps, _, _, _ = IO.load_allocation(os.path.join(d, "allocation.json"))
    L, N, K, D = spec.num_layers, spec.experts_per_layer, spec.top_k, spec.hidden_dim
    w = O.Workload(L, N, K, D, tr.acts.shape[0], gates, tr.acts, tr.scores, tr.selected, np.asarray(fisher))
    tiles, transfer, compute, attention, gate, lookahead, gating, prefetch, seed = ticks
    ref = O.simulate(w, caps, tau, first_gate=fg, tiles=tiles, tile_transfer=transfer, tile_compute=compute,
                     attention=attention, gate=gate, lookahead=lookahead, gating=bool(gating),
                     prefetch=bool(prefetch), seed=seed)
    for k, v in ref.metrics.items():
        assert got[k] == v, (k, got[k], v)
    assert got["tokens"] == w.T
    assert got["on_demand_loads_per_layer"] == ref.od_per_layer.tolist()
    assert got["timeline_events"] == len(ref.timeline)


def test_model_mismatch_is_validation_error(exe, tmp_path):
    import shutil
    for f in ["trace.jsonl", "profiles.json", "threshold.json", "allocation.json"]:
        shutil.copy(os.path.join(DIR, "tiny_t8", f), tmp_path / f)
    shutil.copy(os.path.join(DIR, "odd_d37", "gates.json"), tmp_path / "gates.json")
    r = subprocess.run([exe, str(tmp_path)], capture_output=True, text=True)
    assert r.returncode == 4 and "mismatch" in r.stderr  # require_same_model (moesim_main.cpp:102-104)


@pytest.mark.gpu
def test_python_example_runs():
    r = subprocess.run(["python", os.path.join(ROOT, "examples", "python_decode.py")], capture_output=True, text=True,
                       timeout=300)
    assert r.returncode == 0 and r.stdout.strip().endswith("OK"), r.stdout + r.stderr
