"""First-layer predictive gate trainer on the GPU (inc/prefetch.hpp:194-213,
inc/workload.hpp:186-197).  Contract: bit-exact with the reference — the trained gate's FNV-1a hash
equals the golden produced by the unmodified reference for every case that trains a gate, and the
weights equal the C oracle's at the Mixtral-8x7B width."""
import numpy as np
import pytest

import paper_2408_10284_b200 as P
from conftest import golden_names, load_golden
from helpers import wl_args
from oracle import oracle as O

pytestmark = pytest.mark.gpu


def _trained_cases():
    out = []
    for n in golden_names():
        a = load_golden(n)["workload"]
        if int(a["train_gate"]) and int(a["tokens"]) >= 2:
            out.append(n)
    return out


@pytest.mark.parametrize("name", _trained_cases())
def test_gpu_trainer_matches_reference_golden(name):
    g = load_golden(name)
    a = g["workload"]
    w = O.generate_trace(**wl_args(g))
    with P.Engine(P.ModelSpec(w.L, w.N, w.K, w.D)) as eng:
        W = eng.train_first_gate(w.acts, w.scores, float(a["train_lr"]), int(a["train_steps"]), int(a["train_seed"]))
    assert O.fnv1a(W) == g["hash_first_gate"]


def test_gpu_trainer_matches_oracle_mixtral_width():
    w = O.generate_trace(2, 8, 2, 4096, 9, 0.6, 0.18, 99, 5000, False, [2.0, 1.0], [1.8, 0.9])
    with P.Engine(P.ModelSpec(2, 8, 2, 4096)) as eng:
        W = eng.train_first_gate(w.acts, w.scores, 0.1, 25, 3)
    assert np.array_equal(W, O.train_first_gate(w, lr=0.1, steps=25, seed=3))


def test_gpu_trainer_rejects_empty_training_set():
    w = O.generate_trace(2, 4, 2, 64, 1)
    with P.Engine(P.ModelSpec(2, 4, 2, 64)) as eng:
        with pytest.raises(P.MoeError) as e:
            eng.train_first_gate(w.acts, w.scores)
    assert e.value.code == 1
