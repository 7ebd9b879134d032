"""Extended randomized parity sweep (tools/, evidence run): the tests' case generator
(tests/test_random_gpu.py::_case) over many more seeds; prints failures and a summary line."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402

import paper_2408_10284_b200 as P  # noqa: E402
from oracle import oracle as O  # noqa: E402
from test_random_gpu import _case  # noqa: E402


def run(seed):
    c = _case(seed)
    L, N, K, D, T = c["L"], c["N"], c["K"], c["D"], c["T"]
    w = O.generate_trace(L, N, K, D, T, c["conc"], c["drift"], c["gate_seed"], c["token_seed"])
    fg = O.train_first_gate(w, steps=20) if (c["train"] and T >= 2) else None
    tau = O.calibrate_threshold(w, c["target"])
    alpha, beta = O.generate_profiles(w, tau, fg)
    caps, _ = O.dp_allocate(O.cost_table(alpha, beta, N), c["budget"])
    kw = dict(tiles=c["tiles"], tile_transfer=c["transfer"], tile_compute=c["compute"], attention=c["attention"],
              gate=c["gate"], lookahead=c["lookahead"], gating=c["gating"], prefetch=c["prefetch"], seed=c["seed"])
    ref = O.simulate(w, caps, tau, first_gate=fg, **kw)
    spec = P.ModelSpec(L, N, K, D)
    cfg = P.SimConfig(c["tiles"], c["transfer"], c["compute"], c["attention"], c["gate"], c["lookahead"],
                      P.PolicyFlags(c["gating"], c["prefetch"], True))
    with P.Engine(spec) as eng:
        g = eng.generate_trace(P.SynthConfig(spec, T, c["conc"], c["drift"], c["gate_seed"], c["token_seed"]))
        ok = np.array_equal(g.gates, w.gates) and np.array_equal(g.acts, w.acts) and \
            np.array_equal(g.scores, w.scores) and np.array_equal(g.selected, w.selected)
        eng.load_gates(w.gates, fg)
        r = eng.simulate_trace(w.acts, w.scores, w.fisher, caps, tau, cfg, c["seed"])
    return ok and r.metrics == ref.metrics and np.array_equal(r.timeline, ref.timeline), c


def main():
    lo, hi = int(sys.argv[1]), int(sys.argv[2])
    t0 = time.time()
    bad = []
    for s in range(lo, hi):
        ok, c = run(s)
        if (s - lo + 1) % 1000 == 0:  # progress: a run cut short by a timeout still counts
            print(f"progress seeds {lo}..{s}: {s - lo + 1 - len(bad)} / {s - lo + 1} pass", flush=True)
        if not ok:
            bad.append(s)
            print("MISMATCH", s, c, flush=True)
    print(f"random sweep seeds {lo}..{hi - 1}: {hi - lo - len(bad)} / {hi - lo} bit-exact "
          f"(generate_trace + simulate_trace metrics + timeline), {time.time() - t0:.0f} s", flush=True)


if __name__ == "__main__":
    main()
