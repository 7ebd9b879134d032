"""Diagnostic (tools/, not product): one random-sweep case from tests/test_random_gpu.py, GPU router
outputs and simulate_trace vs the oracle, with and without a preceding generate_trace."""
import sys

import numpy as np

sys.path.insert(0, '.')
sys.path.insert(0, 'tests')
import paper_2408_10284_b200 as P  # noqa: E402
from oracle import oracle as O  # noqa: E402
from test_random_gpu import _case  # noqa: E402

c = _case(int(sys.argv[1]) if len(sys.argv) > 1 else 75)
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
for pre in (False, True):
    with P.Engine(spec) as eng:
        if pre:
            eng.generate_trace(P.SynthConfig(spec, T, c["conc"], c["drift"], c["gate_seed"], c["token_seed"]))
        eng.load_gates(w.gates, fg)
        dec, single, pert, preds = eng.route_trace(w.acts, w.scores, w.fisher, tau, cfg)
        r = eng.simulate_trace(w.acts, w.scores, w.fisher, caps, tau, cfg, c["seed"])
    print("pre-generate", pre, "decisions", np.array_equal(dec, ref.decisions), "preds",
          np.array_equal(preds, ref.predictions), "metrics", r.metrics == ref.metrics, r.metrics["total_latency"],
          ref.metrics["total_latency"])
    bad = np.argwhere((preds != ref.predictions).any(axis=-1))
    for t, l, s in bad[:5]:
        print("  ", t, l, s, preds[t, l, s].tolist(), ref.predictions[t, l, s].tolist())
