"""simulate_trace cost breakdown at the Mixtral-8x7B bench workload (tools/, not product): wall time
of route_trace (H2D of the fp64 trace + one K1 launch + D2H) vs the whole simulate_trace call."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2408_10284_b200 as P  # noqa: E402
from paper_2408_10284_b200 import workloads as W  # noqa: E402

wl = W.mixtral_8x7b(tokens=64)
spec = P.ModelSpec(wl.layers, wl.experts, wl.top_k, wl.hidden)
eng = P.Engine(spec, 0)
tr = eng.generate_trace(P.SynthConfig(spec, wl.tokens, wl.concentration, wl.drift, wl.gate_seed, wl.token_seed, False,
                                      wl.fisher_scales, wl.drift_scales))
tau, _ = P.calibrate_threshold(spec, tr.scores, tr.fisher, wl.target_single_ratio)
alpha, beta = eng.generate_profiles(tr.acts, tr.scores, tr.fisher, tau)
caps, _ = P.dp_allocate(spec, P.build_cost_table(spec, alpha, beta), wl.budget)
cfg = P.SimConfig()
a = torch.from_numpy(np.ascontiguousarray(tr.acts)).pin_memory().numpy()
s = torch.from_numpy(np.ascontiguousarray(tr.scores)).pin_memory().numpy()


def best(fn, n=11):
    b = 1e9
    for _ in range(n):
        t0 = time.perf_counter()
        fn()
        b = min(b, time.perf_counter() - t0)
    return b * 1e3


for name, c in [("default (lookahead 2)", cfg), ("prefetch off", P.SimConfig(policy=P.PolicyFlags(True, False, True)))]:
    r = best(lambda: eng.route_trace(a, s, tr.fisher, tau, c))
    t = best(lambda: eng.simulate_trace(a, s, tr.fisher, caps, tau, c, wl.seed))
    print(f"{name}: route_trace {r:.3f} ms, simulate_trace {t:.3f} ms, engine + timeline ~{t - r:.3f} ms "
          f"({64 / t * 1e3:.0f} tok/s)")
x = torch.empty(a.nbytes // 8, dtype=torch.float64, device="cuda")
h = torch.from_numpy(a.reshape(-1))
print(f"H2D of the 67 MB fp64 trace alone: {best(lambda: (x.copy_(h), torch.cuda.synchronize())):.3f} ms")
