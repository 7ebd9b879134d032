"""generate_trace timing + cProfile (tools/, not product) at the 8x7B 64-token workload."""
import os
import sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2408_10284_b200 as P
from paper_2408_10284_b200 import workloads as W
wl = W.mixtral_8x7b(tokens=64)
spec = P.ModelSpec(wl.layers, wl.experts, wl.top_k, wl.hidden)
eng = P.Engine(spec, 0)
sc = P.SynthConfig(spec, wl.tokens, wl.concentration, wl.drift, wl.gate_seed, wl.token_seed, False, wl.fisher_scales, wl.drift_scales)
for i in range(4):
    t = time.perf_counter(); tr = eng.generate_trace(sc); print("generate_trace call", i, f"{(time.perf_counter()-t)*1e3:.1f} ms")
import cProfile, pstats
cProfile.run("eng.generate_trace(sc)", "/tmp/gp")
pstats.Stats("/tmp/gp").sort_stats("cumtime").print_stats(8)
