"""Per-layer gap probe (tools/, not product): one 8x7B decode with ADAPMOE_GAP_TRACE-style timing of
K1 / host step / FFN / combine per layer (profiling the free-running round trip)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2408_10284_b200 as P
from paper_2408_10284_b200 import workloads as W
wl = W.mixtral_8x7b(tokens=8)
spec = P.ModelSpec(wl.layers, wl.experts, wl.top_k, wl.hidden)
eng = P.Engine(spec, 0)
tr = eng.generate_trace(P.SynthConfig(spec, wl.tokens, wl.concentration, wl.drift, wl.gate_seed, wl.token_seed, False, wl.fisher_scales, wl.drift_scales))
tau, _ = P.calibrate_threshold(spec, tr.scores, tr.fisher, wl.target_single_ratio)
eng.experts_init(wl.ffn, wl.tiles, seed=1, host_alias=16)
cfg = P.SimConfig()
eng.decode_begin([8]*32, tr.fisher, tau, cfg, 0, 8, free_running=True, concentration=wl.concentration)
h = np.zeros((8, 32, 4096), dtype=np.float32)
eng.decode_tokens(tr.acts[:4], tr.scores[:4], h[:4])
os.environ["ADAPMOE_GAP_TRACE"] = "1"
eng.decode_tokens(tr.acts[4:6], tr.scores[4:6], h[4:6])
