#!/usr/bin/env python
"""AdapMoE offloaded-MoE decode on B200 — BASELINE.json metric:
"Mixtral-shape decode tok/s at fixed cache budget; on-demand expert loads/token".

Default workload = BASELINE config 2: Mixtral-8x7B shape (32 layers, 8 experts, top-2, d 4096,
ffn 14336), bf16 experts, batch-1 decode, HBM expert cache capped at 64 of 256 experts (DP-sized,
reference knapsack), all 256 experts in pinned host memory, prefetch lookahead 2, tau calibrated to
a 24% single-expert ratio (reference pipeline: generate -> calibrate -> profile -> allocate).

A step = one decoded token: for each of the 32 layers, K1 (router + pre-gate) -> host tick-model
policy step -> tile copies (on-demand/prefetch) -> K2 SwiGLU over the selected experts -> combine.
  value : tok/s with the token inputs already in HBM (CUDA events on the engine's compute stream)
  e2e   : tok/s through the C ABI with host (pinned) input buffers, one call per token, including
          the H2D of the token's inputs and the D2H of its 32 layer outputs, wall clock
N > 1 GPUs (torchrun): expert parallelism by default (north star): rank r owns experts
e % N == r of every layer, holds / copies / computes only those (its own host link moves them), the
ranks decode ONE token stream and sum their partial layer outputs in rank order after an all_gather
(NCCL over NVLink) — "scaling": "strong".  --replicas runs independent streams instead ("weak").

`--impl reference` times the reference's own CPU implementation of the path (the unmodified moesim
simulate_trace compiled into oracle/_ref) on the same workload and prints its line.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "Mixtral-shape decode tok/s at fixed cache budget; on-demand expert loads/token"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=8)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="mixtral-8x7b", choices=["mixtral-8x7b", "mixtral-8x22b", "tiny"])
    ap.add_argument("--ep", action="store_true",
                    help="expert-parallel over the torchrun ranks (the default when WORLD_SIZE > 1): rank r owns experts "
                         "e % G == r, the ranks decode ONE token stream and combine partial layer outputs (all_gather, "
                         "fixed order)")
    ap.add_argument("--ep-exchange", default="p2p", choices=["p2p", "allgather"],
                    help="EP combine: device-side stores into peer memory (CUDA IPC, NVLink) from the combine "
                         "epilogue, or a torch.distributed all_gather after each call")
    ap.add_argument("--ep-owner", default="balanced", choices=["balanced", "modulo"],
                    help="EP expert placement: balanced by a calibration trace's transfers (ep.balanced_owners) or "
                         "expert e on rank e % N")
    ap.add_argument("--free-running", action="store_true",
                    help="decode with the hidden state flowing through the experts (layer l > 0 routes on layer "
                         "l-1's output; decisions from the gates) instead of replaying the trace")
    ap.add_argument("--replicas", action="store_true",
                    help="N > 1: run independent replicas (one stream per GPU) instead of expert parallelism")
    ap.add_argument("--budget", type=int, default=None)
    ap.add_argument("--layers", type=int, default=None,
                    help="rehearsal: keep only the model's first L layers (budget scaled by L / layers), e.g. the "
                         "8x22B expert-parallel flow on a host that cannot pin all 270 GB of experts")
    ap.add_argument("--batch", type=int, default=1,
                    help="decode streams sharing the cache (BASELINE config 4: 16 / 64; grouped tcgen05 FFN)")
    ap.add_argument("--no-resident-check", action="store_true",
                    help="skip the extra all-resident window (budget = L*N, no host-link traffic) that reports the "
                         "FFN kernel's roofline when every launch covers whole experts")
    ap.add_argument("--trace-tokens", type=int, default=64)
    ap.add_argument("--staging", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--pipeline", action="store_true",
                    help="measure the offline pipeline + ablation grid + artifact files (SURVEY §8(f)) against the "
                         "reference, one JSON line per workload, instead of the decode")
    ap.add_argument("--timeline", default=None,
                    help="record the physical timeline (CUDA-event tile copies, FFN launches, waits, router) over the "
                         "e2e window, write it as JSONL to this path and run the reference's timeline validators")
    ap.add_argument("--store-format", default="xbh", choices=["bf16", "xb12", "xbh"],
                    help="pinned expert store: raw bf16 tiles, XB12 (lossless exponent-coded bf16, 4-bit window "
                         "codes: 75 %% of the bytes over the host link) or XBH (per-tile Huffman-coded exponents: "
                         "~66 %%); coded tiles are decoded into the HBM slot on arrival; identical outputs")
    ap.add_argument("--host-alias", type=int, default=None,
                    help="store only this many distinct experts in host memory (profiling runs; same bytes moved)")
    return ap.parse_args()


def workload(args):
    from paper_2408_10284_b200 import workloads as W
    if args.config == "tiny":
        wl = W.tiny(tokens=max(args.trace_tokens, args.warmup + 2 * args.steps))
    elif args.config == "mixtral-8x22b":
        wl = W.mixtral_8x22b(tokens=max(args.trace_tokens, args.warmup + 2 * args.steps))
    else:
        wl = W.mixtral_8x7b(tokens=max(args.trace_tokens, args.warmup + 2 * args.steps))
    if args.layers is not None:  # rehearsal of a deeper model on a smaller host: its first L layers
        L = args.layers
        budget = wl.budget * L // wl.layers
        wl.name = f"{wl.name} (first {L} of {wl.layers} layers)"
        wl.layers = L
        wl.fisher_scales = wl.fisher_scales[:L]
        wl.drift_scales = wl.drift_scales[:L]
        wl.budget = budget
    if args.budget is not None:
        wl.budget = args.budget
    return wl


# NCCL over NVLink on a multi-GPU node; ADAPMOE_DIST_BACKEND=gloo runs the same flow with several
# ranks sharing one GPU (the single-GPU test box), exchanging through host memory.
BACKEND = os.environ.get("ADAPMOE_DIST_BACKEND", "nccl")


COMM = {"backend": None, "nranks": 1}


def dist_init():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1:
        import torch
        import torch.distributed as dist
        local = local % max(1, torch.cuda.device_count())
        torch.cuda.set_device(local)
        if BACKEND == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(BACKEND)
        # the communicator's own rank count (checked against WORLD_SIZE / --gpus by the caller)
        t = torch.ones(1, device="cuda" if BACKEND == "nccl" else "cpu")
        dist.all_reduce(t)
        COMM.update(backend=dist.get_backend(), nranks=dist.get_world_size(), all_reduce_ranks=int(t.item()),
                    gpus_visible=torch.cuda.device_count())
        if BACKEND == "nccl":
            COMM["nccl_version"] = ".".join(str(v) for v in torch.cuda.nccl.version())
        if COMM["nranks"] != ws or COMM["all_reduce_ranks"] != ws:
            raise SystemExit(f"communicator has {COMM['nranks']} ranks ({COMM['all_reduce_ranks']} in an all_reduce), "
                             f"WORLD_SIZE is {ws}")
    return ws, rank, local


def host_info() -> dict:
    """nproc, CPU model and RAM of this host (with every report)."""
    info = {"nproc": os.cpu_count()}
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                info["cpu_model"] = line.split(":", 1)[1].strip()
                break
        mem = open("/proc/meminfo").read()
        info["ram_gb"] = round(int(mem.split("MemTotal:")[1].split()[0]) / 2**20, 1)
    except Exception:  # noqa: BLE001
        pass
    return info


def fnv1a_i64(arr) -> str:
    """FNV-1a 64 over the raw little-endian bytes of an int64 array (the reference driver's hash)."""
    import numpy as np
    h = 0xcbf29ce484222325
    for b in np.ascontiguousarray(arr, dtype=np.int64).tobytes():
        h = ((h ^ b) * 0x100000001b3) & 0xffffffffffffffff
    return f"{h:016x}"


def spawn_ranks(args) -> None:
    """`bench.py --gpus N` outside torchrun: launch N ranks of this script (one per GPU) through
    torch.distributed.run on 127.0.0.1 and exit with its status.  Under torchrun (WORLD_SIZE set)
    the rank count must equal --gpus."""
    ws = os.environ.get("WORLD_SIZE")
    if ws is not None:
        if int(ws) != args.gpus:
            raise SystemExit(f"bench.py --gpus {args.gpus} launched with WORLD_SIZE={ws}")
        return
    if args.gpus <= 1:
        return
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__)] + sys.argv[1:]
    sys.exit(subprocess.call(cmd))


def barrier(ws):
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()


def max_over_ranks(ws, v: float) -> float:
    if ws == 1:
        return v
    import torch
    import torch.distributed as dist
    t = torch.tensor([v], dtype=torch.float64, device="cuda" if BACKEND == "nccl" else "cpu")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:  # noqa: BLE001
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:  # noqa: BLE001
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 5 + i and r[5 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def measured_peaks():
    try:
        return json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    except Exception:  # noqa: BLE001
        return {}


def h2d_peak_gbs(device: int) -> float:
    """Pinned host -> HBM copy rate of this box's link (1 GiB copies, CUDA events; 3 untimed copies
    bring the link out of its idle state, then the best of 8): the roofline of the expert transfers."""
    import torch
    n = 1 << 30
    src = torch.empty(n, dtype=torch.uint8).pin_memory()
    dst = torch.empty(n, dtype=torch.uint8, device=f"cuda:{device}")
    best = float("inf")
    for i in range(11):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        dst.copy_(src, non_blocking=True)
        b.record()
        torch.cuda.synchronize()
        if i >= 3:
            best = min(best, a.elapsed_time(b))
    del src, dst
    return n / (best * 1e-3) / 1e9


def run_reference_driver(wl, sample_tokens: int, reps: int):
    """The unmodified reference simulate_trace (oracle/_ref/moesim_ref, single thread)."""
    ref = os.path.join(ROOT, "oracle", "_ref", "moesim_ref")
    if not os.path.exists(ref):
        return None
    args = [ref, "mode=bench", f"sample_tokens={sample_tokens}", f"reps={reps}"] + \
           [f"{k}={v}" for k, v in wl.ref_args().items()]
    out = subprocess.run(args, check=True, capture_output=True, text=True).stdout
    return json.loads(out)


def cpu_ffn_baseline(eng, wl, trace, tau, cfg, tok0: int, n_tok: int, gpu_out):
    """the same decode's expert FFN on the host cores (baseline/cpu_ffn.c, OpenMP,
    builder-written — NOT the reference, whose CPU path does no FFN arithmetic): for each (token,
    layer) of a bounded sample, out = x + sum_e w_e SwiGLU_e(x) over the selected experts (the
    reference rule's selections, from K1), reading raw bf16 weights from host memory — the layout a
    CPU-only system keeps (its DRAM is not behind a link, so it gains nothing from coding).  With a
    bf16 store the weights are read in place from the pinned store; with a coded store (XB12 / XBH)
    each selected expert is first expanded into a host bf16 buffer through the GPU decoder, outside
    the timed region.  Also the largest relative difference to the GPU decode's outputs."""
    import ctypes as C

    import numpy as np
    import torch
    lib = C.CDLL(os.path.join(ROOT, "baseline", "libcpu_ffn.so"))
    lib.cpu_moe_layer.argtypes = [C.POINTER(C.c_void_p), C.POINTER(C.c_double), C.c_int, C.c_int, C.c_int, C.c_int,
                                  C.POINTER(C.c_double), C.POINTER(C.c_float), C.c_int]
    fmt, _ = eng.experts_format()
    threads = os.cpu_count() or 1
    acts = np.ascontiguousarray(trace.acts[tok0: tok0 + n_tok])
    scores = trace.scores[tok0: tok0 + n_tok]
    dec, single, _, _ = eng.route_trace(acts, scores, trace.fisher, tau, cfg)
    out = np.zeros((n_tok, wl.layers, wl.hidden), dtype=np.float32)
    ebytes = 3 * wl.ffn * wl.hidden * 2
    if fmt != "bf16":  # two expert-sized staging buffers: device (decode target) and pinned host
        d_buf = torch.empty(ebytes // 2, dtype=torch.int16, device="cuda")
        h_bufs = [torch.empty(ebytes // 2, dtype=torch.int16).pin_memory() for _ in range(wl.top_k)]
    moved = 0
    dt = 0.0
    for t in range(n_tok):
        for l in range(wl.layers):
            sel = [int(e) for e in dec[t, l] if e >= 0]
            den = sum(scores[t, l, e] for e in sel)
            wts = (C.c_double * len(sel))(*[1.0 if len(sel) == 1 else scores[t, l, e] / den for e in sel])
            x = acts[t, l]
            xp, op = x.ctypes.data_as(C.POINTER(C.c_double)), out[t, l].ctypes.data_as(C.POINTER(C.c_float))
            if fmt == "bf16":
                ptrs = [eng.expert_host_ptr(l, e) for e in sel]
            else:
                ptrs = []
                for k, e in enumerate(sel):
                    eng.copy_tiles(l, e, 0, wl.tiles, d_buf.data_ptr())
                    torch.cuda.synchronize()  # the engine's copy + decode stream, then a blocking D2H
                    h_bufs[k].copy_(d_buf)
                    ptrs.append(h_bufs[k].data_ptr())
            t0 = time.perf_counter()
            rc = lib.cpu_moe_layer((C.c_void_p * len(sel))(*ptrs), wts, len(sel), wl.hidden, wl.ffn, wl.tiles, xp, op,
                                   threads)
            dt += time.perf_counter() - t0
            moved += len(sel) * ebytes
            assert rc == 0, rc
    moe_gpu = gpu_out.astype(np.float64) - acts.astype(np.float32).astype(np.float64)
    moe_cpu = out.astype(np.float64) - acts.astype(np.float32).astype(np.float64)
    rel = float(np.abs(moe_cpu - moe_gpu).max() / max(np.abs(moe_gpu).max(), 1e-30))
    where = ("in place from the pinned store" if fmt == "bf16" else
             f"from host bf16 buffers (the {fmt} store's records expanded by the GPU decoder, untimed)")
    return {"value": n_tok / dt, "unit": "tok/s", "cores": threads, "kind": "port",
            "label": "not reference: builder-written CPU SwiGLU (baseline/cpu_ffn.c, OpenMP, fp32 accumulation); "
                     "the reference's CPU path does no FFN arithmetic (inc/simulator.hpp:446-462)",
            "sample": f"{n_tok} tokens x {wl.layers} layers of the e2e window, selected experts' raw bf16 weights read "
                      f"{where} ({moved / 1e9:.1f} GB)",
            "host_read_gbs": moved / dt / 1e9, "max_rel_diff_vs_gpu": rel}


def static_config(args, wl, ws):
    """The bench line's `config`: everything fixed by the command line and the workload (shape, batch,
    budget, mode, store format, parallelism) — identical in both arms.  Values the pipeline derives
    (tau, DP capacities, store sizes) go to the line's `derived` object."""
    B = args.batch
    ep_world = ws if ((args.ep or ws > 1) and not args.replicas) else 1
    if ep_world > 1:
        place = ("experts placed by a calibration trace (ep.balanced_owners)" if args.ep_owner == "balanced"
                 else f"expert e on rank e % {ws}")
        comb = "P2P stores into peer memory from the combine epilogue" if args.ep_exchange == "p2p" else "all_gather"
        par = f"ep{ws} ({place}; combine: {comb})"
    else:
        par = f"replicas x{ws}"
    return {"workload": f"{wl.name} batch-{B} decode, HBM expert cache {wl.budget}/{wl.layers * wl.experts} experts "
                        f"(DP), experts offloaded to pinned host memory" +
                        (f"; {B} token streams share the cache (union policy), grouped tcgen05 FFN" if B > 1 else ""),
            "batch": B, "mode": "free-running" if args.free_running else "trace-replay",
            "layers": wl.layers, "experts": wl.experts, "top_k": wl.top_k, "hidden": wl.hidden, "ffn": wl.ffn,
            "budget": wl.budget, "tiles": wl.tiles, "lookahead": wl.lookahead, "trace_tokens": wl.tokens,
            "store_format": args.store_format, "parallelism": par,
            "l2": "no flush needed: resident experts (>=22 GB) >> 126 MB L2"}


def reference_arm(args):
    ws, rank, _ = dist_init()
    if rank != 0:
        return
    wl = workload(args)
    warm = max(1, args.warmup)
    r = run_reference_driver(wl, wl.tokens, warm + args.steps)
    if r is None:
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/moesim_ref not built (needs /root/reference)"}))
        return
    # simulate_mean_s includes warm-up reps; the per-rep best is the steady number
    per_rep = r["simulate_best_s"]
    value = r["tokens"] / per_rep
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "tok/s", "n_gpus": ws, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": 1e3 * per_rep / r["tokens"], "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "fp64", "data": "synthetic",
        "config": static_config(args, wl, ws),
        "reference_sample": {"tokens": r["tokens"], "what": "the reference simulate_trace over the same trace "
                             "(stream 0 at batch > 1: the reference is batch-1)"},
        "on_demand_loads_per_token": r["on_demand_loads"] / r["tokens"],
        "cpu_baseline": {"value": value, "unit": "tok/s", "cores": 1, "kind": "reference",
                         "sample": f"moesim simulate_trace over the {r['tokens']}-token trace, best of "
                                   f"{warm + args.steps} reps (tick model: no FFN arithmetic, no weight movement)"},
        "e2e": {"value": value, "unit": "tok/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


def ours(args):
    import numpy as np
    import torch

    import paper_2408_10284_b200 as P
    from paper_2408_10284_b200 import ep as EP

    ws, rank, local = dist_init()
    torch.cuda.set_device(local)
    wl = workload(args)
    spec = P.ModelSpec(wl.layers, wl.experts, wl.top_k, wl.hidden)
    cfg = P.SimConfig(wl.tiles, wl.tile_transfer, wl.tile_compute, wl.attention, wl.gate_time, wl.lookahead,
                      P.PolicyFlags(wl.gating, wl.prefetch, True))
    t_setup = time.time()
    eng = P.Engine(spec, local)
    use_ep = (args.ep or ws > 1) and not args.replicas
    ep_world = ws if use_ep else 1
    ep_rank = rank if use_ep else 0
    seed_off = 0 if use_ep else rank  # replicas decode different streams; EP shards share one
    # the reference's offline pipeline on this engine; each stage timed once,
    # like the reference arm times its own (oracle/_ref/moesim_ref mode=bench)
    pipe_ms = {}
    tp = time.perf_counter()
    trace = eng.generate_trace(P.SynthConfig(spec, wl.tokens, wl.concentration, wl.drift, wl.gate_seed,
                                             wl.token_seed + seed_off, False, wl.fisher_scales, wl.drift_scales))
    pipe_ms["generate_trace"], tp = (time.perf_counter() - tp) * 1e3, time.perf_counter()
    tau, realized = P.calibrate_threshold(spec, trace.scores, trace.fisher, wl.target_single_ratio)
    pipe_ms["calibrate_threshold"], tp = (time.perf_counter() - tp) * 1e3, time.perf_counter()
    alpha, beta = eng.generate_profiles(trace.acts, trace.scores, trace.fisher, tau)
    pipe_ms["generate_profiles"], tp = (time.perf_counter() - tp) * 1e3, time.perf_counter()
    caps, exp_loads = P.dp_allocate(spec, P.build_cost_table(spec, alpha, beta), wl.budget)
    pipe_ms["cost_table_and_dp_allocate"] = (time.perf_counter() - tp) * 1e3
    expert_bytes = 3 * wl.ffn * wl.hidden * 2
    W, K, B = args.warmup, args.steps, args.batch
    p2p = ep_world > 1 and args.ep_exchange == "p2p"
    owners = None
    if ep_world > 1:
        # expert placement: balanced by a separate calibration trace of the same model (not the decoded
        # tokens; ep.balanced_owners) or e % G — the same deterministic table on every rank
        if args.ep_owner == "balanced":
            calib = eng.generate_trace(P.SynthConfig(spec, max(wl.tokens, 256), wl.concentration, wl.drift, wl.gate_seed,
                                                     wl.token_seed + 7777, False, wl.fisher_scales, wl.drift_scales))
            eng.load_gates(trace.gates)
            sim = eng.simulate_trace(calib.acts, calib.scores, calib.fisher, caps, tau, cfg, wl.seed)
            owners = EP.balanced_owners(sim.timeline, wl.layers, wl.experts, ep_world)
            del calib
        else:
            owners = np.array([[e % ep_world for e in range(wl.experts)] for _ in range(wl.layers)], dtype=np.int32)
    # host RAM: every expert this rank holds is pinned (an EP shard pins only its own);
    # only a host that cannot hold them aliases blocks (single-GPU 8x22B on a small host)
    held = int((owners == ep_rank).sum()) if owners is not None else wl.layers * wl.experts
    alias = 0
    try:
        avail = int(open("/proc/meminfo").read().split("MemAvailable:")[1].split()[0]) * 1024
        per_rank = int(0.85 * avail / max(1, int(os.environ.get("LOCAL_WORLD_SIZE", ws))))
        # a coded store pins its records only (~0.67 / 0.75 of the bf16 bytes for XBH / XB12)
        held_bytes = {"bf16": 1.0, "xb12": 0.76, "xbh": 0.68}[args.store_format] * expert_bytes
        if per_rank < held * held_bytes:
            alias = max(1, int(per_rank // held_bytes))
    except Exception:  # noqa: BLE001
        pass
    if args.host_alias is not None:
        alias = args.host_alias
    elif alias and ep_world > 1:
        raise SystemExit(f"rank {rank}: the expert-parallel shard needs {held * held_bytes / 1e9:.0f} GB of pinned "
                         f"host memory, {per_rank / 1e9:.0f} GB available per rank (pass --host-alias to alias blocks)")
    link_peak = h2d_peak_gbs(local)
    t0 = time.time()
    eng.experts_init(wl.ffn, wl.tiles, seed=1234, host_alias=alias, expert_owner=owners, rank=ep_rank,
                     store_format=args.store_format)
    t_store = time.time() - t0
    store_info = eng.experts_info()
    store_fmt, store_link_bytes = eng.experts_format()
    # B token streams (config 4): stream b = the reference generator with token_seed + b (same gates)
    acts, scores = trace.acts, trace.scores
    total_tokens = wl.tokens
    if B > 1:
        total_tokens = W + 2 * K
        streams = [trace] + [eng.generate_trace(P.SynthConfig(spec, total_tokens, wl.concentration, wl.drift,
                                                              wl.gate_seed, wl.token_seed + 1000 * seed_off + b, False,
                                                              wl.fisher_scales, wl.drift_scales))
                             for b in range(1, B)]
        acts = np.stack([s.acts[:total_tokens] for s in streams], axis=1)      # [T][B][L][d]
        scores = np.stack([s.scores[:total_tokens] for s in streams], axis=1)  # [T][B][L][N]
        del streams
    else:
        acts, scores = acts[:, None], scores[:, None]

    def begin(capacities):
        eng.decode_begin(capacities, trace.fisher, tau, cfg, wl.seed, total_tokens, args.staging, batch=B,
                         ep_rank=ep_rank, ep_world=ep_world, free_running=args.free_running,
                         concentration=wl.concentration, expert_owner=owners)
        if p2p:  # swap exchange regions (CUDA IPC handles) and connect: outputs come back already summed
            import torch.distributed as dist
            _, handle = eng.decode_ep_export(max(W, K, 1))
            handles = [None] * ep_world
            dist.all_gather_object(handles, handle)
            eng.decode_ep_connect(peer_ptrs=[0] * ep_world, peer_ipc=handles)

    begin(caps)
    # token inputs: device copies for the value window, pinned host copies for the e2e window
    d_acts = torch.from_numpy(np.ascontiguousarray(acts[: W + K])).cuda()
    d_scores = torch.from_numpy(np.ascontiguousarray(scores[: W + K])).cuda()
    d_hidden = torch.zeros((W + K, B, wl.layers, wl.hidden), dtype=torch.float32, device="cuda")
    h_acts = torch.from_numpy(np.ascontiguousarray(acts[W + K: W + 2 * K])).pin_memory()
    h_scores = torch.from_numpy(np.ascontiguousarray(scores[W + K: W + 2 * K])).pin_memory()
    h_hidden = torch.zeros((K, B, wl.layers, wl.hidden), dtype=torch.float32).pin_memory()
    del acts, scores
    torch.cuda.synchronize()
    setup_s = time.time() - t_setup

    def dev_call(a, b):
        step_bytes = B * wl.layers * wl.hidden
        return eng.decode_tokens(d_acts.data_ptr() + a * step_bytes * 8,
                                 d_scores.data_ptr() + a * B * wl.layers * wl.experts * 8,
                                 (d_hidden.data_ptr() + a * step_bytes * 4, b - a), on_device=True)

    # warm-up (untimed)
    if W:
        dev_call(0, W)
    s0 = eng.decode_stats()
    # ---- timed: K tokens, inputs resident in HBM ----
    barrier(ws)
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        if ep_world > 1 and not p2p:
            # the cross-shard combine (all_gather + fixed-order sum) is part of the step
            t_ev0, t_ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            t_ev0.record()
            dev_call(W, W + K)
            combined = EP.combine_partials(d_hidden[W: W + K])
            t_ev1.record()
            torch.cuda.synchronize()
            gpu_ms = t_ev0.elapsed_time(t_ev1)
            del combined
        else:
            gpu_ms = dev_call(W, W + K)
        torch.cuda.synchronize()
    barrier(ws)
    s1 = eng.decode_stats()
    gpu_ms_max = max_over_ranks(ws, gpu_ms)
    # ---- e2e: one C-ABI call per token with pinned host buffers ----
    if args.timeline:
        eng.decode_record_timeline(True)
    barrier(ws)
    torch.cuda.synchronize()
    w0 = time.perf_counter()
    for i in range(K):
        ah = h_acts[i: i + 1].numpy()
        sh = h_scores[i: i + 1].numpy()
        eng.decode_tokens(ah, sh, h_hidden[i: i + 1].numpy())
        if ep_world > 1 and not p2p:
            EP.combine_partials(h_hidden[i: i + 1].cuda(non_blocking=True)).cpu()
    torch.cuda.synchronize()
    e2e_s = max_over_ranks(ws, time.perf_counter() - w0)
    barrier(ws)
    timeline = None
    if args.timeline:
        from paper_2408_10284_b200 import timeline as TLM
        path = args.timeline if ws == 1 else f"{args.timeline}.rank{rank}"
        n_ev = eng.decode_timeline_write(path)
        ev = TLM.load(path)
        copies = [e for e in ev if e["kind"] == "tile_transfer"]
        launches = {e["launch"]: (e["start"], e["end"]) for e in ev if "launch" in e}
        t_lo = min(e["start"] for e in ev)
        t_hi = max(e["end"] for e in ev)
        timeline = {"path": path, "events": n_ev, "window_us": t_hi - t_lo,
                    "link_busy_frac": sum(e["end"] - e["start"] for e in copies) / (t_hi - t_lo),
                    "ffn_busy_frac": sum(b - a for a, b in launches.values()) / (t_hi - t_lo),
                    "tile_copies": len(copies),
                    "on_demand_tiles": sum(1 for e in copies if e["request"] == "on_demand" or e["promoted"]),
                    "causality_problems": len(TLM.check_causality(ev)),
                    "stream_overlap_problems": len(TLM.check_stream_exclusivity(ev))}
    res = eng.decode_end(cfg, total_tokens)
    st_end = res.stats
    resident = None
    hbm_total = torch.cuda.get_device_properties(local).total_memory
    resident_bytes = (held + 32) * expert_bytes
    if not args.no_resident_check and resident_bytes > 0.85 * hbm_total:
        resident = {"skipped": f"all {wl.layers * wl.experts} experts need {resident_bytes / 1e9:.0f} GB of HBM per GPU"}
    elif not args.no_resident_check:
        # same inputs, every expert resident: the FFN launches cover whole experts and nothing waits on
        # the host link, which isolates the kernel's streaming rate inside the decode step
        begin([wl.experts] * wl.layers)
        dev_call(0, W)
        r0 = eng.decode_stats()
        barrier(ws)
        torch.cuda.synchronize()
        g_ms = dev_call(W, W + K)
        torch.cuda.synchronize()
        r1 = eng.decode_stats()
        eng.decode_end(None, None, timeline=False)
        dr = {k: r1[k] - r0[k] for k in r0 if isinstance(r0[k], (int, float))}
        rb = dr["ffn_gate_up_bytes"] + dr["ffn_down_bytes"]
        ach = rb / (dr["ffn_ms"] * 1e-3) / 1e9 if dr["ffn_ms"] > 0 else 0.0
        resident = {"tok_s": ws * B * K / (max_over_ranks(ws, g_ms) * 1e-3), "ms_per_step": g_ms / K,
                    "ffn_achieved_gbs": ach, "ffn_frac": ach / measured_peaks().get("hbm_gbs", 6650.0),
                    "ffn_share_of_step": dr["ffn_ms"] / g_ms if g_ms > 0 else None,
                    "ffn_launches": dr["ffn_launches"], "router_us_per_layer": 1e3 * dr["router_ms"] / max(1, K * wl.layers),
                    "host_wait_k1_ms_per_step": dr["host_sync_ms"] / K, "host_step_ms_per_step": dr["host_step_ms"] / K,
                    "speculative_ffn": {"launches": int(dr["spec_launches"]), "hits": int(dr["spec_hits"])},
                    "budget": wl.layers * wl.experts}
    free = None
    if B == 1 and not args.free_running and ep_world == 1 and not args.no_resident_check:
        # the realistic autoregressive mode beside the trace replay: layer l > 0 routes and computes on
        # layer l-1's output (per-layer K1 + host sync), same budget, same store, CUDA events
        eng.decode_begin(caps, trace.fisher, tau, cfg, wl.seed, total_tokens, args.staging, batch=1,
                         free_running=True, concentration=wl.concentration)
        wf, kf = 2, min(K, 4)
        dev_call(0, wf)
        f0 = eng.decode_stats()
        torch.cuda.synchronize()
        f_ms = dev_call(wf, wf + kf)
        f1 = eng.decode_stats()
        eng.decode_end(None, None, timeline=False)
        df = {k: f1[k] - f0[k] for k in f0 if isinstance(f0[k], (int, float))}
        fb = df["ffn_gate_up_bytes"] + df["ffn_down_bytes"]
        free = {"tok_s": kf / (f_ms * 1e-3), "ms_per_step": f_ms / kf, "tokens": kf,
                "ffn_frac": fb / (df["ffn_ms"] * 1e-3) / 1e9 / measured_peaks().get("hbm_gbs", 6650.0)
                if df["ffn_ms"] > 0 else None,
                "router_launches": int(df["router_launches"]), "host_wait_k1_ms_per_step": df["host_sync_ms"] / kf,
                "speculative_ffn": {"launches": int(df["spec_launches"]), "hits": int(df["spec_hits"])},
                "note": "free-running: decisions from the gates on the evolving hidden state (no reference "
                        "counterpart; per-step parity in tests/test_free_running_gpu.py)"}
    # on-demand loads per token in the timed window (tile 0 of each on-demand expert)
    tl = res.timeline
    od_mask = (tl[:, 1] == 3) & (tl[:, 7] == 0)
    tokens_col = tl[:, 4]
    od_timed = int((od_mask & (tokens_col >= W) & (tokens_col < W + K)).sum())
    act_timed = int((((tl[:, 1] == 2) | ((tl[:, 1] == 3) & (tl[:, 7] == 0))) & (tokens_col >= W) & (tokens_col < W + K)).sum())

    d = {k: s1[k] - s0[k] for k in s0 if isinstance(s0[k], (int, float))}
    per_rank_copy = [int(d["copy_bytes"])]
    per_rank_store = [{"pinned_gb": round(store_info["pinned_bytes"] / 1e9, 2), "experts": held,
                       "numa_node": store_info["numa_node"]}]
    if ws > 1:  # every shard's host-link bytes (EP: the busiest shard bounds the step) and pinned store
        import torch.distributed as dist
        per_rank_copy = [None] * ws
        dist.all_gather_object(per_rank_copy, int(d["copy_bytes"]))
        gathered = [None] * ws
        dist.all_gather_object(gathered, per_rank_store[0])
        per_rank_store = gathered
    ffn_ms = d["ffn_ms"]
    ffn_bytes = d["ffn_gate_up_bytes"] + d["ffn_down_bytes"]
    peaks = measured_peaks()
    hbm_peak = peaks.get("hbm_gbs", 6650.0)
    # DRAM traffic per launch from the committed ncu capture of the same kernel, scaled to this run's
    # mean launch size (traffic / algorithmic bytes is a property of the kernel's access pattern)
    traffic, traffic_src = None, None
    try:
        src = "ncu_r2_traffic.json"
        prof = json.load(open(os.path.join(ROOT, "profiles", src)))
        keys = ["grouped_kernel<0>", "grouped_kernel<1>"] if B > 1 else ["ffn_ring_kernel<1>"]
        alg = sum(prof[k]["algorithmic_bytes"] for k in keys)
        dram = sum((sum(prof[k]["dram_bytes"]) / len(prof[k]["dram_bytes"])) if isinstance(prof[k]["dram_bytes"], list)
                   else prof[k]["dram_bytes"] for k in keys)
        traffic = dram / alg * (ffn_bytes / max(1, d["ffn_launches"]))
        traffic_src = f"profiles/{src}: {', '.join(keys)} DRAM bytes / algorithmic bytes = {dram / alg:.4f}"
    except Exception:  # noqa: BLE001
        pass
    achieved = ffn_bytes / (ffn_ms * 1e-3) / 1e9 if ffn_ms > 0 else 0.0
    copy_gbs = d["copy_bytes"] / (d["copy_busy_ms"] * 1e-3) / 1e9 if d["copy_busy_ms"] > 0 else None

    if rank != 0:
        return
    streams = 1 if ep_world > 1 else ws  # EP shards decode one stream together
    value = streams * B * K / (gpu_ms_max * 1e-3)
    decoded = W + 2 * K
    line = {
        "metric": METRIC, "value": value, "unit": "tok/s", "n_gpus": ws, "steps": K, "warmup": W,
        "ms_per_step": gpu_ms_max / K, "higher_is_better": True, "scaling": "strong" if ep_world > 1 else "weak",
        "vs_baseline": None,
        "dtype": "bf16", "data": "synthetic: reference generator (demo8 settings) trace + counter-based random-init "
                                 "bf16 experts",
        "config": static_config(args, wl, ws),
        "derived": {"tau": tau, "realized_single_ratio": realized, "capacities": [int(c) for c in caps],
                    "dp_expected_loads_per_token": exp_loads, "host_alias": alias,
                    "expert_store_per_rank": per_rank_store, "store_format": store_fmt,
                    "store_link_bytes_per_expert": store_link_bytes / max(1, held)},
        "on_demand_loads_per_token": od_timed / K,
        "experts_activated_per_token": act_timed / K,
        "on_demand_loads_per_token_session": res.metrics["on_demand_loads"] / decoded,
        "roofline": {"bound": "hbm", "kernel": ("K3 grouped tcgen05 SwiGLU (grouped_kernel<0/1>)" if B > 1 else
                                                "K2 TMA bulk-copy ring SwiGLU expert streaming (ffn_ring_kernel)"),
                     "achieved": achieved,
                     "peak": hbm_peak, "unit": "GB/s", "frac": achieved / hbm_peak, "traffic": traffic, "traffic_source": traffic_src,
                     "launches": d["ffn_launches"], "bytes_per_launch": ffn_bytes / max(1, d["ffn_launches"]),
                     "ms_per_launch": ffn_ms / max(1, d["ffn_launches"]),
                     "algorithmic_bytes": "3*d*ffn/tiles*2 B per (expert, tile) segment: every bf16 weight once",
                     "peak_source": "MEASURED_PEAKS.json hbm_gbs" if "hbm_gbs" in peaks else "fallback 6.65 TB/s"},
        # the coded store's tile decode kernel (XB12 / XBH) on the copy engine's decode stream
        "roofline_decode": ({"bound": "hbm", "kernel": f"{store_fmt} tile decode ({'decode_kernel + patch_kernel'})",
                             "achieved": d["record_decode_bytes"] / (d["record_decode_ms"] * 1e-3) / 1e9,
                             "peak": hbm_peak, "unit": "GB/s",
                             "frac": d["record_decode_bytes"] / (d["record_decode_ms"] * 1e-3) / 1e9 / hbm_peak,
                             "launches": d["record_decodes"],
                             "ms_per_launch": d["record_decode_ms"] / d["record_decodes"],
                             "bytes_per_launch": d["record_decode_bytes"] / d["record_decodes"],
                             "algorithmic_bytes": "record bytes read + 2 B per bf16 value written, per tile",
                             "note": "CUDA events on the decode stream; decodes overlap the FFN and the copies"}
                            if d.get("record_decodes") else None),
        "host_link": {"copy_bytes": d["copy_bytes"], "copy_bytes_per_rank": per_rank_copy, "copy_busy_ms": d["copy_busy_ms"], "achieved_gbs": copy_gbs,
                      "tile_copies": d["tile_copies"], "stall_ms": d["stall_ms"],
                      "copy_hidden_frac": (1.0 - d["stall_ms"] / d["copy_busy_ms"]) if d["copy_busy_ms"] > 0 else None,
                      # north-star ">= 90 % of prefetch transfer hidden": prefetches the logical engine
                      # never promoted to on-demand, vs the compute-stream wait on their tiles
                      "prefetch_copy_ms": d["prefetch_copy_ms"], "prefetch_stall_ms": d["prefetch_stall_ms"],
                      "prefetch_tile_copies": d["prefetch_tile_copies"],
                      "prefetch_used_copy_ms": d["prefetch_used_copy_ms"],
                      # of the consumed prefetch copy time, the part the compute stream did not wait for
                      "prefetch_hidden_frac": (1.0 - d["prefetch_stall_ms"] / d["prefetch_used_copy_ms"])
                      if d["prefetch_used_copy_ms"] > 0 else None,
                      "prefetch_wasted_frac": (1.0 - d["prefetch_used_copy_ms"] / d["prefetch_copy_ms"])
                      if d["prefetch_copy_ms"] > 0 else None,
                      "link_busy_frac": d["copy_busy_ms"] / gpu_ms if gpu_ms > 0 else None,
                      "peak_gbs": link_peak, "peak_source": "pinned 1 GiB H2D copies, best of 8 after 3 warm-up copies, measured in this run",
                      "frac": (copy_gbs / link_peak) if copy_gbs else None,
                      # step lower bound if the link were the only cost: bytes moved / link peak
                      "step_bound_ms": d["copy_bytes"] / (link_peak * 1e9) * 1e3 / K,
                      "step_frac_of_link_bound": (d["copy_bytes"] / (link_peak * 1e9) * 1e3 / K) / (gpu_ms / K)
                      if gpu_ms > 0 else None},
        "time_split_ms": {"ffn": ffn_ms, "router": d["router_ms"], "copy_stall": d["stall_ms"], "total": gpu_ms,
                          "host_wait_k1": d["host_sync_ms"], "host_step": d["host_step_ms"]},
        "router": {"launches": int(d["router_launches"]),
                   "groups_per_launch": K * wl.layers * B / max(1, d["router_launches"]),
                   "us_per_launch": 1e3 * d["router_ms"] / max(1, d["router_launches"]),
                   "us_per_layer": 1e3 * d["router_ms"] / max(1, K * wl.layers),
                   "exact_fallback_items": int(d["router_exact_items"])},
        "gpu_launches": int(d["kernels_launched"]),
        "speculative_ffn": {"launches": int(d["spec_launches"]), "hits": int(d["spec_hits"])},
        "clocks": clk.summary(),
        "e2e": {"value": streams * B * K / e2e_s, "unit": "tok/s",
                "h2d_bytes_per_step": int(B * wl.layers * (wl.hidden + wl.experts) * 8),
                "d2h_bytes_per_step": int(B * wl.layers * wl.hidden * 4)},
        "setup_s": {"total": setup_s, "expert_store": t_store},
        "host": host_info(),
        "comm": COMM,
        "slots": {"total": st_end["slots_total"], "staging_high_water": st_end["staging_high_water"]},
    }
    if resident is not None:
        line["all_resident_window"] = resident
    if timeline is not None:
        line["physical_timeline"] = timeline
    if free is not None:
        line["free_running_window"] = free
    if B == 1 and not args.free_running and rank == 0:
        # like-for-like with the reference arm: the same function (simulate_trace: every routing
        # decision + the tick-model cache / transfer engine, no weights moved) on the same 64-token
        # trace, through the C ABI from pinned host buffers (K1 on the GPU, C++ engine), wall clock,
        # best of the reps; metrics must equal the unmodified reference's
        n_sim = min(wl.tokens, trace.acts.shape[0])
        p_acts = torch.from_numpy(np.ascontiguousarray(trace.acts[:n_sim])).pin_memory()
        p_scores = torch.from_numpy(np.ascontiguousarray(trace.scores[:n_sim])).pin_memory()
        best, sim = float("inf"), None
        for _ in range(max(1, args.warmup) + K):
            t0 = time.perf_counter()
            sim = eng.simulate_trace(p_acts.numpy(), p_scores.numpy(), trace.fisher, caps, tau, cfg, wl.seed)
            best = min(best, time.perf_counter() - t0)
        sim_line = {"tok_s": n_sim / best, "ms_per_call": best * 1e3, "tokens": n_sim, "reps": max(1, args.warmup) + K,
                    "h2d_bytes_per_call": int(p_acts.numel() * 8 + p_scores.numel() * 8),
                    "timeline_events": int(len(sim.timeline))}
        if not args.no_cpu_baseline:
            rr = run_reference_driver(wl, n_sim, 5)
            if rr is not None:
                sim_line["reference_tok_s"] = rr["tokens"] / rr["simulate_best_s"]
                sim_line["metrics_equal_reference"] = all(rr["metrics"][k] == v for k, v in sim.metrics.items()) and \
                    rr["metrics"]["on_demand_loads_per_layer"] == [int(v) for v in sim.on_demand_loads_per_layer] and \
                    rr.get("hash_timeline") == fnv1a_i64(sim.timeline)
        line["simulate_trace"] = sim_line
        line["comparison_note"] = ("value / e2e: the physical decode (experts moved over the host link and computed); "
                                   "the reference arm times the reference's tick-model simulate_trace, which moves no "
                                   "weights -- the like-for-like figure is simulate_trace.tok_s vs "
                                   "simulate_trace.reference_tok_s")
    if not args.no_cpu_baseline and ws == 1 and B == 1 and not args.free_running:
        try:
            n_cpu = min(K, 3)
            line["cpu_baseline_ffn"] = cpu_ffn_baseline(eng, wl, trace, tau, cfg, W + K, n_cpu, h_hidden[:n_cpu, 0].numpy())
        except Exception as e:  # noqa: BLE001
            line["cpu_baseline_ffn"] = {"value": None, "unavailable": str(e)[:200]}
    if not args.no_cpu_baseline:
        try:
            r = run_reference_driver(wl, decoded, 20)
            if r is not None and args.free_running:
                line["cpu_baseline"] = {"value": r["tokens"] / r["simulate_best_s"], "unit": "tok/s", "cores": 1,
                                        "kind": "reference",
                                        "sample": f"unmodified moesim simulate_trace over {r['tokens']} replayed tokens "
                                                  "(the reference has no free-running mode)"}
            if r is not None and B == 1 and not args.free_running and "tau" in r:
                ref_ms = {"generate_trace": r["generate_s"] * 1e3, "calibrate_threshold": r["calibrate_s"] * 1e3,
                          "generate_profiles": r["profile_s"] * 1e3, "cost_table_and_dp_allocate": r["allocate_s"] * 1e3}
                line["offline_pipeline"] = {
                    "workload": f"{wl.name}, {wl.tokens}-token trace (first call of each stage, wall clock)",
                    "ours_ms": pipe_ms, "reference_ms": ref_ms,
                    # the stages' outputs equal the unmodified reference's, bit for bit
                    "equal": {"tau": r["tau"] == tau, "alpha": r["alpha"] == [float(v) for v in alpha],
                              "beta": r["beta"] == [float(v) for v in beta],
                              "capacities": r["capacities"] == [int(c) for c in caps]}}
            if r is not None and not args.free_running:
                line["cpu_baseline"] = {"value": r["tokens"] / r["simulate_best_s"], "unit": "tok/s", "cores": 1,
                                        "kind": "reference",
                                        "sample": f"unmodified moesim simulate_trace over the same {r['tokens']} decoded "
                                                  "tokens, best of 20 (tick model: no FFN arithmetic, no weight "
                                                  "movement)"}
                if B == 1:
                    # rank 0 decodes the reference's own stream (token_seed + 0) in every mode, so its
                    # logical trace must equal the reference's: the whole SimMetrics struct
                    # (inc/simulator.hpp:130-166) and the event timeline, hashed like the reference's
                    rm = r["metrics"]
                    ours_m = dict(res.metrics)
                    ours_m["on_demand_loads_per_layer"] = [int(v) for v in res.on_demand_loads_per_layer]
                    ours_m["latency_per_token"] = [int(v) for v in res.latency_per_token[:decoded]]
                    diff = sorted(k for k in rm if rm[k] != ours_m.get(k))
                    ours_hash = fnv1a_i64(res.timeline)
                    line["parity"] = {"tokens": decoded, "metrics_fields": len(rm), "metrics_differ": diff,
                                      "on_demand_loads": [r["on_demand_loads"], res.metrics["on_demand_loads"]],
                                      "timeline_events": [r["timeline_events"], int(len(res.timeline))],
                                      "hash_timeline": [r["hash_timeline"], ours_hash],
                                      "equal": not diff and r["hash_timeline"] == ours_hash
                                      and r["timeline_events"] == len(res.timeline)}
                else:
                    line["cpu_baseline"]["sample"] += ("; the reference is batch-1: it decodes stream 0 only, its "
                                                       "tok/s is per single stream")
        except Exception as e:  # noqa: BLE001
            line["cpu_baseline"] = {"value": None, "unavailable": str(e)[:200]}
    print(json.dumps(line))


def run_reference_mode(wl, mode: str, **extra):
    """The unmodified reference in another mode of oracle/_ref/moesim_ref (compare / save / load)."""
    ref = os.path.join(ROOT, "oracle", "_ref", "moesim_ref")
    if not os.path.exists(ref):
        return None
    args = [ref, f"mode={mode}"] + [f"{k}={v}" for k, v in {**wl.ref_args(), **extra}.items()]
    return json.loads(subprocess.run(args, check=True, capture_output=True, text=True).stdout)


def pipeline_bench(args):
    """SURVEY §8(f) rows on this engine vs the unmodified reference, same workload, wall clock of each
    stage's first call: generate_trace, calibrate_threshold, train_first_gate, generate_profiles,
    cost table + DP, simulate_trace, the 7-row ablation grid (compare_policies) and the artifact files
    (save / load of trace + gates + profiles + threshold + allocation + cost table)."""
    import tempfile

    import numpy as np

    import paper_2408_10284_b200 as P
    from paper_2408_10284_b200 import io as IO
    from paper_2408_10284_b200 import workloads as Wk

    ws, rank, local = dist_init()
    if rank != 0:
        return
    cases = [Wk.tiny(), Wk.mixtral_8x7b(tokens=64), Wk.mixtral_8x7b(tokens=64, train_first_gate=True),
             Wk.mixtral_8x7b(tokens=8, name="mixtral-8x7b-files")]
    for wl in cases:
        spec = P.ModelSpec(wl.layers, wl.experts, wl.top_k, wl.hidden)
        cfg = P.SimConfig(wl.tiles, wl.tile_transfer, wl.tile_compute, wl.attention, wl.gate_time, wl.lookahead,
                          P.PolicyFlags(wl.gating, wl.prefetch, True))
        ms = {}
        with P.Engine(spec, local) as eng:
            t = time.perf_counter()
            tr = eng.generate_trace(P.SynthConfig(spec, wl.tokens, wl.concentration, wl.drift, wl.gate_seed,
                                                  wl.token_seed, False, wl.fisher_scales, wl.drift_scales))
            ms["generate_trace"], t = (time.perf_counter() - t) * 1e3, time.perf_counter()
            tau, realized = P.calibrate_threshold(spec, tr.scores, tr.fisher, wl.target_single_ratio)
            ms["calibrate_threshold"], t = (time.perf_counter() - t) * 1e3, time.perf_counter()
            fg = None
            if wl.train_first_gate:
                fg = eng.train_first_gate(tr.acts, tr.scores, wl.train_lr, wl.train_steps, wl.train_seed)
                eng.load_gates(tr.gates, fg)
                ms["train_first_gate"], t = (time.perf_counter() - t) * 1e3, time.perf_counter()
            alpha, beta = eng.generate_profiles(tr.acts, tr.scores, tr.fisher, tau)
            ms["generate_profiles"], t = (time.perf_counter() - t) * 1e3, time.perf_counter()
            table = P.build_cost_table(spec, alpha, beta)
            caps, total_cost = P.dp_allocate(spec, table, wl.budget)
            ms["cost_table_and_dp_allocate"], t = (time.perf_counter() - t) * 1e3, time.perf_counter()
            sim = eng.simulate_trace(tr.acts, tr.scores, tr.fisher, caps, tau, cfg, wl.seed)
            ms["simulate_trace"], t = (time.perf_counter() - t) * 1e3, time.perf_counter()
            rows = eng.compare_policies(tr.acts, tr.scores, tr.fisher, alpha, beta, tau, cfg, wl.budget, wl.seed)
            ms["compare_policies"] = (time.perf_counter() - t) * 1e3
            files = None
            if wl.tokens <= 8 or wl.hidden <= 256:
                with tempfile.TemporaryDirectory() as d:
                    t = time.perf_counter()
                    IO.save_trace(os.path.join(d, "trace.jsonl"), spec, tr.acts, tr.scores, tr.selected)
                    IO.save_gates(os.path.join(d, "gates.json"), spec, tr.gates, fg, wl.train_lr, wl.train_steps,
                                  wl.train_seed)
                    ph = IO.save_profiles(os.path.join(d, "profiles.json"), spec, alpha, beta, tr.fisher)
                    IO.save_threshold(os.path.join(d, "threshold.json"), tau, wl.target_single_ratio, realized)
                    IO.save_allocation(os.path.join(d, "allocation.json"), caps, wl.budget, total_cost, ph)
                    IO.save_cost_table(os.path.join(d, "cost_table.json"), table)
                    save_ms, t = (time.perf_counter() - t) * 1e3, time.perf_counter()
                    back = IO.load_trace(os.path.join(d, "trace.jsonl"))
                    load_ms = (time.perf_counter() - t) * 1e3
                    size = os.path.getsize(os.path.join(d, "trace.jsonl"))
                    files = {"save_all_ms": save_ms, "load_trace_ms": load_ms, "trace_jsonl_bytes": size,
                             "round_trip_equal": bool(np.array_equal(back.acts, tr.acts)
                                                      and np.array_equal(back.scores, tr.scores))}
        line = {"impl": "ours", "pipeline": wl.name, "tokens": wl.tokens, "ours_ms": ms}
        r = run_reference_driver(wl, wl.tokens, 3)
        if r is not None:
            line["reference_ms"] = {"generate_trace": r["generate_s"] * 1e3, "calibrate_threshold": r["calibrate_s"] * 1e3,
                                    "generate_profiles": r["profile_s"] * 1e3,
                                    "cost_table_and_dp_allocate": r["allocate_s"] * 1e3,
                                    "simulate_trace": r["simulate_best_s"] * 1e3}
            if wl.train_first_gate:
                line["reference_ms"]["train_first_gate"] = r["train_s"] * 1e3
            c = run_reference_mode(wl, "compare")
            line["reference_ms"]["compare_policies"] = c["compare_s"] * 1e3
            cores = os.cpu_count() or 1  # the grid's rows in parallel on every host core
            cj = run_reference_mode(wl, "compare", jobs=cores)
            line["reference_ms"][f"compare_policies_jobs{cores}"] = cj["compare_s"] * 1e3
            line["equal"] = {"tau": r["tau"] == tau, "alpha": r["alpha"] == [float(v) for v in alpha],
                             "beta": r["beta"] == [float(v) for v in beta],
                             "capacities": r["capacities"] == [int(v) for v in caps],
                             "simulate_metrics": all(r["metrics"][k] == v for k, v in sim.metrics.items()),
                             "compare_rows": [(x["metrics"], x["capacities"], x["speedup_vs_baseline"]) for x in rows]
                             == [({k: v for k, v in y["metrics"].items()}, y["capacities"], y["speedup_vs_baseline"])
                                 for y in c["rows"]]}
            if files is not None:
                with tempfile.TemporaryDirectory() as d:
                    s_ = run_reference_mode(wl, "save", dir=d)
                    l_ = run_reference_mode(wl, "load", dir=d)
                files["reference_save_all_ms"] = s_["save_s"] * 1e3
                files["reference_load_trace_ms"] = l_["load_trace_s"] * 1e3
        if files is not None:
            line["files"] = files
        print(json.dumps(line), flush=True)


def main():
    args = parse()
    spawn_ranks(args)
    if args.impl == "reference":
        reference_arm(args)
    elif args.pipeline:
        pipeline_bench(args)
    else:
        ours(args)


if __name__ == "__main__":
    main()
