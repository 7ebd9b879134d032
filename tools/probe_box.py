"""Probe the GPU box: host cores/RAM, PCIe link, pinned H2D/D2H bandwidth, pin cost.

Run under gpurun; prints a JSON summary (also written to gpurun_out/probe.json)."""
import json, os, subprocess, time

def sh(cmd):
    try:
        return subprocess.run(cmd, shell=True, capture_output=True, text=True, timeout=60).stdout.strip()
    except Exception as e:  # noqa: BLE001
        return f"ERR {e}"

out = {}
out["nproc"] = sh("nproc")
out["lscpu_model"] = sh("lscpu | grep 'Model name' | head -1")
out["sockets"] = sh("lscpu | grep -E '^Socket|NUMA node\\(s\\)'")
out["meminfo"] = sh("grep -E 'MemTotal|MemAvailable|HugePages_Total' /proc/meminfo")
out["ulimit_l"] = sh("ulimit -l")
out["pcie"] = sh("nvidia-smi --query-gpu=pcie.link.gen.current,pcie.link.gen.max,pcie.link.width.current,pcie.link.width.max --format=csv")
out["topo"] = sh("nvidia-smi topo -m | head -5")
out["glibc"] = sh("ldd --version | head -1")

import torch
dev = torch.device("cuda:0")
torch.cuda.init()
res = {}
for mb in (16, 88, 256, 1024):
    n = mb << 20
    t0 = time.time()
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    pin_s = time.time() - t0
    d = torch.empty(n, dtype=torch.uint8, device=dev)
    h.fill_(1)
    for _ in range(3):
        d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    reps = max(2, 2048 // mb)
    e0.record()
    for _ in range(reps):
        d.copy_(h, non_blocking=True)
    e1.record(); torch.cuda.synchronize()
    h2d = n * reps / (e0.elapsed_time(e1) / 1e3) / 1e9
    e0.record()
    for _ in range(reps):
        h.copy_(d, non_blocking=True)
    e1.record(); torch.cuda.synchronize()
    d2h = n * reps / (e0.elapsed_time(e1) / 1e3) / 1e9
    res[mb] = {"pin_s": round(pin_s, 4), "h2d_GBps": round(h2d, 2), "d2h_GBps": round(d2h, 2)}
    del h, d
out["copy"] = res
# pin-cost scaling: 8 GiB
t0 = time.time()
big = torch.empty(8 << 30, dtype=torch.uint8, pin_memory=True)
out["pin_8GiB_s"] = round(time.time() - t0, 2)
del big
out["gpu"] = torch.cuda.get_device_name(0)
out["props"] = str(torch.cuda.get_device_properties(0))
print(json.dumps(out, indent=1))
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/probe.json", "w"), indent=1)
