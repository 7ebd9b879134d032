"""Per-launch DRAM traffic and duration of the kernels in ncu reports -> profiles/ncu_r2_traffic.json
(read by bench.py's roofline `traffic`).  Usage: python tools/ncu_traffic.py out.json rep1.ncu-rep ...
Algorithmic bytes per launch come from the caller's kernel table below (weights streamed once)."""
import csv
import json
import subprocess
import sys


def launches(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, units = rows[0], rows[1]
    ki = h.index("Kernel Name")
    want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__registers_per_thread",
            "launch__grid_size"]
    scale = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3,
             "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "register/thread": 1, "": 1}
    for r in rows[2:]:
        d = {"kernel": r[ki].split("(")[0].replace("void ", "").split("::")[-1]}
        for w in want:
            if w in h:
                i = h.index(w)
                d[w] = float(r[i].replace(",", "")) * scale.get(units[i], 1)
        yield d


if __name__ == "__main__":
    res = {}
    for rep in sys.argv[2:]:
        for d in launches(rep):
            k = d["kernel"]
            e = res.setdefault(k, {"report": rep, "duration_us": [], "dram_read_bytes": [], "dram_write_bytes": [],
                                   "registers_per_thread": d.get("launch__registers_per_thread"),
                                   "grid": d.get("launch__grid_size")})
            e["duration_us"].append(d["gpu__time_duration.sum"])
            e["dram_read_bytes"].append(d["dram__bytes_read.sum"])
            e["dram_write_bytes"].append(d["dram__bytes_write.sum"])
    json.dump(res, open(sys.argv[1], "w"), indent=1)
    print(json.dumps({k: (len(v["duration_us"]), sum(v["duration_us"]) / len(v["duration_us"])) for k, v in res.items()}))
