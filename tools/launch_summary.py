"""Summarise an ncu --csv launch list (gpu__time_duration + dram bytes [+ tensor %]) per kernel."""
import collections
import csv
import sys

SCALE_T = {"ns": 1e-3, "nsecond": 1e-3, "us": 1.0, "usecond": 1.0, "ms": 1e3, "msecond": 1e3}
SCALE_B = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}


def summarise(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, mi, vi, ui = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = collections.defaultdict(lambda: collections.defaultdict(float))
    cnt = collections.Counter()
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        k = r[ki].split("(")[0].replace("void ", "").replace("unnamed>::", "")
        v = float(r[vi].replace(",", ""))
        if r[mi] == "gpu__time_duration.sum":
            cnt[k] += 1
            v *= SCALE_T[r[ui]]
        elif r[mi].startswith("dram__bytes"):
            v *= SCALE_B[r[ui]]
        agg[k][r[mi]] += v
    tot = sum(a["gpu__time_duration.sum"] for a in agg.values())
    out = []
    for k, a in sorted(agg.items(), key=lambda x: -x[1]["gpu__time_duration.sum"]):
        t = a["gpu__time_duration.sum"]
        b = a.get("dram__bytes_read.sum", 0) + a.get("dram__bytes_write.sum", 0)
        line = (f"| {k} | {cnt[k]} | {t / cnt[k]:.1f} | {100 * t / tot:.1f} % | {b / 1e6 / cnt[k]:.2f} | "
                f"{b / (t * 1e-6) / 1e9:.0f} |")
        tk = "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"
        if tk in a:
            line += f" {a[tk] / cnt[k]:.1f} |"
        out.append(line)
    return out


if __name__ == "__main__":
    print("| kernel | launches | mean us | share of kernel time | DRAM MB/launch | GB/s | (tensor %) |")
    print("|---|---|---|---|---|---|---|")
    for line in summarise(sys.argv[1]):
        print(line)
