"""Summarise ncu --set full captures and launch lists (profiles/ tables)."""
import csv
import subprocess
import sys
from collections import defaultdict

KEYS = [("gpu__time_duration.sum", "duration"), ("dram__bytes_read.sum", "DRAM read"),
        ("dram__bytes_write.sum", "DRAM write"), ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM %"),
        ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe %"),
        ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "FMA pipe %"),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue %"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
        ("launch__registers_per_thread", "regs"), ("launch__grid_size", "grid"), ("launch__block_size", "block")]


def full(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    h, u, d = rows[0], rows[1], rows[2]
    v = dict(zip(h, d))
    un = dict(zip(h, u))
    st = []
    for k, x in v.items():
        if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio"):
            try:
                st.append((k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")], float(x)))
            except ValueError:
                pass
    st = sorted(st, key=lambda x: -x[1])[:4]
    res = {name: f"{v.get(k, '-')} {un.get(k, '')}".strip() for k, name in KEYS}
    res["kernel"] = v.get("Kernel Name", "")[:60]
    res["stalls"] = ", ".join(f"{a} {b:.2f}" for a, b in st)
    return res


def launches(path):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    t, n = defaultdict(float), defaultdict(int)
    for r in rows[1:]:
        d = dict(zip(h, r))
        try:
            name = d["Kernel Name"].split("(")[0].replace("void ", "")[:48]
            t[name] += float(d["Metric Value"]) / 1e3
            n[name] += 1
        except (KeyError, ValueError):
            pass
    tot = sum(t.values())
    return [(k, n[k], t[k] / n[k], 100 * t[k] / tot) for k in sorted(t, key=lambda x: -t[x])]


if __name__ == "__main__":
    d = sys.argv[1]
    for c in sys.argv[2:]:
        print(f"## {c}")
        r = full(f"{d}/full_{c}.ncu-rep")
        for k, v in r.items():
            print(f"  {k}: {v}")
        print("  launches (kernel, count, mean us, share of GPU time):")
        for k, n, us, sh in launches(f"{d}/launches_{c}.csv")[:6]:
            print(f"    {k:48s} {n:5d} {us:10.1f} {sh:6.1f}%")
