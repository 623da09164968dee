"""Per-source-line warp-stall samples from an ncu report (cuda,sass source page).

  python tools/ncu_lines.py report.ncu-rep [top]
"""
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out))
hdr, cur_file, agg = None, "", {}
for r in rows:
    if r and r[0] == "File Path":
        cur_file = r[1].split("/")[-1]
    elif r and r[0] == "Line No":
        hdr = r
    elif hdr and len(r) == len(hdr) and r[0]:
        ix = hdr.index("Warp Stall Sampling (All Samples)")
        try:
            s = int(r[ix])
        except ValueError:
            continue
        st = {hdr[j]: int(r[j]) for j in range(len(hdr)) if hdr[j].startswith("stall_") and "Not Issued" not in hdr[j]
              and r[j].isdigit() and int(r[j]) > 0}
        agg[(cur_file, int(r[0]))] = (s, r[1].strip(), st)
tot = sum(v[0] for v in agg.values()) or 1
print(f"total samples {tot}")
for (f, ln), (s, src, st) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    big = sorted(st.items(), key=lambda kv: -kv[1])[:3]
    print(f"{100 * s / tot:5.1f}% {f}:{ln:<4} {src[:70]:70s} " + " ".join(f"{k[6:]}={v}" for k, v in big))
