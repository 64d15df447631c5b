"""Per-instruction hot spots of one ncu --set full report (source page, SASS):
top instructions by stall samples and by excess shared-memory wavefronts.
Usage: python scripts/ncu_hot.py <report.ncu-rep> [n]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--print-source", "sass", "--csv"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
idx = {k: i for i, k in enumerate(h)}
data = []
for r in rows[2:]:
    if len(r) < len(h):
        continue
    def f(k):
        try:
            return float(r[idx[k]] or 0)
        except (KeyError, ValueError):
            return 0.0
    data.append((r[idx["Address"]], r[idx["Source"]], f("Warp Stall Sampling (All Samples)"),
                 f("L1 Wavefronts Shared Excessive"), f("stall_mio"), f("stall_short_sb"), f("Instructions Executed")))
tot = sum(d[2] for d in data) or 1
print("top stall-sampled instructions (% of samples, mio, short_sb):")
for d in sorted(data, key=lambda d: -d[2])[:n]:
    print(f"  {d[0]:>6s} {100 * d[2] / tot:5.2f}%  mio {100 * d[4] / tot:4.2f}  ssb {100 * d[5] / tot:4.2f}  {d[1][:90]}")
print("top excess shared wavefronts:")
for d in sorted(data, key=lambda d: -d[3])[:10]:
    if d[3] > 0:
        print(f"  {d[0]:>6s} {d[3]:12.0f}  {d[1][:90]}")
