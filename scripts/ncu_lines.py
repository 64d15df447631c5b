"""Per-source-line stall samples and executed instructions of one ncu report
(kernel built with -lineinfo, captured with --import-source on), summed over
the line ranges given, e.g. the phases of the streamed sweep.
Usage: python scripts/ncu_lines.py <report.ncu-rep> <file-substring> [name:first-last ...]"""
import csv
import io
import subprocess
import sys

rep, fsub = sys.argv[1], sys.argv[2]
ranges = [(a.split(":")[0], *map(int, a.split(":")[1].split("-"))) for a in sys.argv[3:]]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
hdr = None
cur_file = ""
per_line = {}
for r in rows:
    if len(r) == 1 and r[0].startswith("File"):
        cur_file = r[0]
        continue
    if r and r[0] == "#":
        hdr = r
        continue
    if not hdr or len(r) != len(hdr) or fsub not in cur_file:
        continue
    d = dict(zip(hdr, r))
    try:
        line = int(d["#"])
    except ValueError:
        continue
    samp = float(d.get("Warp Stall Sampling (All Samples)", 0) or 0)
    inst = float(d.get("Instructions Executed", 0) or 0)
    per_line[line] = (samp, inst, d.get("Source", "")[:90])
tot_s = sum(v[0] for v in per_line.values()) or 1.0
tot_i = sum(v[1] for v in per_line.values()) or 1.0
print(f"{fsub}: {len(per_line)} lines, {tot_s:.0f} samples, {tot_i:.3g} instructions")
for name, a, b in ranges:
    s = sum(v[0] for k, v in per_line.items() if a <= k <= b)
    i = sum(v[1] for k, v in per_line.items() if a <= k <= b)
    print(f"  {name:24s} lines {a}-{b}: samples {100 * s / tot_s:5.1f}%  instructions {100 * i / tot_i:5.1f}%")
print("top lines:")
for k, v in sorted(per_line.items(), key=lambda x: -x[1][0])[:25]:
    print(f"  {k:5d} {100 * v[0] / tot_s:5.1f}% {100 * v[1] / tot_i:5.1f}%  {v[2]}")
