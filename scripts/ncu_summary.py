"""Summarise one ncu --set full report (first kernel) for profiles/:
key throughput metrics, stall breakdown, top opcodes.
Usage: python scripts/ncu_summary.py <report.ncu-rep> <title> > profiles/<name>.txt"""
import collections
import csv
import io
import subprocess
import sys

rep, title = sys.argv[1], sys.argv[2]


def page(*args):
    out = subprocess.run(["ncu", "-i", rep, *args, "--csv"], capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


raw = page("--page", "raw")
h, units, v = raw[0], raw[1], raw[2]
d = dict(zip(h, v))
u = dict(zip(h, units))
print(title)
print(f"kernel: {d.get('Kernel Name', '')[:140]}")
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "smsp__inst_executed.sum", "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "lts__t_sector_hit_rate.pct",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed"]
for k in keys:
    if k in d:
        print(f"  {k:62s} {d[k]:>16s} {u.get(k, '')}")
stall = {k: float(d[k] or 0) for k in h if k.startswith("smsp__pcsamp_warps_issue_stalled_") and
         not k.endswith("not_issued")}
tot = sum(stall.values()) or 1.0
print("stall samples (% of all samples):")
for k, s in sorted(stall.items(), key=lambda x: -x[1])[:10]:
    print(f"  {k.replace('smsp__pcsamp_warps_issue_stalled_', ''):24s} {100 * s / tot:5.1f}")
src = page("--page", "source", "--print-source", "sass")
if len(src) > 2:
    sh = src[1]
    iE, iS = sh.index("Instructions Executed"), sh.index("Source")
    ops = collections.Counter()
    n = 0.0
    for r in src[2:]:
        if len(r) <= iE or not r[iE]:
            continue
        x = float(r[iE])
        t = r[iS].split()
        if not t:
            continue
        op = (t[1] if t[0].startswith("@") else t[0]).split(".")[0]
        ops[op] += x
        n += x
    print(f"executed warp instructions: {n:.4g}; top opcodes (% of executed):")
    for op, x in ops.most_common(12):
        print(f"  {op:10s} {100 * x / n:5.1f}")
