"""Per-kernel SASS opcode summary of a built library (cuobjdump -sass).

Usage: python scripts/sass_summary.py [LIB] [REGEX] [--top N] [--grep OPCODE_REGEX]
Prints, for every kernel whose demangled name matches REGEX, the instruction
count, the Blackwell-specific opcodes (packed FP32, TMEM, bulk TMA, mbarrier,
cp.async) and the N most frequent opcodes.  --grep lists matching instructions.
"""
import collections
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
args = [a for a in sys.argv[1:] if not a.startswith("--")]
lib = args[0] if args else os.path.join(ROOT, "paper_2011_00162_b200", "libptychodd_cuda.so")
pat = re.compile(args[1] if len(args) > 1 else "sweep_stream_kernel|gather_kernel")
top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 14
grep = re.compile(sys.argv[sys.argv.index("--grep") + 1]) if "--grep" in sys.argv else None

BLACKWELL = ("FADD2", "FMUL2", "FFMA2", "LDTM", "STTM", "UTCBAR", "UTCATOMSWS", "UBLKCP", "UTMALDG", "UTMASTG",
             "SYNCS", "LDGSTS", "UTCHMMA", "UTCQMMA", "UTCIMMA")

sass = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
names = {}
cur = None
ops = collections.defaultdict(collections.Counter)
hits = collections.defaultdict(list)
for line in sass.splitlines():
    m = re.match(r"\s*Function : (\S+)", line)
    if m:
        cur = m.group(1)
        continue
    m = re.match(r"\s*/\*[0-9a-f]{4,}\*/\s+(.*?);", line)
    if m and cur:
        ins = m.group(1).strip()
        toks = ins.split()
        op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
        ops[cur][op.split(".")[0]] += 1
        if grep and grep.search(ins):
            hits[cur].append(ins)
dem = subprocess.run(["c++filt"], input="\n".join(ops), capture_output=True, text=True).stdout.splitlines()
for mangled, name in zip(ops, dem):
    if not pat.search(name):
        continue
    c = ops[mangled]
    n = sum(c.values())
    print(f"{name[:150]}\n  instructions: {n}")
    bw = [(o, c[o]) for o in BLACKWELL if c.get(o)]
    print("  Blackwell-specific: " + (", ".join(f"{o} {k}" for o, k in bw) or "none"))
    print("  top: " + ", ".join(f"{o} {k}" for o, k in c.most_common(top)))
    for h in hits.get(mangled, [])[:60]:
        print("    " + h)
