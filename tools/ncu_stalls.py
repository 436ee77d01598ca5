"""Aggregate per-SASS-instruction stall reasons of an ncu report by opcode (and optionally by
source-line range via --print-source cuda,sass correlation).
usage: python tools/ncu_stalls.py report.ncu-rep kernel_regex [opcode_regex]"""
import collections
import csv
import re
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
opre = re.compile(sys.argv[3]) if len(sys.argv) > 3 else None
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}", "--print-source", "sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out))
hi = next(i for i, r in enumerate(rows[:20]) if "Warp Stall Sampling (All Samples)" in r)
h = rows[hi]
cols = [i for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
tot = collections.Counter()
byop = collections.defaultdict(collections.Counter)
for r in rows[hi + 1:]:
    if len(r) < len(h):
        continue
    op = r[1].split()[0] if r[1].split() else "?"
    if op.startswith("@"):
        op = r[1].split()[1]
    op = op.split(".")[0]
    if opre and not opre.search(op):
        continue
    for i in cols:
        try:
            v = float(r[i] or 0)
        except ValueError:
            continue
        tot[h[i]] += v
        byop[op][h[i]] += v
s = sum(tot.values()) or 1
print("total samples", s)
for k, v in tot.most_common(10):
    print(f"  {k:24s} {v:8.0f} {100*v/s:5.1f}%")
print("by opcode (top 12 by samples):")
for op, c in sorted(byop.items(), key=lambda kv: -sum(kv[1].values()))[:12]:
    t = sum(c.values())
    top = ", ".join(f"{k[6:]}={100*v/t:.0f}%" for k, v in c.most_common(3))
    print(f"  {op:10s} {t:8.0f}  {top}")
