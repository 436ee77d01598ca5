"""Executed SASS instructions by opcode (ncu source page).  usage: python tools/ncu_ops.py rep kernel_regex"""
import collections
import csv
import subprocess
import sys

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "source", "--csv", "-k", f"regex:{sys.argv[2]}",
                      "--print-source", "sass"], capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out))
hi = next(i for i, r in enumerate(rows[:10]) if "Instructions Executed" in r)
h = rows[hi]
iI, iS = h.index("Instructions Executed"), h.index("Source")
c = collections.Counter()
for r in rows[hi + 1:]:
    if len(r) < len(h) or not r[iS].split():
        continue
    op = r[iS].split()
    o = (op[1] if op[0].startswith("@") else op[0]).split(".")[0]
    try:
        c[o] += float(r[iI] or 0)
    except ValueError:
        pass
t = sum(c.values())
print(f"total {t:.4g}")
for o, v in c.most_common(int(sys.argv[3]) if len(sys.argv) > 3 else 20):
    print(f"{o:10s} {v:12.4g} {v / t * 100:5.1f}%")
