"""Warp-stall samples and executed instructions per CUDA source line (ncu source page, cuda+sass
correlation).  usage: python tools/ncu_lines.py report.ncu-rep kernel_regex [top]"""
import csv
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}", "--print-source",
                      "cuda,sass"], capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out))
h = rows[2]
iS = h.index("Warp Stall Sampling (All Samples)")
iI = h.index("Instructions Executed")
src = {}
agg = {}
cur = None
for r in rows[3:]:
    if len(r) < len(h):
        continue
    if r[0] not in ("",):
        cur = int(r[0]) if r[0].isdigit() else None
        if cur is not None:
            src[cur] = r[1]
        continue
    if cur is None:
        continue
    a = agg.setdefault(cur, [0.0, 0.0])
    try:
        a[0] += float(r[iS] or 0)
        a[1] += float(r[iI] or 0)
    except ValueError:
        pass
tot = sum(v[0] for v in agg.values()) or 1
toti = sum(v[1] for v in agg.values()) or 1
print(f"total samples {tot:.0f}, instructions {toti:.3g}")
for ln, (sm, ins) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{ln:5d} {100*sm/tot:5.1f}% samp {100*ins/toti:5.1f}% inst | {src.get(ln, '').strip()[:90]}")
