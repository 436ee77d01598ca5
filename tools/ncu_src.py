"""Summarise an ncu report: per-kernel key metrics and the top source lines by warp-stall samples."""
import csv, subprocess, sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 15
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{kern}", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout.splitlines()
rows = list(csv.reader(out))
hi = next(i for i, r in enumerate(rows[:10]) if "Warp Stall Sampling (All Samples)" in r)
h = rows[hi]
si = h.index("Warp Stall Sampling (All Samples)")
ie = h.index("Instructions Executed")
data = []
for r in rows[hi + 1:]:
    if len(r) > si and r[0] not in ("", "-"):
        try:
            data.append((float(r[si] or 0), r[0], r[1][:110], r[ie]))
        except ValueError:
            pass
tot = sum(d[0] for d in data) or 1
print(kern, "total samples", tot)
for d in sorted(data, reverse=True)[:top]:
    print("%6.0f %5.1f%%  L%s | %s | inst %s" % (d[0], 100 * d[0] / tot, d[1], d[2], d[3]))
