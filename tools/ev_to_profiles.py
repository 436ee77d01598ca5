"""Turn the output of tools/r2_evidence.sh (gpurun_out/ev/) into the committed evidence under profiles/:
bench lines, the ncu launch list, the --set full summaries (+ ncu_traffic.json), the parity summary and
the NEXT-2 part times.  usage: python tools/ev_to_profiles.py [ev_dir] [round_tag]"""
import collections
import json
import os
import re
import shutil
import subprocess
import sys

ev = sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/ev"
tag = sys.argv[2] if len(sys.argv) > 2 else "r2"
prof = "profiles"

for name in ("default", "cfg2b", "cfg3", "cfg5", "cfg4", "reference"):
    src = os.path.join(ev, f"bench_{name}.json")
    line = [x for x in open(src).read().splitlines() if x.startswith("{")][-1]
    json.loads(line)
    with open(os.path.join(prof, f"{tag}_bench_{name}.json"), "w") as fh:
        fh.write(line + "\n")
shutil.copy(os.path.join(ev, "launches_default.csv"), os.path.join(prof, f"{tag}_default_ncu_launches.csv"))
for cfg in ("cfg2", "cfg3", "cfg4"):
    subprocess.run([sys.executable, "tools/ncu_summary.py", os.path.join(ev, f"prof_{cfg}.ncu-rep"), cfg,
                    os.path.join(prof, f"{tag}_{cfg}_ncu_full.md")], check=True)

# parity summary from the LC_PARITY_LOG lines of the GPU suite
agg = collections.OrderedDict()
for ln in open(os.path.join(ev, "parity.jsonl")):
    d = json.loads(ln)
    k = (re.sub(r" v=\d+$", "", d["tag"]), d["direction"])  # per-vector checks of one config together
    a = agg.setdefault(k, {"checks": 0, "rows": 0, "einf": 0.0, "diag": 0.0, "block": 0.0})
    a["checks"] += 1
    a["rows"] += int(d.get("rows", 0))
    a["einf"] = max(a["einf"], d.get("einf", 0.0))
    a["diag"] = max(a["diag"], d.get("diag", 0.0) or 0.0)
    a["block"] = max(a["block"], d.get("block_einf", 0.0) or 0.0)
suite = [x for x in open(os.path.join(ev, "pytest_gpu.log")).read().splitlines() if "passed" in x][-1].strip()
out = [f"# Round-2 GPU parity summary (B200, `pytest -m gpu` with LC_PARITY_LOG, final round-2 build)", "",
       "Every line: the largest value over the checks of that case. E_inf = relative max norm vs the long-double oracle",
       "(PAPER.md:527); diag = per-row |z_i - z*_i| / sum_k |K_ik f_k| (SURVEY C-5); block = round-trip E_inf per 2s-block",
       "(each block against its own max). Gates: E_inf 1e-12 (n <= 1e6) / 1e-11; diag 1e-13; block 1e-13 (random signs) /",
       "1e-10 (all-positive inputs). The `planted` lines are the deliberately corrupted tail block (must exceed the gates);",
       "the `fig3 r=0` lines are the paper's non-decaying round trips (logged, not gated).",
       f"{sum(a['checks'] for a in agg.values())} checks; the suite: {suite} (tests/ -m gpu).", "",
       "| case | direction | checks | rows checked | max E_inf | max diag | max block E_inf |", "|---|---|---|---|---|---|---|"]
for (t, d), a in agg.items():
    out.append(f"| {t} | {d} | {a['checks']} | {a['rows']} | {a['einf']:.2e} | {a['diag']:.2e} | {a['block']:.2e} |")
open(os.path.join(prof, f"{tag}_parity_summary.md"), "w").write("\n".join(out) + "\n")

# NEXT-2 part times
pt = {"note": "NEXT-2 on one B200: device time (CUDA events, 200 reps) of each part of a partitioned single-vector "
              "leg2cheb (tools/part_times.py), parts run alone one after another; partitioned_up_pass = "
              "lc_execute_part phases 0 + 1 (the all-gather of roots and halos between them is not included); on G "
              "GPUs the parts run concurrently"}
for key, pre in (("replicated_up_pass", "part_times"), ("partitioned_up_pass", "part_up")):
    pt[key] = {}
    for nn in ("1e6", "1e7"):
        last = [x for x in open(os.path.join(ev, f"{pre}_{nn}.txt")).read().splitlines() if x.startswith("{")]
        pt[key][nn] = json.loads(last[-1]) if last else None
json.dump(pt, open(os.path.join(prof, f"{tag}_next2_part_times.json"), "w"), indent=1)
print("profiles updated:", tag)
