"""Summarise an `ncu --set full` report into markdown (one table per kernel) and update
profiles/ncu_traffic.json (dram bytes read+write per launch) for bench.py's roofline.traffic.
usage: python tools/ncu_summary.py report.ncu-rep config out.md"""
import csv
import json
import os
import subprocess
import sys

rep, config, out_md = sys.argv[1], sys.argv[2], sys.argv[3]
rows = list(csv.reader(subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                                      text=True).stdout.splitlines()))
h, units = rows[0], rows[1]
M = [("duration", "gpu__time_duration.sum"), ("DRAM read", "dram__bytes_read.sum"),
     ("DRAM write", "dram__bytes_write.sum"), ("SM % peak", "sm__throughput.avg.pct_of_peak_sustained_elapsed"),
     ("fp64 pipe %", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
     ("tensor (DMMA) pipe %", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active"),
     ("shared wavefronts % peak", "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed"),
     ("issue active %", "smsp__issue_active.avg.pct_of_peak_sustained_active"),
     ("achieved occupancy %", "sm__warps_active.avg.pct_of_peak_sustained_active"),
     ("L2 hit rate %", "lts__t_sector_hit_rate.pct"),
     ("grid", "launch__grid_size"), ("block", "launch__block_size"), ("regs/thread", "launch__registers_per_thread"),
     ("dyn smem/CTA", "launch__shared_mem_per_block_dynamic")]
iname = h.index("Kernel Name")
lines = [f"# ncu --set full summary: {os.path.basename(rep)} ({config})", "",
         "Captured with `ncu --set full --clock-control none --import-source on` (one launch per kernel,",
         "serialised, cold caches: absolute times exceed the in-pipeline CUDA-event times).", ""]
traffic = {}
for r in rows[2:]:
    name = r[iname]
    lines += [f"## {name[:80]}", "| metric | value |", "|---|---|"]
    for lab, key in M:
        if key in h:
            i = h.index(key)
            lines.append(f"| {lab} | {r[i]} {units[i]} |")
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    try:
        ir, iw = h.index("dram__bytes_read.sum"), h.index("dram__bytes_write.sum")
        rd = float(r[ir]) * scale.get(units[ir], 1.0)
        wr = float(r[iw]) * scale.get(units[iw], 1.0)
        short = name.split("<")[0].split("(")[0].replace("void ", "").replace("lc::", "").strip()
        traffic[short] = rd + wr
        lines.append(f"| DRAM read+write per launch | {rd + wr:.0f} bytes |")
    except (ValueError, IndexError):
        pass
    lines.append("")
open(out_md, "w").write("\n".join(lines))
tj = os.path.join("profiles", "ncu_traffic.json")
allt = json.load(open(tj)) if os.path.exists(tj) else {}
allt[config] = traffic
json.dump(allt, open(tj, "w"), indent=1, sort_keys=True)
print(open(out_md).read()[:3000])
