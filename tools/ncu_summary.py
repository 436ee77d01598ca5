"""Summarise an `ncu --set full` report (.ncu-rep) into profiles/: a markdown table of the key
metrics per captured kernel, and per-launch DRAM traffic into profiles/ncu_traffic.json
(read by bench.py for roofline.traffic).
usage: python tools/ncu_summary.py report.ncu-rep config_name out.md [launches.csv]"""
import csv
import io
import json
import os
import re
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % peak"),
    ("lts__t_bytes.sum", "L2 bytes"),
    ("sm__throughput.avg.pct_of_peak_sustained_elapsed", "SM % peak"),
    ("sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active", "fp64 pipe %"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__grid_size", "grid"),
    ("launch__block_size", "block"),
    ("launch__registers_per_thread", "regs/thread"),
    ("launch__shared_mem_per_block_dynamic", "dyn smem/CTA"),
    ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "stall long_scoreboard"),
    ("smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio", "stall barrier"),
    ("smsp__average_warps_issue_stalled_wait_per_issue_active.ratio", "stall wait"),
    ("smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio", "stall short_scoreboard"),
    ("smsp__average_warps_issue_stalled_membar_per_issue_active.ratio", "stall membar"),
    ("smsp__average_warps_issue_stalled_sleeping_per_issue_active.ratio", "stall sleeping"),
]
SCALE = {"ns": 1e-9, "us": 1e-6, "ms": 1e-3, "byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3}


def main(rep, config, out_md, launches=None):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    lines = [f"# ncu --set full summary: {os.path.basename(rep)} ({config})", "",
             "Captured with `ncu --set full --clock-control none --import-source on` (one launch per kernel,",
             "serialised, cold-ish caches: absolute times exceed the in-pipeline CUDA-event times).", ""]
    traffic = {}
    kernels = []
    for r in rows[2:]:
        name = re.sub(r"\(.*", "", r[hdr.index("Kernel Name")]).replace("void ", "")
        kernels.append(name)
        vals = {}
        for m, label in METRICS:
            if m in hdr:
                i = hdr.index(m)
                vals[label] = (r[i], units[i])
        rd = float(vals["DRAM read"][0].replace(",", "")) * SCALE.get(vals["DRAM read"][1], 1)
        wr = float(vals["DRAM write"][0].replace(",", "")) * SCALE.get(vals["DRAM write"][1], 1)
        base = re.sub(r"<.*", "", name).split("::")[-1]
        traffic.setdefault(base, rd + wr)
        lines.append(f"## {name}")
        lines.append("| metric | value |")
        lines.append("|---|---|")
        for label, (v, u) in vals.items():
            lines.append(f"| {label} | {v} {u} |")
        lines.append(f"| DRAM read+write per launch | {rd + wr:.0f} bytes |")
        lines.append("")
    if launches:
        lines.append("## Launch list (`--metrics gpu__time_duration.sum --clock-control none`), mean per kernel")
        lrows = [x for x in csv.reader(open(launches)) if len(x) > 10]
        h = lrows[0]
        ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
        agg = {}
        for x in lrows[1:]:
            k = re.sub(r"\(.*", "", x[ki]).replace("void ", "")
            agg.setdefault(k, []).append(float(x[vi].replace(",", "")) * SCALE.get(x[ui], 1) * 1e6)
        tot = sum(sum(v) for k, v in agg.items() if "lc_" in k and "plan" not in k)
        lines.append("| kernel | launches | mean us | share of transform kernels |")
        lines.append("|---|---|---|---|")
        for k, v in agg.items():
            sh = f"{sum(v) / tot:.2f}" if ("lc_" in k and "plan" not in k) else "-"
            lines.append(f"| {k} | {len(v)} | {sum(v) / len(v):.2f} | {sh} |")
        lines.append("")
    open(out_md, "w").write("\n".join(lines) + "\n")
    tp = os.path.join(os.path.dirname(out_md), "ncu_traffic.json")
    d = json.load(open(tp)) if os.path.exists(tp) else {}
    d.setdefault(config, {}).update(traffic)
    json.dump(d, open(tp, "w"), indent=1, sort_keys=True)
    print(out_md, traffic)


if __name__ == "__main__":
    main(*sys.argv[1:])
