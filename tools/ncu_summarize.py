"""Summarize ncu outputs into profiles/ (run here, on the reports gpurun
brought back).

    python tools/ncu_summarize.py launches <launches.csv> <out.txt>
    python tools/ncu_summarize.py full <report.ncu-rep> <out.txt> [traffic_key]
"""
from __future__ import annotations

import csv
import json
import subprocess
import sys
from collections import defaultdict
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]

FULL_METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "launch__shared_mem_per_block_dynamic", "launch__occupancy_limit_registers",
    "smsp__inst_executed.sum", "sm__cycles_elapsed.avg.per_second",
    "smsp__sass_thread_inst_executed_op_dfma_pred_on.sum",
    "smsp__sass_thread_inst_executed_op_dmul_pred_on.sum",
    "smsp__sass_thread_inst_executed_op_dadd_pred_on.sum",
]


def launches(csv_path, out_path):
    rows = list(csv.reader(open(csv_path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi = h.index("Kernel Name"), h.index("Metric Value")
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[hi + 1:]:
        if len(r) > vi:
            agg[r[ki]][0] += 1
            agg[r[ki]][1] += float(r[vi].replace(",", ""))
    tot = sum(v[1] for v in agg.values())
    lines = [f"# ncu launch list ({csv_path}): gpu__time_duration.sum, --clock-control none",
             "# cold-cache, serialised; compare SHARES, not absolute times",
             f"{'launches':>8} {'total ms':>12} {'share':>7}  kernel"]
    for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
        lines.append(f"{v[0]:8d} {v[1] / 1e6:12.3f} {100 * v[1] / tot:6.2f}%  {k[:110]}")
    Path(out_path).write_text("\n".join(lines) + "\n")
    print("\n".join(lines))


def full(rep, out_path, traffic_key=None):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    r = list(csv.reader(raw.splitlines()))
    h, units = r[0], r[1]
    lines = [f"# ncu --set full --clock-control none ({Path(rep).name})"]
    for row in r[2:]:
        name = row[h.index("Kernel Name")] if "Kernel Name" in h else "?"
        lines.append(f"== {name}")
        for w in FULL_METRICS:
            if w in h:
                lines.append(f"  {w:66s} {row[h.index(w)]:>18s} {units[h.index(w)]}")
        st = []
        for i, k in enumerate(h):
            if "pcsamp_warps_issue_stalled" in k and not k.endswith("not_issued"):
                try:
                    st.append((float(row[i].replace(",", "")), k.replace("smsp__pcsamp_warps_issue_stalled_", "")))
                except ValueError:
                    pass
        tot = sum(x for x, _ in st) or 1.0
        lines.append("  stall samples: " + ", ".join(f"{k} {100 * x / tot:.1f}%" for x, k in
                                                     sorted(st, reverse=True)[:8]))
        if traffic_key:
            rd = float(row[h.index("dram__bytes_read.sum")].replace(",", ""))
            wr = float(row[h.index("dram__bytes_write.sum")].replace(",", ""))
            scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
            rd *= scale.get(units[h.index("dram__bytes_read.sum")], 1)
            wr *= scale.get(units[h.index("dram__bytes_write.sum")], 1)
            tf = ROOT / "profiles" / "roofline_traffic.json"
            data = json.loads(tf.read_text()) if tf.exists() else {}
            data[traffic_key] = rd + wr
            tf.write_text(json.dumps(data, indent=1) + "\n")
    Path(out_path).write_text("\n".join(lines) + "\n")
    print("\n".join(lines))


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3])
    else:
        full(sys.argv[2], sys.argv[3], sys.argv[4] if len(sys.argv) > 4 else None)
