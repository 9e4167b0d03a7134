"""Summarise an ncu --set full report (one kernel launch) and an ncu launch
list into a small JSON under profiles/, used by bench.py for the roofline
`traffic` field and by DESIGN.md.

usage: python tools/ncu_summary.py <tag> <report.ncu-rep> [launches.csv]
"""
import csv
import io
import json
import os
import subprocess
import sys

WANT = {
    "gpu__time_duration.sum": "duration",
    "dram__bytes_read.sum": "dram_read",
    "dram__bytes_write.sum": "dram_write",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed": "sm_pct",
    "sm__pipe_tensor_subpipe_imma_cycles_active_realtime.avg": "imma_cycles_realtime",
    "sm__cycles_elapsed.avg": "sm_cycles",
    "sm__cycles_elapsed.avg.per_second": "sm_clock",
    "lts__t_bytes.sum": "l2_bytes",
    "launch__registers_per_thread": "regs",
    "launch__grid_size": "grid",
    "launch__block_size": "block",
    "sm__inst_executed_pipe_tensor_subpipe_imma.avg.pct_of_peak_sustained_active": "imma_inst_pct",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed": "tensor_active_pct",
    "sm__pipe_tensor_cycles_active.avg": "tensor_active_cycles",
    "lts__t_sectors_srcunit_tex_op_read.sum": "l2_read_sectors_from_sm",
    "lts__t_sector_hit_rate.pct": "l2_hit_pct",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active": "alu_pipe_pct",
    "sm__pipe_fmaheavy_cycles_active.avg.pct_of_peak_sustained_elapsed": "fmaheavy_pct",
    "sm__inst_executed.avg.per_cycle_active": "ipc",
    "smsp__issue_active.avg.pct_of_peak_sustained_active": "issue_pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active": "occupancy_pct",
    "sm__inst_executed.sum": "warp_instructions",
}
SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "usecond": 1e-6, "us": 1e-6, "ns": 1e-9,
         "msecond": 1e-3, "ms": 1e-3, "nsecond": 1e-9, "Ghz": 1e9, "GHz": 1e9, "Mhz": 1e6}


def raw(report):
    out = subprocess.run(["ncu", "-i", report, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    h, u, v = rows[0], rows[1], rows[2]
    res = {"kernel": v[h.index("Kernel Name")] if "Kernel Name" in h else None}
    for i, name in enumerate(h):
        key = WANT.get(name)
        if key is None:
            continue
        try:
            val = float(v[i].replace(",", ""))
        except ValueError:
            continue
        res[key] = val * SCALE.get(u[i], 1)
        res[key + "_unit"] = "SI" if u[i] in SCALE else u[i]
    if "dram_read" in res and "dram_write" in res:
        res["dram_traffic_bytes"] = res["dram_read"] + res["dram_write"]
    return res


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = {}
    for r in rows[hi + 1:]:
        if len(r) <= vi:
            continue
        agg.setdefault(r[ki].split("(")[0], []).append(float(r[vi].replace(",", "")) * SCALE.get(r[ui], 1e-9))
    return {k: {"n": len(v), "mean_us": 1e6 * sum(v) / len(v)} for k, v in agg.items()}


if __name__ == "__main__":
    tag, rep = sys.argv[1], sys.argv[2]
    s = {"tag": tag, "report": os.path.basename(rep), "kernel_capture": raw(rep)}
    if len(sys.argv) > 3:
        s["launch_list"] = launches(sys.argv[3])
    os.makedirs("profiles", exist_ok=True)
    json.dump(s, open(os.path.join("profiles", f"ncu_{tag}.json"), "w"), indent=1)
    print(json.dumps(s, indent=1))
