#!/usr/bin/env python3
"""Summarise an ncu --set full report of k_fused into profiles/.

usage: python tools/ncu_summary.py <report.ncu-rep> <config-key> <out.txt> [cell-updates in the launch]
Writes the key metrics (duration, DRAM bytes, throughputs, stall reasons,
registers, occupancy) as text and merges the per-launch DRAM traffic into
profiles/ncu_traffic.json under <config-key> (read by bench.py).
"""
import csv
import io
import json
import os
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__t_sector_hit_rate.pct",
    "lts__t_sectors_srcunit_tex.sum",
    "lts__t_sectors_srcunit_ltcfabric.sum",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum",
    "launch__registers_per_thread",
    "launch__grid_size",
    "launch__block_size",
    "launch__shared_mem_per_block_dynamic",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_branch_resolving_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
]


def main():
    rep, key, out = sys.argv[1:4]
    cells = float(sys.argv[4]) if len(sys.argv) > 4 else None  # cell-updates in the profiled launch
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    name = vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
    m = {}
    for k in KEYS:
        if k in hdr:
            m[k] = (vals[hdr.index(k)], units[hdr.index(k)])
    lines = [f"report: {os.path.basename(rep)}", f"kernel: {name}", f"config: {key}", ""]
    for k in KEYS:
        if k in m:
            lines.append(f"{k:80s} {m[k][0]} {m[k][1]}")

    def to_bytes(v, u):
        f = float(v.replace(",", ""))
        return f * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)

    rd = to_bytes(*m["dram__bytes_read.sum"])
    wr = to_bytes(*m["dram__bytes_write.sum"])
    dur = float(m["gpu__time_duration.sum"][0].replace(",", ""))
    dur_s = dur * {"ns": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3}.get(
        m["gpu__time_duration.sum"][1], 1e-9)
    lines += ["", f"DRAM traffic per launch: {rd + wr:.4e} B (read {rd:.4e}, write {wr:.4e})",
              f"DRAM throughput: {(rd + wr) / dur_s / 1e9:.1f} GB/s over {dur_s * 1e3:.4f} ms"]
    if cells:
        lines.append(f"DRAM bytes per cell-update: {(rd + wr) / cells:.2f} (read {rd / cells:.2f}, "
                     f"write {wr / cells:.2f})")
    open(out, "w").write("\n".join(lines) + "\n")
    tj = os.environ.get("NCU_TRAFFIC_JSON") or os.path.join(os.path.dirname(os.path.abspath(__file__)), "..",
                                                            "profiles", "ncu_traffic.json")
    try:
        t = json.load(open(tj))
    except Exception:
        t = {}
    t[key] = {"bytes_per_launch": rd + wr}
    if cells:
        t[key]["bytes_per_cell_update"] = (rd + wr) / cells
    json.dump(t, open(tj, "w"), indent=1, sort_keys=True)
    print("\n".join(lines))


if __name__ == "__main__":
    main()
