"""Summarise ncu reports (raw page) and launch lists into profiles/.

    python scripts/ncu_summary.py gpurun_out/raycast_v2.ncu-rep [...] --launches gpurun_out/launches.csv
"""

from __future__ import annotations

import csv
import io
import json
import subprocess
import sys
from collections import defaultdict

METRICS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "lts__t_bytes.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__thread_inst_executed_per_inst_executed.ratio",
    "smsp__warps_eligible.avg.per_cycle_active",
    "l1tex__t_sector_hit_rate.pct",
    "lts__t_sector_hit_rate.pct",
    "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
    "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum",
    "launch__registers_per_thread",
    "launch__occupancy_limit_registers",
    "launch__grid_size",
    "launch__block_size",
    "sm__cycles_elapsed.avg.per_second",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_mio_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
]


def raw(rep: str) -> list[dict]:
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")]}
        for m in METRICS:
            if m in hdr:
                i = hdr.index(m)
                d[m] = f"{r[i]} {units[i]}".strip()
        res.append(d)
    return res


def launches(path: str) -> dict:
    agg = defaultdict(lambda: [0, 0.0])
    unit = None
    with open(path) as f:
        lines = [l for l in f if l.startswith('"')]
    rows = list(csv.reader(lines))
    hdr = rows[0]
    ik, iv, iu = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
    for r in rows[1:]:
        name = r[ik].split("(")[0]
        agg[name][0] += 1
        agg[name][1] += float(r[iv].replace(",", ""))
        unit = r[iu]
    total = sum(v[1] for v in agg.values())
    return {"unit": unit, "total": total,
            "kernels": {k: {"launches": n, "time": t, "share": t / total}
                        for k, (n, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])}}


def main():
    args = sys.argv[1:]
    out = {}
    if "--launches" in args:
        i = args.index("--launches")
        out["launch_list"] = launches(args[i + 1])
        args = args[:i] + args[i + 2:]
    for rep in args:
        out[rep.split("/")[-1]] = raw(rep)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
