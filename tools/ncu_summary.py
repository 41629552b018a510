"""Summarise an ncu report (--page raw) into the handful of metrics the roofline argument needs.

    python tools/ncu_summary.py gpurun_out/prof.ncu-rep [--json out.json]
"""

from __future__ import annotations

import csv
import io
import json
import subprocess
import sys

KEYS = [
    "Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed", "l1tex__t_sector_hit_rate.pct",
    "l1tex__throughput.avg.pct_of_peak_sustained_active", "lts__t_sectors_srcunit_tex_op_read.sum",
    "lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum", "launch__registers_per_thread",
    "launch__grid_size", "launch__block_size", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_shared_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_lg_throttle_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
]


def summarise(path: str) -> list[dict]:
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True, check=True)
    rows = list(csv.reader(io.StringIO(out.stdout)))
    hdr, units = rows[0], rows[1]
    res = []
    for vals in rows[2:]:
        d = {}
        for k in KEYS:
            if k in hdr:
                i = hdr.index(k)
                d[k] = f"{vals[i]} {units[i]}".strip()
        # any tensor-pipe metric, every warp-stall reason, the global-load L1 sector counts
        for i, h in enumerate(hdr):
            want = ("pipe_tensor" in h and "pct" in h) or (
                h.startswith("smsp__average_warps_issue_stalled_") and h.endswith("_per_issue_active.ratio")) or (
                h.startswith("l1tex__t_sectors_pipe_lsu_mem_global_op_ld") and h.endswith(".sum")) or (
                h.startswith("l1tex__t_requests_pipe_lsu_mem_global_op_ld") and h.endswith(".sum")) or (
                h in ("sm__warps_active.avg.per_cycle_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
                      "l1tex__m_xbar2l1tex_read_bytes.sum", "lts__t_bytes.sum"))
            if want and h not in d:
                d[h] = f"{vals[i]} {units[i]}".strip()
        res.append(d)
    return res


def main():
    path = sys.argv[1]
    res = summarise(path)
    for d in res:
        for k, v in d.items():
            print(f"{k:80s} {v}")
        print()
    if "--json" in sys.argv:
        with open(sys.argv[sys.argv.index("--json") + 1], "w") as fh:
            json.dump(res, fh, indent=1)


if __name__ == "__main__":
    main()
