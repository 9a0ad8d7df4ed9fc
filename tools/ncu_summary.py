#!/usr/bin/env python
"""Key numbers of an `ncu --page raw --csv` export: tools/ncu_summary.py <raw.csv> [...]."""
import csv
import sys

WANT = [
    "gpu__time_duration.sum", "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "dram__bytes_read.sum", "dram__bytes_write.sum", "lts__t_sectors.sum", "lts__t_sector_hit_rate.pct",
    "l1tex__m_l1tex2xbar_req_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_requests_srcunit_ltcfabric.sum",
    "lts__t_sectors_srcunit_tex_op_read.sum", "lts__t_sectors_srcunit_tex_op_red.sum",
    "lts__t_sectors_srcunit_tex_op_write.sum", "lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum",
    "lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum", "launch__registers_per_thread",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
]


def summary(path):
    rows = list(csv.reader(open(path)))
    hdr, units, vals = rows[0], rows[1], rows[2]
    out = {}
    for h, u, v in zip(hdr, units, vals):
        if h in WANT or (h.startswith("smsp__average_warps_issue_stalled") and h.endswith("per_issue_active.ratio")):
            try:
                out[h] = (float(v), u)
            except ValueError:
                out[h] = (v, u)
    return out


if __name__ == "__main__":
    sums = [summary(p) for p in sys.argv[1:]]
    keys = list(sums[0])
    for k in keys:
        vals = [s.get(k, ("", ""))[0] for s in sums]
        if k.startswith("smsp__average_warps_issue_stalled") and all(isinstance(v, float) and v < 0.3 for v in vals):
            continue
        short = k.replace("smsp__average_warps_issue_stalled_", "stall_").replace("_per_issue_active.ratio", "")
        print(f"{short:75s} {sums[0][k][1]:10s} " + "  ".join(f"{v:>14.4g}" if isinstance(v, float) else str(v) for v in vals))
