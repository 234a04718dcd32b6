"""Summarise an ncu --set full report of one kernel into JSON (for profiles/).

usage: python tools/ncu_summary.py <report.ncu-rep> <algorithmic_bytes_per_launch> > out.json
"""
import csv
import io
import json
import re
import subprocess
import sys

KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "sm__cycles_active.avg", "sm__cycles_elapsed.avg",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
    "l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum",
    "l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum",
    "lts__t_sectors_srcunit_tex_op_read.sum",
    "l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum",
    "sm__warps_active.avg.per_cycle_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
]


def to_bytes(v, unit):
    mult = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    return float(v) * mult.get(unit, 1)


def main():
    rep, alg = sys.argv[1], float(sys.argv[2])
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, u, v = rows[0], rows[1], rows[2]
    d = {h[i]: (v[i].replace(",", ""), u[i]) for i in range(len(h))}
    out = {"report": rep, "kernel": d.get("Kernel Name", ("?",))[0]}
    for k in KEYS:
        if k in d:
            val, unit = d[k]
            try:
                out[k] = {"value": float(val), "unit": unit}
            except ValueError:
                out[k] = {"value": val, "unit": unit}
    stalls = {}
    for k, (val, unit) in d.items():
        m = re.match(r"smsp__average_warps_issue_stalled_(\w+)_per_issue_active\.ratio$", k)
        if m:
            try:
                if float(val) > 0.2:
                    stalls[m.group(1)] = float(val)
            except ValueError:
                pass
    out["stalls_per_issue"] = dict(sorted(stalls.items(), key=lambda x: -x[1]))
    rd = to_bytes(*d["dram__bytes_read.sum"])
    wr = to_bytes(*d["dram__bytes_write.sum"])
    t = float(d["gpu__time_duration.sum"][0])
    tunit = d["gpu__time_duration.sum"][1]
    t_s = t * {"nsecond": 1e-9, "ns": 1e-9, "usecond": 1e-6, "us": 1e-6, "msecond": 1e-3, "ms": 1e-3, "second": 1, "s": 1}[tunit]
    out["traffic_bytes_per_launch"] = rd + wr
    out["algorithmic_bytes_per_launch"] = alg
    out["traffic_over_algorithmic"] = (rd + wr) / alg
    out["duration_s_under_ncu"] = t_s
    out["achieved_algorithmic_GBps_under_ncu"] = alg / t_s / 1e9
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
