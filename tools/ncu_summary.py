"""Summarise an ncu report: per kernel time, DRAM bytes/throughput, L2 hit, occupancy, stalls.

  python tools/ncu_summary.py gpurun_out/prof.ncu-rep [--json out.json]
"""
import csv
import io
import json
import subprocess
import sys

METRICS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
    "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
    "sm__inst_executed_pipe_fp64.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
    "smsp__inst_executed.sum", "l1tex__t_sector_hit_rate.pct",
    "smsp__average_warp_latency_issue_stalled_long_scoreboard",
]
UNITS = {"dram__bytes_read.sum": "MB?", "gpu__time_duration.sum": "us?"}


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--print-units", "base"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr, units, data = rows[0], rows[1], rows[2:]
    return hdr, units, data


def main():
    rep = sys.argv[1]
    hdr, units, data = raw(rep)
    res = []
    for row in data:
        d = dict(zip(hdr, row))
        name = d.get("Kernel Name", "?")
        rec = {"kernel": name[:60]}
        for m in METRICS:
            if m in d:
                try:
                    rec[m] = float(d[m].replace(",", ""))
                except ValueError:
                    rec[m] = d[m]
        res.append(rec)
    for r in res:
        t = r.get("gpu__time_duration.sum", 0) / 1e3
        rb = r.get("dram__bytes_read.sum", 0) / 1e6
        wb = r.get("dram__bytes_write.sum", 0) / 1e6
        print(f"{r['kernel'][:44]:44s} {t:8.1f}us  dram R {rb:7.1f}MB W {wb:7.1f}MB "
              f"{r.get('dram__throughput.avg.pct_of_peak_sustained_elapsed', 0):5.1f}%dram "
              f"L2hit {r.get('lts__t_sector_hit_rate.pct', 0):5.1f} "
              f"warps {r.get('sm__warps_active.avg.pct_of_peak_sustained_active', 0):5.1f}% "
              f"regs {r.get('launch__registers_per_thread', 0):.0f} "
              f"bankc {r.get('l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum', 0):.0f}")
    if "--json" in sys.argv:
        json.dump(res, open(sys.argv[sys.argv.index("--json") + 1], "w"), indent=1)


if __name__ == "__main__":
    main()
