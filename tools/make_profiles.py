"""Turn a gpurun_out/ capture into the committed profiles/ summaries.

  python tools/make_profiles.py <tag> [config]   (reads gpurun_out/{launches,prof,bench}_<tag>.*)

Writes profiles/<tag>_launches.txt (per-launch device times from the
`ncu --metrics gpu__time_duration.sum --clock-control none` pass, with each kernel's share
of the step), profiles/<tag>_ncu_full.txt (per-kernel `ncu --set full` summary: duration,
DRAM bytes, L2 hit rate, occupancy, bank conflicts), profiles/<tag>_bench.json (the bench
line) and profiles/ncu_traffic_cfg<config>.json (DRAM bytes per launch per stage of that
config, read by bench.py for roofline.traffic / dram_frac).
"""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
PROF = os.environ.get("PROF_OUT") or os.path.join(ROOT, "profiles")

import re

# kernel name -> stage of the step (any lattice size): the TMA column kernel's MODE is its
# second template argument (0 = z solve, 1 = y forward, 2 = y inverse, 3/4 = debug z passes)
_COL = {"0": "z_solve", "1": "y_fwd", "2": "y_inv", "3": "z_fwd", "4": "z_inv"}
STAGE_OF = [("k_force_spread", "force_spread"), ("k_drive_spread", "force_spread"),
            ("k_xfwd", "xfwd_rhs_r2c"), ("k_zpass", "z_solve"),
            ("k_xinv", "xinv_c2r"), ("k_interp", "interp_update"), ("k_step_inc", "step_inc"),
            ("k_bin", "binning"), ("k_scan", "binning")]


def stage(name):
    m = re.search(r"k_colfft<(?:\(int\))?\d+, (?:\(int\))?(\d)>", name)
    if m:
        return _COL[m.group(1)]
    m = re.search(r"k_ypass<(?:\(int\))?\d+, (?:\(int\))?(-?1)>", name)
    if m:
        return "y_fwd" if m.group(1) == "-1" else "y_inv"
    for key, st in STAGE_OF:
        if key in name:
            return st
    return name.split("(")[0]


def launches(tag):
    p = os.path.join(OUT, f"launches_{tag}.csv")
    if not os.path.exists(p):
        return None
    rows = list(csv.reader(open(p)))
    hdr, out = None, []
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                out.append((d["Kernel Name"], float(d["Metric Value"].replace(",", "")) / 1e3))
    return out


def ncu_raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--print-units", "base"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    if len(rows) < 3:
        return []
    hdr = rows[0]
    return [dict(zip(hdr, r)) for r in rows[2:]]


def num(d, k):
    try:
        return float(d.get(k, "").replace(",", ""))
    except ValueError:
        return float("nan")


def main():
    tag = sys.argv[1]
    cfg = sys.argv[2] if len(sys.argv) > 2 else "4"
    os.makedirs(PROF, exist_ok=True)
    L = launches(tag)
    if L:
        total = sum(t for _, t in L)
        lines = [f"# ncu --metrics gpu__time_duration.sum --clock-control none ({tag})",
                 "# cold-cache, serialised launches: compare SHARES, not absolute times",
                 f"{'us':>9} {'share':>6}  stage / kernel"]
        if len(L) > 20:           # a whole bench run: per-stage shares first
            agg, cnt = {}, {}
            for k, t in L:
                agg[stage(k)] = agg.get(stage(k), 0.0) + t
                cnt[stage(k)] = cnt.get(stage(k), 0) + 1
            lines.append("# per stage over all launches (us total, launches, mean us, share)")
            for st, t in sorted(agg.items(), key=lambda x: -x[1]):
                lines.append(f"#   {st:16s} {t:10.1f} {cnt[st]:5d} {t / cnt[st]:8.1f} {100 * t / total:5.1f}%")
        for k, t in L:
            lines.append(f"{t:9.1f} {100 * t / total:5.1f}%  {stage(k):14s} {k[:90]}")
        lines.append(f"{total:9.1f}  total over {len(L)} launches")
        open(os.path.join(PROF, f"{tag}_launches.txt"), "w").write("\n".join(lines) + "\n")
    rep = os.path.join(OUT, f"prof_{tag}.ncu-rep")
    if os.path.exists(rep):
        rows = ncu_raw(rep)
        lines = [f"# ncu --set full --clock-control none ({tag}); per launch",
                 f"{'kernel':44s} {'us':>7} {'DRAM R MB':>9} {'DRAM W MB':>9} {'DRAM GB/s':>9} "
                 f"{'L2 hit%':>7} {'warps%':>6} {'regs':>4} {'smem conf':>9}"]
        traffic = {}
        for d in rows:
            name = d.get("Kernel Name", "?")
            us = num(d, "gpu__time_duration.sum") / 1e3
            rb, wb = num(d, "dram__bytes_read.sum"), num(d, "dram__bytes_write.sum")
            gbs = (rb + wb) / (us * 1e-6) / 1e9 if us > 0 else float("nan")
            lines.append(f"{name.split('(')[0][:44]:44s} {us:7.1f} {rb / 1e6:9.1f} {wb / 1e6:9.1f} "
                         f"{gbs:9.0f} {num(d, 'lts__t_sector_hit_rate.pct'):7.1f} "
                         f"{num(d, 'sm__warps_active.avg.pct_of_peak_sustained_active'):6.1f} "
                         f"{num(d, 'launch__registers_per_thread'):4.0f} "
                         f"{num(d, 'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum'):9.0f}")
            st = stage(name)
            traffic.setdefault(st, 0.0)
            traffic[st] += rb + wb
        open(os.path.join(PROF, f"{tag}_ncu_full.txt"), "w").write("\n".join(lines) + "\n")
        json.dump({"source": f"profiles/{tag}_ncu_full.txt (ncu --set full, one step of cfg{cfg})",
                   "unit": "bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum)",
                   "stages": traffic},
                  open(os.path.join(PROF, f"ncu_traffic_cfg{cfg}.json"), "w"), indent=1)
    b = os.path.join(OUT, f"bench_{tag}.json")
    if os.path.exists(b):
        txt = open(b).read().strip().splitlines()
        if txt:
            open(os.path.join(PROF, f"{tag}_bench.json"), "w").write(txt[-1] + "\n")
    print("\n".join(sorted(f for f in os.listdir(PROF) if tag in f)))


if __name__ == "__main__":
    main()
