"""Pipe-level summary of the kernels in an ncu --set full report (dev tool): per launch the
L1 data-pipe wavefronts (shared / global), their share of the pipe's peak, smem bank
conflicts, executed warp instructions by class (fp64, integer/ALU, memory, other), issue
activity, warps per scheduler and the top stall reasons per issued instruction.

  python tools/ncu_pipes.py report.ncu-rep [kernel-regex]
"""
import csv
import io
import subprocess
import sys


def raw(rep, kern):
    args = ["ncu", "-i", rep, "--page", "raw", "--csv"]
    if kern:
        args += ["-k", f"regex:{kern}"]
    out = subprocess.run(args, capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[2:]


def opclasses(rep, kname, idx):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name",
                          f"regex:{kname}", "--launch-skip", str(idx), "--launch-count", "1",
                          "--print-source", "sass"], capture_output=True, text=True).stdout
    lines = out.splitlines()
    r = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
    h = r[0]
    ix = {k: i for i, k in enumerate(h)}
    cls, seen = {}, set()
    for row in r[1:]:
        if len(row) < len(h) or row[0] == "Address" or row[0] in seen:
            continue
        seen.add(row[0])
        src = row[ix["Source"]].split()
        op = (src[1] if src and src[0].startswith("@") else (src[0] if src else "?")).split(".")[0]
        n = float((row[ix["Instructions Executed"]] or "0").replace(",", ""))
        if op in ("DADD", "DFMA", "DMUL", "DSETP", "DMMA", "DMNMX", "MUFU"):
            c = "fp64/mufu"
        elif op.startswith(("LD", "ST", "RED", "ATOM", "SHFL", "UTMA", "SYNCS", "UBLKCP")):
            c = "memory"
        elif op in ("BRA", "BAR", "BSYNC", "BSSY", "EXIT", "NOP", "YIELD", "WARPSYNC", "CALL", "RET"):
            c = "control"
        else:
            c = "int/alu"
        cls[c] = cls.get(c, 0.0) + n
    return cls


def main():
    rep = sys.argv[1]
    kern = sys.argv[2] if len(sys.argv) > 2 else ""
    h, rows = raw(rep, kern)
    ix = {k: i for i, k in enumerate(h)}

    def g(r, k):
        try:
            return float(r[ix[k]].replace(",", ""))
        except (KeyError, ValueError):
            return float("nan")
    count = {}
    for r in rows:
        name = r[ix["Kernel Name"]]
        short = name.split("(")[0].replace("void ", "")
        base = short.split("<")[0]
        k = count.get(base, 0)
        count[base] = k + 1
        us = g(r, "gpu__time_duration.sum")
        print(f"== {short}  {us:.1f} us")
        sh = g(r, "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum")
        pipe = g(r, "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed")
        lg = g(r, "SM_A.TriageCompute.l1tex__data_pipe_lsu_wavefronts_mem_lgds.avg") * 148
        conf = g(r, "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum")
        print(f"   L1 data pipe {pipe:5.1f}% of peak: shared {sh / 1e6:6.2f} M wavefronts "
              f"(bank conflicts {conf / 1e6:5.2f} M), global {lg / 1e6:6.2f} M")
        inst = g(r, "smsp__inst_executed.sum")
        cls = opclasses(rep, base, k)
        tot = sum(cls.values()) or 1.0
        mix = ", ".join(f"{c} {100 * v / tot:.0f}%" for c, v in sorted(cls.items(), key=lambda x: -x[1]))
        issue = g(r, "sm__inst_issued.avg.pct_of_peak_sustained_active")
        warps = g(r, "sm__warps_active.avg.pct_of_peak_sustained_active")
        dram = g(r, "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed")
        print(f"   {inst / 1e6:6.1f} M warp instructions ({mix}); issue {issue:4.1f}% of peak, "
              f"warps active {warps:4.1f}%, DRAM {dram:4.1f}% of peak")
        st = [(k2[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")], g(r, k2))
              for k2 in h if k2.startswith("smsp__average_warps_issue_stalled_") and
              k2.endswith("_per_issue_active.ratio")]
        st = sorted([s for s in st if s[1] == s[1] and s[0] not in ("selected",)], key=lambda x: -x[1])[:5]
        print("   stalls per issue: " + ", ".join(f"{a} {b:.2f}" for a, b in st))


if __name__ == "__main__":
    main()
