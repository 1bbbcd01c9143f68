"""Top SASS lines of one kernel from an ncu report: stall samples and smem bank conflicts.

  python tools/ncu_source.py report.ncu-rep <kernel-regex> [N]
"""
import csv
import io
import subprocess
import sys

rep, kern = sys.argv[1], sys.argv[2]
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
skip = int(sys.argv[4]) if len(sys.argv) > 4 else 0      # n-th matching launch
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name",
                      f"regex:{kern}", "--launch-skip", str(skip), "--launch-count", "1",
                      "--print-source", "sass"], capture_output=True, text=True).stdout
lines = out.splitlines()
# first line = kernel name row
rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
hdr, data = rows[0], rows[1:]
ix = {h: i for i, h in enumerate(hdr)}


def f(r, k):
    try:
        return float(r[ix[k]].replace(",", "")) if k in ix and ix[k] < len(r) and r[ix[k]] else 0.0
    except ValueError:
        return 0.0


tot = sum(f(r, "Warp Stall Sampling (All Samples)") for r in data) or 1.0
print(f"total stall samples {tot:.0f}")
stall_cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
agg = {c: sum(f(r, c) for r in data) for c in stall_cols}
print("stall mix:", ", ".join(f"{k[6:]} {100 * v / tot:.1f}%" for k, v in
                              sorted(agg.items(), key=lambda kv: -kv[1])[:8]))
ex = sorted(data, key=lambda r: -f(r, "L1 Wavefronts Shared Excessive"))[:8]
print("-- smem excessive wavefronts")
for r in ex:
    if f(r, "L1 Wavefronts Shared Excessive") > 0:
        print(f"  {f(r, 'L1 Wavefronts Shared Excessive'):10.0f} / {f(r, 'L1 Wavefronts Shared'):10.0f}  {r[ix['Source']][:90]}")
print("-- top stall lines")
for r in sorted(data, key=lambda r: -f(r, "Warp Stall Sampling (All Samples)"))[:top]:
    s = f(r, "Warp Stall Sampling (All Samples)")
    top_st = sorted(((c, f(r, c)) for c in stall_cols), key=lambda kv: -kv[1])[:2]
    print(f"  {100 * s / tot:5.1f}%  {r[ix['Address']]:>6} {r[ix['Source']][:70]:70s} "
          + " ".join(f"{c[6:]}={v:.0f}" for c, v in top_st))
