"""Per-source-line stall samples of one kernel: ncu SASS samples mapped through nvdisasm line info.

  python tools/ncu_lines.py report.ncu-rep <kernel-regex> [skip] [top] [--so path] [--inst]

--inst ranks lines by executed warp instructions instead of stall samples.

The .so must be the build that was profiled (same sources); the kernel's SASS offsets
(address - first address) are matched to `nvdisasm -g` line annotations.
"""
import collections
import csv
import glob
import io
import os
import re
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def sass_rows(rep, kern, skip):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--kernel-name",
                          f"regex:{kern}", "--launch-skip", str(skip), "--launch-count", "1",
                          "--print-source", "sass"], capture_output=True, text=True).stdout
    lines = out.splitlines()
    name = lines[0]
    rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
    data = []
    for r in rows[1:]:
        if r and r[0] == "Kernel Name":      # next kernel's section
            break
        data.append(r)
    return name, rows[0], data


def line_map(so, mangled_hint):
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(so)], cwd=tmp, capture_output=True)
    best = {}
    for cub in glob.glob(os.path.join(tmp, "*.cubin")):
        txt = subprocess.run(["nvdisasm", "-g", "-c", cub], capture_output=True, text=True).stdout
        cur, curline, funcs = None, None, {}
        for l in txt.splitlines():
            m = re.match(r"\s*\.text\.(\S+):", l)
            if m:
                cur = m.group(1)
                funcs[cur] = {}
                continue
            m = re.search(r'//## File "([^"]+)", line (\d+)', l)
            if m:
                curline = f"{os.path.basename(m.group(1))}:{m.group(2)}"
                continue
            m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", l)
            if m and cur:
                funcs[cur][int(m.group(1), 16)] = curline
        for f, mp in funcs.items():
            if all(h in f for h in mangled_hint):
                best[f] = mp
    return best


def main():
    rep, kern = sys.argv[1], sys.argv[2]
    skip = int(sys.argv[3]) if len(sys.argv) > 3 else 0
    top = int(sys.argv[4]) if len(sys.argv) > 4 else 25
    so = os.path.join(ROOT, "paper_math_0301321_b200", "libib_b200.so")
    if "--so" in sys.argv:
        so = sys.argv[sys.argv.index("--so") + 1]
    name, hdr, data = sass_rows(rep, kern, skip)
    ix = {h: i for i, h in enumerate(hdr)}
    addr0 = int(data[0][ix["Address"]], 16)
    hints = [h for h in sys.argv[5:] if not h.startswith("--") and h != so] or [kern.split("<")[0]]
    maps = line_map(so, hints)
    if not maps:
        print("no function matched", hints)
        return
    if len(maps) > 1:
        # choose the map whose offsets cover the sampled range best
        n = len(data)
        maps = {k: v for k, v in maps.items() if len(v) == n} or maps
    fname, mp = next(iter(maps.items()))
    print(name[:120])
    print("function", fname[:100])
    agg = collections.Counter()
    stall = collections.defaultdict(collections.Counter)
    cols = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
    tot = 0.0
    for r in data:
        off = int(r[ix["Address"]], 16) - addr0
        col = "Instructions Executed" if "--inst" in sys.argv else "Warp Stall Sampling (All Samples)"
        s = float((r[ix[col]] or "0").replace(",", ""))
        ln = mp.get(off, "?")
        agg[ln] += s
        tot += s
        for c in cols:
            v = r[ix[c]]
            if v:
                stall[ln][c[6:]] += float(v)
    for ln, s in agg.most_common(top):
        mix = ", ".join(f"{k} {v:.0f}" for k, v in stall[ln].most_common(3))
        print(f"{100 * s / max(tot, 1):5.1f}%  {s:12.0f}  {ln:22s} {mix}")


if __name__ == "__main__":
    main()
