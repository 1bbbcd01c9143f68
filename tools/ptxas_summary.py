"""Rebuild libib_b200.so with -Xptxas -v and print registers / stack / spills per kernel."""
import os
import re
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_math_0301321_b200 import _build  # noqa: E402

flt = sys.argv[1] if len(sys.argv) > 1 else ""
cmd = [_build.nvcc(), *_build.ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
       "-shared", "-cudart", "shared", "-Xptxas=-v", "-o", "/tmp/ptxas_probe.so", *_build.sources()]
out = subprocess.run(cmd, capture_output=True, text=True).stderr
cur = None
rows = {}
for line in out.splitlines():
    m = re.search(r"Compiling entry function '(\S+)'", line)
    if m:
        cur = m.group(1)
        rows[cur] = {}
        continue
    if cur is None:
        continue
    m = re.search(r"(\d+) bytes stack frame, (\d+) bytes spill stores", line)
    if m:
        rows[cur]["stack"], rows[cur]["spill"] = int(m.group(1)), int(m.group(2))
    m = re.search(r"Used (\d+) registers", line)
    if m:
        rows[cur]["regs"] = int(m.group(1))
for k, v in rows.items():
    dem = subprocess.run(["c++filt", k], capture_output=True, text=True).stdout.strip()
    dem = re.sub(r"\(.*", "", dem)
    if flt in dem:
        print(f"{v.get('regs', '?'):>4} regs  stack {v.get('stack', 0):>4}  spill {v.get('spill', 0):>4}  {dem}")
