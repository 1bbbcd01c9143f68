"""Per-stage timing of one config in stage mode (dev tool): python tools/stage_bench_cfg.py cfg steps"""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from gen import make_config
from paper_math_0301321_b200 import IBContext, IB_OPT_STAGE_TIMING
k = sys.argv[1] if len(sys.argv) > 1 else "4"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 20
cfg = make_config(k)
c = IBContext.from_config(cfg)
c.step(5)
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize(); s.record(); c.step(steps); e.record(); torch.cuda.synchronize()
graph_ms = s.elapsed_time(e) / steps
c.set_option(IB_OPT_STAGE_TIMING, 1)
c.stage_times(reset=True)
c.step(steps)
st = c.stage_times()
lib = os.environ.get("IB_B200_LIB", "default")
print(json.dumps({"lib": lib[-12:], "cfg": k, "graph_ms": round(graph_ms, 4),
                  "stages_us": {a: round(1e3 * b / steps, 1) for a, b in st.items()}}))
