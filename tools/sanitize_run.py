"""Small workload for compute-sanitizer (memcheck / racecheck / initcheck / synccheck):
configs 1 and 2 (32^3 and 64^3: both the pencil and the TMA column kernels), 2 steps each
through the graph path and the stage-timed path, plus every debug entry point.

  compute-sanitizer --tool memcheck python tools/sanitize_run.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from gen import make_config  # noqa: E402
from paper_math_0301321_b200 import IBContext, IB_OPT_PRESSURE, IB_OPT_STAGE_TIMING  # noqa: E402

for k in (1, 2):
    cfg = make_config(k)
    with IBContext.from_config(cfg) as c:
        c.step(2)
        c.set_option(IB_OPT_STAGE_TIMING, 1)
        c.set_option(IB_OPT_PRESSURE, 1)
        c.step(1)
        u, p = c.get_fields(want_p=True)
        X = c.get_positions()
        f = c.debug_force()
        F = c.debug_spread(f)
        U = c.debug_interp(u)
        r = c.debug_rhs(u, F)
        un, pn = c.debug_fluid(u, F)
        sp = c.debug_fft(u[0])
        assert np.isfinite(u).all() and np.isfinite(X).all() and np.isfinite(U).all()
        print(f"cfg{k}: ok |u|={np.abs(u).max():.3e} |p|={np.abs(p).max():.3e}", flush=True)
