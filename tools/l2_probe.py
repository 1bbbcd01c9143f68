"""Dev: per-plane stage times vs the number of z planes (pure fluid, 256 x 256 x N3): when the
spectra fit in L2 (small N3) the passes show their SM-bound cost."""
import json, os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
from gen import random_divfree_velocity
from paper_math_0301321_b200 import IBContext, IB_OPT_STAGE_TIMING
for n3 in (256, 128, 64, 32, 16):
    shape = (256, 256, n3)
    c = IBContext(shape, 1 / 256, 1.0, 1e-3, 1.25e-4)
    c.set_velocity(random_divfree_velocity(shape, 3, 0.01, np.random.default_rng(1)))
    c.step(3)
    c.set_option(IB_OPT_STAGE_TIMING, 1)
    c.stage_times(reset=True)
    c.step(20)
    st = c.stage_times()
    print(json.dumps({"N3": n3, "us_per_plane": {k: round(1e3 * v / 20 / n3, 3) for k, v in st.items() if v > 0}}))
    c.close()
