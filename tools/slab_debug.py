"""Dev: LocalSlabs vs the one-context step, step by step (first differing points, counts)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import torch
from gen import small_sheet_config, make_config
from paper_math_0301321_b200 import IBContext
from paper_math_0301321_b200.slab import LocalSlabs

P = int(sys.argv[1]) if len(sys.argv) > 1 else 4
which = sys.argv[2] if len(sys.argv) > 2 else "sheet"
cfg = small_sheet_config(N=64, n1=40, n2=30, seed=61, u_amp=0.2) if which == "sheet" else make_config(int(which))
s = LocalSlabs(cfg, P)
c = IBContext.from_config(cfg)
for n in range(1, 13):
    s.step(1)
    c.step(1)
    counts = [int(r.count_send.item()) for r in s.ranks]
    Xs = [s.get_positions(r) for r in range(P)]
    Xc = c.get_positions()
    us, _ = s.get_fields()
    uc, _ = c.get_fields()
    eu = np.linalg.norm(us - uc) / np.linalg.norm(uc)
    d = [np.max(np.abs(X - Xc)) for X in Xs]
    rep_ok = all(np.array_equal(Xs[0], X) for X in Xs[1:])
    print(f"step {n}: counts {counts} sum {sum(counts)} np {cfg.np_}  u {eu:.2e}  maxdX per rank {['%.1e' % v for v in d]} replicas equal {rep_ok}")
    if max(d) > 1e-12:
        for r in range(P):
            bad = np.flatnonzero(np.abs(Xs[r] - Xc).max(1) > 1e-12)
            if bad.size:
                i = bad[0]
                print(f"   rank {r}: {bad.size} bad, first {i}: slab {Xs[r][i]} one-ctx {Xc[i]}  z-plane {np.floor(Xc[i,2]*64)}")
