"""Profiling driver: one warm-up IB step then `--steps` steps of a config (default cfg4).

Used under ncu:  ncu --set full -s <launches to skip> -c <n> python tools/prof_step.py
Launch order per step: force_spread (drive included), xfwd, y_fwd, z_solve,
y_inv, xinv, interp, step counter.  ib_create issues 1 launch (tables).
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="4")
    ap.add_argument("--steps", type=int, default=1)
    ap.add_argument("--warmup", type=int, default=1)
    a = ap.parse_args()
    from gen import make_config
    from paper_math_0301321_b200 import IBContext
    cfg = make_config(a.config)
    c = IBContext.from_config(cfg)
    c.step(a.warmup)
    c.step(a.steps)
    print("launches", c.launch_count())
    c.close()


if __name__ == "__main__":
    main()
