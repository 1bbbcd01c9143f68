"""Linearity and frequency-sweep experiments on the synthetic basilar-membrane strip, run as
independent GPU replicas (PAPER.md 1080-1085: "increasing the force by
a factor of 10 resulted in basilar membrane displacements almost exactly ten times bigger";
PAPER.md 1151-1167: the peak of the travelling wave moves toward the stapes as the input
frequency rises).

Every time step runs through the C-ABI (`ib_step`); this module only schedules replicas and
post-processes positions read back every `every` steps (the analysis of SPEC.md 413-450):

  centerline  normal displacement of the strip's middle row, d_i = (X_i - X_i^0) . n_i^0,
              at arclength stations s_i of the rest centre line;
  envelope    pointwise max |d_i| over a window of snapshots;
  peak        station of the envelope maximum (ties -> the smallest station);
  linearity   per-station envelope ratio against the drive scale.

Replicas: `python -m paper_math_0301321_b200.experiments linearity|sweep [...]`; under
torchrun each rank runs its share of the replicas on its own GPU (no communication but the
final gather of results on rank 0).
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time
from typing import List, Sequence

import numpy as np


# ------------------------------------------------------------------ analysis (host, numpy)
def strip_rows(cfg, patch: int = 0):
    """(indices of the middle row i2 = n2 // 2 of patch `patch`, n1)."""
    p = cfg.patches[patch]
    mid = p.n2 // 2
    return p.first + mid * p.n1 + np.arange(p.n1), p.n1


def rest_frame(cfg, patch: int = 0):
    """Arclength stations s_i and unit rest normals n_i of the middle row (normal = the cross
    product of the central-difference tangents along i1 and i2 at rest)."""
    p = cfg.patches[patch]
    P = cfg.X[p.first:p.first + p.n1 * p.n2].reshape(p.n2, p.n1, 3)
    mid = p.n2 // 2
    t1 = np.gradient(P[mid], axis=0)
    lo, hi = max(mid - 1, 0), min(mid + 1, p.n2 - 1)
    t2 = P[hi] - P[lo]
    n = np.cross(t1, t2)
    n /= np.linalg.norm(n, axis=1, keepdims=True)
    seg = np.linalg.norm(np.diff(P[mid], axis=0), axis=1)
    s = np.concatenate([[0.0], np.cumsum(seg)])
    return s, n


def centerline(X, X0, rows, normals):
    """Normal displacement of the middle row: d_i = (X_i - X0_i) . n_i."""
    return np.einsum("ij,ij->i", X[rows] - X0[rows], normals)


def envelope(profiles: Sequence[np.ndarray]) -> np.ndarray:
    """Pointwise max |d_i| over the snapshots of a window."""
    return np.max(np.abs(np.asarray(profiles)), axis=0)


def peak_location(env: np.ndarray, stations: np.ndarray) -> float:
    """Station of the global envelope maximum (ties -> the smallest station)."""
    return float(stations[int(np.argmax(env))])


def linearity(env_a: np.ndarray, env_b: np.ndarray, scale: float, floor: float = 0.01) -> dict:
    """Per-station ratio env_b / env_a against `scale`, where env_a exceeds `floor` x its
    peak; returns the max relative deviation and the mean ratio."""
    mask = env_a > floor * env_a.max()
    ratio = env_b[mask] / env_a[mask]
    return {"max_dev": float(np.max(np.abs(ratio / scale - 1.0))), "mean_ratio": float(ratio.mean()),
            "stations": int(mask.sum())}


# ------------------------------------------------------------------ replicas (GPU)
def run_replica(cfg, steps: int, every: int, window_start: int = 0, patch: int = 0):
    """Run cfg for `steps` IB steps on the current CUDA device; return (stations, envelope
    over snapshots at steps >= window_start, steps/s of the device run)."""
    from .ib import IBContext
    rows, _ = strip_rows(cfg, patch)
    s, n = rest_frame(cfg, patch)
    X0 = cfg.X.copy()
    prof = []
    with IBContext.from_config(cfg) as c:
        t0 = time.perf_counter()
        done = 0
        while done < steps:
            k = min(every, steps - done)
            c.step(k)
            done += k
            if done >= window_start:
                prof.append(centerline(c.get_positions(), X0, rows, n))
        dt = time.perf_counter() - t0
    return s, envelope(prof), steps / dt


def _scaled(cfg, amp_scale: float = 1.0, period: int = None):
    import copy
    c = copy.copy(cfg)
    c.drive_amp = cfg.drive_amp * amp_scale
    if period is not None:
        c.drive_period = int(period)
    return c


def _share(items: List, rank: int, ws: int) -> List:
    return [x for i, x in enumerate(items) if i % ws == rank]


def _dist():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def _gather(obj, ws):
    if ws == 1:
        return [obj]
    import torch.distributed as dist
    out = [None] * ws
    dist.all_gather_object(out, obj)
    return out


def main(argv=None):
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    ap.add_argument("kind", choices=["linearity", "sweep"])
    ap.add_argument("--config", default="3")
    ap.add_argument("--steps", type=int, default=400)
    ap.add_argument("--every", type=int, default=10)
    ap.add_argument("--window-start", type=int, default=0)
    ap.add_argument("--amp", type=float, default=1e-6, help="total drive amplitude of the base run")
    ap.add_argument("--scale", type=float, default=10.0)
    ap.add_argument("--periods", default="50,100,200", help="drive periods (steps) for sweep")
    args = ap.parse_args(argv)
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from gen import make_config
    import torch
    ws, rank, local = _dist()
    torch.cuda.set_device(local)
    if ws > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    base = make_config(args.config)
    n_drive = base.drive_idx.size
    base.drive_amp = args.amp / n_drive
    if args.kind == "linearity":
        runs = [("x1", _scaled(base, 1.0)), (f"x{args.scale:g}", _scaled(base, args.scale))]
    else:
        runs = [(f"T{p}", _scaled(base, 1.0, int(p))) for p in args.periods.split(",")]
    mine = {}
    for name, cfg in _share(runs, rank, ws):
        s, env, sps = run_replica(cfg, args.steps, args.every, args.window_start)
        mine[name] = {"stations": s.tolist(), "env": env.tolist(), "steps_per_s": sps}
    allres = {}
    for d in _gather(mine, ws):
        allres.update(d)
    if rank == 0:
        out = {"kind": args.kind, "config": args.config, "steps": args.steps, "replicas": len(runs),
               "gpus": ws, "steps_per_s": {k: v["steps_per_s"] for k, v in allres.items()}}
        if args.kind == "linearity":
            a, b = (np.array(allres[k]["env"]) for k, _ in runs)
            out["linearity"] = linearity(a, b, args.scale)
            out["peak_env_x1"] = float(a.max())
        else:
            st = np.array(allres[runs[0][0]]["stations"])
            out["peaks"] = {k: peak_location(np.array(allres[k]["env"]), st) for k, _ in runs}
        print(json.dumps(out), flush=True)
    if ws > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
