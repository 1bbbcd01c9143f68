#!/usr/bin/env python
"""Benchmark of the B200 IB time step (BASELINE.json metric: IB time steps/s at 256^3, fp64).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config 4] [--impl ours|reference]

One "step" = one full IB time step (force, spread, fluid solve, interpolate, update) of
BASELINE.json configs[3] (256^3 grid, 2,097,152 Lagrangian points), synthetic seeded
inputs (gen/).  N > 1: one process per GPU (torchrun), each running an independent
replica (DESIGN.md §7 "replicas only"; no data-path collective), timed on the device and
reduced as the max over ranks; value = total steps of all ranks / time.
`--impl reference` times the CPU oracle (the reference arm of this tier) on the host.
Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "IB time steps/sec at 256^3 grid (fp64); per-stage achieved HBM GB/s vs peak"
UNIT = "steps/s"
SORT_PERIOD = 32          # steps between re-binnings inside ib_step (csrc ib_internal.cuh)


# ------------------------------------------------------------------ algorithmic bytes
def dims(N):
    """(N1, N2, N3) from an int (cubic lattice) or a 3-sequence (x, y, z)."""
    return tuple(int(v) for v in N) if isinstance(N, (tuple, list)) else (int(N),) * 3


def grid_name(N) -> str:
    n1, n2, n3 = dims(N)
    return f"{n1}^3" if n1 == n2 == n3 else f"{n1}x{n2}x{n3}"


def stage_bytes(N, np_: int, nd: int = 0) -> dict:
    """Compulsory HBM bytes per launch of each stage (DESIGN.md §5 byte model).
    V = N1 N2 N3 cells, C = N2 N3 (N1/2+1) complex modes per component."""
    n1, n2, n3 = dims(N)
    V = n1 * n2 * n3
    C = n2 * n3 * (n1 // 2 + 1)
    return {
        # X (24) + neighbour X (24, cached) + per-point k/L0 (32) -> 80 B/pt; F band RMW
        # is on-chip (L2 atomics) and not counted
        "force_spread": 80 * np_,
        "xfwd_rhs_r2c": 24 * V + 24 * V + 48 * C,     # read u, read F, write r^ (x-spectrum)
        "y_fwd": 96 * C,                              # read + write 3 complex components
        "z_solve": 96 * C,
        "y_inv": 96 * C,
        "xinv_c2r": 48 * C + 24 * V,                  # read spectrum, write u^{n+1}
        "interp_update": 48 * np_,                    # read X, write X (u band from L2)
    }


def load_peaks() -> dict:
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return {"hbm_gbs": float(d["hbm_gbs"]), "source": "measured (MEASURED_PEAKS.json)"}
    return {"hbm_gbs": 6650.0, "source": "fallback (B200_PROFILING.md)"}


def cfg_key(k) -> str:
    return f"cfg{k}"


def ncu_traffic(stage: str, config) -> float | None:
    """dram__bytes_read.sum + dram__bytes_write.sum per launch of `stage` for THIS config from
    its committed ncu --set full summary (profiles/ncu_traffic_cfg<k>.json), else None."""
    p = os.path.join(ROOT, "profiles", f"ncu_traffic_{cfg_key(config)}.json")
    if not os.path.exists(p):
        return None
    try:
        d = json.load(open(p))
        v = d.get("stages", {}).get(stage)
        return None if v is None else float(v)
    except Exception:
        return None


def ncu_source(config) -> str | None:
    p = os.path.join(ROOT, "profiles", f"ncu_traffic_{cfg_key(config)}.json")
    if not os.path.exists(p):
        return None
    try:
        return json.load(open(p)).get("source")
    except Exception:
        return None


def cpu_model() -> str:
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            if line.startswith("Model name:"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


# ------------------------------------------------------------------ clocks
class ClockSampler:
    """SM clocks and throttle reasons sampled DURING the timed region (NVML every ~10 ms,
    nvidia-smi as a fallback), summarised as {"sm_mhz": median, "sm_max_mhz", "reasons"}."""
    REASONS = {0x4: "sw_power_cap", 0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown",
               0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown"}
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int, period_s: float = 0.01):
        self.idx = gpu_index
        self.period = period_s
        self.sm, self.mx, self.reasons = [], [], set()
        self.source = None
        self._stop = threading.Event()
        self._t = None
        self._nvml = None
        try:
            import pynvml
            pynvml.nvmlInit()
            vis = os.environ.get("CUDA_VISIBLE_DEVICES")
            phys = int(vis.split(",")[gpu_index]) if vis and vis.split(",")[0].isdigit() else gpu_index
            self._h = pynvml.nvmlDeviceGetHandleByIndex(phys)
            self._nvml = pynvml
            self.source = "nvml"
        except Exception:
            self.source = "nvidia-smi"

    def _sample_nvml(self):
        p = self._nvml
        self.sm.append(float(p.nvmlDeviceGetClockInfo(self._h, p.NVML_CLOCK_SM)))
        self.mx.append(float(p.nvmlDeviceGetMaxClockInfo(self._h, p.NVML_CLOCK_SM)))
        try:
            bits = p.nvmlDeviceGetCurrentClocksEventReasons(self._h)
        except Exception:
            bits = p.nvmlDeviceGetCurrentClocksThrottleReasons(self._h)
        for b, nm in self.REASONS.items():
            if bits & b:
                self.reasons.add(nm)

    def _sample_smi(self):
        out = subprocess.run(["nvidia-smi", f"--id={self.idx}", f"--query-gpu={self.Q}",
                              "--format=csv,noheader,nounits"], capture_output=True, text=True,
                             timeout=5).stdout.strip()
        if not out:
            return
        r = [x.strip() for x in out.split(",")]
        if r[1].replace(".", "").isdigit():
            self.sm.append(float(r[1]))
        if r[2].replace(".", "").isdigit():
            self.mx.append(float(r[2]))
        for k, nm in enumerate(["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown",
                                "sw_power_cap"]):
            if len(r) > 5 + k and r[5 + k].lower().startswith("active"):
                self.reasons.add(nm)

    def _run(self):
        while not self._stop.is_set():
            try:
                self._sample_nvml() if self._nvml else self._sample_smi()
            except Exception:
                pass
            self._stop.wait(self.period)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._t:
            self._t.join(timeout=6)

    def summary(self) -> dict:
        if not self.sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no clock samples"],
                    "samples": 0, "source": self.source}
        return {"sm_mhz": float(np.median(self.sm)), "sm_max_mhz": max(self.mx) if self.mx else None,
                "reasons": sorted(self.reasons), "samples": len(self.sm), "source": self.source}


# ------------------------------------------------------------------ distributed helpers
def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def reduce_max(x: float) -> float:
    """Max over ranks (the timed region's duration); identity without a process group."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()):
        return float(x)
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([float(x)], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def job_throughput(ws: int, steps: int, ms_max: float) -> float:
    """Whole-job steps/s: every rank runs `steps` steps of its own replica; the job takes the
    slowest rank's device time (ms_max, the max over ranks)."""
    return ws * steps / (ms_max / 1e3)


def barrier():
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized():
        dist.barrier()


# ------------------------------------------------------------------ reference arm (oracle)
def run_reference(args, ws, rank):
    if rank != 0:
        return 0
    import oracle
    from gen import make_config
    oracle.set_threads(os.cpu_count() or 1)
    cfg = make_config(args.config)
    o = oracle.Oracle.from_config(cfg)
    k = max(1, min(args.steps, args.ref_max_steps))
    w = min(args.warmup, 1)
    o.step(w)
    t0 = time.perf_counter()
    o.step(k)
    dt = time.perf_counter() - t0
    v = k / dt
    sample = f"{k} full IB steps of cfg{args.config} ({grid_name(cfg.N)}, {cfg.np_} points) after {w} warm-up"
    line = {"metric": METRIC, "value": v, "unit": UNIT, "impl": "reference", "n_gpus": ws,
            "steps": k, "warmup": w, "ms_per_step": 1e3 * dt / k, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(cfg, args.config),
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": oracle.get_threads(),
                             "kind": "oracle", "sample": sample, "cpu_model": cpu_model(),
                             "host_cpus": os.cpu_count()},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


def workload_config(cfg, k):
    src = (f"BASELINE.json configs[{int(k) - 1}]" if k != "4h" else
           "half-cube variant of BASELINE.json configs[3] (PAPER.md 1003-1007)")
    return {"workload": f"{src} ({cfg.name}): {grid_name(cfg.N)} periodic grid, "
                        f"{cfg.np_} Lagrangian points",
            "N": cfg.N if isinstance(cfg.N, int) else list(cfg.N),
            "lagrangian_points": cfg.np_, "global_batch": 1,
            "parallelism": "replicas", "l2": "inputs larger than L2 (u + spectrum >> 126 MB)"
            if np.prod(dims(cfg.N)) >= 128 ** 3 * 4 else "working set fits in L2 (no flush)"}


# ------------------------------------------------------------------ our arm
def run_ours(args, ws, rank, local):
    import torch
    from gen import make_config
    from paper_math_0301321_b200 import IBContext, IB_OPT_STAGE_TIMING
    from paper_math_0301321_b200 import ib as ibmod

    torch.cuda.set_device(local)
    cfg = make_config(args.config)
    N, npts = cfg.N, cfg.np_
    ctx = IBContext.from_config(cfg)
    stream = torch.cuda.Stream()
    ctx.set_stream(stream.cuda_stream)
    with torch.cuda.stream(stream):
        ctx.step(args.warmup)                              # untimed warm-up
        ctx.launch_count(reset=True)
        # (A) the headline: the product path (CUDA-graph replays), device-timed
        barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with ClockSampler(local) as clk:
            e0.record(stream)
            ctx.step(args.steps)
            e1.record(stream)
            torch.cuda.synchronize()
        barrier()
        ms = e0.elapsed_time(e1)
        launches = ctx.launch_count(reset=True)
        # (B) per-stage CUDA events on the context stream (graph off while recording them)
        ctx.set_option(IB_OPT_STAGE_TIMING, 1)
        ctx.stage_times(reset=True)
        torch.cuda.synchronize()
        f0, f1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        f0.record(stream)
        ctx.step(args.steps)
        f1.record(stream)
        torch.cuda.synchronize()
        ms_staged = f0.elapsed_time(f1)
        stages = ctx.stage_times(reset=True)
        ctx.set_option(IB_OPT_STAGE_TIMING, 0)
    ms_max = reduce_max(ms)
    value = job_throughput(ws, args.steps, ms_max)

    # per-stage roofline against the measured HBM copy peak: algorithmic bytes (DESIGN.md §5
    # model) and, beside them, the ncu-measured DRAM bytes of this config's committed capture
    peaks = load_peaks()
    sb = stage_bytes(N, npts)
    per_stage = {}
    for k, t in stages.items():
        avg = t / args.steps
        gbs = sb[k] / (avg / 1e3) / 1e9 if avg > 0 else None
        nb = ncu_traffic(k, args.config)
        dgbs = nb / (avg / 1e3) / 1e9 if (nb is not None and avg > 0) else None
        per_stage[k] = {"ms": avg, "alg_bytes": sb[k], "gbs": gbs,
                        "frac": gbs / peaks["hbm_gbs"] if gbs else None,
                        "dram_bytes": nb, "dram_gbs": dgbs,
                        "dram_frac": dgbs / peaks["hbm_gbs"] if dgbs else None}
    # the re-binning (counting sort of the points by cell) runs every 32 steps outside the
    # step graph; timed here on its own and reported amortised
    rb0, rb1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    nrb = 5
    with torch.cuda.stream(stream):
        ctx.rebin()
        rb0.record(stream)
        for _ in range(nrb):
            ctx.rebin()
        rb1.record(stream)
    torch.cuda.synchronize()
    rebin_ms = rb0.elapsed_time(rb1) / nrb
    per_stage["rebin_amortized"] = {"ms": rebin_ms / SORT_PERIOD, "ms_per_call": rebin_ms,
                                    "period_steps": SORT_PERIOD}
    dom = max(stages, key=lambda k: stages[k])
    avg_dom = stages[dom] / args.steps
    achieved = sb[dom] / (avg_dom / 1e3) / 1e9
    step_bytes = sum(sb.values())
    ms_step = ms_max / args.steps
    ncu_step = [ncu_traffic(k, args.config) for k in stages]
    ncu_step_bytes = sum(ncu_step) if all(v is not None for v in ncu_step) else None
    nb_dom = ncu_traffic(dom, args.config)
    roof = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peaks["hbm_gbs"],
            "unit": "GB/s", "frac": achieved / peaks["hbm_gbs"], "traffic": nb_dom,
            "dram_frac": (nb_dom / (avg_dom / 1e3) / 1e9 / peaks["hbm_gbs"]) if nb_dom else None,
            "traffic_source": ncu_source(args.config),
            "peak_source": peaks["source"],
            "timing": "kernel: mean per-stage CUDA-event time over a second timed region of "
                      f"{args.steps} steps (stage events, no graph; {ms_staged / args.steps:.4f} "
                      "ms/step there)",
            "step": {"alg_bytes": step_bytes, "ms": ms_step,
                     "gbs": step_bytes / (ms_step / 1e3) / 1e9,
                     "frac": step_bytes / (ms_step / 1e3) / 1e9 / peaks["hbm_gbs"],
                     "dram_bytes": ncu_step_bytes,
                     "dram_frac": (ncu_step_bytes / (ms_step / 1e3) / 1e9 / peaks["hbm_gbs"])
                     if ncu_step_bytes else None,
                     "ms_incl_rebin": ms_step + rebin_ms / SORT_PERIOD}}

    # end-to-end through the C-ABI with pinned host buffers: per step H2D (u, X), step,
    # D2H (u, X)
    ke = max(2, min(args.steps, args.e2e_steps))
    n1, n2, n3 = dims(N)
    hu = torch.empty((3, n3, n2, n1), dtype=torch.float64).pin_memory()
    hX = torch.empty((npts, 3), dtype=torch.float64).pin_memory()
    ctx.get_fields_into(hu)
    ctx.get_positions_into(hX)
    torch.cuda.synchronize()
    barrier()
    t0 = time.perf_counter()
    for _ in range(ke):
        ibmod.ib_set_velocity(ctx.ctx, hu, dims(N))
        ibmod.ib_set_positions(ctx.ctx, hX)
        ctx.step(1)
        ctx.get_fields_into(hu)
        ctx.get_positions_into(hX)
    torch.cuda.synchronize()
    te = reduce_max(time.perf_counter() - t0)
    e2e = {"value": ws * ke / te, "unit": UNIT, "h2d_bytes_per_step": hu.numel() * 8 + hX.numel() * 8,
           "d2h_bytes_per_step": hu.numel() * 8 + hX.numel() * 8, "steps": ke,
           "path": "ib_set_velocity + ib_set_positions (pinned host) -> ib_step(1) -> "
                   "ib_get_fields + ib_get_positions (pinned host)"}
    ctx.close()

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(args)

    if rank == 0:
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_max / args.steps,
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
                "dtype": "f64", "data": "synthetic", "config": workload_config(cfg, args.config),
                "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "clocks": clk.summary(),
                "gpu_launches": launches,
                "throughput": {"cells_per_s": value * int(np.prod(dims(N))), "points_per_s": value * npts,
                               "steps_per_s_incl_rebin": ws * 1e3 / roof["step"]["ms_incl_rebin"]},
                "stages": per_stage}
        print(json.dumps(line), flush=True)
    return 0


def run_slab(args, ws, rank, local):
    """--mode slab: the z-slab decomposition.  N = 1: P slab contexts on one
    GPU with device copies in place of the collectives (an emulation: it measures the
    decomposed kernels plus the copies, not NVLink); N > 1: one slab per GPU, NCCL
    all-to-all / all-gather between the phases (total work fixed: strong scaling)."""
    import torch
    from gen import make_config
    from paper_math_0301321_b200 import slab as slabmod
    torch.cuda.set_device(local)
    cfg = make_config(args.config)
    stream = torch.cuda.Stream()
    with torch.cuda.stream(stream):
        if ws == 1:
            P = args.slab_P
            run = slabmod.LocalSlabs(cfg, P, stream, fused=args.slab_fused)
            par = (f"slab{P} emulated on 1 GPU, fused transposes (peer stores from the y-forward "
                   f"and z-solve kernels; device copies for the ghost planes and records)"
                   if args.slab_fused else
                   f"slab{P} emulated on 1 GPU (device copies in place of collectives)")
        else:
            P = ws
            run = slabmod.DistSlab(cfg)
            stream = run.stream
            par = f"slab{P} over {ws} GPUs (NCCL all-to-all / all-gather)"
        run.step(args.warmup)
        barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with ClockSampler(local) as clk:
            e0.record(stream)
            run.step(args.steps)
            e1.record(stream)
            torch.cuda.synchronize()
        barrier()
        ms = reduce_max(e0.elapsed_time(e1))
        run.close()
    value = args.steps / (ms / 1e3)                  # whole-lattice steps per second
    if rank == 0:
        wc = workload_config(cfg, args.config)
        wc["parallelism"] = par
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": ws, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": wc, "mode": "slab", "slab_P": P, "slab_fused": bool(args.slab_fused and ws == 1),
                "clocks": clk.summary(),
                "note": "not the headline: --mode replicas (default) is; see DESIGN.md §10"}
        print(json.dumps(line), flush=True)
    return 0


def cpu_baseline(args):
    """The oracle as it stands, on this host's cores, on a bounded sample: IB steps of the
    same config until about 10 s have passed (at least one step) on all cores, then one
    step on a single thread (1 thread is the baseline, all cores beside it)."""
    import oracle
    from gen import make_config
    ncores = os.cpu_count() or 1
    oracle.set_threads(ncores)
    cfg = make_config(args.config)
    o = oracle.Oracle.from_config(cfg)
    k, t0 = 0, time.perf_counter()
    while k < 1 or (time.perf_counter() - t0 < 10.0 and k < 50):
        o.step(1)
        k += 1
    dt = time.perf_counter() - t0
    one = None
    if not args.no_cpu_1thread:
        oracle.set_threads(1)
        k1, t1 = 0, time.perf_counter()
        while k1 < 1 or (time.perf_counter() - t1 < 5.0 and k1 < 50):
            o.step(1)
            k1 += 1
        d1 = time.perf_counter() - t1
        one = {"value": k1 / d1, "unit": UNIT, "cores": 1,
               "sample": f"{k1} full IB step(s) of cfg{args.config}, {d1:.1f} s"}
        oracle.set_threads(ncores)
    return {"value": k / dt, "unit": UNIT, "cores": oracle.get_threads(), "kind": "oracle",
            "cpu_model": cpu_model(), "host_cpus": ncores,
            "sample": f"{k} full IB steps of cfg{args.config} ({grid_name(cfg.N)}, {cfg.np_} points), "
                      f"{dt:.1f} s on {ncores} threads",
            "one_thread": one}


def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="4", help="1..5 (BASELINE.json configs) or 4h (half-cube)")
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--mode", choices=["replicas", "slab"], default="replicas",
                    help="replicas (default, the headline): one independent IB run per GPU; "
                         "slab: the z-slab decomposition of one lattice")
    ap.add_argument("--slab-P", type=int, default=4, help="slabs emulated on one GPU (--mode slab, N = 1)")
    ap.add_argument("--slab-fused", action="store_true",
                    help="--mode slab, N = 1: fused transposes (ib_slab_set_peers) instead of copies")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-cpu-1thread", action="store_true")
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--ref-max-steps", type=int, default=6)
    args = ap.parse_args(argv)
    if args.warmup < 3 and args.impl == "ours":
        args.warmup = 3                                    # timing rule: W >= 3
    ws, rank, local = dist_env()
    if args.impl == "reference":
        return run_reference(args, ws, rank)      # rank 0 only; no process group needed
    if ws > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    try:
        if args.mode == "slab":
            return run_slab(args, ws, rank, local)
        return run_ours(args, ws, rank, local)
    finally:
        if ws > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    sys.exit(main())
