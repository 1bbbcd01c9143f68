"""Multi-process (world_size 2, gloo on CPU) checks of bench.py's replica plumbing: the
max-over-ranks timing reduction, the barrier, the whole-job aggregate, and the reference arm
under torchrun (rank 0 alone prints; the other ranks exit 0).  DESIGN.md §7: replicas only."""
import json
import os
import socket
import subprocess
import sys

import pytest
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, ws, port, out):
    import torch.distributed as dist
    sys.path.insert(0, ROOT)
    import bench
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank,
                            world_size=ws)
    try:
        bench.barrier()
        m = bench.reduce_max(10.0 + 5.0 * rank)      # rank 1 is the slow one
        out[rank] = m
        bench.barrier()
    finally:
        dist.destroy_process_group()


def test_reduce_max_over_two_gloo_ranks():
    ws, port = 2, _free_port()
    with mp.Manager() as man:
        out = man.dict()
        mp.spawn(_worker, args=(ws, port, out), nprocs=ws, join=True)
        assert dict(out) == {0: 15.0, 1: 15.0}


def test_job_throughput_is_whole_job_over_slowest_rank():
    sys.path.insert(0, ROOT)
    import bench
    # 2 replicas x 100 steps, slowest rank 200 ms -> 1000 steps/s for the whole job
    assert bench.job_throughput(2, 100, 200.0) == pytest.approx(1000.0)
    assert bench.job_throughput(1, 100, 200.0) == pytest.approx(500.0)


def test_reference_arm_under_torchrun_prints_once():
    port = _free_port()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port), "bench.py", "--impl",
           "reference", "--gpus", "2", "--config", "1", "--steps", "2", "--warmup", "1"]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["unit"] == "steps/s" and d["value"] > 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["e2e"]["h2d_bytes_per_step"] == 0
