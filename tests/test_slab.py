"""Slab decomposition of the IB step along z.

GPU: P slab contexts in one process (device copies in place of the collectives,
paper_math_0301321_b200.slab.LocalSlabs) against the oracle at checkpoints 1, 2 and 10 on
BASELINE.json configs[2] (128^3) and configs[3] (256^3) and a small sheet, P = 2, 4 (8).
CPU: the exchange plumbing (exchange_dist over torch.distributed) on a gloo world of size 2
against the single-process exchange (exchange_local) on the same buffers.
"""
import os
import socket

import numpy as np
import pytest
import torch

from gen import make_config, small_sheet_config
from parity import rel_l2, step_parity


# ------------------------------------------------------------------ exchange plumbing (CPU)
class _FakeRank:
    """The SlabRank buffer attributes on CPU tensors, filled from a seed per rank."""

    def __init__(self, N, P, rank, cap=64):
        from paper_math_0301321_b200.slab import slab_shapes
        g = torch.Generator().manual_seed(1000 + rank)
        sh = slab_shapes(N, P)
        self.P, self.rank, self.cap = P, rank, cap
        self.s2 = torch.randn(sh["s2"], generator=g, dtype=torch.float64)
        self.z = torch.zeros(sh["z"], dtype=torch.float64)
        self.edge_send = torch.randn(sh["edge_send"], generator=g, dtype=torch.float64)
        self.edge_recv = torch.zeros(sh["edge_recv"], dtype=torch.float64)
        k = 5 + 7 * rank
        self.pack_send = torch.zeros((cap, 4), dtype=torch.float64)
        self.pack_send[:k] = torch.randn((k, 4), generator=g, dtype=torch.float64)
        self.pack_recv = torch.zeros((P, cap, 4), dtype=torch.float64)
        self.count_send = torch.tensor([k], dtype=torch.int64)
        self.count_recv = torch.zeros(P, dtype=torch.int64)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, ws, port, N, q):
    import torch.distributed as dist
    from paper_math_0301321_b200.slab import exchange_dist, exchange_local
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    try:
        me = _FakeRank(N, ws, rank)
        ref = [_FakeRank(N, ws, r) for r in range(ws)]       # every rank's buffers, locally
        ok = True
        for ph in range(4):
            exchange_dist(me, ph)
            exchange_local(ref, ph)
            for name in ("s2", "z", "edge_recv", "count_recv"):
                ok &= torch.equal(getattr(me, name), getattr(ref[rank], name))
            for r in range(ws):
                k = int(ref[r].count_send[0])
                ok &= torch.equal(me.pack_recv[r, :k], ref[rank].pack_recv[r, :k])
        # after the forward and the backward transpose s2 is back to its start
        ok &= torch.equal(me.s2, _FakeRank(N, ws, rank).s2)
        q.put((rank, bool(ok)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("N", [(64, 64, 64), (64, 128, 32)])
def test_slab_exchange_plumbing_gloo_world2(N):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    ps = [ctx.Process(target=_worker, args=(r, 2, port, N, q)) for r in range(2)]
    for p in ps:
        p.start()
    res = dict(q.get(timeout=120) for _ in ps)
    for p in ps:
        p.join(timeout=60)
    assert res == {0: True, 1: True}


def test_slab_transpose_is_the_z_pencil_layout():
    """After the y -> z exchange, rank q's z[c][src][ky][zl] holds S2 row ky = q Ky + ky of
    plane z = src L + zl: the z pass's 5-D view (x, zl, ky, src, comp) reads whole pencils."""
    from paper_math_0301321_b200.slab import exchange_local
    N, P = (64, 64, 64), 4
    ranks = [_FakeRank(N, P, r) for r in range(P)]
    exchange_local(ranks, 0)
    L, Ky = 64 // P, 64 // P
    # global S2 [comp][ky][z] from the ranks' local S2 [comp][ky][zl]
    glob = torch.cat([r.s2.reshape(3, 64, L, -1, 2) for r in ranks], dim=2)   # [3][ky][z]
    for q in range(P):
        zq = ranks[q].z                                      # [3][src][Ky][L]
        pencil = zq.permute(0, 2, 1, 3, 4, 5).reshape(3, Ky, 64, -1, 2)
        assert torch.equal(pencil, glob[:, q * Ky:(q + 1) * Ky])


# ------------------------------------------------------------------ GPU parity
@pytest.fixture(scope="module")
def slabm():
    from paper_math_0301321_b200 import _build, ib
    _build.build()
    ib.load()
    from paper_math_0301321_b200 import slab
    return slab


def _slab_parity(slabm, olib, cfg, P):
    rep = step_parity(olib, cfg, lambda: slabm.LocalSlabs(cfg, P), check_U=False)
    return rep


@pytest.mark.gpu
@pytest.mark.parametrize("P", [2, 4, 8])
def test_slab_small_sheet_matches_oracle(slabm, olib, P):
    # dt 2.5e-4: the sheet's stiffest springs and tethers are unstable at dt 1e-3 on h = 1/64
    cfg = small_sheet_config(N=64, n1=40, n2=30, seed=61, u_amp=0.2, dt=2.5e-4)
    print(_slab_parity(slabm, olib, cfg, P))


@pytest.mark.gpu
@pytest.mark.parametrize("P", [2, 4])
def test_slab_config3_matches_oracle(slabm, olib, P):
    print(_slab_parity(slabm, olib, make_config(3), P))


@pytest.mark.gpu
@pytest.mark.slow
@pytest.mark.parametrize("P", [2, 4])
def test_slab_config4_matches_oracle(slabm, olib, P):
    print(_slab_parity(slabm, olib, make_config(4), P))


@pytest.mark.gpu
def test_slab_replicas_agree_and_match_the_whole_lattice(slabm):
    """Every rank's replica of X is the same after the all-gather, and the decomposed step
    agrees with the one-context step to fp64 summation order."""
    from paper_math_0301321_b200 import IBContext
    cfg = small_sheet_config(N=(64, 128, 64), n1=30, n2=24, seed=62, u_amp=0.3, dt=2.5e-4)
    with slabm.LocalSlabs(cfg, 4) as s, IBContext.from_config(cfg) as c:
        s.step(6)
        c.step(6)
        Xs = [s.get_positions(r) for r in range(4)]
        for X in Xs[1:]:
            assert np.array_equal(X, Xs[0])
        us, _ = s.get_fields()
        uc, _ = c.get_fields()
        assert rel_l2(us, uc) < 1e-13
        assert rel_l2(Xs[0] - cfg.X, c.get_positions() - cfg.X) < 1e-11
        assert s.n == c.n == 6


@pytest.mark.gpu
@pytest.mark.parametrize("P", [2, 4, 8])
def test_fused_slab_small_sheet_matches_oracle(slabm, olib, P):
    """Fused transposes (ib_slab_set_peers): the y-forward and z-solve kernels store the
    transposed blocks straight into the other ranks' buffers, no exchange after phases 0-1."""
    cfg = small_sheet_config(N=64, n1=40, n2=30, seed=61, u_amp=0.2, dt=2.5e-4)
    print(step_parity(olib, cfg, lambda: slabm.LocalSlabs(cfg, P, fused=True), check_U=False))


@pytest.mark.gpu
@pytest.mark.parametrize("shape,P", [((64, 128, 64), 4), ((128, 64, 256), 2), ((64, 64, 512), 8)])
def test_fused_slab_equals_exchange_slab(slabm, shape, P):
    """The fused step against the exchange step on anisotropic lattices (z tiles of 8 and 4
    columns, L from 8 to 256): u and X agree to fp64 summation order (spread atomics)."""
    cfg = small_sheet_config(N=shape, n1=30, n2=24, seed=63, u_amp=0.3, dt=2.5e-4)
    with slabm.LocalSlabs(cfg, P) as a, slabm.LocalSlabs(cfg, P, fused=True) as b:
        a.step(4)
        b.step(4)
        ua, _ = a.get_fields()
        ub, _ = b.get_fields()
        assert rel_l2(ub, ua) < 1e-13
        assert rel_l2(b.get_positions() - cfg.X, a.get_positions() - cfg.X) < 1e-11
        b.set_fused(False)                          # back to the exchange mode
        b.step(2)
        a.step(2)
        assert rel_l2(b.get_fields()[0], a.get_fields()[0]) < 1e-13


@pytest.mark.gpu
@pytest.mark.slow
def test_fused_slab_config4_matches_oracle(slabm, olib):
    print(step_parity(olib, make_config(4), lambda: slabm.LocalSlabs(make_config(4), 4, fused=True),
                      check_U=False))


@pytest.mark.gpu
def test_slab_rejects_bad_decompositions(slabm):
    from paper_math_0301321_b200.ib import IBError
    for N, P in (((64, 64, 64), 16), ((64, 64, 64), 3), ((32, 64, 64), 2)):
        with pytest.raises(IBError):
            slabm.SlabRank(N, 1 / N[0], 1.0, 0.01, 1e-3, P, 0, 10)


@pytest.mark.gpu
@pytest.mark.parametrize("fused", [False, True])
def test_distslab_nccl_world1_matches_oracle(slabm, olib, fused):
    """The torch.distributed path (DistSlab: NCCL all_to_all_single / all_gather_into_tensor
    between the phases) in a world of one rank on the box's one GPU, against the oracle at
    steps 1, 2, 10.  (Several ranks need several GPUs; the exchange layout for P = 2 is
    covered by the gloo test above and by LocalSlabs.)"""
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()))
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        cfg = small_sheet_config(N=64, n1=40, n2=30, seed=63, u_amp=0.2, dt=2.5e-4)

        class _Run:
            def __init__(self):
                self.d = slabm.DistSlab(cfg, fused=fused)

            def step(self, k):
                self.d.step(k)

            @property
            def n(self):
                return self.d.rank.n

            def get_fields(self):
                return self.d.rank.get_fields()

            def get_positions(self):
                return self.d.rank.get_positions()

            def close(self):
                self.d.close()

        print(step_parity(olib, cfg, _Run, check_U=False))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_slab_window_plate_matches_oracle(slabm, olib):
    """Fixed rim points and the surface-normal drive (PAPER.md 914-922, 988-993) through the
    slab phases: the normal comes from every rank's replica of X^n; fixed points are owned
    like any other and never move (bitwise)."""
    from gen import window_config
    cfg = window_config(N=64, m=40, seed=9, u_amp=0.05, dt=2.5e-4)
    print(_slab_parity(slabm, olib, cfg, 2))
    with slabm.LocalSlabs(cfg, 2) as s:
        s.step(5)
        X = s.get_positions(1)
    fixed = cfg.fixed.astype(bool)
    assert np.array_equal(X[fixed], cfg.X[fixed])


@pytest.mark.gpu
def test_slab_phases_must_come_in_order(slabm):
    from paper_math_0301321_b200.ib import IBError, IB_ESTATE
    cfg = small_sheet_config(N=64, n1=8, n2=6, seed=64, dt=2.5e-4)
    r = slabm.SlabRank.from_config(cfg, 2, 0)
    try:
        with pytest.raises(IBError) as e:
            r.phase(1)
        assert e.value.code == IB_ESTATE
        r.phase(0)
        with pytest.raises(IBError):
            r.phase(0)
    finally:
        r.close()
