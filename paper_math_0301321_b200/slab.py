"""The IB step over P z-slabs of the lattice.

The paper partitions its fluid and material grids over processors (PAPER.md 801-807); on
B200s the partition is one z-slab per GPU.  Every arithmetic step runs in libib_b200.so
(`ib_slab_phase`); this module owns the exchange buffers (torch device memory) and moves
them between the phases:

  after phase 0   all-to-all per component: s2 [dst][Ky][L] -> z [src][Ky][L]  (y -> z transpose)
  after phase 1   all-to-all per component: z -> s2                          (z -> y transpose)
  after phase 2   all-gather of the edge planes (ghost planes of u)
  after phase 3   all-gather of the owned points' X^{n+1} records (replicated X)

With fused=True the first two exchanges disappear: the y-forward and z-solve kernels store
the transposed blocks straight into the peers' s2 / z buffers (ib_slab_set_peers).

`LocalSlabs` runs P slab contexts in one process on one GPU with device copies in place of
the collectives (the parity harness: the decomposition is checked against the oracle on a
single GPU); `DistSlab` is one rank of a torch.distributed job (NCCL across GPUs) using the
same buffers and phase sequence.  `exchange_local` and `exchange_dist` are written over
plain torch tensors, so the exchange plumbing is testable on CPU with gloo.
"""
from __future__ import annotations

import ctypes as C
from typing import List, Sequence

import numpy as np

from .ib import IBContext, IBError, IB_EINVAL, _check, dims, load


def slab_shapes(N, P: int):
    """Exchange-buffer shapes (element type float64; complex stored as pairs) of one rank."""
    n1, n2, n3 = dims(N)
    L, Ky, Pc = n3 // P, n2 // P, n1 // 2 + 2
    return {
        "s2": (3, P, Ky, L, Pc, 2),          # [comp][dst][Ky][L][Pc] complex (y pass output)
        "z": (3, P, Ky, L, Pc, 2),           # [comp][src][Ky][L][Pc] complex (z pass input)
        "edge_send": (3, 3, n2, n1),         # [last, first, second owned plane][comp]
        "edge_recv": (P, 3, 3, n2, n1),
    }


class SlabRank(IBContext):
    """Rank `rank` of P z-slabs (ib_slab_create) with its exchange buffers as torch tensors
    on `device`.  np_cap bounds the structure size (the record buffers are np_cap long)."""

    def __init__(self, N, h, rho, mu, dt, P: int, rank: int, np_cap: int, device="cuda"):
        import torch
        self.dims = dims(N)
        self.N = self.dims
        self.h, self.rho, self.mu, self.dt = float(h), float(rho), float(mu), float(dt)
        self.P, self.rank = int(P), int(rank)
        n1, n2, n3 = self.dims
        self.ctx = load().ib_slab_create(n1, n2, n3, self.h, self.rho, self.mu, self.dt, self.P,
                                         self.rank)
        if not self.ctx:
            raise IBError(IB_EINVAL, load().ib_last_error().decode())
        self.np = 0
        info = (C.c_int32 * 8)()
        _check(load().ib_slab_info(self.ctx, info, 8))
        self.L, self.Ky = int(info[2]), int(info[3])
        f64 = dict(dtype=torch.float64, device=device)
        sh = slab_shapes(self.dims, self.P)
        self.s2 = torch.zeros(sh["s2"], **f64)
        self.z = torch.zeros(sh["z"], **f64)
        self.edge_send = torch.zeros(sh["edge_send"], **f64)
        self.edge_recv = torch.zeros(sh["edge_recv"], **f64)
        self.cap = max(1, int(np_cap))
        self.pack_send = torch.zeros((self.cap, 4), **f64)
        self.pack_recv = torch.zeros((self.P, self.cap, 4), **f64)
        self.count_send = torch.zeros(1, dtype=torch.int64, device=device)
        self.count_recv = torch.zeros(self.P, dtype=torch.int64, device=device)
        p = lambda t: C.c_void_p(t.data_ptr())
        _check(load().ib_slab_set_buffers(self.ctx, p(self.s2), p(self.z), p(self.edge_send),
                                          p(self.edge_recv), p(self.pack_send), p(self.pack_recv),
                                          p(self.count_send), p(self.count_recv), self.cap))

    @classmethod
    def from_config(cls, cfg, P: int, rank: int, device="cuda"):
        o = cls(cfg.N, cfg.h, cfg.rho, cfg.mu, cfg.dt, P, rank, cfg.np_, device)
        o.set_structure(cfg.X, cfg.patches, cfg.stiffness)
        if cfg.u0 is not None:
            o.set_velocity(cfg.u0)                # the whole lattice; the rank keeps its planes
        if cfg.drive_idx is not None:
            o.set_drive(cfg.drive_idx, cfg.drive_dir, cfg.drive_amp, cfg.drive_period)
        if getattr(cfg, "fixed", None) is not None:
            o.set_fixed(cfg.fixed)
        return o

    @property
    def fshape(self):                             # owned planes
        n1, n2, _ = self.dims
        return (3, self.L, n2, n1)

    def phase(self, k: int):
        _check(load().ib_slab_phase(self.ctx, int(k)))

    def sync(self):
        _check(load().ib_slab_sync(self.ctx))

    def step(self, nsteps=1):
        raise IBError(-5, "slab ranks step through LocalSlabs / DistSlab")

    def get_fields(self, want_p=False):
        if want_p:
            raise IBError(-5, "slab context: no pressure output")
        u = np.empty(self.fshape)
        _check(load().ib_get_fields(self.ctx, u.ctypes.data_as(C.c_void_p), None))
        return u, None


# ------------------------------------------------------------------ exchanges
def exchange_local(ranks: Sequence, phase: int, counts=None) -> None:
    """The exchange after `phase` between P ranks of one process (device copies standing in
    for the collectives; objects with the SlabRank buffer attributes)."""
    if phase == 0:                                 # y -> z transpose
        for r in ranks:
            for q in ranks:
                q.z[:, r.rank].copy_(r.s2[:, q.rank])
    elif phase == 1:                               # z -> y transpose
        for r in ranks:
            for q in ranks:
                r.s2[:, q.rank].copy_(q.z[:, r.rank])
    elif phase == 2:                               # ghost planes: all-gather of the edges
        for q in ranks:
            for r in ranks:
                q.edge_recv[r.rank].copy_(r.edge_send)
    elif phase == 3:                               # replicated X: all-gather of the records
        if counts is None:
            counts = [int(r.count_send.item()) for r in ranks]
        for q in ranks:
            for r in ranks:
                q.count_recv[r.rank].copy_(r.count_send[0])
                k = counts[r.rank]
                if k:
                    q.pack_recv[r.rank, :k].copy_(r.pack_send[:k])


def exchange_dist(rank, phase: int, group=None) -> None:
    """The same exchange as exchange_local for ONE rank of a torch.distributed job."""
    import torch
    import torch.distributed as dist
    if phase == 0:
        for c in range(3):
            dist.all_to_all_single(rank.z[c], rank.s2[c], group=group)
    elif phase == 1:
        for c in range(3):
            dist.all_to_all_single(rank.s2[c], rank.z[c], group=group)
    elif phase == 2:
        # output viewed as the concatenation along dim 0 (what every backend accepts)
        dist.all_gather_into_tensor(rank.edge_recv.view(-1, *rank.edge_send.shape[1:]),
                                    rank.edge_send, group=group)
    elif phase == 3:
        dist.all_gather_into_tensor(rank.count_recv, rank.count_send, group=group)
        k = int(rank.count_recv.max().item())
        if k:
            tmp = torch.empty((rank.P * k, 4), dtype=rank.pack_send.dtype, device=rank.pack_send.device)
            dist.all_gather_into_tensor(tmp, rank.pack_send[:k].contiguous(), group=group)
            rank.pack_recv[:, :k].copy_(tmp.view(rank.P, k, 4))


# ------------------------------------------------------------------ drivers
def set_peers(rank, s2_ptrs: Sequence[int], z_ptrs: Sequence[int]) -> None:
    """Fused transposes for `rank` (ib_slab_set_peers): phase 0 / 1 store straight into the
    peers' z / s2 buffers (device pointers valid in this process); empty lists switch back
    to the exchange mode."""
    P = len(s2_ptrs)
    arr = C.c_void_p * max(P, 1)
    _check(load().ib_slab_set_peers(rank.ctx, P, arr(*s2_ptrs) if P else None,
                                    arr(*z_ptrs) if P else None))


class LocalSlabs:
    """P slab ranks of one lattice in one process on the current GPU, all on one stream.

    fused=True: the y-forward and z-solve kernels store the transposed blocks straight into
    the other ranks' buffers (ib_slab_set_peers) — no copies after phases 0 and 1; the one
    stream orders the ranks' phases."""

    def __init__(self, cfg, P: int, stream=None, fused: bool = False):
        import torch
        self.cfg = cfg
        self.P = int(P)
        self.ranks: List[SlabRank] = [SlabRank.from_config(cfg, P, r) for r in range(P)]
        # one NON-default torch stream for the phases and the copies: a NULL handle (torch's
        # legacy default stream) would select each context's own stream (ib_set_stream)
        self.stream = stream if stream is not None else torch.cuda.Stream()
        assert self.stream.cuda_stream != 0, "LocalSlabs needs a non-default stream"
        for r in self.ranks:
            r.set_stream(self.stream.cuda_stream)
        self.set_fused(fused)

    def set_fused(self, fused: bool):
        """Switch between fused transposes (peer stores) and the exchange copies."""
        self.fused = bool(fused)
        s2 = [q.s2.data_ptr() for q in self.ranks] if self.fused else []
        z = [q.z.data_ptr() for q in self.ranks] if self.fused else []
        for r in self.ranks:
            set_peers(r, s2, z)

    def step(self, nsteps: int = 1):
        import torch
        with torch.cuda.stream(self.stream):
            for _ in range(int(nsteps)):
                for ph in range(5):
                    for r in self.ranks:
                        r.phase(ph)
                    if ph < 4 and not (self.fused and ph < 2):
                        exchange_local(self.ranks, ph)
        for r in self.ranks:
            r.sync()

    @property
    def n(self):
        return self.ranks[0].n

    def get_fields(self):
        """u of the whole lattice, [3][N3][N2][N1] (the ranks' owned planes stacked)."""
        return np.concatenate([r.get_fields()[0] for r in self.ranks], axis=1), None

    def get_positions(self, rank: int = 0):
        return self.ranks[rank].get_positions()

    def launch_count(self, reset=False):
        return sum(r.launch_count(reset) for r in self.ranks)

    def close(self):
        for r in self.ranks:
            r.close()

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


def _peer_views(t, group):
    """Every rank's copy of buffer t as a tensor mapped into this process: CUDA IPC handles
    (torch's tensor sharing) exchanged with all_gather_object; this rank's own entry is t."""
    import torch.distributed as dist
    from torch.multiprocessing.reductions import reduce_tensor
    P, me = dist.get_world_size(group), dist.get_rank(group)
    if P == 1:
        return [t]
    shared = [None] * P
    dist.all_gather_object(shared, reduce_tensor(t), group=group)
    return [t if d == me else shared[d][0](*shared[d][1]) for d in range(P)]


class DistSlab:
    """This process's rank of a P-GPU slab decomposition (torch.distributed, NCCL).

    fused=True: the y-forward and z-solve kernels store the transposed blocks straight into
    the peers' buffers (mapped with CUDA IPC; NVLink peer stores), and a one-element NCCL
    all-reduce on the phase stream orders the ranks after phases 0 and 1 instead of the two
    all-to-alls.  Only a world of one rank (peers = itself) is exercised on this pool's
    one-GPU boxes; the IPC mapping across GPUs is untested here."""

    def __init__(self, cfg, group=None, fused: bool = False):
        import torch
        import torch.distributed as dist
        self.group = group
        P, rank = dist.get_world_size(group), dist.get_rank(group)
        self.rank = SlabRank.from_config(cfg, P, rank)
        self.stream = torch.cuda.Stream()          # non-default: see LocalSlabs
        self.rank.set_stream(self.stream.cuda_stream)
        self.fused = bool(fused)
        if self.fused:
            self._s2 = _peer_views(self.rank.s2, group)      # keep the mappings alive
            self._z = _peer_views(self.rank.z, group)
            set_peers(self.rank, [t.data_ptr() for t in self._s2], [t.data_ptr() for t in self._z])
            self._tick = torch.zeros(1, dtype=torch.float64, device=self.rank.s2.device)

    def step(self, nsteps: int = 1):
        import torch
        import torch.distributed as dist
        with torch.cuda.stream(self.stream):      # the collectives wait on this stream
            for _ in range(int(nsteps)):
                for ph in range(5):
                    self.rank.phase(ph)
                    if ph < 4:
                        if self.fused and ph < 2:  # peer stores landed on every rank
                            dist.all_reduce(self._tick, group=self.group)
                        else:
                            exchange_dist(self.rank, ph, self.group)
        self.rank.sync()

    def close(self):
        self.rank.close()
