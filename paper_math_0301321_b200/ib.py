"""Thin ctypes binding of the C-ABI in include/ib.h (argument marshalling only).

Every step of the IB method runs in libib_b200.so's sm_100a kernels; this module only
checks dtypes/shapes and passes pointers.  Arrays may be numpy arrays (host) or torch
tensors (host or CUDA; torch is used for device memory and streams only).  There is no
CPU fallback: if the library is missing or no CUDA device is present, calls raise.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional, Sequence

import numpy as np

from . import _build

IB_OK, IB_EINVAL, IB_ENOMEM, IB_ECUDA, IB_ENONFINITE, IB_ESTATE, IB_EDEGENERATE = 0, -1, -2, -3, -4, -5, -6
IB_WRAP1, IB_WRAP2, IB_STRETCH1, IB_STRETCH2, IB_BEND1, IB_BEND2, IB_TETHER = 1, 2, 4, 8, 16, 32, 64
IB_OPT_PRESSURE, IB_OPT_STAGE_TIMING, IB_OPT_GRAPH = 1, 2, 3

EXPORTS = ("ib_create", "ib_create3", "ib_destroy", "ib_set_stream", "ib_set_option", "ib_set_structure",
           "ib_set_positions", "ib_set_velocity", "ib_set_drive", "ib_set_fixed", "ib_step", "ib_get_fields",
           "ib_get_positions", "ib_rebin", "ib_get_step", "ib_set_step", "ib_num_points", "ib_stage_times",
           "ib_launch_count", "ib_last_error", "ib_debug_force", "ib_debug_spread",
           "ib_debug_interp", "ib_debug_rhs", "ib_debug_fluid", "ib_debug_project",
           "ib_debug_fft", "ib_debug_ifft", "ib_slab_create", "ib_slab_info", "ib_slab_set_buffers", "ib_slab_set_peers",
           "ib_slab_phase", "ib_slab_sync")


class IBError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


class ib_patch(C.Structure):
    _fields_ = [("first", C.c_int64), ("n1", C.c_int32), ("n2", C.c_int32),
                ("flags", C.c_uint32), ("pad_", C.c_uint32), ("param_off", C.c_int64)]


_lib = None


def library_path() -> str:
    return _build.SO


def load(path: Optional[str] = None):
    """Load libib_b200.so (raises if it has not been built — no fallback)."""
    global _lib
    if _lib is not None:
        return _lib
    path = path or os.environ.get("IB_B200_LIB") or _build.SO   # env: dev-only variant builds
    if not os.path.exists(path):
        raise ImportError(f"{path} not found: build it with __graft_entry__.build() "
                          "(the IB step has no CPU fallback)")
    L = C.CDLL(path)
    p, d, i32, i64 = C.c_void_p, C.c_double, C.c_int32, C.c_int64
    L.ib_create.restype = p
    L.ib_create.argtypes = [i32, d, d, d, d]
    L.ib_create3.restype = p
    L.ib_create3.argtypes = [i32, i32, i32, d, d, d, d]
    L.ib_destroy.argtypes = [p]
    L.ib_set_stream.argtypes = [p, p]
    L.ib_set_option.argtypes = [p, i32, i64]
    L.ib_set_structure.argtypes = [p, p, i64, p, i32, p, i64]
    L.ib_set_positions.argtypes = [p, p]
    L.ib_set_velocity.argtypes = [p, p]
    L.ib_set_drive.argtypes = [p, p, i64, p, d, i32]
    L.ib_set_fixed.argtypes = [p, p]
    L.ib_step.argtypes = [p, i32]
    L.ib_get_fields.argtypes = [p, p, p]
    L.ib_get_positions.argtypes = [p, p]
    L.ib_rebin.argtypes = [p]
    L.ib_get_step.restype = i64
    L.ib_get_step.argtypes = [p]
    L.ib_set_step.argtypes = [p, i64]
    L.ib_num_points.restype = i64
    L.ib_num_points.argtypes = [p]
    L.ib_stage_times.argtypes = [p, p, i32, p, i32, i32]
    L.ib_launch_count.restype = i64
    L.ib_launch_count.argtypes = [p, i32]
    L.ib_last_error.restype = C.c_char_p
    L.ib_debug_force.argtypes = [p, p]
    L.ib_debug_spread.argtypes = [p, p, p]
    L.ib_debug_interp.argtypes = [p, p, p]
    L.ib_debug_rhs.argtypes = [p, p, p, p]
    L.ib_debug_fluid.argtypes = [p, p, p, p, p]
    L.ib_debug_fft.argtypes = [p, p, p]
    L.ib_debug_project.argtypes = [p, p, p, p]
    L.ib_debug_ifft.argtypes = [p, p, p]
    L.ib_slab_create.restype = p
    L.ib_slab_create.argtypes = [i32, i32, i32, d, d, d, d, i32, i32]
    L.ib_slab_info.argtypes = [p, p, i32]
    L.ib_slab_set_buffers.argtypes = [p, p, p, p, p, p, p, p, p, i64]
    L.ib_slab_set_peers.argtypes = [p, i32, p, p]
    L.ib_slab_phase.argtypes = [p, i32]
    L.ib_slab_sync.argtypes = [p]
    for name in EXPORTS:
        if name not in ("ib_create", "ib_create3", "ib_slab_create", "ib_destroy", "ib_get_step", "ib_num_points",
                        "ib_launch_count", "ib_last_error"):
            getattr(L, name).restype = C.c_int
    _lib = L
    return L


def _check(rc: int):
    if rc != IB_OK:
        raise IBError(rc, load().ib_last_error().decode())


def _ptr(a, dtype=np.float64, size: Optional[int] = None, writable=False):
    """Pointer of a contiguous numpy array or torch tensor (host or CUDA); None passes NULL."""
    if a is None:
        return None
    if isinstance(a, np.ndarray):
        if a.dtype != dtype or not a.flags.c_contiguous:
            raise TypeError(f"need a C-contiguous {np.dtype(dtype)} array")
        if writable and not a.flags.writeable:
            raise TypeError("output array is read-only")
        n = a.size
        ptr = a.ctypes.data
    else:   # torch.Tensor
        import torch
        tdt = {np.float64: torch.float64, np.int64: torch.int64, np.uint8: torch.uint8}[dtype]
        if a.dtype != tdt or not a.is_contiguous():
            raise TypeError(f"need a contiguous {tdt} tensor")
        n = a.numel()
        ptr = a.data_ptr()
    if size is not None and n != size:
        raise ValueError(f"expected {size} elements, got {n}")
    return C.c_void_p(ptr)


# ------------------------------------------------------------------ C-named functions
def dims(N):
    """(N1, N2, N3) from an int (cubic lattice) or a 3-sequence (x, y, z)."""
    if isinstance(N, (tuple, list)):
        return tuple(int(v) for v in N)
    return int(N), int(N), int(N)


def ib_create(N: int, h: float, rho: float, mu: float, dt: float) -> int:
    ctx = load().ib_create(int(N), float(h), float(rho), float(mu), float(dt))
    if not ctx:
        raise IBError(IB_EINVAL, load().ib_last_error().decode())
    return ctx


def ib_create3(N1: int, N2: int, N3: int, h: float, rho: float, mu: float, dt: float) -> int:
    ctx = load().ib_create3(int(N1), int(N2), int(N3), float(h), float(rho), float(mu), float(dt))
    if not ctx:
        raise IBError(IB_EINVAL, load().ib_last_error().decode())
    return ctx


def ib_destroy(ctx: int) -> None:
    load().ib_destroy(ctx)


def ib_set_stream(ctx, stream_handle: int) -> None:
    _check(load().ib_set_stream(ctx, C.c_void_p(stream_handle) if stream_handle else None))


def ib_set_option(ctx, option: int, value: int) -> None:
    _check(load().ib_set_option(ctx, int(option), int(value)))


def _patch_array(patches: Sequence) -> C.Array:
    arr = (ib_patch * max(1, len(patches)))()
    for k, p in enumerate(patches):
        arr[k] = ib_patch(int(p.first), int(p.n1), int(p.n2), int(p.flags), 0, int(p.param_off))
    return arr


def ib_set_structure(ctx, points, patches: Sequence, stiffness) -> None:
    npts = (points.size if isinstance(points, np.ndarray) else points.numel()) // 3
    pa = _patch_array(patches)
    nst = stiffness.size if isinstance(stiffness, np.ndarray) else stiffness.numel()
    _check(load().ib_set_structure(ctx, _ptr(points, size=3 * npts), npts, C.cast(pa, C.c_void_p),
                                   len(patches), _ptr(stiffness) if nst else None, nst))


def ib_set_positions(ctx, points) -> None:
    _check(load().ib_set_positions(ctx, _ptr(points, size=3 * load().ib_num_points(ctx))))


def ib_set_velocity(ctx, u, N) -> None:
    n1, n2, n3 = dims(N)
    _check(load().ib_set_velocity(ctx, _ptr(u, size=3 * n1 * n2 * n3)))


def ib_set_drive(ctx, idx, direction, amp_per_point: float, period_steps: int) -> None:
    """direction None: surface-normal drive (the unit normal of each point's patch at X^n)."""
    n = 0 if idx is None else (idx.size if isinstance(idx, np.ndarray) else idx.numel())
    _check(load().ib_set_drive(ctx, _ptr(idx, np.int64) if n else None, n,
                               _ptr(direction, size=3 * n) if (n and direction is not None) else None,
                               float(amp_per_point), int(period_steps)))


def ib_set_fixed(ctx, mask) -> None:
    """mask: uint8 [np] (1 = the point never moves) or None to clear."""
    _check(load().ib_set_fixed(ctx, None if mask is None else _ptr(mask, np.uint8,
                                                                    size=int(load().ib_num_points(ctx)))))


def ib_step(ctx, nsteps: int) -> None:
    _check(load().ib_step(ctx, int(nsteps)))


def ib_get_fields(ctx, u_out=None, p_out=None, N=None) -> None:
    n1, n2, n3 = dims(N)
    V = n1 * n2 * n3
    _check(load().ib_get_fields(ctx, _ptr(u_out, size=3 * V, writable=True),
                                _ptr(p_out, size=V, writable=True)))


def ib_get_positions(ctx, X_out) -> None:
    _check(load().ib_get_positions(ctx, _ptr(X_out, size=3 * load().ib_num_points(ctx),
                                             writable=True)))


def ib_get_step(ctx) -> int:
    return int(load().ib_get_step(ctx))


def ib_set_step(ctx, n: int) -> None:
    _check(load().ib_set_step(ctx, int(n)))


def ib_stage_times(ctx, reset: bool = False) -> dict:
    ms = (C.c_double * 16)()
    names = C.create_string_buffer(512)
    n = load().ib_stage_times(ctx, C.cast(ms, C.c_void_p), 16, C.cast(names, C.c_void_p), 512,
                              1 if reset else 0)
    keys = names.raw.split(b"\0")[:n]
    return {k.decode(): ms[i] for i, k in enumerate(keys)}


def ib_launch_count(ctx, reset: bool = False) -> int:
    return int(load().ib_launch_count(ctx, 1 if reset else 0))


# ------------------------------------------------------------------ convenience object
class IBContext:
    """Owning wrapper: `IBContext(N, h, rho, mu, dt)` + the ib_* calls as methods.  N is an
    int (N^3 lattice, ib_create) or (N1, N2, N3) (ib_create3); fields are [3][N3][N2][N1]."""

    def __init__(self, N, h, rho, mu, dt):
        self.dims = dims(N)
        self.N = self.dims if isinstance(N, (tuple, list)) else int(N)
        self.h, self.rho, self.mu, self.dt = float(h), float(rho), float(mu), float(dt)
        if isinstance(N, (tuple, list)):
            self.ctx = ib_create3(*self.dims, h, rho, mu, dt)
        else:
            self.ctx = ib_create(N, h, rho, mu, dt)
        self.np = 0

    @property
    def fshape(self):
        n1, n2, n3 = self.dims
        return (3, n3, n2, n1)

    @property
    def V(self):
        n1, n2, n3 = self.dims
        return n1 * n2 * n3

    @classmethod
    def from_config(cls, cfg):
        o = cls(cfg.N, cfg.h, cfg.rho, cfg.mu, cfg.dt)
        o.set_structure(cfg.X, cfg.patches, cfg.stiffness)
        if cfg.u0 is not None:
            o.set_velocity(cfg.u0)
        if cfg.drive_idx is not None:
            o.set_drive(cfg.drive_idx, cfg.drive_dir, cfg.drive_amp, cfg.drive_period)
        if getattr(cfg, "fixed", None) is not None:
            o.set_fixed(cfg.fixed)
        return o

    def close(self):
        if self.ctx:
            ib_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    # state
    def set_structure(self, X, patches, stiffness):
        X = np.ascontiguousarray(X, dtype=np.float64) if isinstance(X, np.ndarray) else X
        st = np.ascontiguousarray(stiffness, dtype=np.float64) if isinstance(stiffness, np.ndarray) else stiffness
        ib_set_structure(self.ctx, X, patches, st)
        self.np = int(load().ib_num_points(self.ctx))

    def set_positions(self, X):
        ib_set_positions(self.ctx, np.ascontiguousarray(X, dtype=np.float64) if isinstance(X, np.ndarray) else X)

    def set_velocity(self, u):
        ib_set_velocity(self.ctx, np.ascontiguousarray(u, dtype=np.float64) if isinstance(u, np.ndarray) else u, self.dims)

    def set_drive(self, idx, direction, amp, period):
        ib_set_drive(self.ctx, np.ascontiguousarray(idx, dtype=np.int64),
                     None if direction is None else np.ascontiguousarray(direction, dtype=np.float64),
                     amp, period)

    def set_fixed(self, mask):
        ib_set_fixed(self.ctx, None if mask is None else np.ascontiguousarray(mask, dtype=np.uint8))

    def set_option(self, opt, value):
        ib_set_option(self.ctx, opt, value)

    def set_stream(self, handle):
        ib_set_stream(self.ctx, handle)

    def step(self, nsteps=1):
        ib_step(self.ctx, nsteps)

    @property
    def n(self):
        return ib_get_step(self.ctx)

    def set_step(self, n):
        ib_set_step(self.ctx, n)

    def get_fields(self, want_p=False):
        u = np.empty(self.fshape)
        p = np.empty(self.fshape[1:]) if want_p else None
        ib_get_fields(self.ctx, u, p, self.dims)
        return u, p

    def get_fields_into(self, u_out=None, p_out=None):
        ib_get_fields(self.ctx, u_out, p_out, self.dims)

    def get_positions(self):
        X = np.empty((self.np, 3))
        ib_get_positions(self.ctx, X)
        return X

    def get_positions_into(self, X_out):
        ib_get_positions(self.ctx, X_out)

    def rebin(self):
        """Re-bin the points by cell now (asynchronous on the context stream)."""
        _check(load().ib_rebin(self.ctx))

    def stage_times(self, reset=False):
        return ib_stage_times(self.ctx, reset)

    def launch_count(self, reset=False):
        return ib_launch_count(self.ctx, reset)

    # test-only single-stage entry points
    def debug_force(self):
        out = np.empty((self.np, 3))
        _check(load().ib_debug_force(self.ctx, _ptr(out)))
        return out

    def debug_spread(self, f_node):
        f = np.ascontiguousarray(f_node, dtype=np.float64)
        F = np.empty(self.fshape)
        _check(load().ib_debug_spread(self.ctx, _ptr(f, size=3 * self.np), _ptr(F)))
        return F

    def debug_interp(self, u):
        u = np.ascontiguousarray(u, dtype=np.float64)
        U = np.empty((self.np, 3))
        _check(load().ib_debug_interp(self.ctx, _ptr(u, size=3 * self.V), _ptr(U)))
        return U

    def debug_rhs(self, u, F):
        u = np.ascontiguousarray(u, dtype=np.float64)
        F = np.ascontiguousarray(F, dtype=np.float64)
        r = np.empty(self.fshape)
        _check(load().ib_debug_rhs(self.ctx, _ptr(u, size=3 * self.V), _ptr(F, size=3 * self.V), _ptr(r)))
        return r

    def debug_fluid(self, u, F, want_p=True):
        u = np.ascontiguousarray(u, dtype=np.float64)
        F = np.ascontiguousarray(F, dtype=np.float64)
        un = np.empty(self.fshape)
        p = np.empty(self.fshape[1:]) if want_p else None
        _check(load().ib_debug_fluid(self.ctx, _ptr(u, size=3 * self.V), _ptr(F, size=3 * self.V),
                                     _ptr(un), _ptr(p)))
        return un, p

    def debug_project(self, rhat, want_p=True):
        """S3c on a half spectrum rhat [3][N3][N2][N1/2+1] (complex) -> (uhat, phat)."""
        n1, n2, n3 = self.dims
        r = np.ascontiguousarray(np.stack([np.asarray(rhat).real, np.asarray(rhat).imag], -1),
                                 dtype=np.float64)
        u = np.empty((3, n3, n2, n1 // 2 + 1, 2))
        p = np.empty((n3, n2, n1 // 2 + 1, 2)) if want_p else None
        _check(load().ib_debug_project(self.ctx, _ptr(r, size=r.size), _ptr(u), _ptr(p)))
        return u[..., 0] + 1j * u[..., 1], (None if p is None else p[..., 0] + 1j * p[..., 1])

    def debug_ifft(self, X):
        """Unnormalised inverse DFT of a half spectrum [N3][N2][N1/2+1] -> real [N3][N2][N1]."""
        n1, n2, n3 = self.dims
        xin = np.ascontiguousarray(np.stack([np.asarray(X).real, np.asarray(X).imag], -1),
                                   dtype=np.float64)
        out = np.empty((n3, n2, n1))
        _check(load().ib_debug_ifft(self.ctx, _ptr(xin, size=xin.size), _ptr(out)))
        return out

    def debug_fft(self, x):
        n1, n2, n3 = self.dims
        x = np.ascontiguousarray(x, dtype=np.float64)
        out = np.empty((n3, n2, n1 // 2 + 1, 2))
        _check(load().ib_debug_fft(self.ctx, _ptr(x, size=self.V), _ptr(out)))
        return out[..., 0] + 1j * out[..., 1]
