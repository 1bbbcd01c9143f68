"""CPU oracle of the IB time step — TEST INFRASTRUCTURE, not product code.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / `--impl reference`
legs may import this package.  It wraps liboracle.so (plain fp64 C, oracle/ib_oracle.c,
written from PAPER.md §3.2) with ctypes and shares no code with the CUDA
path.  Parity status of each function: see DESIGN.md §4 (all pinned; the coupled
trajectory physics of PAPER.md lines 1096-1182 is "parity unpinned").
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SO = os.path.join(_HERE, "liboracle.so")
_SRC = [os.path.join(_HERE, "ib_oracle.c")]
_lock = threading.Lock()
_lib = None


def build(force: bool = False) -> str:
    """Compile liboracle.so with gcc (contraction off; OpenMP over independent outputs)."""
    newest = max(os.path.getmtime(p) for p in _SRC + [os.path.join(_HERE, "ib_oracle.h")])
    if force or not os.path.exists(_SO) or os.path.getmtime(_SO) < newest:
        tmp = _SO + f".tmp{os.getpid()}"
        cmd = ["gcc", "-O2", "-std=c11", "-ffp-contract=off", "-fno-fast-math", "-fopenmp",
               "-fPIC", "-shared", "-o", tmp] + _SRC + ["-lm"]
        subprocess.check_call(cmd)
        os.replace(tmp, _SO)
    return _SO


def lib():
    global _lib
    with _lock:
        if _lib is None:
            build()
            L = C.CDLL(_SO)
            d, i32, i64, u32, p = C.c_double, C.c_int32, C.c_int64, C.c_uint32, C.c_void_p
            L.ibo_phi.restype = d
            L.ibo_phi.argtypes = [d]
            L.ibo_set_threads.argtypes = [C.c_int]
            L.ibo_get_threads.restype = C.c_int
            n3 = [i32, i32, i32]
            L.ibo_force.argtypes = [p, i64, i32, p, p, p, p, p, p, i64, p, p, d, i32, i64, p]
            L.ibo_spread.argtypes = n3 + [d, p, p, i64, p]
            L.ibo_interp.argtypes = n3 + [d, p, p, i64, p]
            L.ibo_advect.argtypes = n3 + [d, p, p]
            L.ibo_rhs.argtypes = n3 + [d, d, d, p, p, p]
            L.ibo_fft3.argtypes = n3 + [p, p, C.c_int]
            L.ibo_solve.argtypes = n3 + [d, d, d, d, p, p, p]
            L.ibo_fluid_step.argtypes = n3 + [d, d, d, d, p, p, p, p]
            L.ibo_step.restype = C.c_int
            L.ibo_step.argtypes = n3 + [d, d, d, d, p, p, p, i64, i32, p, p, p, p, p, p,
                                        i64, p, p, d, i32, i64, i32, i32, p]
            _lib = L
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _f64(a, shape=None):
    a = np.ascontiguousarray(a, dtype=np.float64)
    if shape is not None:
        a = a.reshape(shape)
    return a


def dims(N):
    """(N1, N2, N3) = lattice points along x, y, z from an int (cubic) or a 3-sequence."""
    if isinstance(N, (tuple, list, np.ndarray)):
        n1, n2, n3 = (int(v) for v in N)
        return n1, n2, n3
    return int(N), int(N), int(N)


def fshape(N):
    """Field array shape [3][N3][N2][N1]."""
    n1, n2, n3 = dims(N)
    return (3, n3, n2, n1)


def set_threads(n: int) -> None:
    lib().ibo_set_threads(int(n))


def get_threads() -> int:
    return int(lib().ibo_get_threads())


def phi(r) -> np.ndarray:
    L = lib()
    r = np.asarray(r, dtype=np.float64)
    return np.vectorize(L.ibo_phi, otypes=[np.float64])(r)


class _Structure:
    """Flat patch arrays in the oracle's own argument convention."""

    def __init__(self, patches, stiffness):
        self.first = np.array([p.first for p in patches], dtype=np.int64)
        self.n1 = np.array([p.n1 for p in patches], dtype=np.int32)
        self.n2 = np.array([p.n2 for p in patches], dtype=np.int32)
        self.flags = np.array([p.flags for p in patches], dtype=np.uint32)
        self.off = np.array([p.param_off for p in patches], dtype=np.int64)
        self.stiff = _f64(stiffness if len(stiffness) else np.zeros(1))
        self.npatch = len(patches)

    def args(self):
        return (self.npatch, _ptr(self.first), _ptr(self.n1), _ptr(self.n2), _ptr(self.flags),
                _ptr(self.off), _ptr(self.stiff))


def force(X, patches, stiffness, step=0, drive_idx=None, drive_dir=None, drive_amp=0.0,
          drive_period=1) -> np.ndarray:
    X = _f64(X, (-1, 3))
    S = _Structure(patches, stiffness)
    nd = 0 if drive_idx is None else len(drive_idx)
    di = np.ascontiguousarray(drive_idx, dtype=np.int64) if nd else None
    dd = _f64(drive_dir, (-1, 3)) if (nd and drive_dir is not None) else None   # None: normal
    out = np.zeros_like(X)
    lib().ibo_force(_ptr(X), X.shape[0], *S.args(), nd, _ptr(di), _ptr(dd), float(drive_amp),
                    int(drive_period), int(step), _ptr(out))
    return out


def spread(N, h, X, Fnode) -> np.ndarray:
    X = _f64(X, (-1, 3)); Fn = _f64(Fnode, (-1, 3))
    F = np.empty(fshape(N))
    lib().ibo_spread(*dims(N), h, _ptr(X), _ptr(Fn), X.shape[0], _ptr(F))
    return F


def interp(N, h, u, X) -> np.ndarray:
    X = _f64(X, (-1, 3)); u = _f64(u, fshape(N))
    U = np.empty_like(X)
    lib().ibo_interp(*dims(N), h, _ptr(u), _ptr(X), X.shape[0], _ptr(U))
    return U


def advect(N, h, u) -> np.ndarray:
    u = _f64(u, fshape(N))
    a = np.empty_like(u)
    lib().ibo_advect(*dims(N), h, _ptr(u), _ptr(a))
    return a


def rhs(N, h, rho, dt, u, F) -> np.ndarray:
    u = _f64(u, fshape(N)); F = _f64(F, fshape(N))
    r = np.empty_like(u)
    lib().ibo_rhs(*dims(N), h, rho, dt, _ptr(u), _ptr(F), _ptr(r))
    return r


def fft3(x: np.ndarray, sign: int = -1) -> np.ndarray:
    """Unnormalised 3-D DFT of a complex [N3][N2][N1] array with the oracle's radix-2 FFT."""
    x = np.asarray(x, dtype=np.complex128)
    n3, n2, n1 = x.shape
    re = np.ascontiguousarray(x.real); im = np.ascontiguousarray(x.imag)
    lib().ibo_fft3(n1, n2, n3, _ptr(re), _ptr(im), int(sign))
    return re + 1j * im


def solve(N, h, rho, mu, dt, r, want_p=True):
    r = _f64(r, fshape(N))
    u = np.empty_like(r)
    p = np.empty(fshape(N)[1:]) if want_p else None
    lib().ibo_solve(*dims(N), h, rho, mu, dt, _ptr(r), _ptr(u), _ptr(p))
    return u, p


def fluid_step(N, h, rho, mu, dt, u, F, want_p=True):
    u = _f64(u, fshape(N)); F = _f64(F, fshape(N))
    un = np.empty_like(u)
    p = np.empty(fshape(N)[1:]) if want_p else None
    lib().ibo_fluid_step(*dims(N), h, rho, mu, dt, _ptr(u), _ptr(F), _ptr(un), _ptr(p))
    return un, p


class Oracle:
    """Stateful oracle with the same call sequence as the product binding
    (create / set_structure / set_velocity / set_drive / step / get_*).  N is an int (cubic
    lattice) or (N1, N2, N3)."""

    def __init__(self, N, h, rho, mu, dt):
        self.dims = dims(N)
        self.N = N if not isinstance(N, (tuple, list)) else tuple(int(v) for v in N)
        self.h, self.rho, self.mu, self.dt = float(h), float(rho), float(mu), float(dt)
        self.u = np.zeros(fshape(N))
        self.p = np.zeros(fshape(N)[1:])
        self.p_steps = None              # [nsteps][N3][N2][N1] when step(..., p_every=True)
        self.X = np.zeros((0, 3))
        self.S = _Structure([], np.zeros(0))
        self.nd = 0
        self.di = self.dd = None
        self.amp, self.period = 0.0, 1
        self.fixed = None                # uint8 [np] or None
        self.n = 0

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

    def set_structure(self, X, patches, stiffness):
        self.X = _f64(X, (-1, 3)).copy()
        self.S = _Structure(patches, stiffness)

    def set_positions(self, X):
        self.X = _f64(X, (-1, 3)).copy()

    def set_velocity(self, u):
        self.u = _f64(u, fshape(self.dims)).copy()

    def set_drive(self, idx, direction, amp, period):
        """direction None: surface-normal drive (normal of each point's patch at X^n)."""
        self.nd = len(idx)
        self.di = np.ascontiguousarray(idx, dtype=np.int64)
        self.dd = None if direction is None else _f64(direction, (-1, 3))
        self.amp, self.period = float(amp), int(period)

    def set_fixed(self, mask):
        self.fixed = None if mask is None else np.ascontiguousarray(mask, dtype=np.uint8)

    def step(self, nsteps=1, p_every=False):
        """nsteps IB steps; p_every: keep p^{n+1} of every step in self.p_steps."""
        pbuf = np.empty((int(nsteps),) + fshape(self.dims)[1:]) if p_every else self.p
        st = lib().ibo_step(*self.dims, self.h, self.rho, self.mu, self.dt, _ptr(self.u),
                            _ptr(pbuf), _ptr(self.X), self.X.shape[0], *self.S.args(),
                            self.nd, _ptr(self.di), _ptr(self.dd), self.amp, self.period,
                            self.n, int(nsteps), 1 if p_every else 0, _ptr(self.fixed))
        if p_every:
            self.p_steps = pbuf
            if nsteps:
                self.p = pbuf[-1].copy()
        if st:
            self.n += st - 1
            raise FloatingPointError(f"oracle: non-finite state at step {self.n}")
        self.n += int(nsteps)

    def get_fields(self):
        return self.u.copy(), self.p.copy()

    def get_positions(self):
        return self.X.copy()

    def force(self):
        return force(self.X, [], np.zeros(0)) if self.S.npatch == 0 else _force_state(self)


def _force_state(o: Oracle):
    out = np.zeros_like(o.X)
    lib().ibo_force(_ptr(o.X), o.X.shape[0], *o.S.args(), o.nd, _ptr(o.di), _ptr(o.dd),
                    o.amp, o.period, o.n, _ptr(out))
    return out
