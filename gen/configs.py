"""BASELINE.json configs 1-5 as seeded numpy arrays (input recipe: DESIGN.md §3).

Geometry lives in the periodic unit cube [0,1)^3 (h = 1/N).  Structures are given as
structured Lagrangian patches, the paper's rectangular parameter lattice Q
(§3.2 "Q = {(i1 dq1, i2 dq2)}", lines 697-710): point (i1, i2) of a patch is
X[first + i2*n1 + i1].

Link families (one stiffness block each, indexed by the link's lower-index endpoint i):
  STRETCH1: (i1,i2)-(i1+1,i2)   STRETCH2: (i1,i2)-(i1,i2+1)
  BEND1:    (i1,i2)-(i1+2,i2)   BEND2:    (i1,i2)-(i1,i2+2)
  WRAP1/WRAP2 make the i1 / i2 direction periodic.
  TETHER:   point i tied to the anchor Y_i with nodal stiffness kt_i.
Stiffness block of a patch, starting at param_off, in this order: for each link family
present (STRETCH1, STRETCH2, BEND1, BEND2) k[n1*n2] then L0[n1*n2]; for TETHER kt[n1*n2]
then Y[n1*n2*3].  Forces are nodal (f * dq folded in, PAPER.md eq:discreteF lines
712-720; reading Z12).
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

WRAP1, WRAP2 = 1, 2
STRETCH1, STRETCH2, BEND1, BEND2 = 4, 8, 16, 32
TETHER = 64
# (flag, axis, offset) in block order
FAMILIES = ((STRETCH1, 1, 1), (STRETCH2, 2, 1), (BEND1, 1, 2), (BEND2, 2, 2))

CONFIG_STEPS = {1: 10, 2: 100, 3: 400, 4: 200, 5: 50}


@dataclass
class Patch:
    first: int
    n1: int
    n2: int
    flags: int
    param_off: int


@dataclass
class Config:
    name: str
    N: int
    h: float
    rho: float
    mu: float
    dt: float
    steps: int
    X: np.ndarray                      # [np][3] float64
    patches: List[Patch]
    stiffness: np.ndarray              # float64
    u0: Optional[np.ndarray] = None    # [3][N][N][N] float64 (x fastest) or None (= rest)
    drive_idx: Optional[np.ndarray] = None   # int64 [nd]
    drive_dir: Optional[np.ndarray] = None   # float64 [nd][3]
    drive_amp: float = 0.0             # amplitude per driven point
    drive_period: int = 1              # steps
    fixed: Optional[np.ndarray] = None  # uint8 [np]: 1 = point never moves (window plates)
    info: dict = field(default_factory=dict)

    @property
    def np_(self) -> int:
        return int(self.X.shape[0])


# --------------------------------------------------------------------------- helpers
def _norm_rows(d: np.ndarray) -> np.ndarray:
    """Plain IEEE order sqrt((dx*dx + dy*dy) + dz*dz), no FMA (reading Z13)."""
    return np.sqrt((d[..., 0] * d[..., 0] + d[..., 1] * d[..., 1]) + d[..., 2] * d[..., 2])


def _rest_lengths(P: np.ndarray, n1: int, n2: int, axis: int, off: int, wrap: bool) -> np.ndarray:
    """Rest length of every link of one family, from rest positions P[n2][n1][3]."""
    if axis == 1:
        Q = np.roll(P, -off, axis=1)
    else:
        Q = np.roll(P, -off, axis=0)
    L = _norm_rows(Q - P)
    if not wrap:
        if axis == 1:
            L[:, n1 - off:] = 0.0
        else:
            L[n2 - off:, :] = 0.0
    return L


class _Builder:
    def __init__(self):
        self.X: list = []
        self.patches: List[Patch] = []
        self.stiff: list = []
        self.np = 0
        self.nstiff = 0

    def add(self, P: np.ndarray, flags: int, blocks: list) -> Patch:
        """P: [n2][n1][3] positions; blocks: list of flat float64 arrays in block order."""
        n2, n1 = P.shape[0], P.shape[1]
        p = Patch(self.np, n1, n2, flags, self.nstiff)
        self.patches.append(p)
        self.X.append(P.reshape(-1, 3))
        for b in blocks:
            b = np.ascontiguousarray(b, dtype=np.float64).reshape(-1)
            self.stiff.append(b)
            self.nstiff += b.size
        self.np += n1 * n2
        return p

    def arrays(self):
        X = np.ascontiguousarray(np.concatenate(self.X, axis=0), dtype=np.float64)
        S = (np.ascontiguousarray(np.concatenate(self.stiff), dtype=np.float64)
             if self.stiff else np.zeros(0))
        return X, S


# --------------------------------------------------------------------------- velocity
def _dims(N):
    """(N1, N2, N3) from an int (cubic lattice) or a 3-sequence (x, y, z)."""
    if isinstance(N, (tuple, list)):
        return tuple(int(v) for v in N)
    return int(N), int(N), int(N)


def random_divfree_velocity(N, K: int, amplitude: float, rng: np.random.Generator,
                            h: float = None) -> np.ndarray:
    """Seeded random discretely divergence-free field (reading Z19).

    A vector potential A with random Fourier coefficients on the modes 0 < |k|^2 <= K^2
    (half-space representatives, loops k1, k2, k3 from -K to K, k3 outermost) is evaluated
    on the grid; u = D0 x A (centred-difference curl) so that D0 . u = 0 up to rounding;
    u is then scaled so that its RMS speed sqrt(mean |u|^2) equals `amplitude`.
    N is an int (N^3 lattice) or (N1, N2, N3); h defaults to 1/N1.
    Returns [3][N3][N2][N1] (component, z, y, x), x fastest.
    """
    n1, n2, n3 = _dims(N)
    h = 1.0 / n1 if h is None else h
    spec = np.zeros((3, n3, n2, n1 // 2 + 1), dtype=np.complex128)
    scale = n1 * n2 * n3 / 2.0
    for k3 in range(-K, K + 1):
        for k2 in range(-K, K + 1):
            for k1 in range(-K, K + 1):
                if not (0 < k1 * k1 + k2 * k2 + k3 * k3 <= K * K):
                    continue
                if not (k3 > 0 or (k3 == 0 and k2 > 0) or (k3 == 0 and k2 == 0 and k1 > 0)):
                    continue
                a = rng.standard_normal(3)
                b = rng.standard_normal(3)
                c = (a - 1j * b) * scale          # Re(c e^{i theta}) = a cos + b sin
                if k1 > 0:
                    spec[:, k3 % n3, k2 % n2, k1] += c
                elif k1 < 0:
                    spec[:, (-k3) % n3, (-k2) % n2, -k1] += np.conj(c)
                else:
                    spec[:, k3 % n3, k2 % n2, 0] += c
                    spec[:, (-k3) % n3, (-k2) % n2, 0] += np.conj(c)
    A = np.fft.irfftn(spec, s=(n3, n2, n1), axes=(1, 2, 3))   # A[c][z][y][x]
    inv2h = 1.0 / (2.0 * h)

    def d0(f, ax):   # ax: 0 = x, 1 = y, 2 = z on a [z][y][x] array
        a = {0: 2, 1: 1, 2: 0}[ax]
        return (np.roll(f, -1, axis=a) - np.roll(f, 1, axis=a)) * inv2h

    u = np.empty_like(A)
    u[0] = d0(A[2], 1) - d0(A[1], 2)
    u[1] = d0(A[0], 2) - d0(A[2], 0)
    u[2] = d0(A[1], 0) - d0(A[0], 1)
    rms = math.sqrt(float(np.mean(u[0] ** 2 + u[1] ** 2 + u[2] ** 2)))
    u *= amplitude / rms
    return np.ascontiguousarray(u)


# --------------------------------------------------------------------------- geometry
def _helix(n1: int, th_max: float = 5.0 * math.pi, z0: float = 0.35):
    """Centre-line C(theta), frame (t, n, e) of the helix of BASELINE.json cfg3: theta in
    [0, th_max] (2.5 turns by default), radius 0.35 -> 0.1, pitch 0.12, starting at z0."""
    i = np.arange(n1, dtype=np.float64)
    th = th_max * i / (n1 - 1)
    R = 0.35 - 0.25 * th / th_max
    dR = -0.25 / th_max
    C = np.stack([0.5 + R * np.cos(th), 0.5 + R * np.sin(th),
                  z0 + 0.12 * th / (2.0 * math.pi)], axis=-1)
    dC = np.stack([dR * np.cos(th) - R * np.sin(th), dR * np.sin(th) + R * np.cos(th),
                   np.full_like(th, 0.12 / (2.0 * math.pi))], axis=-1)
    t = dC / np.linalg.norm(dC, axis=-1, keepdims=True)
    radial = np.stack([np.cos(th), np.sin(th), np.zeros_like(th)], axis=-1)
    n = np.cross(t, radial)
    n /= np.linalg.norm(n, axis=-1, keepdims=True)
    e = np.cross(n, t)
    return C, t, n, e


def _strip(n1: int, n2: int, **hx):
    C, t, n, e = _helix(n1, **hx)
    i = np.arange(n1, dtype=np.float64)
    w = 0.01 + 0.03 * i / (n1 - 1)
    j = np.arange(n2, dtype=np.float64)
    off = (j / (n2 - 1) - 0.5)[:, None] * w[None, :]            # [n2][n1]
    P = C[None, :, :] + off[:, :, None] * e[None, :, :]
    return np.ascontiguousarray(P), n


def _walls(n1: int, n2: int, a: float = 0.045, **hx):
    C, t, n, e = _helix(n1, **hx)
    out = []
    for base in (0.0, math.pi):
        psi = base + math.pi * (np.arange(n2, dtype=np.float64) + 0.5) / n2
        P = (C[None, :, :] + a * (np.cos(psi)[:, None, None] * e[None, :, :]
                                  + np.sin(psi)[:, None, None] * n[None, :, :]))
        out.append(np.ascontiguousarray(P))
    return out


def _spacing(P: np.ndarray, axis: int) -> np.ndarray:
    """Central-difference rest spacing along i1 (axis=1) or i2 (axis=0); one-sided at ends."""
    d = np.empty(P.shape[:2])
    if axis == 1:
        d[:, 1:-1] = np.linalg.norm(P[:, 2:] - P[:, :-2], axis=-1) / 2
        d[:, 0] = np.linalg.norm(P[:, 1] - P[:, 0], axis=-1)
        d[:, -1] = np.linalg.norm(P[:, -1] - P[:, -2], axis=-1)
    else:
        d[1:-1, :] = np.linalg.norm(P[2:] - P[:-2], axis=-1) / 2
        d[0, :] = np.linalg.norm(P[1] - P[0], axis=-1)
        d[-1, :] = np.linalg.norm(P[-1] - P[-2], axis=-1)
    return d


def _spring_blocks(P_rest, n1, n2, flags, kfun):
    """k and L0 blocks for each link family present in `flags` (block order)."""
    blocks = []
    for fam, axis, off in FAMILIES:
        if not flags & fam:
            continue
        wrap = bool(flags & (WRAP1 if axis == 1 else WRAP2))
        L0 = _rest_lengths(P_rest, n1, n2, axis, off, wrap)
        k = kfun(fam) * np.ones((n2, n1))
        k = np.where(L0 > 0, k, 0.0)
        blocks += [k, L0]
    return blocks


# --------------------------------------------------------------------------- configs
def _cfg1() -> Config:
    N = 32
    h = 1.0 / N
    rng = np.random.default_rng(1)
    n = 48
    s = 1.0 / 64
    xi = rng.standard_normal(n * n).reshape(n, n)                  # order i2*48 + i1
    i1 = np.arange(n, dtype=np.float64)[None, :]
    i2 = np.arange(n, dtype=np.float64)[:, None]
    P = np.stack(np.broadcast_arrays(0.5 + (i1 - 23.5) * s, 0.5 + (i2 - 23.5) * s,
                                     0.5 + 0.05 * h * xi), axis=-1)
    flags = STRETCH1 | STRETCH2
    k = np.ones((n, n))
    L0 = np.full((n, n), h / 2)
    k1 = k.copy(); k1[:, -1] = 0.0
    L1 = L0.copy(); L1[:, -1] = 0.0
    k2 = k.copy(); k2[-1, :] = 0.0
    L2 = L0.copy(); L2[-1, :] = 0.0
    b = _Builder()
    b.add(P, flags, [k1, L1, k2, L2])
    X, S = b.arrays()
    return Config("cfg1", N, h, 1.0, 0.01, 1e-3, CONFIG_STEPS[1], X, b.patches, S)


def _cfg2() -> Config:
    N = 64
    h = 1.0 / N
    rng = np.random.default_rng(2)
    u0 = random_divfree_velocity(N, 4, 0.01, rng)
    n1, n2 = 256, 128
    phi = 2 * math.pi * np.arange(n1) / n1
    th = math.pi * (np.arange(n2) + 0.5) / n2

    def sphere(R):
        return np.stack([0.5 + R * np.sin(th)[:, None] * np.cos(phi)[None, :],
                         0.5 + R * np.sin(th)[:, None] * np.sin(phi)[None, :],
                         0.5 + R * np.cos(th)[:, None] * np.ones(n1)[None, :]], axis=-1)
    P = np.ascontiguousarray(sphere(0.25))
    P0 = np.ascontiguousarray(sphere(0.20))
    flags = WRAP1 | STRETCH1 | STRETCH2 | BEND1 | BEND2
    kk = {STRETCH1: 10.0, STRETCH2: 10.0, BEND1: 0.1, BEND2: 0.1}
    b = _Builder()
    b.add(P, flags, _spring_blocks(P0, n1, n2, flags, lambda f: kk[f]))
    X, S = b.arrays()
    return Config("cfg2", N, h, 1.0, 0.005, 5e-4, CONFIG_STEPS[2], X, b.patches, S, u0=u0)


def _helix_config(name, N, mu, dt, steps, n1, n2, nw2, walls: bool, jitter_rng=None,
                  u0=None, **hx) -> Config:
    h = 1.0 / _dims(N)[0]
    P, nrm = _strip(n1, n2, **hx)
    flags = STRETCH1 | STRETCH2
    s = np.arange(n1, dtype=np.float64) / (n1 - 1)
    kprof = np.broadcast_to(100.0 ** (-s)[None, :], (n2, n1))        # reading Z2
    blocks = []
    for fam, axis, off in FAMILIES[:2]:
        L0 = _rest_lengths(P, n1, n2, axis, off, False)
        blocks += [np.where(L0 > 0, kprof, 0.0), L0]
    wall_P = _walls(n1, nw2, **hx) if walls else []
    kt = []
    for W in wall_P:
        dA = _spacing(W, 1) * _spacing(W, 0)
        kt.append(1.0e4 * dA)                                         # reading Z1
    if jitter_rng is not None:                                        # reading Z18
        for bi in (0, 2):
            blocks[bi] = blocks[bi] * (1.0 + 0.01 * jitter_rng.uniform(-1.0, 1.0, blocks[bi].shape))
            blocks[bi] = np.where(blocks[bi + 1] > 0, blocks[bi], 0.0)
        kt = [k * (1.0 + 0.01 * jitter_rng.uniform(-1.0, 1.0, k.shape)) for k in kt]
    b = _Builder()
    strip = b.add(P, flags, blocks)
    for W, k in zip(wall_P, kt):
        b.add(W, TETHER, [k, W.reshape(-1, 3)])
    X, S = b.arrays()
    idx = strip.first + np.arange(n2, dtype=np.int64) * n1             # basal row i1 = 0
    ddir = np.repeat(nrm[0][None, :], n2, axis=0)
    cfg = Config(name, N, h, 1.0, mu, dt, steps, X, b.patches, S, u0=u0,
                 drive_idx=idx, drive_dir=np.ascontiguousarray(ddir),
                 drive_amp=1e-3 / n2, drive_period=200)                # reading Z3
    return cfg


def _cfg3() -> Config:
    return _helix_config("cfg3", 128, 0.002, 2.5e-4, CONFIG_STEPS[3], 2048, 32, 0, False)


def _cfg4() -> Config:
    return _helix_config("cfg4", 256, 1e-3, 1.25e-4, CONFIG_STEPS[4], 8192, 64, 96, True)


def _cfg5() -> Config:
    rng = np.random.default_rng(5)
    u0 = random_divfree_velocity(512, 8, 1e-3, rng)
    return _helix_config("cfg5", 512, 5e-4, 6.25e-5, CONFIG_STEPS[5], 16384, 128, 192, True,
                         jitter_rng=rng, u0=u0)


def _cfg4h() -> Config:
    """The paper's half-cube box (256 x 256 x 128, PAPER.md 1003-1007) with
    cfg4's physics and mesh sizes: strip 8192 x 64 and two tethered duct walls 8192 x 96
    (2,097,152 points) on a 1.25-turn helix of the same radius law and pitch, starting at
    z = 0.125 so that it fits the [0, 1) x [0, 1) x [0, 0.5) domain."""
    return _helix_config("cfg4h", (256, 256, 128), 1e-3, 1.25e-4, 200, 8192, 64, 96, True,
                         th_max=2.5 * math.pi, z0=0.125)


_MAKERS = {1: _cfg1, 2: _cfg2, 3: _cfg3, 4: _cfg4, 5: _cfg5, "4h": _cfg4h}


def make_config(k) -> Config:
    """BASELINE.json configs[k-1] as arrays (k = 1..5); k = "4h": the half-cube variant."""
    return _MAKERS[k if k == "4h" else int(k)]()


# --------------------------------------------------------------------------- small cases
def random_points(n: int, rng: np.random.Generator, lo: float = 0.0, hi: float = 1.0) -> np.ndarray:
    return np.ascontiguousarray(rng.uniform(lo, hi, size=(n, 3)))


def small_sheet_config(N=16, n1: int = 12, n2: int = 10, seed: int = 0,
                       flags: int = STRETCH1 | STRETCH2 | BEND1 | BEND2,
                       tether: bool = True, drive: bool = True, u_amp: float = 0.0,
                       rho: float = 1.0, mu: float = 0.01, dt: float = 1e-3,
                       spacing: float = None, noise: float = 0.3) -> Config:
    """A small stressed sheet (+ optional tethered patch and drive) for parity tests.
    N is an int or (N1, N2, N3); h = 1/N1 (the domain is [0, N1 h) x [0, N2 h) x [0, N3 h))."""
    rng = np.random.default_rng(seed)
    h = 1.0 / _dims(N)[0]
    s = h / 2 if spacing is None else spacing
    i1 = np.arange(n1, dtype=np.float64)[None, :]
    i2 = np.arange(n2, dtype=np.float64)[:, None]
    P = np.stack(np.broadcast_arrays(0.37 + i1 * s, 0.41 + i2 * s, 0.5 + 0 * i1), axis=-1)
    P = np.ascontiguousarray(P + noise * h * rng.standard_normal(P.shape))
    blocks = []
    for fam, axis, off in FAMILIES:
        if not flags & fam:
            continue
        wrap = bool(flags & (WRAP1 if axis == 1 else WRAP2))
        L0 = _rest_lengths(P, n1, n2, axis, off, wrap) * rng.uniform(0.7, 1.1, (n2, n1))
        k = rng.uniform(0.5, 2.0, (n2, n1))
        blocks += [np.where(L0 > 0, k, 0.0), L0]
    b = _Builder()
    b.add(P, flags, blocks)
    if tether:
        m1, m2 = 7, 5
        T = np.stack(np.broadcast_arrays(0.2 + np.arange(m1)[None, :] * s,
                                         0.75 + np.arange(m2)[:, None] * s,
                                         0.3 + 0 * np.arange(m1)[None, :]), axis=-1)
        T = np.ascontiguousarray(T)
        Y = T.reshape(-1, 3) + 0.2 * h * rng.standard_normal((m1 * m2, 3))
        b.add(T, TETHER, [rng.uniform(10.0, 50.0, m1 * m2), Y])
    X, S = b.arrays()
    u0 = random_divfree_velocity(N, 3, u_amp, rng) if u_amp > 0 else None
    name = "sheet" + ("x".join(str(v) for v in N) if isinstance(N, (tuple, list)) else str(N))
    cfg = Config(name, N, h, rho, mu, dt, 10, X, b.patches, S, u0=u0)
    if drive:
        cfg.drive_idx = np.arange(0, n1, 3, dtype=np.int64)
        d = rng.standard_normal((cfg.drive_idx.size, 3))
        cfg.drive_dir = np.ascontiguousarray(d / np.linalg.norm(d, axis=1, keepdims=True))
        cfg.drive_amp = 0.05
        cfg.drive_period = 8
    return cfg


def window_config(N=32, m: int = 24, seed: int = 0, rho: float = 1.0, mu: float = 0.01,
                  dt: float = 1e-3, amp: float = 2e-3, period: int = 8, k: float = 1.0,
                  u_amp: float = 0.0) -> Config:
    """An oval-window-like plate (PAPER.md 914-922, 988-993): an m x m
    rectangular grid at spacing h/2 with stretch links of uniform stiffness k, tilted out of
    the lattice planes; its points outside the inscribed circle are fixed (a circular plate
    in a rectangular piece of bone); a sinusoidal force of total amplitude `amp` orthogonal
    to the plate surface (the normal recomputed from X^n each step) is distributed uniformly
    over the free disc points.  Rest lengths are the initial spacings, and the disc starts
    bulged by a seeded random normal displacement so that the plate is stressed."""
    rng = np.random.default_rng(seed)
    h = 1.0 / _dims(N)[0]
    s = h / 2
    e1 = np.array([0.96, 0.28, 0.0])
    e2 = np.array([-0.1, 0.35, 0.93])
    e2 -= e1 * (e1 @ e2); e2 /= np.linalg.norm(e2)
    nrm = np.cross(e1, e2)
    i1 = np.arange(m, dtype=np.float64)[None, :, None]
    i2 = np.arange(m, dtype=np.float64)[:, None, None]
    c = (m - 1) / 2.0
    P = 0.47 + (i1 - c) * s * e1 + (i2 - c) * s * e2                 # [m][m][3]
    rr = np.sqrt((i1[..., 0] - c) ** 2 + (i2[..., 0] - c) ** 2)     # [m][m]
    disc = rr <= c
    flags = STRETCH1 | STRETCH2
    blocks = []
    for fam, axis, off in FAMILIES[:2]:
        L0 = _rest_lengths(np.ascontiguousarray(P), m, m, axis, off, False)
        blocks += [np.where(L0 > 0, k, 0.0), L0]
    bulge = 0.15 * h * rng.standard_normal((m, m)) * disc
    P = np.ascontiguousarray(P + bulge[..., None] * nrm)
    b = _Builder()
    b.add(P, flags, blocks)
    X, S = b.arrays()
    u0 = random_divfree_velocity(N, 3, u_amp, rng) if u_amp > 0 else None
    name = "window" + ("x".join(str(v) for v in N) if isinstance(N, (tuple, list)) else str(N))
    cfg = Config(name, N, h, rho, mu, dt, 10, X, b.patches, S, u0=u0)
    cfg.fixed = np.ascontiguousarray((~disc).reshape(-1).astype(np.uint8))
    cfg.drive_idx = np.flatnonzero(disc.reshape(-1)).astype(np.int64)
    cfg.drive_dir = None                                     # surface-normal drive
    cfg.drive_amp = amp / cfg.drive_idx.size
    cfg.drive_period = period
    return cfg


def decaying_shear_config(N=16, m: int = 3, A: float = 1.0, npts: int = 40, seed: int = 0,
                          rho: float = 1.0, mu: float = 0.1, dt: float = 1e-2) -> Config:
    """Free points (one patch, no links: F = 0) in the shear mode u = A sin(2 pi m y) e_x
    sampled on the lattice, y_j = j h (an input only; the closed-form step lives in
    tests/test_oracle_force_step.py).  Points are seeded uniformly in the box."""
    rng = np.random.default_rng(seed)
    n1, n2, n3 = _dims(N)
    h = 1.0 / n1
    X = np.ascontiguousarray(rng.uniform(0.0, 1.0, (npts, 3)) * np.array([n1, n2, n3]) * h)
    u0 = np.zeros((3, n3, n2, n1))
    u0[0] = A * np.sin(2.0 * np.pi * m * np.arange(n2) / n2)[None, :, None]
    name = "shear" + ("x".join(str(v) for v in N) if isinstance(N, (tuple, list)) else str(N))
    return Config(name, N, h, rho, mu, dt, 2, X, [Patch(0, npts, 1, 0, 0)], np.zeros(0), u0=u0,
                  info={"m": m, "A": A})
