"""Pins of the oracle's delta function, spread and interpolate (CPU only).

Each pin comes from the paper's definitions, not from the oracle's code:
phi closed forms (PAPER.md 745-759, tests/golden/phi_closed_forms.txt), the
alternative closed form of the 1<=|r|<=2 branch, moment identities, a brute-force
full-lattice sum of delta_h with no support window (eq:discreteF, PAPER.md 712-723),
conservation, adjointness and reproduction of constants/linear fields (eq:discreteX,
PAPER.md 725-734).
"""
import math
import os

import numpy as np
import pytest

GOLD = os.path.join(os.path.dirname(__file__), "golden", "phi_closed_forms.txt")


def test_phi_golden_closed_forms(olib):
    rows = [l.split() for l in open(GOLD) if l.strip() and not l.startswith("#")]
    assert len(rows) >= 9
    for r, a, b, c, d in rows:
        r = float(r)
        want = (float(a) + float(b) * math.sqrt(float(c))) / float(d)
        for s in (r, -r):
            assert abs(olib.phi(s) - want) <= 2e-16, (s, olib.phi(s), want)


def test_phi_second_branch_alternative_form(olib):
    # 1 <= |r| <= 2: 1/2 - phi(2-|r|) == (5 - 2|r| - sqrt(-7 + 12|r| - 4 r^2))/8 (Peskin;
    # algebra: substitute s = 2 - |r| into the first branch).
    r = np.random.default_rng(0).uniform(1.0, 2.0, 2000)
    alt = (5 - 2 * r - np.sqrt(-7 + 12 * r - 4 * r * r)) / 8
    assert np.max(np.abs(olib.phi(r) - alt)) < 4e-16
    assert np.max(np.abs(olib.phi(-r) - alt)) < 4e-16


def test_phi_moment_identities(olib):
    r = np.random.default_rng(1).uniform(-3, 3, 4000)
    j = np.arange(-6, 7)[None, :]
    P = olib.phi(r[:, None] - j)
    assert np.max(np.abs(P.sum(1) - 1.0)) < 1e-15                       # partition of unity
    even = (j % 2 == 0)
    assert np.max(np.abs((P * even).sum(1) - 0.5)) < 1e-15              # even/odd sums 1/2
    assert np.max(np.abs(((r[:, None] - j) * P).sum(1))) < 1e-15        # first moment 0
    assert np.max(np.abs((P * P).sum(1) - 3.0 / 8.0)) < 1e-15           # sum phi^2 = 3/8
    assert np.all(P >= 0)


def test_phi_continuity_and_support(olib):
    eps = 1e-9
    for a in (1.0, 2.0):
        assert abs(olib.phi(a - eps) - olib.phi(a + eps)) < 1e-8
        # C^1: one-sided difference quotients agree
        dl = (olib.phi(a) - olib.phi(a - eps)) / eps
        dr = (olib.phi(a + eps) - olib.phi(a)) / eps
        assert abs(dl - dr) < 1e-5
    assert olib.phi(2.0 + 1e-12) == 0.0 and olib.phi(7.3) == 0.0


def _brute_delta(N, h, x, X):
    """delta_h(x - X) on the whole periodic lattice, no window: sum over periodic images."""
    def phi1(r):
        a = np.abs(r)
        out = np.zeros_like(a)
        m1 = a <= 1
        out[m1] = (3 - 2 * a[m1] + np.sqrt(1 + 4 * a[m1] - 4 * a[m1] ** 2)) / 8
        m2 = (a > 1) & (a < 2)
        out[m2] = (5 - 2 * a[m2] - np.sqrt(-7 + 12 * a[m2] - 4 * a[m2] ** 2)) / 8
        return out
    L = N * h
    w = []
    for ax in range(3):
        acc = np.zeros(N)
        for img in (-2, -1, 0, 1, 2):
            acc += phi1((x - (X[ax] + img * L)) / h)
        w.append(acc)
    return np.einsum("k,j,i->kji", w[2], w[1], w[0]) / h ** 3


def test_spread_matches_brute_force_lattice_sum(olib):
    rng = np.random.default_rng(2)
    N, h = 8, 1.0 / 8
    X = rng.uniform(-0.3, 1.3, (7, 3))              # unwrapped positions, incl. outside [0,1)
    X[0] = [0.25, 0.5, 0.75]                        # exactly on lattice nodes
    X[1] = [0.0, 1.0 - 1e-17, 0.5 + 0.5 * h]
    Fn = rng.standard_normal((7, 3))
    F = olib.spread(N, h, X, Fn)
    x = np.arange(N) * h
    want = np.zeros((3, N, N, N))
    for q in range(7):
        d = _brute_delta(N, h, x, X[q])
        for c in range(3):
            want[c] += Fn[q, c] * d
    assert np.max(np.abs(F - want)) <= 1e-13 * np.max(np.abs(want))


def test_spread_single_point_on_node(olib):
    N, h = 16, 1.0 / 16
    X = np.array([[5 * h, 7 * h, 9 * h]])
    F = olib.spread(N, h, X, np.array([[1.0, -2.0, 0.5]]))
    assert F[0, 9, 7, 5] == pytest.approx(0.125 * N ** 3, rel=1e-15)
    assert F[1, 9, 7, 5] == pytest.approx(-0.25 * N ** 3, rel=1e-15)
    assert F[0, 9, 7, 6] == pytest.approx(0.5 * 0.5 * 0.25 * N ** 3, rel=1e-15)
    assert F[0, 9, 7, 7] == 0.0                                   # phi(2) = 0
    assert np.count_nonzero(F[0]) == 27                           # 3x3x3 support on a node


def test_spread_conservation_cancellation_and_shift(olib):
    rng = np.random.default_rng(3)
    N, h = 16, 1.0 / 16
    X = rng.uniform(0, 1, (300, 3))
    Fn = rng.standard_normal((300, 3))
    F = olib.spread(N, h, X, Fn)
    tot = F.reshape(3, -1).sum(1) * h ** 3
    assert np.allclose(tot, Fn.sum(0), rtol=0, atol=1e-12 * np.abs(Fn).sum())
    # opposite forces at the same point cancel
    F2 = olib.spread(N, h, np.vstack([X[:5], X[:5]]), np.vstack([Fn[:5], -Fn[:5]]))
    assert np.max(np.abs(F2)) < 1e-12
    # lattice-vector shift equivariance (exact shifts by 3h, -2h, 5h)
    s = np.array([3, -2, 5])
    Fs = olib.spread(N, h, X + s * h, Fn)
    assert np.max(np.abs(Fs - np.roll(F, shift=(s[2], s[1], s[0]), axis=(1, 2, 3)))) < 1e-9


def test_interp_constants_linear_and_adjoint(olib):
    rng = np.random.default_rng(4)
    N, h = 16, 1.0 / 16
    X = rng.uniform(0.25, 0.75, (200, 3))
    c = np.array([0.3, -1.7, 2.5])
    u = np.broadcast_to(c[:, None, None, None], (3, N, N, N)).copy()
    U = olib.interp(N, h, u, X)
    assert np.max(np.abs(U - c)) < 1e-15 * 8
    # locally linear field (no wrap inside the support): U = a + b.X (first moment = 0)
    x = np.arange(N) * h
    zz, yy, xx = np.meshgrid(x, x, x, indexing="ij")
    a, b = rng.standard_normal(3), rng.standard_normal((3, 3))
    lin = np.stack([a[i] + b[i, 0] * xx + b[i, 1] * yy + b[i, 2] * zz for i in range(3)])
    U = olib.interp(N, h, lin, X)
    want = a[None, :] + X @ b.T
    assert np.max(np.abs(U - want)) < 1e-13
    # adjointness: h^3 <S f, v> = <f, S* v>
    f = rng.standard_normal((200, 3))
    v = rng.standard_normal((3, N, N, N))
    lhs = h ** 3 * np.sum(olib.spread(N, h, X, f) * v)
    rhs = np.sum(f * olib.interp(N, h, v, X))
    assert abs(lhs - rhs) <= 1e-12 * max(abs(lhs), 1.0)


def test_spread_interp_anisotropic_conservation_and_adjoint(olib):
    # on a 16 x 8 x 32 lattice: h^3 sum F = sum f, adjointness, constants reproduced,
    # and periodic wrap on each axis with its own length
    shape, h = (16, 8, 32), 1.0 / 16
    rng = np.random.default_rng(21)
    L = np.array(shape) * h
    X = rng.uniform(-0.3, 1.3, (300, 3)) * L
    f = rng.standard_normal((300, 3))
    F = olib.spread(shape, h, X, f)
    assert F.shape == (3, 32, 8, 16)
    assert np.allclose(F.reshape(3, -1).sum(1) * h ** 3, f.sum(0), rtol=0, atol=1e-12 * np.abs(f).sum())
    u = rng.standard_normal((3, 32, 8, 16))
    U = olib.interp(shape, h, u, X)
    assert abs(np.sum(F * u) * h ** 3 - np.sum(f * U)) <= 1e-12 * np.sum(np.abs(f * U))
    c = np.ones((3, 32, 8, 16)) * np.array([0.3, -1.0, 2.0])[:, None, None, None]
    assert np.allclose(olib.interp(shape, h, c, X), [0.3, -1.0, 2.0], rtol=0, atol=1e-14)
    # a shift by the period N_a h along any axis changes nothing (to rounding of X + L)
    for a in range(3):
        Xs = X.copy(); Xs[:, a] += L[a]
        assert np.allclose(olib.spread(shape, h, Xs, f), F, rtol=0, atol=1e-11 * np.abs(F).max())
