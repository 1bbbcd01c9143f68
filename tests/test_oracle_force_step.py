"""Pins of the oracle's Lagrangian force and whole time step (CPU only).

Force (spring law per DESIGN.md): rest -> 0, Newton's third law,
Hooke by hand, energy gradient by central differences, tether linearity, drive phase.
Whole step (eq:discreteX 725-734): rest fixed point, rigid
translation by a uniform flow, boundedness on configs 1-2.
"""
import numpy as np
import pytest

from gen import (BEND1, BEND2, STRETCH1, STRETCH2, TETHER, WRAP1, Patch, make_config,
                 small_sheet_config)


def _energy(X, cfg):
    """Spring + tether energy E = sum 1/2 k (|d| - L0)^2 + sum 1/2 kt |X - Y|^2, written
    from the patch description (independent of the oracle's gather loop)."""
    E = 0.0
    for p in cfg.patches:
        P = X[p.first:p.first + p.n1 * p.n2].reshape(p.n2, p.n1, 3)
        b = p.param_off
        npts = p.n1 * p.n2
        for fam, axis, off in ((STRETCH1, 1, 1), (STRETCH2, 2, 1), (BEND1, 1, 2), (BEND2, 2, 2)):
            if not p.flags & fam:
                continue
            k = cfg.stiffness[b:b + npts].reshape(p.n2, p.n1)
            L0 = cfg.stiffness[b + npts:b + 2 * npts].reshape(p.n2, p.n1)
            b += 2 * npts
            wrap = bool(p.flags & (WRAP1 if axis == 1 else 2))
            for i2 in range(p.n2):
                for i1 in range(p.n1):
                    j1, j2 = (i1 + off, i2) if axis == 1 else (i1, i2 + off)
                    if not wrap and (j1 >= p.n1 or j2 >= p.n2):
                        continue
                    d = P[j2 % p.n2, j1 % p.n1] - P[i2, i1]
                    E += 0.5 * k[i2, i1] * (np.linalg.norm(d) - L0[i2, i1]) ** 2
        if p.flags & TETHER:
            kt = cfg.stiffness[b:b + npts]
            Y = cfg.stiffness[b + npts:b + 4 * npts].reshape(-1, 3)
            E += 0.5 * np.sum(kt * np.sum((P.reshape(-1, 3) - Y) ** 2, axis=1))
    return E


def test_force_rest_is_exactly_zero(olib):
    for k in (3,):
        cfg = make_config(k)
        F = olib.force(cfg.X, cfg.patches, cfg.stiffness)
        assert np.max(np.abs(F)) == 0.0          # L0 computed in the same IEEE order (Z13)


def test_force_newton_third_law_and_energy_gradient(olib):
    cfg = small_sheet_config(N=16, n1=6, n2=5, seed=3, drive=False, tether=True)
    F = olib.force(cfg.X, cfg.patches, cfg.stiffness)
    sheet = cfg.patches[0]
    Fs = olib.force(cfg.X, cfg.patches[:1], cfg.stiffness)
    assert np.max(np.abs(Fs.sum(0))) < 1e-13 * np.max(np.abs(Fs))      # springs only: sum = 0
    # F = -dE/dX by central differences
    eps = 1e-7
    rng = np.random.default_rng(0)
    for _ in range(12):
        i, c = int(rng.integers(cfg.X.shape[0])), int(rng.integers(3))
        Xp = cfg.X.copy(); Xp[i, c] += eps
        Xm = cfg.X.copy(); Xm[i, c] -= eps
        g = (_energy(Xp, cfg) - _energy(Xm, cfg)) / (2 * eps)
        assert abs(-g - F[i, c]) <= 1e-6 * max(1.0, np.max(np.abs(F)))
    assert sheet.flags & BEND1


def test_force_hooke_by_hand(olib):
    # two points, one STRETCH1 link k = 3, L0 = 0.1, stretched to 0.25 along (1, 2, 2)/3
    X = np.array([[0.1, 0.2, 0.3], [0.1 + 0.25 / 3, 0.2 + 0.5 / 3, 0.3 + 0.5 / 3]])
    stiff = np.array([3.0, 0.0, 0.1, 0.0])                  # k[2], L0[2]
    F = olib.force(X, [Patch(0, 2, 1, STRETCH1, 0)], stiff)
    want = 3.0 * (0.25 - 0.1) * np.array([1, 2, 2]) / 3
    assert np.allclose(F[0], want, rtol=1e-14, atol=0) and np.allclose(F[1], -want, rtol=1e-14)


def test_force_wrap_ring_and_tether_linear(olib):
    n = 8
    th = 2 * np.pi * np.arange(n) / n
    X = np.stack([0.5 + 0.2 * np.cos(th), 0.5 + 0.2 * np.sin(th), 0.5 + 0 * th], 1)
    L0 = np.full(n, 0.1)
    F = olib.force(X, [Patch(0, n, 1, STRETCH1 | WRAP1, 0)], np.concatenate([np.ones(n), L0]))
    chord = 2 * 0.2 * np.sin(np.pi / n)
    radial = -(X - 0.5) / 0.2
    mag = 2 * (chord - 0.1) * np.sin(np.pi / n)             # two links, inward resultant
    assert np.allclose(F, mag * radial, atol=1e-15)
    # tether: F = kt (Y - X), exactly linear in the displacement
    Y = X + 0.01
    kt = np.linspace(1, 2, n)
    S = np.concatenate([kt, Y.reshape(-1)])
    F1 = olib.force(X, [Patch(0, n, 1, TETHER, 0)], S)
    assert np.allclose(F1, kt[:, None] * 0.01, rtol=1e-12)
    F2 = olib.force(Y - 0.03, [Patch(0, n, 1, TETHER, 0)], S)
    assert np.allclose(F2, kt[:, None] * 0.03, rtol=1e-12)


def test_drive_phase(olib):
    X = np.zeros((3, 3)) + 0.5
    idx = np.array([1]); d = np.array([[0.0, 0.6, 0.8]])
    for n, s in ((0, 0.0), (2, 1.0), (4, 0.0), (6, -1.0), (8 + 2, 1.0)):
        F = olib.force(X, [], np.zeros(0), step=n, drive_idx=idx, drive_dir=d,
                       drive_amp=2.0, drive_period=8)
        assert np.allclose(F[1], 2.0 * s * d[0], atol=1e-15) and not F[[0, 2]].any()


def test_step_rest_fixed_point(olib):
    cfg = make_config(3)                      # rest geometry; drive sin(0) = 0 at n = 0
    o = olib.Oracle.from_config(cfg)
    o.step(1)
    u, p = o.get_fields()
    assert np.max(np.abs(u)) == 0.0
    assert np.array_equal(o.get_positions(), cfg.X)


def test_step_uniform_translation(olib):
    # spring-only structure at rest, uniform u = c: u unchanged, X^n = X^0 + n dt c
    cfg = small_sheet_config(N=16, n1=6, n2=5, seed=4, drive=False, tether=False, noise=0.0)
    # put the springs at rest: L0 = current lengths
    o = olib.Oracle(cfg.N, cfg.h, cfg.rho, cfg.mu, cfg.dt)
    import gen.configs as gc
    P = cfg.X.reshape(5, 6, 3)
    blocks = []
    for fam, axis, off in gc.FAMILIES:
        L0 = gc._rest_lengths(P, 6, 5, axis, off, False)
        blocks += [np.where(L0 > 0, 1.0, 0.0), L0]
    o.set_structure(cfg.X, cfg.patches, np.concatenate([b.ravel() for b in blocks]))
    c = np.array([0.3, -0.2, 0.1])
    o.set_velocity(np.broadcast_to(c[:, None, None, None], (3, 16, 16, 16)))
    o.step(5)
    u, _ = o.get_fields()
    assert np.max(np.abs(u - c[:, None, None, None])) < 1e-15
    assert np.max(np.abs(o.get_positions() - (cfg.X + 5 * cfg.dt * c))) < 1e-15


@pytest.mark.parametrize("k,steps,umax,dmax", [(1, 10, 0.1, 0.05), (2, 20, 20.0, 2.0)])
def test_configs_stay_bounded(olib, k, steps, umax, dmax):
    # cfg2's open lat-long poles carry unbalanced meridian tension (reading Z16):
    # a strong but bounded polar jet (max|u| oscillates in 1.5-7), not a blow-up.
    cfg = make_config(k)
    o = olib.Oracle.from_config(cfg)
    o.step(steps)
    u, _ = o.get_fields()
    disp = np.max(np.abs(o.get_positions() - cfg.X))
    assert np.isfinite(u).all() and np.max(np.abs(u)) < umax
    assert disp < dmax * cfg.h


# ---------------------------------------------------------------- window plates
def test_window_fixed_points_never_move_and_free_points_do(olib):
    from gen import window_config
    cfg = window_config(N=16, m=16, seed=3, u_amp=0.05)
    o = olib.Oracle.from_config(cfg)
    X0 = cfg.X.copy()
    o.step(5)
    fixed = cfg.fixed.astype(bool)
    assert fixed.any() and (~fixed).any()
    assert np.array_equal(o.X[fixed], X0[fixed])                 # bitwise: never updated
    assert np.min(np.abs(o.X[~fixed] - X0[~fixed]).max(1)) > 0    # every free point moved


def test_window_normal_drive_is_orthogonal_to_the_plate(olib):
    # a flat plate in the plane spanned by e1, e2: every driven force is along e1 x e2 and of
    # the prescribed magnitude amp * sin(2 pi n / T) (PAPER.md 988-993)
    from gen import window_config
    cfg = window_config(N=16, m=12, seed=4, amp=3e-3, period=8)
    i = np.arange(cfg.X.shape[0])
    m = 12
    e1 = cfg.X[1] - cfg.X[0]; e2 = cfg.X[m] - cfg.X[0]
    flat = cfg.X[0] + (i % m)[:, None] * e1 + (i // m)[:, None] * e2   # undo the bulge
    step = 2                                                   # sin(2 pi 2/8) = 1
    f_drive = olib.force(flat, cfg.patches, cfg.stiffness * 0.0, step, cfg.drive_idx, None,
                         cfg.drive_amp, cfg.drive_period)
    nrm = np.cross(e1, e2); nrm /= np.linalg.norm(nrm)
    fd = f_drive[cfg.drive_idx]
    along = fd @ nrm
    assert np.allclose(np.abs(along), cfg.drive_amp, rtol=1e-13, atol=0)
    assert np.max(np.linalg.norm(fd - along[:, None] * nrm, axis=1)) < 1e-15 * cfg.drive_amp * 10
    assert np.all(f_drive[cfg.fixed.astype(bool)] == 0.0)      # no drive on the bony rim
    f0 = olib.force(flat, cfg.patches, cfg.stiffness * 0.0, 0, cfg.drive_idx, None,
                    cfg.drive_amp, cfg.drive_period)
    assert np.max(np.abs(f0)) == 0.0                            # t = 0 -> sin 0 = 0


def test_window_fixed_points_still_spread_their_force(olib):
    # total spread force equals the total nodal force including the fixed rim's reactions
    from gen import window_config
    cfg = window_config(N=16, m=16, seed=5)
    f = olib.force(cfg.X, cfg.patches, cfg.stiffness, 2, cfg.drive_idx, None, cfg.drive_amp,
                   cfg.drive_period)
    fixed = cfg.fixed.astype(bool)
    assert np.abs(f[fixed]).max() > 0                          # the rim pulls back on the disc
    F = olib.spread(16, cfg.h, cfg.X, f)
    assert np.allclose(F.reshape(3, -1).sum(1) * cfg.h ** 3, f.sum(0), rtol=0,
                       atol=1e-13 * np.abs(f).sum())


# ---------------------------------------------------------------- time coupling (eq:discreteX)
@pytest.mark.parametrize("N,m", [(16, 3), ((16, 32, 8), 5)])
def test_step_interpolates_new_velocity_at_old_positions(olib, N, m):
    """Pins the time levels of eq:discreteX (PAPER.md 725-734, lines 729-730): X^{n+1} =
    X^n + dt sum_x u^{n+1}(x) delta_h(x - X^n) h^3.  Free points (F = 0) in the shear mode
    u^0 = A sin(2 pi m y) e_x: u^{n+1} = g u^n with the closed-form viscous gain g
    (tests/closed_forms.py), so X_x^1 - X_x^0 = dt g A S(Y) and X_x^2 - X_x^1 = dt g^2 A S(Y)
    with S(Y) = sum_b phi(j_b - Y/h) sin(2 pi m j_b/N2).  Interpolating u^n instead of u^{n+1}
    misses by the factor 1 - g (0.18-0.24 here)."""
    import closed_forms as cf
    from gen import decaying_shear_config
    cfg = decaying_shear_config(N=N, m=m, seed=8)
    o = olib.Oracle.from_config(cfg)
    X0 = cfg.X.copy()
    for n in (1, 2):
        o.step(1)
        want, g = cf.shear_positions(cfg, n)
        assert 0.15 < 1.0 - g < 0.8
        # the fluid: u^n = g^n u^0 (advection 0, projection inactive)
        assert np.max(np.abs(o.u - g ** n * cfg.u0)) <= 1e-14 * cfg.info["A"]
        d_got, d_want = o.X - X0, want - X0
        assert np.max(np.abs(d_got - d_want)) <= 1e-12 * np.max(np.abs(d_want))
        assert np.max(np.abs(o.X[:, 1:] - X0[:, 1:])) <= 1e-16
    # the wrong coupling (u^n at X^n) would have given dt A S(Y) in the first step
    o1 = olib.Oracle.from_config(cfg)
    o1.step(1)
    wrong = cfg.dt * cfg.info["A"] * cf.shear_interp(X0[:, 1], o1.dims[1], cfg.h, m)
    assert np.max(np.abs((o1.X[:, 0] - X0[:, 0]) - wrong)) > 0.15 * np.max(np.abs(wrong))
