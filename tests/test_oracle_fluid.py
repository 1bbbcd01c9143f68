"""Pins of the oracle's fluid step (CPU only).

Pins come from the discrete system itself (PAPER.md eq:discreteNS1-2, lines 659-695):
a physical-space residual built from independent np.roll difference operators
(eq:differenceOps, lines 641-655), the closed-form single-mode decay, divergence,
zero-mode bookkeeping, gradient forcing, Stokes linearity, and — for the FFT — the
direct O(N^6) DFT on 8^3 and numpy's FFT.
"""
import numpy as np
import pytest


# ---- independent difference operators on [z][y][x] arrays (axis a: 0=x, 1=y, 2=z) ----
def _ax(a):
    return {0: -1, 1: -2, 2: -3}[a]


def Dp(f, a, h):
    return (np.roll(f, -1, _ax(a)) - f) / h


def Dm(f, a, h):
    return (f - np.roll(f, 1, _ax(a))) / h


def D0(f, a, h):
    return (np.roll(f, -1, _ax(a)) - np.roll(f, 1, _ax(a))) / (2 * h)


def lap(f, h):
    return sum(Dp(Dm(f, a, h), a, h) for a in range(3))


def div0(u, h):
    return sum(D0(u[a], a, h) for a in range(3))


def test_fft_equals_direct_dft_8cubed(olib):
    rng = np.random.default_rng(10)
    N = 8
    x = rng.standard_normal((N, N, N)) + 1j * rng.standard_normal((N, N, N))
    j = np.arange(N)
    W = np.exp(-2j * np.pi * np.outer(j, j) / N)              # direct DFT matrix
    direct = np.einsum("az,by,cx,zyx->abc", W, W, W, x)       # O(N^6)
    got = olib.fft3(x, -1)
    assert np.max(np.abs(got - direct)) < 1e-13 * np.max(np.abs(direct))
    inv = np.einsum("az,by,cx,zyx->abc", W.conj(), W.conj(), W.conj(), x)
    assert np.max(np.abs(olib.fft3(x, +1) - inv)) < 1e-13 * np.max(np.abs(inv))


@pytest.mark.parametrize("N", [16, 32, 64])
def test_fft_matches_numpy_and_round_trip(olib, N):
    rng = np.random.default_rng(N)
    x = rng.standard_normal((N, N, N)) + 1j * rng.standard_normal((N, N, N))
    X = olib.fft3(x, -1)
    ref = np.fft.fftn(x)
    assert np.max(np.abs(X - ref)) < 1e-13 * np.max(np.abs(ref))
    back = olib.fft3(X, +1) / N ** 3
    assert np.max(np.abs(back - x)) < 1e-14 * np.max(np.abs(x)) * np.log2(N)
    # Parseval
    assert abs(np.sum(np.abs(X) ** 2) / N ** 3 - np.sum(np.abs(x) ** 2)) < 1e-11 * np.sum(np.abs(x) ** 2)


def test_fft_single_mode_is_one_spike(olib):
    N = 16
    k = (3, 5, 11)  # (kx, ky, kz)
    j = np.arange(N)
    zz, yy, xx = np.meshgrid(j, j, j, indexing="ij")
    x = np.exp(2j * np.pi * (k[0] * xx + k[1] * yy + k[2] * zz) / N)
    X = olib.fft3(x, -1)
    assert abs(X[k[2], k[1], k[0]] - N ** 3) < 1e-9
    X[k[2], k[1], k[0]] = 0
    assert np.max(np.abs(X)) < 1e-9


def test_advection_constant_and_closed_forms(olib):
    N, h = 16, 1.0 / 16
    u = np.zeros((3, N, N, N)); u[0], u[1], u[2] = 0.3, -0.2, 0.7
    assert np.max(np.abs(olib.advect(N, h, u))) == 0.0
    x = np.arange(N) * h
    zz, yy, xx = np.meshgrid(x, x, x, indexing="ij")
    for c in (0.4, -0.4):
        u = np.stack([np.sin(2 * np.pi * yy), c + 0 * yy, 0 * yy])
        a = olib.advect(N, h, u)
        sy = np.sin(2 * np.pi * x)
        if c > 0:
            want1 = c * (sy - np.roll(sy, 1)) / h          # backward difference D_y^-
        else:
            want1 = c * (np.roll(sy, -1) - sy) / h          # forward difference D_y^+
        assert np.max(np.abs(a[0] - want1[None, :, None])) < 1e-12
        assert np.max(np.abs(a[1])) == 0 and np.max(np.abs(a[2])) == 0


def test_advection_mixed_sign_separable(olib):
    # u = (f(y), g(z), k(x)): adv_x = g(z) * upwind_y(f); adv_y = k(x) * upwind_z(g);
    # adv_z = f(y) * upwind_x(k); upwind by the sign of the advecting component (PAPER.md 676-691)
    rng = np.random.default_rng(11)
    N, h = 8, 1.0 / 8
    f, g, k = rng.standard_normal(N), rng.standard_normal(N), rng.standard_normal(N)
    g[2] = 0.0                                                   # a tie (u_k = 0)
    zz, yy, xx = np.meshgrid(np.arange(N), np.arange(N), np.arange(N), indexing="ij")
    u = np.stack([f[yy], g[zz], k[xx]]).astype(float)
    a = olib.advect(N, h, u)

    want0 = g[zz] * np.where(g[zz] < 0, ((np.roll(f, -1) - f) / h)[yy], ((f - np.roll(f, 1)) / h)[yy])
    want1 = k[xx] * np.where(k[xx] < 0, ((np.roll(g, -1) - g) / h)[zz], ((g - np.roll(g, 1)) / h)[zz])
    want2 = f[yy] * np.where(f[yy] < 0, ((np.roll(k, -1) - k) / h)[xx], ((k - np.roll(k, 1)) / h)[xx])
    for got, want in zip(a, (want0, want1, want2)):
        assert np.max(np.abs(got - want)) < 1e-13 * np.max(np.abs(want))


def _rand(N, seed):
    return np.random.default_rng(seed).standard_normal((3, N, N, N))


@pytest.mark.parametrize("N", [8, 16])
def test_solve_physical_space_residual(olib, N):
    h, rho, mu, dt = 1.0 / N, 1.3, 0.02, 1e-2
    r = _rand(N, 12)
    u, p = olib.solve(N, h, rho, mu, dt, r)
    gp = np.stack([D0(p, a, h) for a in range(3)])
    res = rho * u / dt + gp - mu * np.stack([lap(u[a], h) for a in range(3)]) - r
    assert np.max(np.abs(res)) < 1e-12 * np.max(np.abs(r))
    assert np.max(np.abs(div0(u, h))) < 1e-12 * np.max(np.abs(u)) / h


@pytest.mark.parametrize("N", [8, 16, 32, 64])
def test_single_mode_viscous_decay(olib, N):
    # u0 = A (sin 2 pi m y, 0, 0), F = 0: advection vanishes, projection inactive:
    # u^n = A (1 + mu dt (4/h^2) sin^2(pi m/N)/rho)^-n
    h, rho, mu, dt, A, m = 1.0 / N, 1.0, 0.01, 1e-3, 0.7, 3
    y = np.arange(N) * h
    u = np.zeros((3, N, N, N))
    u[0] = A * np.sin(2 * np.pi * m * y)[None, :, None]
    F = np.zeros_like(u)
    g = 1.0 / (1.0 + mu * dt * 4.0 / h ** 2 * np.sin(np.pi * m / N) ** 2 / rho)
    for n in range(1, 6):
        u, _ = olib.fluid_step(N, h, rho, mu, dt, u, F)
        want = A * g ** n * np.sin(2 * np.pi * m * y)[None, :, None]
        assert np.max(np.abs(u[0] - want)) <= 1e-10 * A * g ** n
        assert np.max(np.abs(u[1:])) < 1e-15


def test_divergence_zero_mode_and_uniform_force(olib):
    N, h, rho, mu, dt = 16, 1.0 / 16, 1.0, 0.01, 1e-3
    rng = np.random.default_rng(13)
    u = 0.1 * rng.standard_normal((3, N, N, N))
    F = rng.standard_normal((3, N, N, N))
    un, p = olib.fluid_step(N, h, rho, mu, dt, u, F)
    assert np.max(np.abs(div0(un, h))) <= 1e-10 * max(1.0, np.max(np.abs(un)) / h)
    # zero-mode momentum: mean(u') = mean(u) - dt mean(adv) + dt mean(F)/rho
    adv = olib.advect(N, h, u)
    want = u.mean((1, 2, 3)) - dt * adv.mean((1, 2, 3)) + dt * F.mean((1, 2, 3)) / rho
    assert np.max(np.abs(un.mean((1, 2, 3)) - want)) < 1e-14
    # uniform force and uniform velocity: u' = u + dt G/rho
    G = np.array([0.5, -1.0, 2.0]); c = np.array([0.1, 0.2, -0.3])
    uu = np.broadcast_to(c[:, None, None, None], (3, N, N, N)).copy()
    FF = np.broadcast_to(G[:, None, None, None], (3, N, N, N)).copy()
    un, p = olib.fluid_step(N, h, rho, mu, dt, uu, FF)
    assert np.max(np.abs(un - (c + dt * G / rho)[:, None, None, None])) < 1e-14
    assert np.max(np.abs(p)) < 1e-10


def test_gradient_forcing_goes_to_pressure(olib):
    N, h, rho, mu, dt = 16, 1.0 / 16, 1.0, 0.01, 1e-3
    phi = np.random.default_rng(14).standard_normal((N, N, N))
    F = np.stack([D0(phi, a, h) for a in range(3)])
    un, p = olib.fluid_step(N, h, rho, mu, dt, np.zeros_like(F), F)
    assert np.max(np.abs(un)) < 1e-12 * np.max(np.abs(F))
    for a in range(3):                                  # p = phi up to D0's null space
        assert np.max(np.abs(D0(p - phi, a, h))) < 1e-11 * np.max(np.abs(F))


def test_stokes_path_linearity(olib):
    N, h, rho, mu, dt = 8, 1.0 / 8, 1.0, 0.05, 1e-2
    r1, r2 = _rand(N, 15), _rand(N, 16)
    u1, p1 = olib.solve(N, h, rho, mu, dt, r1)
    u2, p2 = olib.solve(N, h, rho, mu, dt, r2)
    u3, p3 = olib.solve(N, h, rho, mu, dt, 2.0 * r1 - 3.0 * r2)
    assert np.max(np.abs(u3 - (2 * u1 - 3 * u2))) < 1e-12 * np.max(np.abs(u3))
    assert np.max(np.abs(p3 - (2 * p1 - 3 * p2))) < 1e-12 * np.max(np.abs(p3))


def test_nyquist_null_space_integer_decision(olib):
    # r = checkerboard along x (pure Nyquist mode, s = 0): no pressure, u = r/d
    N, h, rho, mu, dt = 8, 1.0 / 8, 1.0, 0.01, 1e-3
    x = np.arange(N)
    r = np.zeros((3, N, N, N))
    r[0] = ((-1.0) ** x)[None, None, :]
    u, p = olib.solve(N, h, rho, mu, dt, r)
    d = rho / dt + mu * 4 / h ** 2 * 1.0        # sin^2(pi (N/2)/N) = 1
    assert np.max(np.abs(u[0] - r[0] / d)) < 1e-15 * N
    assert np.max(np.abs(p)) == 0.0


# ---------------------------------------------------------------- anisotropic lattices
# (the paper's half-cube model is 256 x 256 x 128, PAPER.md 1003-1007)
@pytest.mark.parametrize("shape", [(8, 4, 2), (4, 8, 16), (16, 2, 8)])
def test_fft_equals_direct_dft_anisotropic(olib, shape):
    n1, n2, n3 = shape
    rng = np.random.default_rng(sum(shape))
    x = rng.standard_normal((n3, n2, n1)) + 1j * rng.standard_normal((n3, n2, n1))

    def W(n):
        j = np.arange(n)
        return np.exp(-2j * np.pi * np.outer(j, j) / n)
    direct = np.einsum("az,by,cx,zyx->abc", W(n3), W(n2), W(n1), x)
    got = olib.fft3(x, -1)
    assert np.max(np.abs(got - direct)) < 1e-13 * np.max(np.abs(direct))


@pytest.mark.parametrize("shape", [(8, 16, 4), (16, 8, 32)])
def test_solve_physical_space_residual_anisotropic(olib, shape):
    n1, n2, n3 = shape
    h, rho, mu, dt = 1.0 / 16, 1.1, 0.03, 1e-2
    r = np.random.default_rng(13).standard_normal((3, n3, n2, n1))
    u, p = olib.solve(shape, h, rho, mu, dt, r)
    gp = np.stack([D0(p, a, h) for a in range(3)])
    res = rho * u / dt + gp - mu * np.stack([lap(u[a], h) for a in range(3)]) - r
    assert np.max(np.abs(res)) < 1e-12 * np.max(np.abs(r))
    assert np.max(np.abs(div0(u, h))) < 1e-12 * np.max(np.abs(u)) / h


@pytest.mark.parametrize("axis", [0, 1, 2])
def test_single_mode_decay_anisotropic(olib, axis):
    # u_c = A sin(2 pi m j_a / N_a) along axis a (c != a): advection and projection vanish;
    # u^n = A (1 + mu dt (4/h^2) sin^2(pi m/N_a)/rho)^-n
    shape = (16, 8, 32)
    h, rho, mu, dt, A, m = 1.0 / 16, 1.0, 0.02, 1e-3, 0.5, 3
    n = shape[axis]
    j = np.arange(n)
    prof = A * np.sin(2 * np.pi * m * j / n)
    bshape = [1, 1, 1]
    bshape[2 - axis] = n
    u = np.zeros((3, shape[2], shape[1], shape[0]))
    c = (axis + 1) % 3
    u[c] = prof.reshape(bshape)
    F = np.zeros_like(u)
    g = 1.0 / (1.0 + mu * dt * 4.0 / h ** 2 * np.sin(np.pi * m / n) ** 2 / rho)
    for k in range(1, 4):
        u, _ = olib.fluid_step(shape, h, rho, mu, dt, u, F)
        assert np.max(np.abs(u[c] - g ** k * prof.reshape(bshape))) <= 1e-10 * A * g ** k
        assert np.max(np.abs(u[(c + 1) % 3])) == 0.0 and np.max(np.abs(u[(c + 2) % 3])) == 0.0
