"""GPU parity: the CUDA path through the C-ABI against the CPU oracle, element by element.

Tolerances: single stages with a deterministic order 1e-13 relative;
atomic stages (spread) 1e-13; full IB step rel-L2 <= 1e-11 after 1 step and <= 1e-9
after 10 steps on u and X (BASELINE.json north_star), plus the interpolated velocity U
and the displacement X - X0 (reading Z4).
"""
import numpy as np
import pytest

from gen import make_config, random_divfree_velocity, random_points, small_sheet_config
from parity import rel_l2, step_parity

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ibm():
    from paper_math_0301321_b200 import _build, ib
    _build.build()
    ib.load()
    return ib


def _ctx(ibm, N, rho=1.0, mu=0.01, dt=1e-3, X=None, patches=None, stiff=None):
    c = ibm.IBContext(N, 1.0 / N, rho, mu, dt)
    if X is not None:
        c.set_structure(X, patches, stiff)
    return c


def _points_only(X):
    """A structure of free points (one patch, no links) so debug spread/interp see X."""
    from gen import Patch
    return [Patch(0, X.shape[0], 1, 0, 0)], np.zeros(0)


# ------------------------------------------------------------------ single stages
@pytest.mark.parametrize("N", [8, 16, 32, 64, 128])
def test_fft_matches_oracle_and_numpy(ibm, olib, N):
    rng = np.random.default_rng(N)
    x = rng.standard_normal((N, N, N))
    with _ctx(ibm, N) as c:
        got = c.debug_fft(x)
    ref = np.fft.rfftn(x)
    assert np.max(np.abs(got - ref)) < 1e-13 * np.max(np.abs(ref)) * np.log2(N)
    if N <= 32:
        orc = olib.fft3(x.astype(complex), -1)[:, :, : N // 2 + 1]
        assert np.max(np.abs(got - orc)) < 1e-13 * np.max(np.abs(orc)) * np.log2(N)


@pytest.mark.parametrize("N", [8, 16, 32])
def test_rhs_matches_oracle(ibm, olib, N):
    rng = np.random.default_rng(1)
    u = rng.standard_normal((3, N, N, N))
    u[0, 0, 0, :] = 0.0                      # ties u_k = 0 (reading Z5)
    F = rng.standard_normal((3, N, N, N))
    h, rho, dt = 1.0 / N, 1.3, 2e-3
    with ibm.IBContext(N, h, rho, 0.01, dt) as c:
        r = c.debug_rhs(u, F)
    ref = olib.rhs(N, h, rho, dt, u, F)
    assert np.max(np.abs(r - ref)) <= 1e-13 * np.max(np.abs(ref))


@pytest.mark.parametrize("N", [8, 16, 32, 64])
def test_fluid_step_matches_oracle(ibm, olib, N):
    rng = np.random.default_rng(2)
    u = random_divfree_velocity(N, 3, 0.3, rng) + 0.05 * rng.standard_normal((3, N, N, N))
    F = rng.standard_normal((3, N, N, N)) * 50
    h, rho, mu, dt = 1.0 / N, 1.0, 0.02, 1e-3
    with ibm.IBContext(N, h, rho, mu, dt) as c:
        un, p = c.debug_fluid(u, F)
    ref_u, ref_p = olib.fluid_step(N, h, rho, mu, dt, u, F)
    assert rel_l2(un, ref_u) < 1e-13
    assert rel_l2(p, ref_p) < 1e-12


@pytest.mark.parametrize("N,npts,cluster", [(16, 1000, False), (32, 5000, True), (64, 20000, True)])
def test_spread_matches_oracle(ibm, olib, N, npts, cluster):
    rng = np.random.default_rng(3)
    if cluster:   # heavy per-cell fan-in (many points per cell) + points outside [0,1)
        centres = rng.uniform(-0.2, 1.2, (npts // 50, 3))
        X = centres[rng.integers(0, len(centres), npts)] + rng.uniform(0, 0.3 / N, (npts, 3))
    else:
        X = random_points(npts, rng)
    f = rng.standard_normal((npts, 3))
    f[::7] = 0.0
    patches, st = _points_only(X)
    with _ctx(ibm, N, X=X, patches=patches, stiff=st) as c:
        F = c.debug_spread(f)
    ref = olib.spread(N, 1.0 / N, X, f)
    assert rel_l2(F, ref) < 1e-13
    tot = F.reshape(3, -1).sum(1) / N ** 3
    assert np.allclose(tot, f.sum(0), rtol=0, atol=1e-11 * np.abs(f).sum())


@pytest.mark.parametrize("N,npts", [(16, 777), (64, 20000)])
def test_interp_matches_oracle_and_adjoint(ibm, olib, N, npts):
    rng = np.random.default_rng(4)
    X = random_points(npts, rng, -0.5, 1.5)
    u = rng.standard_normal((3, N, N, N))
    patches, st = _points_only(X)
    with _ctx(ibm, N, X=X, patches=patches, stiff=st) as c:
        U = c.debug_interp(u)
        f = rng.standard_normal((npts, 3))
        F = c.debug_spread(f)
    ref = olib.interp(N, 1.0 / N, u, X)
    assert rel_l2(U, ref) < 1e-14
    lhs = np.sum(F * u) / N ** 3
    rhs = np.sum(f * U)
    assert abs(lhs - rhs) <= 1e-12 * max(1.0, abs(lhs))


def _clustered_points(N, rng):
    """Points laid out warp by warp (index order) so that the tensor-core interp sees every
    grouping case: one 32-member group (4 MMA row blocks), uneven groups (9, 8, 7, 5, 3),
    exactly 8 groups (the MMA limit), 9 groups (per-point fallback), cells on the periodic
    edge (wrapped support), and a partial last warp (non-live lanes)."""
    h = 1.0 / N
    warps = [[32], [9, 8, 7, 5, 3], [4] * 8, [3, 3, 3, 3, 4, 4, 4, 4, 4], [13, 7]]
    pts = []
    cell = 0
    for sizes in warps:
        for m in sizes:
            c = np.array([(7 * cell) % N, (3 * cell + 1) % N, (5 * cell + 2) % N])
            if cell % 3 == 0:
                c[cell % 3] = N - 1                 # support wraps around the box
            cell += 1
            pts.append((c + rng.uniform(0.0, 1.0, size=(m, 3))) * h)
    return np.ascontiguousarray(np.concatenate(pts))


@pytest.mark.parametrize("shuffle", [False, True])
def test_interp_grouping_cases_match_oracle(ibm, olib, shuffle):
    N = 32
    rng = np.random.default_rng(11)
    X = _clustered_points(N, rng)
    if shuffle:
        X = X[rng.permutation(X.shape[0])]
    u = rng.standard_normal((3, N, N, N))
    patches, st = _points_only(X)
    with _ctx(ibm, N, X=X, patches=patches, stiff=st) as c:
        U = c.debug_interp(u)
        f = rng.standard_normal((X.shape[0], 3))
        F = c.debug_spread(f)
    ref = olib.interp(N, 1.0 / N, u, X)
    assert rel_l2(U, ref) < 1e-14
    assert np.max(np.abs(U - ref)) <= 1e-13 * np.max(np.abs(ref))
    Fo = olib.spread(N, 1.0 / N, X, f)
    assert rel_l2(F, Fo) < 1e-13


@pytest.mark.parametrize("step", [0, 3, 5])
def test_force_matches_oracle(ibm, olib, step):
    cfg = small_sheet_config(N=16, n1=12, n2=10, seed=5)
    with ibm.IBContext.from_config(cfg) as c:
        c.set_step(step)
        f = c.debug_force()
    ref = olib.force(cfg.X, cfg.patches, cfg.stiffness, step, cfg.drive_idx, cfg.drive_dir,
                     cfg.drive_amp, cfg.drive_period)
    assert rel_l2(f, ref) < 1e-14


def test_force_at_rest_is_exactly_zero(ibm):
    cfg = make_config(3)
    with ibm.IBContext.from_config(cfg) as c:
        assert np.max(np.abs(c.debug_force())) == 0.0


# ------------------------------------------------------------------ whole step
def _parity(ibm, olib, cfg, steps=(1, 1, 8), tol=(1e-11, 1e-11, 1e-9), elem=1e-10):
    """GPU (one context) vs oracle at checkpoints 1, 2 and 10: see parity.step_parity."""
    return step_parity(olib, cfg, lambda: ibm.IBContext.from_config(cfg), steps, tol, elem)


@pytest.mark.parametrize("k", [1, 2, 3])
def test_config_step_parity(ibm, olib, k):
    print(_parity(ibm, olib, make_config(k)))


@pytest.mark.slow
def test_config4_step_parity(ibm, olib):
    print(_parity(ibm, olib, make_config(4)))


@pytest.mark.slow
def test_config5_step_parity(ibm, olib):
    """BASELINE.json configs[4]: 512^3, 8.4M points, random initial flow; checkpoints after
    1, 2 and 10 steps (1e-11, 1e-11, 1e-9).  The oracle needs ~30 s per step here."""
    print(_parity(ibm, olib, make_config(5)))


@pytest.mark.parametrize("N,m", [(16, 3), ((16, 32, 8), 5), (64, 7)])
def test_step_time_coupling_closed_form(ibm, N, m):
    """eq:discreteX's time levels on the GPU (PAPER.md 725-734): free points in the decaying
    shear mode move by dt g^{n+1} A S(Y) per step (tests/closed_forms.py; the same pin as
    tests/test_oracle_force_step.py::test_step_interpolates_new_velocity_at_old_positions)."""
    import closed_forms as cf
    from gen import decaying_shear_config
    cfg = decaying_shear_config(N=N, m=m, seed=9, npts=300)
    with ibm.IBContext.from_config(cfg) as c:
        for n in (1, 2):
            c.step(1)
            want, g = cf.shear_positions(cfg, n)
            u, _ = c.get_fields()
            X = c.get_positions()
            assert np.max(np.abs(u - g ** n * cfg.u0)) <= 1e-14 * cfg.info["A"]
            d_want = want - cfg.X
            assert np.max(np.abs((X - cfg.X) - d_want)) <= 1e-12 * np.max(np.abs(d_want))


def test_small_sheet_with_tethers_drive_and_flow(ibm, olib):
    cfg = small_sheet_config(N=32, n1=20, n2=14, seed=6, u_amp=0.2)
    print(_parity(ibm, olib, cfg))


def test_pure_fluid_and_pressure(ibm, olib):
    N = 32
    rng = np.random.default_rng(7)
    u0 = random_divfree_velocity(N, 4, 0.5, rng)
    o = olib.Oracle(N, 1.0 / N, 1.0, 0.01, 1e-3)
    o.set_velocity(u0)
    with ibm.IBContext(N, 1.0 / N, 1.0, 0.01, 1e-3) as c:
        c.set_velocity(u0)
        c.set_option(ibm.IB_OPT_PRESSURE, 1)
        c.step(3)
        o.step(3)
        ug, pg = c.get_fields(want_p=True)
    uo, po = o.get_fields()
    assert rel_l2(ug, uo) < 1e-12
    assert rel_l2(pg, po) < 1e-10


def test_device_pointers_roundtrip(ibm):
    import torch
    cfg = make_config(1)
    N = cfg.N
    with ibm.IBContext.from_config(cfg) as c:
        u = torch.randn(3, N, N, N, dtype=torch.float64, device="cuda") * 1e-3
        c.set_velocity(u)
        out = torch.empty_like(u)
        c.get_fields_into(out)
        assert torch.equal(out, u)
        X = torch.empty(cfg.X.shape[0], 3, dtype=torch.float64, device="cuda")
        c.get_positions_into(X)
        assert np.array_equal(X.cpu().numpy(), cfg.X)


def test_error_codes(ibm):
    from gen import Patch, STRETCH1
    with ibm.IBContext(16, 1 / 16, 1, 0.01, 1e-3) as c:
        X = np.array([[0.5, 0.5, 0.5], [0.5, 0.5, 0.5]])
        with pytest.raises(ibm.IBError) as e:
            c.set_structure(X, [Patch(0, 2, 1, STRETCH1, 0)], np.array([1.0, 0, 0.1, 0]))
        assert e.value.code == ibm.IB_EDEGENERATE
        with pytest.raises(ibm.IBError) as e:
            c.set_structure(np.array([[np.nan, 0, 0]]), [Patch(0, 1, 1, 0, 0)], np.zeros(0))
        assert e.value.code == ibm.IB_EINVAL
        with pytest.raises(ibm.IBError) as e:
            c.get_fields(want_p=True)
        assert e.value.code == ibm.IB_ESTATE
        # blow-up is detected and reported
        X = np.array([[0.5, 0.5, 0.5], [0.52, 0.5, 0.5]])
        c.set_structure(X, [Patch(0, 2, 1, STRETCH1, 0)], np.array([1e30, 0, 1e-6, 0]))
        with pytest.raises(ibm.IBError) as e:
            c.step(50)
        assert e.value.code == ibm.IB_ENONFINITE


@pytest.mark.parametrize("N", [16, 64])
def test_nonfinite_step_reported_as_in_single_steps(ibm, N):
    """The first non-finite step reported by a multi-step graph run (the step index read on
    the device) equals the step at which single steps first fail, with the pencil (N = 16)
    and the TMA (N = 64) x inverse."""
    import re
    from gen import Patch, STRETCH1
    X = np.array([[0.5, 0.5, 0.5], [0.52, 0.5, 0.5]])

    def make(c):
        c.set_structure(X, [Patch(0, 2, 1, STRETCH1, 0)], np.array([1e30, 0, 1e-6, 0]))

    with ibm.IBContext(N, 1 / N, 1, 0.01, 1e-3) as c:
        make(c)
        with pytest.raises(ibm.IBError) as e:
            c.step(50)
        assert e.value.code == ibm.IB_ENONFINITE
        first_graph = int(re.search(r"first at step (\d+)", str(e.value)).group(1))
    with ibm.IBContext(N, 1 / N, 1, 0.01, 1e-3) as c:
        make(c)
        first_single = None
        for k in range(50):
            try:
                c.step(1)
            except ibm.IBError as e1:
                assert e1.code == ibm.IB_ENONFINITE
                first_single = int(re.search(r"first at step (\d+)", str(e1)).group(1))
                assert first_single == k
                break
    assert first_single is not None and first_graph == first_single


def test_empty_structure_and_smallest_grid(ibm, olib):
    with ibm.IBContext(8, 1 / 8, 1.0, 0.1, 1e-2) as c:
        c.step(2)
        u, _ = c.get_fields()
        assert np.max(np.abs(u)) == 0.0
        assert c.get_positions().shape == (0, 3)


@pytest.mark.parametrize("k", [1, 2, 3, 4, 5])
def test_config_full_length_stays_finite_and_bounded(ibm, k):
    """Each BASELINE.json config for its stated step count (10/100/400/200/50) on the GPU:
    ib_step reports no non-finite state, and velocity / displacement stay bounded."""
    cfg = make_config(k)
    with ibm.IBContext.from_config(cfg) as c:
        c.step(cfg.steps)
        assert c.n == cfg.steps
        u, _ = c.get_fields()
        X = c.get_positions()
    assert np.isfinite(u).all() and np.isfinite(X).all()
    umax = float(np.max(np.abs(u)))
    dmax = float(np.max(np.abs(X - cfg.X)))
    print(f"cfg{k}: {cfg.steps} steps, max|u| {umax:.3e}, max|X-X0| {dmax:.3e}")
    assert umax < 100.0 and dmax < 0.5 * cfg.N * cfg.h


# ---------------------------------------------------------------- anisotropic lattices
# N1 x N2 x N3 boxes such as the paper's 256 x 256 x 128 half-cube
# (PAPER.md 1003-1007).  Shapes mix the TMA column passes (pencil >= 64) with the cp.async
# pencil kernels (pencil < 64) on each axis.
ANISO = [(32, 64, 16), (64, 32, 128), (16, 16, 64), (128, 64, 32),
         (512, 16, 8), (256, 8, 64), (256, 64, 256)]   # 512-wide x rows (two TMA boxes), tuned group counts


@pytest.mark.parametrize("shape", [(256, 64, 256), (128, 128, 128), (64, 64, 64)])
def test_column_pass_rings_repeatable(ibm, shape):
    """Regression for the ring-ownership rule of the TMA column passes (fluid_tma.cu ColCfg):
    with more consumer groups than stages divide, a group could pass a stage's mbarrier
    parity test one phase early (about 1 run in 60 faulted or went wrong on 256x64x256).
    The forward passes (x, y, z) and the product inverse passes (z, y, x) run 50 times each;
    they have no atomics, so every repeat must be bitwise identical to the first run, which
    matches numpy's FFT."""
    n1, n2, n3 = shape
    x = np.random.default_rng(5).standard_normal((n3, n2, n1))
    ref = np.fft.rfftn(x)
    with ibm.IBContext(shape, 1.0 / n1, 1.0, 0.01, 1e-3) as c:
        f0 = c.debug_fft(x)
        i0 = c.debug_ifft(ref)
        assert rel_l2(f0, ref) < 1e-13
        assert rel_l2(i0, x * (n1 * n2 * n3)) < 1e-13
        for _ in range(50):
            assert np.array_equal(c.debug_fft(x), f0)
            assert np.array_equal(c.debug_ifft(ref), i0)


@pytest.mark.slow
@pytest.mark.parametrize("shape", [(256, 64, 256), (128, 128, 128), (64, 64, 64), (512, 16, 8)])
def test_tma_rings_stress(ibm, olib, shape):
    """Every TMA ring of the fluid step under repetition: the whole
    fluid solve (x forward, y forward, z forward + solve + z inverse, y inverse, x inverse
    through ib_debug_fluid) 500 times on the multi-group shapes.  The passes are
    deterministic, so every repeat must reproduce the first result bit for bit; the first
    result matches the oracle's fluid step."""
    n1, n2, n3 = shape
    rng = np.random.default_rng(51)
    u = rng.standard_normal((3, n3, n2, n1))
    F = rng.standard_normal((3, n3, n2, n1)) * 10
    h, rho, mu, dt = 1.0 / n1, 1.0, 0.02, 1e-3
    with ibm.IBContext(shape, h, rho, mu, dt) as c:
        u0, p0 = c.debug_fluid(u, F)
        ref_u, _ = olib.fluid_step(shape, h, rho, mu, dt, u, F, want_p=False)
        assert rel_l2(u0, ref_u) < 1e-13
        for _ in range(500):
            un, pn = c.debug_fluid(u, F)
            assert np.array_equal(un, u0) and np.array_equal(pn, p0)


@pytest.mark.parametrize("shape", ANISO)
def test_fft_anisotropic(ibm, shape):
    n1, n2, n3 = shape
    x = np.random.default_rng(n1 + n2 + n3).standard_normal((n3, n2, n1))
    with ibm.IBContext(shape, 1.0 / n1, 1.0, 0.01, 1e-3) as c:
        got = c.debug_fft(x)
    ref = np.fft.rfftn(x)
    assert got.shape == ref.shape
    assert np.max(np.abs(got - ref)) < 1e-13 * np.max(np.abs(ref)) * np.log2(n1 * n2 * n3)


@pytest.mark.parametrize("shape", ANISO)
def test_fluid_step_anisotropic(ibm, olib, shape):
    n1, n2, n3 = shape
    rng = np.random.default_rng(31)
    h = 1.0 / n1
    u = random_divfree_velocity(shape, 3, 0.3, rng) + 0.05 * rng.standard_normal((3, n3, n2, n1))
    F = rng.standard_normal((3, n3, n2, n1)) * 50
    rho, mu, dt = 1.0, 0.02, 1e-3
    with ibm.IBContext(shape, h, rho, mu, dt) as c:
        un, p = c.debug_fluid(u, F)
        r = c.debug_rhs(u, F)
    ref_u, ref_p = olib.fluid_step(shape, h, rho, mu, dt, u, F)
    assert rel_l2(r, olib.rhs(shape, h, rho, dt, u, F)) < 1e-14
    assert rel_l2(un, ref_u) < 1e-13
    assert rel_l2(p, ref_p) < 1e-12


@pytest.mark.parametrize("shape", [(32, 64, 16), (64, 32, 128)])
def test_spread_interp_anisotropic(ibm, olib, shape):
    n1, n2, n3 = shape
    h = 1.0 / n1
    rng = np.random.default_rng(32)
    L = np.array(shape) * h
    centres = rng.uniform(-0.2, 1.2, (60, 3)) * L
    X = centres[rng.integers(0, 60, 6000)] + rng.uniform(0, 0.4 * h, (6000, 3))
    f = rng.standard_normal((6000, 3))
    u = rng.standard_normal((3, n3, n2, n1))
    patches, st = _points_only(X)
    with ibm.IBContext(shape, h, 1.0, 0.01, 1e-3) as c:
        c.set_structure(X, patches, st)
        F = c.debug_spread(f)
        U = c.debug_interp(u)
    assert rel_l2(F, olib.spread(shape, h, X, f)) < 1e-13
    assert rel_l2(U, olib.interp(shape, h, u, X)) < 1e-14


@pytest.mark.parametrize("shape", [(32, 64, 16), (64, 64, 128)])
def test_step_parity_anisotropic_with_pressure_every_step(ibm, olib, shape):
    """Full IB steps on an anisotropic box (sheet with all link families, tethers, drive,
    flow), and the pressure of EVERY step: ib_step(1) + ib_get_fields(p) per step against
    the oracle's per-step pressure history."""
    cfg = small_sheet_config(N=shape, n1=20, n2=14, seed=33, u_amp=0.2)
    o = olib.Oracle.from_config(cfg)
    with ibm.IBContext.from_config(cfg) as c:
        c.set_option(ibm.IB_OPT_PRESSURE, 1)
        ps = []
        for _ in range(4):
            c.step(1)
            ps.append(c.get_fields(want_p=True)[1])
        o.step(4, p_every=True)
        ug, _ = c.get_fields()
        Xg = c.get_positions()
    assert rel_l2(ug, o.u) < 1e-11 and rel_l2(Xg, o.X) < 1e-11
    for k in range(4):
        assert rel_l2(ps[k], o.p_steps[k]) < 1e-10, k


@pytest.mark.slow
def test_halfcube_step_parity(ibm, olib):
    """The 256 x 256 x 128 half-cube workload (gen make_config("4h")): checkpoints 1, 2, 10."""
    print(_parity(ibm, olib, make_config("4h")))


# ---------------------------------------------------------------- window plates
@pytest.mark.parametrize("N", [32, (32, 64, 16)])
def test_window_plate_parity(ibm, olib, N):
    """Fixed rim points (never move, bitwise) + surface-normal sinusoidal drive on the free
    disc (PAPER.md 914-922, 988-993) against the oracle after 1 and 10 steps."""
    from gen import window_config
    cfg = window_config(N=N, m=24, seed=7, u_amp=0.05)
    print(_parity(ibm, olib, cfg))
    with ibm.IBContext.from_config(cfg) as c:
        c.step(10)
        X = c.get_positions()
        f = c.debug_force()
    fixed = cfg.fixed.astype(bool)
    assert np.array_equal(X[fixed], cfg.X[fixed])
    ref = olib.force(X, cfg.patches, cfg.stiffness, 10, cfg.drive_idx, None, cfg.drive_amp,
                     cfg.drive_period)
    assert rel_l2(f, ref) < 1e-13


def test_normal_drive_rejects_a_line_patch(ibm):
    from gen import Patch, STRETCH1
    X = np.array([[0.5, 0.5, 0.5], [0.52, 0.5, 0.5], [0.54, 0.5, 0.5]])
    with ibm.IBContext(16, 1 / 16, 1, 0.01, 1e-3) as c:
        c.set_structure(X, [Patch(0, 3, 1, STRETCH1, 0)], np.array([1.0, 1.0, 0.0, 0.02, 0.02, 0.0]))
        with pytest.raises(ibm.IBError) as e:
            c.set_drive(np.array([1]), None, 1e-3, 8)
        assert e.value.code == ibm.IB_EINVAL


# ---------------------------------------------------------------- experiments
def test_linearity_experiment_on_the_strip(ibm):
    """PAPER.md 1080-1085: in the linear regime a 10x drive gives 10x the membrane response.
    cfg3's strip driven with total amplitude 1e-7 vs 1e-6 for 200 steps: the centre-line
    envelopes agree with the scale to 1 % wherever the base envelope exceeds 1 % of its peak."""
    from paper_math_0301321_b200 import experiments as ex
    base = make_config(3)
    base.drive_amp = 1e-7 / base.drive_idx.size
    s, ea, _ = ex.run_replica(ex._scaled(base, 1.0), 200, 10)
    _, eb, _ = ex.run_replica(ex._scaled(base, 10.0), 200, 10)
    rep = ex.linearity(ea, eb, 10.0)
    print(rep, ea.max())
    assert ea.max() > 0 and rep["stations"] > 10
    assert rep["max_dev"] <= 0.01


@pytest.mark.parametrize("shape", [64, (16, 16, 64), (64, 32, 128)])
def test_project_alone_matches_oracle_solve(ibm, olib, shape):
    """S3c in isolation (ib_debug_project): the GPU's per-mode solve of r^ = rfftn(r) against
    rfftn of the oracle's solve of r (numpy's FFT as a library step)."""
    n1, n2, n3 = (shape,) * 3 if isinstance(shape, int) else shape
    r = np.random.default_rng(41).standard_normal((3, n3, n2, n1))
    h, rho, mu, dt = 1.0 / n1, 1.2, 0.03, 2e-3
    with ibm.IBContext(shape, h, rho, mu, dt) as c:
        uh, ph = c.debug_project(np.fft.rfftn(r, axes=(1, 2, 3)))
    u, p = olib.solve(shape, h, rho, mu, dt, r)
    assert rel_l2(uh, np.fft.rfftn(u, axes=(1, 2, 3))) < 1e-13
    assert rel_l2(ph, np.fft.rfftn(p)) < 1e-12


@pytest.mark.parametrize("shape", [64, (32, 64, 128), (256, 64, 64)])
def test_inverse_fft_alone(ibm, olib, shape):
    """S3d in isolation (ib_debug_ifft): the product inverse passes on X = rfftn(x) give the
    unnormalised inverse V x; cross-checked against the oracle's radix-2 FFT on the full
    Hermitian spectrum."""
    n1, n2, n3 = (shape,) * 3 if isinstance(shape, int) else shape
    x = np.random.default_rng(43).standard_normal((n3, n2, n1))
    X = np.fft.rfftn(x)
    with ibm.IBContext(shape, 1.0 / n1, 1.0, 0.01, 1e-3) as c:
        got = c.debug_ifft(X)
    V = n1 * n2 * n3
    assert rel_l2(got, V * x) < 1e-14 * np.log2(V)
    if V <= 64 ** 3:
        full = np.fft.fftn(x)
        assert rel_l2(got, olib.fft3(full, +1).real) < 1e-14 * np.log2(V)


def test_checkpoint_resume_matches_straight_run(ibm):
    """the state is (u, X, n); saving it with ib_get_fields/positions/step and
    restoring it in a fresh context with ib_set_velocity/structure/step resumes the run (to
    the fp64 atomic-order tolerance, not bitwise)."""
    cfg = small_sheet_config(N=32, n1=20, n2=14, seed=44, u_amp=0.2)
    with ibm.IBContext.from_config(cfg) as a:
        a.step(10)
        u_ref, _ = a.get_fields()
        X_ref = a.get_positions()
    with ibm.IBContext.from_config(cfg) as b:
        b.step(4)
        u4, _ = b.get_fields()
        X4 = b.get_positions()
        n4 = b.n
    with ibm.IBContext.from_config(cfg) as r:       # fresh context, restored state
        r.set_structure(X4, cfg.patches, cfg.stiffness)
        r.set_drive(cfg.drive_idx, cfg.drive_dir, cfg.drive_amp, cfg.drive_period)
        r.set_velocity(u4)
        r.set_step(n4)
        r.step(6)
        assert r.n == 10
        u, _ = r.get_fields()
        X = r.get_positions()
    assert rel_l2(u, u_ref) < 1e-12 and rel_l2(X - cfg.X, X_ref - cfg.X) < 1e-10


@pytest.mark.slow
def test_strip_experiment_observables_match_oracle(ibm, olib):
    """SURVEY 8(f) row 3 against the oracle: the cfg3 strip driven for 100 steps (period 50,
    total drive 1e-3 as BASELINE.json configs[2]) on the GPU and on the oracle, the centre-line
    normal displacement (experiments.centerline) compared station by station every 10 steps
    (max |d_gpu - d_oracle| <= 1e-9 max |d_oracle|), then the envelopes and their peak."""
    from paper_math_0301321_b200 import experiments as ex
    cfg = ex._scaled(make_config(3), 1.0, 50)
    rows, _ = ex.strip_rows(cfg)
    s, n = ex.rest_frame(cfg)
    X0 = cfg.X.copy()
    o = olib.Oracle.from_config(cfg)
    pg, po = [], []
    with ibm.IBContext.from_config(cfg) as c:
        for _ in range(10):
            c.step(10)
            o.step(10)
            dg = ex.centerline(c.get_positions(), X0, rows, n)
            do = ex.centerline(o.get_positions(), X0, rows, n)
            assert np.max(np.abs(dg - do)) <= 1e-9 * np.max(np.abs(do)), c.n
            pg.append(dg)
            po.append(do)
    eg, eo = ex.envelope(pg), ex.envelope(po)
    assert eo.max() > 0
    assert np.max(np.abs(eg - eo)) <= 1e-9 * eo.max()
    assert ex.peak_location(eg, s) == ex.peak_location(eo, s)


def test_spread_interp_degenerate_positions(ibm, olib):
    """Points exactly on lattice nodes, on cell faces and edges (floor(X/h) exact, the window
    j0 = floor - 1 .. + 2 with phi(+-2) = 0 at its ends, reading Z8), exactly on
    the periodic boundary, negative and far outside the box (indices mod N), and many
    points coinciding: spread and interpolation against the oracle, plus adjointness."""
    N = 32
    h = 1.0 / N
    rng = np.random.default_rng(71)
    nodes = rng.integers(-3 * N, 4 * N, (200, 3)) * h                 # on nodes, any period
    faces = rng.integers(0, N, (200, 3)) * h
    faces[:, 0] += 0.5 * h                                              # x between nodes
    edges = np.array([[0.0, 0.0, 0.0], [1.0, 1.0, 1.0], [1.0 - 1e-16, 0.5, 0.5],
                      [-1e-300, 0.25, 0.75], [31 * h, 31 * h, 31 * h], [-h, -h, -h]])
    same = np.tile([[0.4375, 0.5, 0.53125]], (70, 1))                  # 70 coincident points
    X = np.ascontiguousarray(np.concatenate([nodes, faces, edges, same]))
    f = rng.standard_normal(X.shape)
    u = rng.standard_normal((3, N, N, N))
    patches, st = _points_only(X)
    with _ctx(ibm, N, X=X, patches=patches, stiff=st) as c:
        F = c.debug_spread(f)
        U = c.debug_interp(u)
    Fo = olib.spread(N, h, X, f)
    Uo = olib.interp(N, h, u, X)
    assert rel_l2(F, Fo) < 1e-13
    assert np.max(np.abs(U - Uo)) <= 1e-13 * np.max(np.abs(Uo))
    assert abs(np.sum(F * u) * h ** 3 - np.sum(f * U)) <= 1e-12 * np.sum(np.abs(f * U))


@pytest.mark.parametrize("shape", [(64, 64, 512), (128, 64, 512), (64, 512, 64)])
def test_z512_column_passes(ibm, olib, shape):
    """512-long z (and y) pencils: the 3-pass plan whose radix-2 first pass is folded into
    the second pass's loads (fluid_tma.cu fft_inplace): forward FFT vs numpy, the fluid step
    vs the oracle, and the per-mode solve alone (S3c) vs the oracle's solve."""
    n1, n2, n3 = shape
    rng = np.random.default_rng(81)
    x = rng.standard_normal((n3, n2, n1))
    h, rho, mu, dt = 1.0 / n1, 1.0, 0.02, 1e-3
    u = random_divfree_velocity(shape, 3, 0.3, rng) + 0.05 * rng.standard_normal((3, n3, n2, n1))
    F = rng.standard_normal((3, n3, n2, n1)) * 50
    with ibm.IBContext(shape, h, rho, mu, dt) as c:
        got = c.debug_fft(x)
        un, p = c.debug_fluid(u, F)
        r = rng.standard_normal((3, n3, n2, n1))
        uh, ph = c.debug_project(np.fft.rfftn(r, axes=(1, 2, 3)))
        for _ in range(20):                           # deterministic passes: bitwise repeats
            assert np.array_equal(c.debug_fft(x), got)
    ref = np.fft.rfftn(x)
    assert np.max(np.abs(got - ref)) < 1e-13 * np.max(np.abs(ref)) * np.log2(x.size)
    ref_u, ref_p = olib.fluid_step(shape, h, rho, mu, dt, u, F)
    assert rel_l2(un, ref_u) < 1e-13 and rel_l2(p, ref_p) < 1e-12
    us, ps = olib.solve(shape, h, rho, mu, dt, r)
    assert rel_l2(uh, np.fft.rfftn(us, axes=(1, 2, 3))) < 1e-13
