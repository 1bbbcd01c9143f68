"""Generator self-checks (input recipe) and oracle thread invariance."""
import numpy as np
import pytest

from gen import make_config, random_divfree_velocity


@pytest.mark.parametrize("k,np_,N", [(1, 2304, 32), (2, 32768, 64), (3, 65536, 128),
                                     (4, 2097152, 256)])
def test_config_counts(k, np_, N):
    cfg = make_config(k)
    assert cfg.X.shape == (np_, 3) and cfg.N == N and cfg.h == 1.0 / N
    assert np.isfinite(cfg.X).all() and np.isfinite(cfg.stiffness).all()
    last = cfg.patches[-1]
    assert last.first + last.n1 * last.n2 == np_
    if k >= 3:
        assert cfg.drive_idx.size == {3: 32, 4: 64}[k]
        assert abs(cfg.drive_amp * cfg.drive_idx.size - 1e-3) < 1e-18


def test_divfree_velocity_recipe():
    N = 32
    u = random_divfree_velocity(N, 4, 0.01, np.random.default_rng(7))
    inv2h = N / 2.0
    d0 = lambda f, a: (np.roll(f, -1, a) - np.roll(f, 1, a)) * inv2h
    div = d0(u[0], 2) + d0(u[1], 1) + d0(u[2], 0)
    assert np.max(np.abs(div)) < 1e-15 * N * 10
    assert abs(np.sqrt(np.mean(np.sum(u * u, 0))) - 0.01) < 1e-15
    # band-limited: no energy above |k| = 4 (plus the curl's own symbol)
    spec = np.abs(np.fft.fftn(u[0]))
    k = np.fft.fftfreq(N, 1.0 / N)
    kk = k[:, None, None] ** 2 + k[None, :, None] ** 2 + k[None, None, :] ** 2
    assert spec[kk > 16].max() < 1e-12 * spec.max()


def test_cfg4_tether_stiffness_density_reading():
    cfg = make_config(4)
    wall = cfg.patches[1]
    npts = wall.n1 * wall.n2
    kt = cfg.stiffness[wall.param_off:wall.param_off + npts]
    # reading Z1: kt = 1e4 * dA, dA ~ (0.05-0.17 h) x 0.38 h  -> mean ~ 6e-3
    assert 1e-3 < kt.mean() < 2e-2 and kt.min() > 0


def test_oracle_thread_count_invariance(olib):
    cfg = make_config(1)
    outs = []
    for t in (1, 3):
        olib.set_threads(t)
        o = olib.Oracle.from_config(cfg)
        o.step(2)
        outs.append((o.get_fields()[0], o.get_positions()))
    olib.set_threads(1)
    assert np.array_equal(outs[0][0], outs[1][0]) and np.array_equal(outs[0][1], outs[1][1])
