"""Analysis functions of the linearity / frequency-sweep experiments (
SPEC.md 413-450 examples), CPU only; the GPU replicas are exercised in test_gpu_parity.py."""
import numpy as np
import pytest

from paper_math_0301321_b200 import experiments as ex
from gen import make_config


def test_centerline_rest_and_uniform_normal_offset():
    cfg = make_config(3)
    rows, n1 = ex.strip_rows(cfg)
    s, n = ex.rest_frame(cfg)
    assert rows.size == n1 == s.size and np.all(np.diff(s) > 0)
    assert np.allclose(np.linalg.norm(n, axis=1), 1.0)
    assert np.max(np.abs(ex.centerline(cfg.X, cfg.X, rows, n))) == 0.0       # rest -> 0
    X = cfg.X.copy()
    X[rows] += 2e-4 * n                                                       # offset delta
    assert np.allclose(ex.centerline(X, cfg.X, rows, n), 2e-4, rtol=0, atol=1e-15)


def test_envelope_of_a_standing_wave_and_window_monotonicity():
    s = np.linspace(0, 3, 200)
    snaps = [np.sin(s) * np.cos(w) for w in np.linspace(0, 2 * np.pi, 400)]
    env = ex.envelope(snaps)
    assert np.max(np.abs(env - np.abs(np.sin(s)))) <= 0.02
    assert np.all(ex.envelope(snaps[:100]) <= env)                  # widening never decreases
    assert np.array_equal(ex.envelope(snaps[:1]), np.abs(snaps[0]))


def test_peak_location_and_tie_rule():
    st = np.linspace(0, 1, 11)
    assert ex.peak_location(np.exp(-((st - 0.3) / 0.1) ** 2), st) == pytest.approx(0.3)
    two = np.zeros(11); two[2] = two[7] = 1.0
    assert ex.peak_location(two, st) == pytest.approx(0.2)
    assert ex.peak_location(np.arange(11.0), st) == pytest.approx(1.0)


def test_linearity_report():
    rng = np.random.default_rng(0)
    a = rng.uniform(0.0, 1.0, 50)
    assert ex.linearity(a, a, 1.0)["max_dev"] == 0.0
    assert ex.linearity(a, 10 * a, 10.0)["max_dev"] < 1e-15
    assert ex.linearity(a, 11 * a, 10.0)["max_dev"] == pytest.approx(0.1)
