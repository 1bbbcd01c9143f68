"""Shared GPU-vs-oracle comparison of whole IB steps (tests only)."""
import numpy as np


def rel_l2(a, b):
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    nb = np.linalg.norm(b)
    na = np.linalg.norm(a - b)
    if nb == 0.0:
        return 0.0 if na == 0.0 else np.inf
    return na / nb


def _max_rel(a, b, scale):
    """max |a - b| / scale (element-wise check beside the rel-L2 norms)."""
    d = float(np.max(np.abs(np.asarray(a) - np.asarray(b)))) if np.size(b) else 0.0
    if scale == 0.0:
        return 0.0 if d == 0.0 else np.inf
    return d / scale


def step_parity(olib, cfg, make_gpu, steps=(1, 1, 8), tol=(1e-11, 1e-11, 1e-9), elem=1e-10,
                check_U=True):
    """GPU vs oracle after each batch of `steps` (checkpoints 1, 2 and 10 by default).

    At every checkpoint, on the same seeded inputs (BASELINE.json north_star tolerances;
    DESIGN.md reading Z4):
      u        rel-L2 <= tol, and element-wise max|du| <= elem * max|u|
      X        rel-L2 <= tol
      X - X0   rel-L2 <= max(tol, 10 * fp64 floor) (floor ~ 8 ulp(max|X0|)/rms|X - X0|), and
               element-wise max|d(X - X0)| <= elem * max|X - X0| + 8 ulp(max|X0|)
      U        the interpolated velocity at the checkpoint's positions (ib_debug_interp vs the
               oracle's interp), rel-L2 <= min(tol, 1e-11) and element-wise <= elem * max|U|
    Checkpoints where both sides are exactly at rest (cfg3/cfg4 step 1: zero drive at t = 0)
    compare 0 with 0 and pass; the step-2 checkpoint is the first non-trivial one there."""
    o = olib.Oracle.from_config(cfg)
    c = make_gpu()
    X0 = cfg.X.copy()
    ulp0 = np.spacing(np.max(np.abs(X0))) if X0.size else 0.0
    report = []
    done = 0
    for k, t in zip(steps, tol):
        o.step(k)
        c.step(k)
        done += k
        uo, _ = o.get_fields()
        ug, _ = c.get_fields()
        Xo, Xg = o.get_positions(), c.get_positions()
        e_u, e_X = rel_l2(ug, uo), rel_l2(Xg, Xo)
        e_d = rel_l2(Xg - X0, Xo - X0)
        m_u = _max_rel(ug, uo, float(np.max(np.abs(uo))))
        dd = Xo - X0
        m_d = float(np.max(np.abs((Xg - X0) - dd))) if dd.size else 0.0
        if check_U and X0.size:
            Ug = c.debug_interp(ug)
            Uo = olib.interp(cfg.N, cfg.h, uo, Xo)
            e_U = rel_l2(Ug, Uo)
            m_U = _max_rel(Ug, Uo, float(np.max(np.abs(Uo))))
        else:
            e_U = m_U = 0.0
        report.append({"cfg": cfg.name, "step": done, "u": e_u, "u_max": m_u, "X": e_X, "X-X0": e_d,
                       "U": e_U, "U_max": m_U})
        assert e_u <= t, (cfg.name, done, "u", e_u)
        assert m_u <= elem, (cfg.name, done, "u element-wise", m_u)
        assert e_X <= t, (cfg.name, done, "X", e_X)
        disp = np.sqrt(np.mean(dd ** 2)) if dd.size else 0.0
        floor = 8 * ulp0 / disp if disp > 0 else 0.0
        assert e_d <= max(t, 10 * floor), (cfg.name, done, "X-X0", e_d, floor)
        assert m_d <= elem * (float(np.max(np.abs(dd))) if dd.size else 0.0) + 8 * ulp0, \
            (cfg.name, done, "X-X0 element-wise", m_d)
        assert e_U <= min(t, 1e-11), (cfg.name, done, "U", e_U)
        assert m_U <= elem, (cfg.name, done, "U element-wise", m_U)
        assert c.n == o.n == done
    c.close()
    return report
