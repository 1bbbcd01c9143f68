"""Closed forms the tests pin the oracle (and the GPU path) to.  Written from the paper's
formulas, independently of oracle/ (no import of it): Peskin's phi in the alternative
closed form of its second branch (reading Z9), and the one-step solution of the
decaying shear mode.
"""
import numpy as np


def phi(r):
    """Peskin's 4-point function (PAPER.md 745-759), second branch in closed form:
    |r| <= 1: (3 - 2|r| + sqrt(1 + 4|r| - 4r^2))/8;  1 <= |r| <= 2: (5 - 2|r| -
    sqrt(-7 + 12|r| - 4r^2))/8;  0 beyond."""
    a = np.abs(np.asarray(r, dtype=np.float64))
    out = np.zeros_like(a)
    m1 = a <= 1.0
    m2 = (a > 1.0) & (a <= 2.0)
    out[m1] = (3.0 - 2.0 * a[m1] + np.sqrt(1.0 + 4.0 * a[m1] - 4.0 * a[m1] ** 2)) / 8.0
    out[m2] = (5.0 - 2.0 * a[m2] - np.sqrt(-7.0 + 12.0 * a[m2] - 4.0 * a[m2] ** 2)) / 8.0
    return out


def shear_gain(N2, h, rho, mu, dt, m):
    """Amplification g of the mode A sin(2 pi m y) e_x over one step of eq:discreteNS1-2
    with F = 0: advection vanishes (u_x is constant along x, u_y = u_z = 0), the projection
    is inactive (the D0 symbol along x is 0 for this mode), and the implicit viscous update
    (rho/dt - mu D+D-) u^{n+1} = rho u^n / dt gives g = (1 + mu dt 4 sin^2(pi m/N2)/(rho h^2))^-1."""
    return 1.0 / (1.0 + mu * dt * 4.0 * np.sin(np.pi * m / N2) ** 2 / (rho * h * h))


def shear_interp(Y, N2, h, m):
    """sum_b phi(j_b - Y/h) sin(2 pi m j_b / N2), j_b = floor(Y/h) - 1 + b, b = 0..3: the
    y part of interpolating sin(2 pi m y) at height Y (the x and z weights sum to 1)."""
    Y = np.asarray(Y, dtype=np.float64)
    j0 = np.floor(Y / h) - 1.0
    s = np.zeros_like(Y)
    for b in range(4):
        j = j0 + b
        s += phi(j - Y / h) * np.sin(2.0 * np.pi * m * (np.mod(j, N2)) / N2)
    return s


def shear_positions(cfg, steps):
    """X^n of free points in the decaying shear mode (eq:discreteX, PAPER.md 725-734):
    X_x^{k+1} = X_x^k + dt g^{k+1} A shear_interp(Y), i.e. u^{k+1} = g^{k+1} u^0 interpolated at
    X^k; Y and Z never change (u_y = u_z = 0)."""
    n2 = cfg.N if isinstance(cfg.N, int) else cfg.N[1]
    g = shear_gain(n2, cfg.h, cfg.rho, cfg.mu, cfg.dt, cfg.info["m"])
    X = cfg.X.copy()
    s = shear_interp(X[:, 1], n2, cfg.h, cfg.info["m"])
    for k in range(steps):
        X[:, 0] = X[:, 0] + cfg.dt * g ** (k + 1) * cfg.info["A"] * s
    return X, g
