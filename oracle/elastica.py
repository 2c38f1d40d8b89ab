"""Planar elastica of the gravity-loaded cantilever (§4.1; Bickley 1934 / Shield 1992
as cited there) -- the analytical master curve of SURVEY.md §8(f) N2.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

The boundary value problem, in the paper's notation (s = s/L, (x, y) = (x/L, y/L)):

    theta''(s) + Gamma (1 - s) cos theta = 0,   theta(0) = 0,  theta'(1) = 0,
    x'(s) = cos theta,  x(0) = 0,     y'(s) = sin theta,  y(0) = 0,

with Gamma = Gamma*_gb = rho A* g L^3 / (D w).  theta is the slope angle measured
from the undeformed (horizontal) axis towards the load, so y is the deflection in the direction of g.

Solved by shooting: for a trial root curvature k = theta'(0) the initial value problem is integrated
with the classical fourth-order Runge-Kutta method on a uniform grid of n steps, and k is found by
bisection on theta'(1) = 0.  theta'(1) is increasing in k (a stiffer root bends more at the tip side),
which brackets the root in [0, Gamma / 2 * max(1, ...)]: the linear solution has k = Gamma / 2 and
the cos theta <= 1 factor only lowers the load, so k in [0, Gamma / 2].
"""
from __future__ import annotations

import math


def _rhs(s, th, dth, gamma):
    # (theta, theta', x, y)' = (theta', -Gamma (1 - s) cos theta, cos theta, sin theta)
    return dth, -gamma * (1.0 - s) * math.cos(th), math.cos(th), math.sin(th)


def integrate(gamma: float, k0: float, n: int = 2000):
    """RK4 from s = 0 to 1 with theta(0) = 0, theta'(0) = k0.  Returns (theta(1), theta'(1), x(1), y(1))."""
    h = 1.0 / n
    th, dth, x, y = 0.0, k0, 0.0, 0.0
    for i in range(n):
        s = i * h
        a1 = _rhs(s, th, dth, gamma)
        a2 = _rhs(s + 0.5 * h, th + 0.5 * h * a1[0], dth + 0.5 * h * a1[1], gamma)
        a3 = _rhs(s + 0.5 * h, th + 0.5 * h * a2[0], dth + 0.5 * h * a2[1], gamma)
        a4 = _rhs(s + h, th + h * a3[0], dth + h * a3[1], gamma)
        th += h / 6.0 * (a1[0] + 2 * a2[0] + 2 * a3[0] + a4[0])
        dth += h / 6.0 * (a1[1] + 2 * a2[1] + 2 * a3[1] + a4[1])
        x += h / 6.0 * (a1[2] + 2 * a2[2] + 2 * a3[2] + a4[2])
        y += h / 6.0 * (a1[3] + 2 * a2[3] + 2 * a3[3] + a4[3])
    return th, dth, x, y


def solve(gamma: float, n: int = 2000, tol: float = 1e-14):
    """Equilibrium of the elastica for load parameter Gamma >= 0.  Returns a dict with the root
    curvature k = theta'(0), the tip slope theta(1), the tip position (x(1), y(1)) and the aspect
    ratio H / W = y(1) / x(1) of the deformed shape ("the aspect ratio H/W")."""
    if gamma == 0.0:
        return {"gamma": 0.0, "k0": 0.0, "theta_tip": 0.0, "x_tip": 1.0, "y_tip": 0.0, "HW": 0.0}
    lo, hi = 0.0, 0.5 * gamma
    # theta'(1; k) is increasing in k: theta'(1; 0) < 0 (the load bends the beam back), theta'(1; G/2) >= 0
    f_lo = integrate(gamma, lo, n)[1]
    f_hi = integrate(gamma, hi, n)[1]
    if not (f_lo <= 0.0 <= f_hi):
        raise RuntimeError(f"elastica: root not bracketed for Gamma = {gamma} ({f_lo}, {f_hi})")
    for _ in range(200):
        mid = 0.5 * (lo + hi)
        f = integrate(gamma, mid, n)[1]
        if f < 0.0:
            lo = mid
        else:
            hi = mid
        if hi - lo <= tol * max(1.0, hi):
            break
    k = 0.5 * (lo + hi)
    th, dth, x, y = integrate(gamma, k, n)
    return {"gamma": gamma, "k0": k, "theta_tip": th, "x_tip": x, "y_tip": y, "HW": y / x if x > 0 else math.inf}


def gamma_of(E: float, nu: float, rho: float, g: float, L: float, h: float) -> float:
    """Gamma*_gb = rho A* g L^3 / (D w) with A* = w h and D = E h^3 / (12 (1 - nu^2));
    the width w cancels (plane strain, unit depth)."""
    D = E * h ** 3 / (12.0 * (1.0 - nu * nu))
    return rho * h * g * L ** 3 / D


def g_for_gamma(gamma: float, E: float, nu: float, rho: float, L: float, h: float) -> float:
    return gamma / gamma_of(E, nu, rho, 1.0, L, h)
