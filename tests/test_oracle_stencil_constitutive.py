"""Pins of oracle O1 (quadratic B-spline stencil) and O3 (Neo-Hookean) against closed forms,
golden values and invariants (§8(c).3b G1, G3-G5)."""
import numpy as np
import pytest

import oracle
import synth
from conftest import read_golden


def test_g1_bspline_weights_golden():
    for f, w0, w1, w2, d0, d1, d2 in read_golden("g1_bspline_weights.txt"):
        w, dw = oracle.bspline1(f, dx=0.5)
        np.testing.assert_allclose(w, [w0, w1, w2], rtol=0, atol=1e-15)
        np.testing.assert_allclose(dw * 0.5, [d0, d1, d2], rtol=0, atol=1e-15)


@pytest.mark.parametrize("dim", [2, 3])
def test_knot_weights(dim):
    # particle exactly on a node: per-axis (1/8, 3/4, 1/8); centre 9/16 (2D), 27/64 (3D)
    grid = synth.Grid(dim, (0.0, 0.0, 0.0), 0.1, (10, 10, 10 if dim == 3 else 1))
    x = np.full(dim, 0.5)
    idx, N, gN, xip = oracle.stencil(grid, x)
    assert len(N) == 3 ** dim
    centre = np.argmin(np.abs(xip).sum(axis=1))
    assert N[centre] == pytest.approx((3 / 4) ** dim, abs=1e-15)
    assert N.max() == N[centre]
    assert sorted(set(np.round(N, 15)))[0] == pytest.approx((1 / 8) ** dim, abs=1e-15)


@pytest.mark.parametrize("dim", [2, 3])
def test_partition_of_unity_and_linear_completeness(dim):
    # Σ N = 1; Σ N x_i = x; Σ N (x_i-x)(x_i-x)^T = dx^2/4 I; Σ ∇N = 0; Σ x_i ∇N^T = I  (App. B.1)
    rng = np.random.default_rng(7)
    dx = 0.037
    grid = synth.Grid(dim, (-0.3, 0.1, 0.2), dx, (40, 40, 40 if dim == 3 else 1))
    worst = 0.0
    for _ in range(500):
        x = np.asarray(grid.origin[:dim]) + rng.uniform(2.0, 37.0, size=dim) * dx
        idx, N, gN, xip = oracle.stencil(grid, x)
        xi = xip + x
        assert (N >= 0).all()
        checks = [
            (N.sum() - 1.0),
            np.abs(N @ xi - x).max() / dx,
            np.abs((xip.T * N) @ xip - dx * dx / 4 * np.eye(dim)).max() / dx ** 2,
            np.abs(gN.sum(axis=0)).max() * dx,
            np.abs(xi.T @ gN - np.eye(dim)).max(),
        ]
        worst = max(worst, max(abs(c) for c in checks))
    assert worst < 1e-12


def test_out_of_domain():
    grid = synth.Grid(2, (0.0, 0.0, 0.0), 0.1, (10, 10, 1))
    assert oracle.stencil(grid, np.array([0.04, 0.5])) is None     # X = 0.4 -> base = -1
    assert oracle.stencil(grid, np.array([0.15, 0.5])) is not None  # base = 1
    assert oracle.stencil(grid, np.array([0.86, 0.5])) is None     # base + 2 = 10 > 9


def test_g3_lame_golden():
    (E, nu, mu, lam), = read_golden("g3_lame.txt")
    m, l = oracle.lame(E, nu)
    assert m == pytest.approx(mu, rel=1e-14)
    assert l == pytest.approx(lam, rel=1e-14)


@pytest.mark.parametrize("name,d", [("g4_neohookean_2d.txt", 2), ("g5_neohookean_3d.txt", 3)])
def test_neohookean_golden(name, d):
    rows = {r[0]: np.array(r[1:]) for r in read_golden(name)}
    mu, lam = oracle.lame(1e5, 0.3)
    F = rows["F"].reshape(d, d)
    dF = rows["dF"].reshape(d, d)
    assert oracle.psi(F, mu, lam) == pytest.approx(rows["Psi"][0], rel=1e-12)
    np.testing.assert_allclose(oracle.P(F, mu, lam).ravel(), rows["P"], rtol=1e-12, atol=1e-9)
    np.testing.assert_allclose(oracle.dP(F, dF, mu, lam).ravel(), rows["dP"], rtol=1e-12, atol=1e-9)


def _rot(d, rng):
    q, r = np.linalg.qr(rng.normal(size=(d, d)))
    q = q * np.sign(np.diag(r))
    if np.linalg.det(q) < 0:
        q[:, 0] *= -1
    return q


@pytest.mark.parametrize("d", [2, 3])
def test_neohookean_invariants_and_fd(d):
    rng = np.random.default_rng(3)
    mu, lam = oracle.lame(2e5, 0.35)
    I = np.eye(d)
    assert oracle.psi(I, mu, lam) == 0.0
    assert np.abs(oracle.P(I, mu, lam)).max() == 0.0
    R = _rot(d, rng)
    assert abs(oracle.psi(R, mu, lam)) < 1e-9 * mu
    # rotation invariance of Psi: Psi(RF) = Psi(F)
    F = I + rng.normal(0, 0.1, (d, d))
    assert oracle.psi(R @ F, mu, lam) == pytest.approx(oracle.psi(F, mu, lam), rel=1e-12)
    # inverted F -> +inf
    Finv = F.copy()
    Finv[0] *= -1
    if np.linalg.det(Finv) < 0:
        assert np.isinf(oracle.psi(Finv, mu, lam))
    # P = dPsi/dF by central differences
    h = 1e-6
    Pfd = np.zeros((d, d))
    for a in range(d):
        for b in range(d):
            E = np.zeros((d, d))
            E[a, b] = h
            Pfd[a, b] = (oracle.psi(F + E, mu, lam) - oracle.psi(F - E, mu, lam)) / (2 * h)
    Pa = oracle.P(F, mu, lam)
    assert np.abs(Pfd - Pa).max() / np.abs(Pa).max() < 1e-8
    # dP = dP/dF : dF by central differences
    dF = rng.normal(0, 1.0, (d, d))
    eps = 1e-6
    dPfd = (oracle.P(F + eps * dF, mu, lam) - oracle.P(F - eps * dF, mu, lam)) / (2 * eps)
    dPa = oracle.dP(F, dF, mu, lam)
    assert np.abs(dPfd - dPa).max() / np.abs(dPa).max() < 1e-8
    # bilinear symmetry: dF2 : dP(dF1) = dF1 : dP(dF2) (Hessian of Psi is symmetric)
    dF2 = rng.normal(0, 1.0, (d, d))
    s1 = (dF2 * oracle.dP(F, dF, mu, lam)).sum()
    s2 = (dF * oracle.dP(F, dF2, mu, lam)).sum()
    assert s1 == pytest.approx(s2, rel=1e-12)
    # at F = I: dP = mu (dF + dF^T) + lam tr(dF) I exactly
    lin = mu * (dF + dF.T) + lam * np.trace(dF) * I
    assert np.abs(oracle.dP(I, dF, mu, lam) - lin).max() <= 1e-12 * np.abs(lin).max()
