"""Pins of oracle O2 (APIC P2G), O8 (G2P + F + advection), O9 (Π) and O10 (I + T) against
golden values, conservation laws and completeness identities (
G2)."""
import numpy as np
import pytest

import oracle
import synth
from conftest import read_golden


def _cross2(x, p):
    return x[..., 0] * p[..., 1] - x[..., 1] * p[..., 0]


def test_g2_single_particle_p2g_golden():
    grid = synth.Grid(2, (0.0, 0.0, 0.0), 0.1, (10, 10, 1))
    pt = synth.Particles(np.array([[0.23, 0.47]]), np.array([[1.0, -0.5]]), np.eye(2)[None].copy(),
                         np.array([[[0.001, 0.002], [-0.003, 0.0005]]]), np.array([2.0]), np.array([1e-3]),
                         np.zeros(1, np.int32), np.zeros(1, np.uint8))
    sc = synth.Scene(grid, pt, [(1e5, 0.3)], 1e-3)
    gs = oracle.p2g(sc)
    for i, j, m, px, py in read_golden("g2_p2g_single_particle.txt"):
        n = int(i) * 10 + int(j)
        assert gs.m[n] == pytest.approx(m, rel=1e-12)
        np.testing.assert_allclose(gs.p[n], [px, py], rtol=1e-12)
    assert gs.m.sum() == pytest.approx(2.0, rel=1e-14)
    np.testing.assert_allclose(gs.p.sum(axis=0), [2.0, -1.0], rtol=1e-14)
    k = np.stack(np.meshgrid(np.arange(10), np.arange(10), indexing="ij"), -1).reshape(-1, 2) * 0.1
    assert _cross2(k, gs.p).sum() == pytest.approx(-1.18, rel=1e-12)


def test_single_particle_at_node():
    # one particle on a node, v = (1, 0), B = 0 -> centre mass 9/16 m, all active v = (1, 0)
    grid = synth.Grid(2, (0.0, 0.0, 0.0), 0.1, (10, 10, 1))
    pt = synth.make_particles(np.array([[0.5, 0.5]]), 1e-2, 100.0)
    pt.v[:] = [1.0, 0.0]
    gs = oracle.p2g(synth.Scene(grid, pt, [(1e5, 0.3)], 1e-3))
    assert gs.m[55] == pytest.approx(9 / 16 * pt.m[0], rel=1e-15)
    act = gs.active.astype(bool)
    assert act.sum() == 9
    np.testing.assert_allclose(gs.v[act], np.tile([1.0, 0.0], (9, 1)), rtol=0, atol=1e-15)


@pytest.mark.parametrize("dim", [2, 3])
def test_p2g_conservation_and_angular_momentum(dim):
    sc = synth.random_fixture(dim=dim, seed=11, cells=(4, 3, 3))
    pt = sc.particles
    gs = oracle.p2g(sc)
    d = dim
    assert gs.m.sum() == pytest.approx(pt.m.sum(), rel=1e-14)
    np.testing.assert_allclose(gs.p.sum(axis=0), (pt.m[:, None] * pt.v).sum(axis=0), rtol=1e-13, atol=1e-14)
    # f_ext = m_i g  (partition of unity)
    np.testing.assert_allclose(gs.fext, gs.m[:, None] * np.asarray(sc.gravity[:d])[None], rtol=1e-15, atol=0)
    # node positions
    shp = oracle.node_shape(sc.grid)
    k = np.stack(np.meshgrid(*[np.arange(s) for s in shp], indexing="ij"), -1).reshape(-1, d)
    xi = np.asarray(sc.grid.origin[:d]) + k * sc.grid.dx
    # angular momentum (APIC exactness)
    if d == 2:
        Lg = _cross2(xi, gs.p).sum()
        Lp = (_cross2(pt.x, pt.m[:, None] * pt.v) + pt.m * (pt.B[:, 1, 0] - pt.B[:, 0, 1])).sum()
        assert Lg == pytest.approx(Lp, rel=1e-12)
    else:
        Lg = np.cross(xi, gs.p).sum(axis=0)
        Bt = pt.B
        extra = np.stack([Bt[:, 2, 1] - Bt[:, 1, 2], Bt[:, 0, 2] - Bt[:, 2, 0], Bt[:, 1, 0] - Bt[:, 0, 1]], -1)
        Lp = (np.cross(pt.x, pt.m[:, None] * pt.v) + pt.m[:, None] * extra).sum(axis=0)
        np.testing.assert_allclose(Lg, Lp, rtol=1e-12, atol=1e-13 * np.abs(Lp).max())
    # stress scatter: Σ f^σ = 0 and Σ f^σ ⊗ x_i = -Σ V0 P F^T (symmetric)
    assert np.abs(gs.fsig.sum(axis=0)).max() <= 1e-12 * np.abs(gs.fsig).max()
    M = gs.fsig.T @ xi
    tau = np.zeros((d, d))
    for p in range(pt.n):
        mu, lam = oracle.lame(*sc.materials[pt.mat[p]])
        tau += pt.V0[p] * oracle.P(pt.F[p], mu, lam) @ pt.F[p].T
    np.testing.assert_allclose(M, -tau, rtol=1e-11, atol=1e-12 * np.abs(tau).max())
    np.testing.assert_allclose(tau, tau.T, rtol=1e-10, atol=1e-12 * np.abs(tau).max())


@pytest.mark.parametrize("dim", [2, 3])
def test_apic_affine_round_trip(dim):
    # particles with v_p = A x_p + c, B_p = (dx^2/4) A transfer an exactly affine grid field
    sc = synth.random_fixture(dim=dim, seed=12, cells=(3, 3, 3))
    rng = np.random.default_rng(5)
    d = dim
    A = rng.normal(size=(d, d))
    c = rng.normal(size=d)
    pt = sc.particles
    pt.v = pt.x @ A.T + c
    pt.B = np.broadcast_to(sc.grid.dx ** 2 / 4 * A, pt.B.shape).copy()
    gs = oracle.p2g(sc)
    act = gs.active.astype(bool)
    shp = oracle.node_shape(sc.grid)
    k = np.stack(np.meshgrid(*[np.arange(s) for s in shp], indexing="ij"), -1).reshape(-1, d)
    xi = np.asarray(sc.grid.origin[:d]) + k * sc.grid.dx
    np.testing.assert_allclose(gs.v[act], xi[act] @ A.T + c, rtol=0, atol=1e-12)


@pytest.mark.parametrize("dim", [2, 3])
def test_g2p_completeness(dim):
    sc = synth.random_fixture(dim=dim, seed=13, cells=(3, 4, 3))
    d = dim
    rng = np.random.default_rng(9)
    shp = oracle.node_shape(sc.grid)
    k = np.stack(np.meshgrid(*[np.arange(s) for s in shp], indexing="ij"), -1).reshape(-1, d)
    xi = np.asarray(sc.grid.origin[:d]) + k * sc.grid.dx
    pt0 = sc.particles
    # uniform v0 -> v_p = v0, B_p = 0, F unchanged (up to (I + dt*0)), x shifted by dt v0
    v0 = rng.normal(size=d)
    pt = oracle.g2p(sc, np.tile(v0, (xi.shape[0], 1)))
    np.testing.assert_allclose(pt.v, np.tile(v0, (pt0.n, 1)), rtol=0, atol=1e-14)
    assert np.abs(pt.B).max() < 1e-15
    np.testing.assert_allclose(pt.F, pt0.F, rtol=0, atol=1e-14)
    np.testing.assert_allclose(pt.x, pt0.x + sc.dt * v0, rtol=0, atol=1e-14)
    # affine v_i = A x_i + c -> v_p = A x_p + c, grad v = A, B_p = dx^2/4 A, F <- (I + dt A) F
    A = rng.normal(size=(d, d))
    c = rng.normal(size=d)
    pt = oracle.g2p(sc, xi @ A.T + c)
    np.testing.assert_allclose(pt.v, pt0.x @ A.T + c, rtol=0, atol=1e-12)
    np.testing.assert_allclose(pt.B, np.broadcast_to(sc.grid.dx ** 2 / 4 * A, pt.B.shape), rtol=0, atol=1e-13)
    np.testing.assert_allclose(pt.F, np.einsum("ab,pbc->pac", np.eye(d) + sc.dt * A, pt0.F), rtol=0, atol=1e-12)
    # zero field: v = 0, B = 0, x and F unchanged;  dt = 0: x unchanged
    pt = oracle.g2p(sc, np.zeros((xi.shape[0], d)))
    assert np.abs(pt.v).max() == 0 and np.abs(pt.B).max() == 0
    np.testing.assert_array_equal(pt.x, pt0.x)
    np.testing.assert_array_equal(pt.F, pt0.F)
    pt = oracle.g2p(sc, xi @ A.T + c, dt=0.0)
    np.testing.assert_array_equal(pt.x, pt0.x)


def _coarse_fine_pair(dim, r=4, offset=0.0):
    """A fine grid (dx_s) with a uniform active node set and a coarse grid dx_b = r dx_s."""
    dxs = 0.01
    dxb = r * dxs
    nf = 6 * r + 1
    grid_s = synth.Grid(dim, tuple([0.2 + offset * dxs] * dim + [0.0] * (3 - dim)), dxs,
                        tuple([nf] * dim + [1] * (3 - dim)))
    grid_b = synth.Grid(dim, tuple([0.2 - 4 * dxb] * dim + [0.0] * (3 - dim)), dxb,
                        tuple([15] * dim + [1] * (3 - dim)))
    return grid_s, grid_b


def _nodes(grid):
    d = grid.dim
    shp = oracle.node_shape(grid)
    k = np.stack(np.meshgrid(*[np.arange(s) for s in shp], indexing="ij"), -1).reshape(-1, d)
    return k, np.asarray(grid.origin[:d]) + k * grid.dx


@pytest.mark.parametrize("dim", [2, 3])
def test_projection_constant_and_linear(dim):
    rng = np.random.default_rng(21)
    for r, off in ((2, 0.0), (4, 0.37), (4, 0.5), (8, 0.0)):
        gS, gB = _coarse_fine_pair(dim, r, off)
        kS, xS = _nodes(gS)
        kB, xB = _nodes(gB)
        nS = xS.shape[0]
        act = np.ones(nS, np.uint8)
        # constant field: exact for ANY masses (ε_tol = 0)
        m = rng.uniform(0.5, 2.0, nS)
        c = rng.normal(size=dim)
        gsf = oracle.GridState(m, None, np.tile(c, (nS, 1)), None, None, act)
        vb, num, den = oracle.project(gS, gsf, gB, 0.0)
        cov = den > 0
        np.testing.assert_allclose(vb[cov], np.tile(c, (cov.sum(), 1)), rtol=0, atol=1e-13)
        # linear field, uniform fine mass: exact on coarse nodes whose support is fully covered
        A = rng.normal(size=(dim, dim))
        gsf = oracle.GridState(np.ones(nS), None, xS @ A.T + c, None, None, act)
        vb, num, den = oracle.project(gS, gsf, gB, 0.0)
        lo = np.asarray(gS.origin[:dim]) + 1.5 * gB.dx
        hi = np.asarray(gS.origin[:dim]) + (gS.dims[0] - 1) * gS.dx - 1.5 * gB.dx
        full = np.all((xB >= lo - 1e-12) & (xB <= hi + 1e-12), axis=1)
        assert full.sum() >= 1
        np.testing.assert_allclose(vb[full], xB[full] @ A.T + c, rtol=0, atol=1e-13)


def test_projection_hand_case_and_vacuum():
    # 1 coarse node support, two fine nodes with masses m1, m2 and velocities v1, v2 -> weighted mean
    gB = synth.Grid(2, (0.0, 0.0, 0.0), 0.1, (10, 10, 1))
    gS = synth.Grid(2, (0.5, 0.5, 0.0), 0.05, (3, 3, 1))
    m = np.zeros(9)
    v = np.zeros((9, 2))
    act = np.zeros(9, np.uint8)
    m[0], m[4] = 2.0, 3.0   # fine nodes at (0.5, 0.5) and (0.55, 0.55)
    v[0], v[4] = [1.0, 0.0], [0.0, 1.0]
    act[[0, 4]] = 1
    vb, num, den = oracle.project(gS, oracle.GridState(m, None, v, None, None, act), gB, 0.0)
    # coarse node (5,5) at (0.5,0.5): N_B(0.5,0.5) = 9/16; N_B(0.55,0.55) = (0.75-0.25)^2... per axis
    w_on = 0.75
    w_half = 0.75 - 0.5 ** 2       # f - 1 = 0.5 cells -> 0.5
    N0 = w_on * w_on
    N1 = w_half * w_half
    I = 5 * 10 + 5
    assert den[I] == pytest.approx(2.0 * N0 + 3.0 * N1, rel=1e-15)
    np.testing.assert_allclose(vb[I], (2.0 * N0 * np.array([1, 0]) + 3.0 * N1 * np.array([0, 1])) / den[I],
                               rtol=1e-15)
    # vacuum: with eps_tol > 0, an empty coarse node returns 0
    vb2, _, den2 = oracle.project(gS, oracle.GridState(m, None, v, None, None, act), gB, 1e-12)
    assert np.all(vb2[den2 == 0] == 0)


@pytest.mark.parametrize("dim", [2, 3])
def test_interp_time_reproduces_linear(dim):
    rng = np.random.default_rng(31)
    gS, gB = _coarse_fine_pair(dim, 4, 0.37)
    kS, xS = _nodes(gS)
    kB, xB = _nodes(gB)
    A0, A1 = rng.normal(size=(2, dim, dim))
    c0, c1 = rng.normal(size=(2, dim))
    v0 = xB @ A0.T + c0
    v1 = xB @ A1.T + c1
    targets = np.arange(xS.shape[0])
    for alpha in (0.0, 0.25, 1.0):
        out = oracle.interp(gB, v0, v1, alpha, gS, targets)
        exp = (1 - alpha) * (xS @ A0.T + c0) + alpha * (xS @ A1.T + c1)
        np.testing.assert_allclose(out, exp, rtol=0, atol=1e-12)
    # endpoint identities and linearity in alpha on arbitrary coarse fields
    w0 = rng.normal(size=v0.shape)
    w1 = rng.normal(size=v0.shape)
    o0 = oracle.interp(gB, w0, w1, 0.0, gS, targets)
    o1 = oracle.interp(gB, w0, w1, 1.0, gS, targets)
    oh = oracle.interp(gB, w0, w1, 0.3, gS, targets)
    # endpoints (PAPER.md:352 with alpha = 0 / 1): T_0 = I(v^n) and T_1 = I(v^{n+1}) whatever the other
    # field is -- compared with the single-field interpolation (both endpoints set to the same field)
    np.testing.assert_array_equal(o0, oracle.interp(gB, w0, 100.0 * w1 + 7.0, 0.0, gS, targets))
    np.testing.assert_allclose(o0, oracle.interp(gB, w0, w0, 0.5, gS, targets), rtol=0, atol=1e-14)
    np.testing.assert_array_equal(o1, oracle.interp(gB, -3.0 * w0, w1, 1.0, gS, targets))
    np.testing.assert_allclose(o1, oracle.interp(gB, w1, w1, 0.5, gS, targets), rtol=0, atol=1e-14)
    assert np.abs(o0 - o1).max() > 0.1  # the two endpoints differ, so the checks above see alpha
    np.testing.assert_allclose(oh, 0.7 * o0 + 0.3 * o1, rtol=0, atol=1e-14)
