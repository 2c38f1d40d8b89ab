"""Pins of the oracle's Schwarz frame (O11-O12): arbitration rules, exact reproduction of uniform
translation for any M and resolution ratio, free fall as the converged frame (pins the temporal
interpolation alpha = m / M), contraction of the interface residuals, parity mode
(PAPER.md:294-301, 436-501)."""
import numpy as np
import pytest

import oracle
import synth
from oracle import schwarz as S


def _translating_pair(dim, c, M=4):
    coarse, fine = synth.c1_cantilever(g=0.0) if dim == 2 else (None, None)
    for sc in (coarse, fine):
        sc.particles.v[:] = c
        sc.gravity = (0.0, 0.0, 0.0)
    fine.dt = coarse.dt / M
    return coarse, fine


# ---------------------------------------------------------------------------------------------
# O11 Gamma selection (Eq. boundary_grid_set): pins of its own
# ---------------------------------------------------------------------------------------------

def _one_boundary_particle_scene(dim, x_p, m_p=2.0):
    """A block of ordinary particles plus one marked boundary particle at x_p."""
    sc = synth.random_fixture(dim=dim, cells=(4, 4, 3) if dim == 3 else (6, 5, 1), seed=71, dx=0.1)
    pt = sc.particles
    pt.boundary[:] = 0
    pt.x[0] = x_p
    pt.m[0] = m_p
    pt.boundary[0] = 1
    return sc


@pytest.mark.parametrize("dim", [2, 3])
def test_gamma_one_boundary_particle_touches_its_stencil_only(dim):
    """One P^∂ particle sitting exactly on a grid node: its boundary mass lands on exactly its 3^d
    stencil nodes with the knot weights (1/8, 3/4, 1/8) per axis (golden G1 at f = 1), so
    m^∂ = m_p (3/4)^d at the node, m_p (3/4)^(d-1)/8 at face neighbours, ..., and sums to m_p."""
    sc = _one_boundary_particle_scene(dim, None)
    g = sc.grid
    k = np.array([3, 3, 2][:dim])
    sc.particles.x[0] = np.asarray(g.origin[:dim]) + g.dx * k
    mb = oracle.boundary_mass(sc)
    nz = np.flatnonzero(mb)
    assert nz.size == 3 ** dim
    knot = {-1: 1 / 8, 0: 3 / 4, 1: 1 / 8}
    shp = oracle.node_shape(g)
    for i in nz:
        ki = np.array(np.unravel_index(i, shp))
        off = ki - k
        assert np.all(np.abs(off) <= 1)
        assert mb[i] == pytest.approx(2.0 * np.prod([knot[int(o)] for o in off]), rel=1e-15)
    assert mb.sum() == pytest.approx(2.0, rel=1e-15)
    # Gamma (threshold 1e-6 x median mass): exactly those 3^d nodes
    gs = oracle.p2g(sc)
    gam, tau = S.gamma_set(sc, gs, 1e-6)
    assert set(np.flatnonzero(gam)) == set(nz)


def test_gamma_counts_only_marked_particles():
    """m^∂ equals the P2G mass (pinned by golden G2 and conservation) of the marked subset alone: an
    oracle that treated every particle as a boundary particle fails this."""
    sc = synth.random_fixture(dim=2, cells=(8, 6, 1), seed=72, dx=0.1)
    rng = np.random.default_rng(3)
    sc.particles.boundary[:] = (rng.random(sc.particles.n) < 0.3).astype(np.uint8)
    mb = oracle.boundary_mass(sc)
    sub = synth.Scene(sc.grid, sc.particles.subset(sc.particles.boundary.astype(bool)), sc.materials, sc.dt)
    np.testing.assert_allclose(mb, oracle.p2g(sub).m, rtol=1e-14, atol=0)
    assert mb.sum() < 0.5 * oracle.p2g(sc).m.sum()


def test_gamma_threshold_is_relative_to_the_median_mass():
    """tau_Gamma = tau_rel x median particle mass (R11): a boundary particle whose stencil
    weight at a corner node is w gives that node m_p w; the node is in Gamma iff m_p w > tau."""
    sc = _one_boundary_particle_scene(2, None, m_p=1.0)
    g = sc.grid
    k = np.array([3, 3])
    sc.particles.x[0] = np.asarray(g.origin[:2]) + g.dx * k
    gs = oracle.p2g(sc)
    med = oracle.median(sc.particles.m)
    corner = 1 / 64  # (1/8)^2
    for tau_rel, expect in ((0.999 * corner / med, 9), (1.001 * corner / med, 5)):
        gam, tau = S.gamma_set(sc, gs, tau_rel)
        assert tau == pytest.approx(tau_rel * med)
        assert int(gam.sum()) == expect  # corners drop out first (faces carry 3/32)


def test_receivers_hand_case_1d_overlap():
    """A hand-computed pair: coarse dx = 0.2, fine dx = 0.1, both marked at their artificial cuts.
    The fine nodes at x = 0.4 and the coarse node at x = 0.4 coincide; whichever carries the larger
    raw nodal mass donates (tie -> B), the other side receives, never both."""
    # fine block x in [0, 0.6], coarse block x in [0.3, 1.2] (2D strips, one row of cells)
    fine = synth.random_fixture(dim=2, cells=(6, 2, 1), seed=73, dx=0.1, F_sigma=0.0, B_scale=0.0)
    coarse = synth.random_fixture(dim=2, cells=(5, 1, 1), seed=74, dx=0.2, F_sigma=0.0, B_scale=0.0)
    coarse.particles.x[:, 0] += 0.2
    for sc, cut, side in ((fine, 0.6, -1), (coarse, 0.2 + 0.0, +1)):
        x = sc.particles.x[:, 0]
        sc.particles.boundary[:] = (np.abs(x - (x.max() if side < 0 else x.min())) < sc.grid.dx).astype(np.uint8)
    lo = np.minimum(fine.particles.x.min(0), coarse.particles.x.min(0)) - 0.6
    for sc in (fine, coarse):
        sc.grid = synth.grid_around(np.vstack([fine.particles.x, coarse.particles.x]), sc.grid.dx, 4, 2,
                                    align_origin=(0.0, 0.0))
    gsB, gsS = oracle.p2g(coarse), oracle.p2g(fine)
    hatB, hatS = S.receivers(coarse, fine, gsB, gsS, 1e-6)
    gB, _ = S.gamma_set(coarse, gsB, 1e-6)
    gS, _ = S.gamma_set(fine, gsS, 1e-6)
    assert hatB.sum() > 0 and hatS.sum() > 0
    xs, _ = S.node_positions(fine.grid)
    cidx = S.coincident_coarse_index(coarse.grid, xs, 1e-9)
    amb = np.flatnonzero(gS & (cidx >= 0) & gB[np.maximum(cidx, 0)])
    assert amb.size > 0
    for j in amb:
        I = cidx[j]
        assert not (hatB[I] and hatS[j])
        if gsB.m[I] >= gsS.m[j]:
            assert not hatB[I]
        else:
            assert not hatS[j]
    # receivers are a subset of Gamma on each side
    assert np.all(gB[hatB]) and np.all(gS[hatS])


def test_receivers_disjoint_and_tie_to_B():
    coarse, fine = synth.c1_cantilever()
    gsB = oracle.p2g(coarse)
    gsS = oracle.p2g(fine)
    hatB, hatS = S.receivers(coarse, fine, gsB, gsS, 1e-6)
    assert hatB.sum() > 0 and hatS.sum() > 0
    # every receiver is an active node of its own grid
    assert np.all(gsB.active[hatB]) and np.all(gsS.active[hatS])
    # coincident nodes are never receivers on both sides
    xs, _ = S.node_positions(fine.grid)
    cidx = S.coincident_coarse_index(coarse.grid, xs, 1e-9 * fine.grid.dx)
    both = hatS & (cidx >= 0)
    assert not np.any(hatB[cidx[both]])


def test_arbitration_tie_goes_to_background():
    # hand case: one coincident boundary node with equal masses on both grids -> B donates, S receives
    coarse, fine = synth.c1_cantilever()
    gsB = oracle.p2g(coarse)
    gsS = oracle.p2g(fine)
    gB, _ = S.gamma_set(coarse, gsB, 1e-6)
    gS, _ = S.gamma_set(fine, gsS, 1e-6)
    xs, _ = S.node_positions(fine.grid)
    cidx = S.coincident_coarse_index(coarse.grid, xs, 1e-9 * fine.grid.dx)
    amb = np.flatnonzero(gS & (cidx >= 0) & gB[np.maximum(cidx, 0)])
    assert amb.size > 0
    j = amb[0]
    I = cidx[j]
    gsS.m[j] = gsB.m[I]          # force a tie
    hatB, hatS = S.receivers(coarse, fine, gsB, gsS, 1e-6)
    assert not hatB[I]
    gsS.m[j] = 2.0 * gsB.m[I]    # S heavier -> S donates, B receives (if eligible)
    hatB2, hatS2 = S.receivers(coarse, fine, gsB, gsS, 1e-6)
    assert not hatS2[j]


@pytest.mark.parametrize("M", [1, 4])
def test_uniform_translation_is_reproduced_exactly(M):
    c = np.array([0.3, -0.2])
    coarse, fine = _translating_pair(2, c, M)
    x0c = coarse.particles.x.copy()
    x0f = fine.particles.x.copy()
    res = S.schwarz_step(coarse, fine, M, parity_fixed_k=2)
    # exact up to the solver tolerance (Newton / PCG at 1e-12 relative)
    for pt, x0 in ((res.coarse_particles, x0c), (res.fine_particles, x0f)):
        np.testing.assert_allclose(pt.v, np.tile(c, (pt.n, 1)), rtol=0, atol=1e-10)
        np.testing.assert_allclose(pt.x, x0 + coarse.dt * c, rtol=0, atol=1e-12)
        np.testing.assert_allclose(pt.F, np.broadcast_to(np.eye(2), pt.F.shape), rtol=0, atol=1e-10)
    assert res.r_B[-1] < 1e-10 and res.r_S[-1] < 1e-10


def _falling_pair(M, c=(0.3, -0.2), g=(0.5, -9.81)):
    coarse, fine = synth.c1_cantilever(g=0.0)
    for sc in (coarse, fine):
        sc.particles.v[:] = np.asarray(c)
        sc.gravity = (g[0], g[1], 0.0)
    fine.dt = coarse.dt / M
    return coarse, fine, np.asarray(c), np.asarray(g)


def free_fall_closed_form(x0, c, g, dt, n):
    """n backward-Euler steps of free fall: v_m = c + m dt g, x_m = x_{m-1} + dt v_m."""
    return x0 + n * dt * c + dt * dt * g * n * (n + 1) / 2, c + n * dt * g


@pytest.mark.parametrize("M", [2, 4])
def test_free_fall_is_the_converged_frame(M):
    # Uniform free fall is a fixed point of the whole frame only if the fine receivers get the
    # coarse velocity at the sub-step's own time, (1 - alpha) v_B^n + alpha v_B^(n+1) with alpha = m/M
    # (Eq. temporal_interp): backward Euler then gives every fine particle
    # v = c + m dt g after sub-step m.  The iteration starts from Pi(v_S^n) = c on the coarse receivers
    # (R16), so it converges to that closed form instead of reproducing it at k = 1.
    coarse, fine, c, g = _falling_pair(M)
    x0c, x0f = coarse.particles.x.copy(), fine.particles.x.copy()
    res = S.schwarz_step(coarse, fine, M, eps_conv=1e-10, k_max=200)
    assert res.converged and res.iters < 60
    xf, vf = free_fall_closed_form(x0f, c, g, fine.dt, M)
    xc, vc = free_fall_closed_form(x0c, c, g, coarse.dt, 1)
    np.testing.assert_allclose(res.fine_particles.v, np.tile(vf, (fine.particles.n, 1)), rtol=0, atol=1e-8)
    np.testing.assert_allclose(res.coarse_particles.v, np.tile(vc, (coarse.particles.n, 1)), rtol=0, atol=1e-8)
    np.testing.assert_allclose(res.fine_particles.x, xf, rtol=0, atol=1e-10)
    np.testing.assert_allclose(res.coarse_particles.x, xc, rtol=0, atol=1e-10)
    np.testing.assert_allclose(res.fine_particles.F, np.broadcast_to(np.eye(2), res.fine_particles.F.shape),
                               rtol=0, atol=1e-9)


def test_cantilever_frame_converges_with_contracting_residuals():
    coarse, fine = synth.c1_cantilever()
    # clamp: fine nodes with x <= 0 fixed in all components (R17)
    gsS = oracle.p2g(fine)
    xs, _ = S.node_positions(fine.grid)
    mask = np.repeat((xs[:, 0] <= 1e-12)[:, None], 2, axis=1).astype(np.uint8)
    user_S = S.UserBC(mask, np.zeros_like(xs))
    res = S.schwarz_step(coarse, fine, 4, eps_conv=1e-5, k_max=30, user_S=user_S)
    assert res.converged
    assert res.iters >= 2
    # the interface residuals contract (geometric convergence of the alternating method)
    rB = np.array(res.r_B)
    assert rB[-1] < rB[0]
    # the beam sags (gravity) and the clamp holds
    assert res.fine_particles.x[:, 1].mean() < fine.particles.x[:, 1].mean()
