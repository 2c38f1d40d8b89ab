"""GPU parity on BASELINE.json configs[1..3] (C2 Hertz, C3 inclusion, C4 fold), the
configs that are parity-test cases rather than bench lines: every hot-path kernel on each config's
fine and coarse subdomain (P2G, gradient + energy, Jacobi diagonal, HVP, G2P; 1e-11), and one whole
Schwarz frame (Alg. 1) with the config's loads and boundary conditions against the
oracle frame (fixed K and fixed Newton x PCG counts on both sides, R18; the north_star's full-step
bar 1e-8 on displacements, velocities and F).  C4 also runs as its fp32 variant (R14: 1e-4).

Boundary conditions (R17):
* C2: rigid frictionless plane, v_y = 0 at nodes with y <= 0 on both grids; body load = the first
  frame of the linear ramp to g_max = 5.49 m/s^2 (here the full g_max, to load the contact).
* C3: rollers, v_x = 0 at coarse nodes with x <= 0, v_x = 0.01 m/s at coarse nodes with x >= 1.
* C4: coarse nodes with x <= 0 clamped, nodes with x >= 1 driven at the t = 0 velocity of the
  circular arc about the crease axis (x = 0.5, z = 0.02, parallel to y), theta = pi t / (100 dT);
  gravity -9.81 in z.  Reduced band y in [0, 1/16] (SURVEY.md §8(d) oracle budget).
"""
import functools

import numpy as np
import pytest

import oracle
import synth
from oracle import schwarz as OS
from gpu_helpers import make_sub, random_u, rel_linf

pytestmark = pytest.mark.gpu

TOL = 1e-11
FIXED = dict(max_newton=2, max_cg=40, fixed_iters=1)


@pytest.fixture(scope="module")
def ctx():
    from paper_2605_09097_b200 import osmpm
    c = osmpm.Context(0)
    yield c
    c.close()


def _c2():
    coarse, fine = synth.c2_hertz()
    for sc in (coarse, fine):
        sc.gravity = (0.0, -5.49, 0.0)
    return coarse, fine


def _c4():
    return synth.c4_fold(y_extent=1.0 / 16)


CONFIGS = {"c2": _c2, "c3": lambda: synth.c3_inclusion(256), "c4": _c4}


def _bcs(name, scene, dT):
    """(node indices, per-node component bit mask, per-node velocity (n, d)) of the config's physical
    boundary conditions on `scene`'s node box."""
    xs, _ = OS.node_positions(scene.grid)
    d = scene.grid.dim
    if name == "c2":
        sel = np.flatnonzero(xs[:, 1] <= 1e-12)
        return sel, np.full(sel.size, 2, np.uint8), np.zeros((sel.size, d))
    if name == "c3":
        lo = np.flatnonzero(xs[:, 0] <= 1e-12)
        hi = np.flatnonzero(xs[:, 0] >= 1.0 - 1e-12)
        vel = np.zeros((lo.size + hi.size, d))
        vel[lo.size:, 0] = 0.01
        return np.concatenate([lo, hi]), np.full(lo.size + hi.size, 1, np.uint8), vel
    if name == "c4":
        lo = np.flatnonzero(xs[:, 0] <= 1e-12)
        hi = np.flatnonzero(xs[:, 0] >= 1.0 - 1e-12)
        omega = np.pi / (100 * dT)
        r = xs[hi] - np.array([0.5, 0.0, 0.02])
        vel = np.zeros((lo.size + hi.size, 3))
        vel[lo.size:, 0] = -omega * r[:, 2]       # omega (-y) x r
        vel[lo.size:, 2] = omega * r[:, 0]
        return np.concatenate([lo, hi]), np.full(lo.size + hi.size, 7, np.uint8), vel
    raise KeyError(name)


def _user_bc(scene, sel, bits, vel):
    nn, d = oracle.n_nodes(scene.grid), scene.grid.dim
    mask = np.zeros((nn, d), np.uint8)
    v = np.zeros((nn, d))
    for c in range(d):
        on = (bits >> c) & 1 == 1
        mask[sel[on], c] = 1
        v[sel[on], c] = vel[on, c]
    return OS.UserBC(mask, v)


@pytest.mark.parametrize("which", ["fine", "coarse"])
@pytest.mark.parametrize("name", list(CONFIGS))
def test_config_kernel_parity(ctx, name, which):
    coarse, fine = CONFIGS[name]()
    sc = fine if which == "fine" else coarse
    d = sc.grid.dim
    ref = oracle.p2g(sc)
    sub = make_sub(ctx, sc)
    sub.p2g()
    out = sub.read_grid()
    np.testing.assert_array_equal(out["active"], ref.active)
    for k, r in (("m", ref.m), ("p", ref.p), ("v", ref.v), ("fext", ref.fext)):
        assert rel_linf(out[k], r) <= TOL, k
    assert np.abs(out["fsig"]).max() <= TOL * np.abs(ref.m).max()    # F = I: no stress force
    u = random_u(ref.active, d, 2e-3 * sc.grid.dx, 11)
    g, E = sub.newton_gradient(u)
    assert rel_linf(g, oracle.gradient(sc, ref, u)) <= TOL
    E_ref, _ = oracle.energy(sc, ref, u)
    assert abs(E - E_ref) <= TOL * abs(E_ref)
    assert rel_linf(sub.newton_diag(), oracle.diag(sc, ref, u)) <= TOL
    dv = np.random.default_rng(12).normal(size=u.shape) * sc.grid.dx
    assert rel_linf(sub.newton_hvp(dv), oracle.hvp(sc, ref, u, dv)) <= TOL
    vg = np.zeros((ref.m.shape[0], d))
    # |dt grad v| ~ 0.05: F stays invertible
    vg[ref.active.astype(bool)] = np.random.default_rng(13).normal(size=(int(ref.active.sum()), d)) * (
        0.05 * sc.grid.dx / sc.dt)
    sub.set_grid_velocity(vg)
    sub.g2p()
    sub.sync()
    po = sub.read_particles()
    pr = oracle.g2p(sc, vg)
    for k, r in (("x", pr.x), ("v", pr.v), ("F", pr.F), ("B", pr.B)):
        assert rel_linf(po[k], r) <= TOL, k


@functools.lru_cache(maxsize=None)
def _oracle_frame(name, K):
    coarse, fine = CONFIGS[name]()
    M = coarse.meta["M"]
    bcB = _bcs(name, coarse, coarse.dt)
    bcS = _bcs(name, fine, coarse.dt)
    return OS.schwarz_step(coarse, fine, M, parity_fixed_k=K,
                           user_B=_user_bc(coarse, *bcB), user_S=_user_bc(fine, *bcS),
                           newton_coarse=oracle.default_settings(**FIXED),
                           newton_fine=oracle.default_settings(**FIXED))


def _frame(ctx, name, precision=0, K=2):
    from paper_2605_09097_b200 import osmpm
    coarse, fine = CONFIGS[name]()
    M = coarse.meta["M"]
    dT = coarse.dt
    bcB = _bcs(name, coarse, dT)
    bcS = _bcs(name, fine, dT)
    ref = _oracle_frame(name, K)
    sb = make_sub(ctx, coarse, precision=precision)      # the coupler pairs subdomains of one precision
    ss = make_sub(ctx, fine, precision=precision)
    for sub, (sel, bits, vel) in ((sb, bcB), (ss, bcS)):
        if sel.size:
            sub.set_dirichlet(sel, bits, vel)
    st = osmpm.schwarz_settings(M=M, parity_fixed_k=K, eps_tol=-1.0, coarse=osmpm.newton_settings(**FIXED),
                                fine=osmpm.newton_settings(**FIXED))
    cpl = osmpm.Coupler(sb, ss, st)
    rep = cpl.step()
    return coarse, fine, ref, rep, sb.read_particles(), ss.read_particles()


@pytest.mark.parametrize("name", list(CONFIGS))
def test_config_frame_parity(ctx, name):
    coarse, fine, ref, rep, co, fo = _frame(ctx, name)
    assert rep.n_recv_B == ref.n_recv_B and rep.n_recv_S == ref.n_recv_S
    assert rep.n_recv_B > 0 and rep.n_recv_S > 0
    assert rep.iters == 2
    for out, r, x0 in ((fo, ref.fine_particles, fine.particles.x), (co, ref.coarse_particles, coarse.particles.x)):
        assert np.abs(r.x - x0).max() > 0          # the loads moved something
        assert rel_linf(out["x"] - x0, r.x - x0) <= 1e-8
        assert rel_linf(out["v"], r.v) <= 1e-8
        assert rel_linf(out["F"] - np.eye(fine.grid.dim), r.F - np.eye(fine.grid.dim)) <= 1e-8
    np.testing.assert_allclose(np.array(rep.r_B[:2]), np.array(ref.r_B), rtol=1e-6, atol=1e-12)
    np.testing.assert_allclose(np.array(rep.r_S[:2]), np.array(ref.r_S), rtol=1e-6, atol=1e-12)


def test_c4_fp32_frame(ctx):
    """fp32 variant (R14): 1e-4 on the solved velocities.  Positions and F are stored in fp32, so a
    displacement x - x0 carries an absolute rounding of up to (sub-steps + 1) * eps32 * max|x| (one
    rounding per advection): bounded by that plus 1e-4 of its size.  F - I: the same storage term
    plus 1e-3 of its size -- the fixed 2 x 40 Newton x PCG solves are far from converged, so the
    fp32 HVP's rounding moves the Krylov iterates, and grad v amplifies the node-to-node part of that
    velocity difference (measured 0.5-1.8e-4 of max|F - I| on the coarse subdomain, whose driven edge
    reaches |F - I| = 0.89)."""
    from paper_2605_09097_b200 import osmpm
    coarse, fine, ref, rep, co, fo = _frame(ctx, "c4", precision=osmpm.F32)
    assert rep.n_recv_B == ref.n_recv_B and rep.n_recv_S == ref.n_recv_S
    eps32 = float(np.finfo(np.float32).eps)
    for out, r, sc, nsub in ((fo, ref.fine_particles, fine, 2 * fine.meta["M"]), (co, ref.coarse_particles, coarse, 1)):
        x0 = sc.particles.x
        assert rel_linf(out["v"], r.v) <= 1e-4
        for k, a0, rr, rel in (("x", x0, r.x, 1e-4), ("F", np.eye(3), r.F, 1e-3)):
            bound = (nsub + 1) * eps32 * np.abs(rr).max() + rel * np.abs(rr - a0).max()
            assert np.abs(out[k] - rr).max() <= bound, k


@pytest.mark.parametrize("name,slabs,nccl", [("c4", 2, False), ("c4", 3, False), ("c3", 2, False), ("c3", 4, False),
                                             ("c3", 2, True), ("c4", 1, True)])
def test_config_frame_parity_decomposed_fine(name, slabs, nccl):
    """The Schwarz frame with the FINE subdomain split into x-slabs (here `slabs` local
    slabs on one GPU: the same slab layout, halo sums, Gamma_S / arbitration over owned + ghost nodes,
    Pi partial sums and residual reductions as the multi-rank path, minus NCCL) and the coarse
    subdomain whole (decompose = 0): equal to the oracle frame at 1e-8 with the same receiver sets.
    `nccl`: on a one-rank NCCL communicator, so that the coupler's Gamma_B broadcast, the OR of the
    taken-over coarse nodes, the Pi partial sums and the residual norms go through NCCL."""
    from paper_2605_09097_b200 import osmpm
    coarse, fine = CONFIGS[name]()
    M = coarse.meta["M"]
    dT = coarse.dt
    ref = _oracle_frame(name, 2)
    ctx = osmpm.Context(0)
    if nccl:
        ctx.init_comm(0, 1, osmpm.comm_unique_id())
    if slabs > 1:
        ctx.set_local_slabs(slabs)
    sb = osmpm.Subdomain(ctx, coarse.grid, coarse.dt, coarse.particles, coarse.materials, coarse.gravity,
                         decompose=False)
    ss = osmpm.Subdomain(ctx, fine.grid, fine.dt, fine.particles, fine.materials, fine.gravity)
    assert ss.decomp()[0] == slabs
    for sub, sc in ((sb, coarse), (ss, fine)):
        sel, bits, vel = _bcs(name, sc, dT)
        if sel.size:
            sub.set_dirichlet(sel, bits, vel)
    st = osmpm.schwarz_settings(M=M, parity_fixed_k=2, eps_tol=-1.0, coarse=osmpm.newton_settings(**FIXED),
                                fine=osmpm.newton_settings(**FIXED))
    rep = osmpm.Coupler(sb, ss, st).step()
    assert rep.n_recv_B == ref.n_recv_B and rep.n_recv_S == ref.n_recv_S and rep.iters == 2
    co, fo = sb.read_particles(), ss.read_particles()
    for out, r, x0 in ((fo, ref.fine_particles, fine.particles.x), (co, ref.coarse_particles, coarse.particles.x)):
        assert rel_linf(out["x"] - x0, r.x - x0) <= 1e-8
        assert rel_linf(out["v"], r.v) <= 1e-8
        assert rel_linf(out["F"] - np.eye(fine.grid.dim), r.F - np.eye(fine.grid.dim)) <= 1e-8
    ctx.close()
