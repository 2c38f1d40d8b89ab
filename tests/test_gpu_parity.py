"""GPU parity: the CUDA path (through the C ABI) against the fp64 oracle on identical seeded
inputs, element by element (tolerance rel L∞ <= 1e-11 per kernel output in fp64,
<= 1e-8 on Newton-converged solutions, <= 1e-4 for the fp32 variant; north_star)."""
import numpy as np
import pytest

import oracle
import synth
from gpu_helpers import make_sub, random_u, rel_linf

pytestmark = pytest.mark.gpu

TOL = 1e-11

FIXTURES = {
    # several tiles per axis and ragged tails (3D tiles are 4^3 cells, 2D tiles 8^2 cells)
    "3d": dict(dim=3, cells=(10, 9, 7), seed=101),
    "2d": dict(dim=2, cells=(21, 17, 1), seed=102),
    "3d_dense": dict(dim=3, cells=(6, 5, 9), seed=103, ppa=3),
}


@pytest.fixture(scope="module")
def ctx():
    from paper_2605_09097_b200 import osmpm
    c = osmpm.Context(0)
    yield c
    c.close()


def _scene(name):
    return synth.random_fixture(**FIXTURES[name])


@pytest.mark.parametrize("name", list(FIXTURES))
def test_p2g_parity(ctx, name):
    sc = _scene(name)
    ref = oracle.p2g(sc)
    sub = make_sub(ctx, sc)
    sub.p2g()
    out = sub.read_grid()
    np.testing.assert_array_equal(out["active"], ref.active)
    assert rel_linf(out["m"], ref.m) <= TOL
    assert rel_linf(out["p"], ref.p) <= TOL
    assert rel_linf(out["v"], ref.v) <= TOL
    assert rel_linf(out["fext"], ref.fext) <= TOL
    assert rel_linf(out["fsig"], ref.fsig) <= TOL


@pytest.mark.parametrize("name", list(FIXTURES))
def test_gradient_hvp_diag_parity(ctx, name):
    sc = _scene(name)
    d = sc.grid.dim
    ref = oracle.p2g(sc)
    sub = make_sub(ctx, sc)
    sub.p2g()
    u = random_u(ref.active, d, 2e-3 * sc.grid.dx, 7)
    g, E = sub.newton_gradient(u)
    g_ref = oracle.gradient(sc, ref, u)
    E_ref, _ = oracle.energy(sc, ref, u)
    assert rel_linf(g, g_ref) <= TOL
    assert abs(E - E_ref) <= TOL * abs(E_ref)
    dg = sub.newton_diag()
    assert rel_linf(dg, oracle.diag(sc, ref, u)) <= TOL
    rng = np.random.default_rng(8)
    for trial in range(2):
        dv = rng.normal(size=u.shape) * sc.grid.dx
        y = sub.newton_hvp(dv)
        assert rel_linf(y, oracle.hvp(sc, ref, u, dv)) <= TOL


@pytest.mark.parametrize("name", ["3d", "2d"])
def test_g2p_parity(ctx, name):
    sc = _scene(name)
    d = sc.grid.dim
    ref = oracle.p2g(sc)
    sub = make_sub(ctx, sc)
    sub.p2g()
    rng = np.random.default_rng(9)
    vg = np.zeros((ref.m.shape[0], d))
    vg[ref.active.astype(bool)] = rng.normal(size=(int(ref.active.sum()), d))
    sub.set_grid_velocity(vg)
    sub.g2p()
    sub.sync()
    out = sub.read_particles()
    pref = oracle.g2p(sc, vg)
    for k, r in (("x", pref.x), ("v", pref.v), ("F", pref.F), ("B", pref.B)):
        assert rel_linf(out[k], r) <= TOL, k


@pytest.mark.parametrize("name", ["3d", "2d"])
def test_implicit_solve_parity_converged(ctx, name):
    from paper_2605_09097_b200 import osmpm
    sc = synth.random_fixture(**{**FIXTURES[name], "cells": (5, 4, 4) if name == "3d" else (9, 8, 1)})
    ref = oracle.p2g(sc)
    kw = dict(newton_rtol=1e-12, cg_rtol=1e-12, max_cg=4000, max_newton=50)
    u_ref, st_ref = oracle.implicit_solve(sc, ref, oracle.default_settings(**kw))
    sub = make_sub(ctx, sc)
    sub.p2g()
    st = sub.implicit_solve(osmpm.newton_settings(**kw))
    assert st.status == 0 and st_ref.status == 0
    # converged at newton_rtol on both sides, not accepted at the round-off floor (R8)
    assert st.floor_accept == st_ref.floor_accept == 0
    assert st.ls_failures == st_ref.ls_failures == 0
    v = sub.read_grid_velocity()
    act = ref.active.astype(bool)
    v_ref = np.where(act[:, None], u_ref / sc.dt, 0.0)
    assert rel_linf(v, v_ref) <= 1e-8


def test_implicit_solve_parity_fixed_iterations(ctx):
    from paper_2605_09097_b200 import osmpm
    sc = synth.random_fixture(dim=3, cells=(5, 5, 4), seed=104)
    ref = oracle.p2g(sc)
    kw = dict(max_newton=3, max_cg=20, fixed_iters=1)
    u_ref, st_ref = oracle.implicit_solve(sc, ref, oracle.default_settings(**kw))
    sub = make_sub(ctx, sc)
    sub.p2g()
    st = sub.implicit_solve(osmpm.newton_settings(**kw))
    assert st.newton_iters == 3 and st.cg_iters == 60
    v = sub.read_grid_velocity()
    act = ref.active.astype(bool)
    assert rel_linf(v, np.where(act[:, None], u_ref / sc.dt, 0.0)) <= 1e-9


@pytest.mark.parametrize("variant", [0, 1])
def test_fixed_iteration_solve_parity_both_pcg_variants(ctx, variant):
    """R22: standard and single-reduction PCG, each against the oracle running the same variant, fixed
    3 x 20 and converged."""
    from paper_2605_09097_b200 import osmpm
    sc = synth.random_fixture(dim=3, cells=(5, 5, 4), seed=104)
    ref = oracle.p2g(sc)
    act = ref.active.astype(bool)
    for kw, tol in ((dict(max_newton=3, max_cg=20, fixed_iters=1), 1e-9),
                    (dict(newton_rtol=1e-12, cg_rtol=1e-12, max_cg=4000, max_newton=50), 1e-8)):
        u_ref, st_ref = oracle.implicit_solve(sc, ref, oracle.default_settings(cg_variant=variant, **kw))
        sub = make_sub(ctx, sc)
        sub.p2g()
        st = sub.implicit_solve(osmpm.newton_settings(cg_variant=variant, **kw))
        assert st.status == 0 and st_ref.status == 0
        if kw.get("fixed_iters"):
            assert st.cg_iters == st_ref.cg_iters == 60
        assert rel_linf(sub.read_grid_velocity(), np.where(act[:, None], u_ref / sc.dt, 0.0)) <= tol
        sub.close()


def test_fixed_mode_line_search_failure_parity(ctx):
    """R8 fixed-iteration policy on both sides: no trial accepted -> alpha = 0, counted, u unchanged."""
    from paper_2605_09097_b200 import osmpm
    sc = synth.random_fixture(dim=3, cells=(3, 2, 2), seed=58)
    ref = oracle.p2g(sc)
    kw = dict(max_newton=4, max_cg=0, fixed_iters=1, energy_noise_rtol=-1.0)
    u_ref, st_ref = oracle.implicit_solve(sc, ref, oracle.default_settings(**kw))
    sub = make_sub(ctx, sc)
    sub.p2g()
    st = sub.implicit_solve(osmpm.newton_settings(**kw))
    assert st.status == 0 and st.ls_failures == st_ref.ls_failures == 4 and st.ls_halvings == st_ref.ls_halvings
    act = ref.active.astype(bool)
    assert rel_linf(sub.read_grid_velocity(), np.where(act[:, None], u_ref / sc.dt, 0.0)) <= 1e-14
    sub.close()


@pytest.mark.parametrize("fixed", [1, 0])
def test_negative_curvature_parity(ctx, fixed):
    """R7 on both sides: an indefinite tangent (F = 0.3 I) stops PCG at p^T H p <= 0, counted."""
    from paper_2605_09097_b200 import osmpm
    sc = synth.random_fixture(dim=2, cells=(4, 4, 1), seed=59, F_sigma=0.0)
    sc.particles.F[:] = np.diag([0.3, 0.3])
    sc.dt = 1.0
    ref = oracle.p2g(sc)
    kw = dict(max_newton=2, max_cg=30, fixed_iters=fixed, guess=1)
    u_ref, st_ref = oracle.implicit_solve(sc, ref, oracle.default_settings(**kw), raise_on_error=False)
    sub = make_sub(ctx, sc)
    sub.p2g()
    st = sub.implicit_solve(osmpm.newton_settings(**kw), raise_on_error=False)
    assert st.negcurv == st_ref.negcurv >= 1 and st.cg_iters == st_ref.cg_iters
    # same outcome (the two status enums number differently: GPU 4 / oracle 3 = Newton not converged)
    ORC2GPU = {0: 0, 3: 4, 4: 5}
    assert st.status == ORC2GPU[st_ref.status]
    if st.status == 0:
        act = ref.active.astype(bool)
        assert rel_linf(sub.read_grid_velocity(), np.where(act[:, None], u_ref / sc.dt, 0.0)) <= 1e-9
    sub.close()


def test_dirichlet_parity(ctx):
    from paper_2605_09097_b200 import osmpm
    sc = synth.random_fixture(dim=2, cells=(10, 8, 1), seed=105)
    ref = oracle.p2g(sc)
    d = 2
    nn = ref.m.shape[0]
    rng = np.random.default_rng(3)
    act = np.flatnonzero(ref.active)
    sel = rng.choice(act, size=len(act) // 5, replace=False)
    masks = rng.integers(1, 4, size=sel.size).astype(np.uint8)
    vel = rng.normal(size=(sel.size, d))
    dm = np.zeros((nn, d), np.uint8)
    dv = np.zeros((nn, d))
    for i, mk, vv in zip(sel, masks, vel):
        for a in range(d):
            if (mk >> a) & 1:
                dm[i, a] = 1
                dv[i, a] = vv[a]
    kw = dict(newton_rtol=1e-12, cg_rtol=1e-12, max_cg=4000)
    u_ref, _ = oracle.implicit_solve(sc, ref, oracle.default_settings(**kw), dirichlet_mask=dm, dirichlet_v=dv)
    sub = make_sub(ctx, sc)
    sub.set_dirichlet(sel, masks, vel)
    sub.p2g()
    sub.implicit_solve(osmpm.newton_settings(**kw))
    v = sub.read_grid_velocity()
    assert rel_linf(v, np.where(ref.active[:, None].astype(bool), u_ref / sc.dt, 0.0)) <= 1e-8


def test_transmit_parity(ctx):
    from paper_2605_09097_b200 import osmpm
    # fine subdomain inside a coarse one, r = 4
    fine = synth.random_fixture(dim=3, cells=(8, 8, 6), seed=106, dx=0.025)
    coarse = synth.random_fixture(dim=3, cells=(6, 6, 5), seed=107, dx=0.1)
    coarse.particles.x -= 0.1  # cover the fine block
    coarse.grid = synth.grid_around(coarse.particles.x, 0.1, 4, 3)
    rf = oracle.p2g(fine)
    rc = oracle.p2g(coarse)
    sf = make_sub(ctx, fine)
    scs = make_sub(ctx, coarse)
    sf.p2g()
    scs.p2g()
    nb = rc.m.shape[0]
    # Pi of the fine v^n onto every coarse node
    out = osmpm.transmit(sf, scs, osmpm.FINE_TO_COARSE, alpha=0.0, eps_tol=1e-12)
    vb_ref, num, den = oracle.project(fine.grid, rf, coarse.grid, eps_tol=1e-12)
    assert rel_linf(out, vb_ref) <= TOL
    # I + T with the coarse v^n and a set v^{n+1}
    rng = np.random.default_rng(4)
    v1 = np.zeros((nb, 3))
    v1[rc.active.astype(bool)] = rng.normal(size=(int(rc.active.sum()), 3))
    scs.set_grid_velocity(v1)
    targets = np.flatnonzero(rf.active)
    for alpha in (0.0, 0.25, 1.0):
        o = osmpm.transmit(scs, sf, osmpm.COARSE_TO_FINE, alpha=alpha, targets=targets)
        r = oracle.interp(coarse.grid, rc.v, v1, alpha, fine.grid, targets)
        assert rel_linf(o, r) <= TOL


@pytest.mark.parametrize("dim,dxf,dxc", [(3, 0.025, 0.1), (2, 0.04, 0.1), (2, 1 / 30, 0.11), (3, 0.03, 0.075)])
def test_projection_gather_parity_and_reproducibility(ctx, dim, dxf, dxc):
    """Pi as the separable gather: equal to the oracle's plain scatter at 1e-11 for
    integer (4), non-integer (2.5, 3.3) ratios and unaligned grid origins, in 2D and 3D, and bitwise
    identical across calls (no atomics)."""
    from paper_2605_09097_b200 import osmpm
    cells = (8, 8, 6) if dim == 3 else (12, 10, 1)
    fine = synth.random_fixture(dim=dim, cells=cells, seed=110 + dim, dx=dxf)
    coarse = synth.random_fixture(dim=dim, cells=(5, 5, 4) if dim == 3 else (6, 6, 1), seed=120 + dim, dx=dxc)
    coarse.particles.x -= 0.37 * dxc
    coarse.grid = synth.grid_around(coarse.particles.x, dxc, 4, dim)
    rf = oracle.p2g(fine)
    sf = make_sub(ctx, fine)
    scs = make_sub(ctx, coarse)
    sf.p2g()
    scs.p2g()
    out = osmpm.transmit(sf, scs, osmpm.FINE_TO_COARSE, alpha=0.0, eps_tol=1e-12)
    ref = oracle.project(fine.grid, rf, coarse.grid, eps_tol=1e-12)[0]
    assert np.abs(ref).max() > 0
    assert rel_linf(out, ref) <= TOL
    again = osmpm.transmit(sf, scs, osmpm.FINE_TO_COARSE, alpha=0.0, eps_tol=1e-12)
    assert np.array_equal(out, again)


def test_transmit_rejects_targets_outside_the_box(ctx):
    """Host targets are validated before any work; device targets are skipped and latched."""
    import torch
    from paper_2605_09097_b200 import osmpm
    fine = synth.random_fixture(dim=3, cells=(6, 6, 4), seed=130, dx=0.025)
    coarse = synth.random_fixture(dim=3, cells=(4, 4, 3), seed=131, dx=0.1)
    coarse.particles.x -= 0.1
    coarse.grid = synth.grid_around(coarse.particles.x, 0.1, 4, 3)
    sf = make_sub(ctx, fine)
    scs = make_sub(ctx, coarse)
    sf.p2g()
    scs.p2g()
    nb = oracle.n_nodes(coarse.grid)
    for bad in (-1, nb):
        with pytest.raises(osmpm.OsmpmError) as e:
            osmpm.transmit(sf, scs, osmpm.FINE_TO_COARSE, alpha=0.0, targets=np.array([0, bad], np.int64))
        assert e.value.code == 1
    tg = torch.tensor([3, nb + 5, 7], dtype=torch.int64, device="cuda")
    out = osmpm.transmit(sf, scs, osmpm.FINE_TO_COARSE, alpha=0.0, targets=tg, device="cuda")
    with pytest.raises(osmpm.OsmpmError) as e:
        scs.sync()
    assert e.value.code == 1 and "target 1" in str(e.value)
    assert float(out[1].abs().max()) == 0.0
    scs.sync()  # the latch was cleared by the report


def test_empty_and_single_particle(ctx):
    sc = synth.random_fixture(dim=3, cells=(1, 1, 1), ppa=1, seed=108)
    sub = make_sub(ctx, sc)
    sub.p2g()
    ref = oracle.p2g(sc)
    assert rel_linf(sub.read_grid()["m"], ref.m) <= TOL
    empty = synth.random_fixture(dim=2, cells=(2, 2, 1), seed=109)
    empty.particles = empty.particles.subset(np.zeros(empty.particles.n, bool))
    sub = make_sub(ctx, empty)
    sub.p2g()
    assert np.abs(sub.read_grid()["m"]).max() == 0.0


def test_out_of_domain_is_reported(ctx):
    from paper_2605_09097_b200 import osmpm
    sc = synth.random_fixture(dim=2, cells=(3, 3, 1), seed=110)
    sc.particles.x[5, 0] = sc.grid.origin[0] + 0.4 * sc.grid.dx  # base = -1
    with pytest.raises(osmpm.OsmpmError) as ei:
        make_sub(ctx, sc)
    assert ei.value.code == 2 and "particle 5" in str(ei.value)


def test_fp32_variant_within_1e_4(ctx):
    from paper_2605_09097_b200 import osmpm
    sc = _scene("3d")
    d = 3
    ref = oracle.p2g(sc)
    sub = make_sub(ctx, sc, precision=osmpm.F32)
    sub.p2g()
    out = sub.read_grid()
    assert rel_linf(out["m"], ref.m) <= 1e-4
    assert rel_linf(out["p"], ref.p) <= 1e-4
    u = random_u(ref.active, d, 2e-3 * sc.grid.dx, 7)
    g, E = sub.newton_gradient(u)
    assert rel_linf(g, oracle.gradient(sc, ref, u)) <= 1e-4
    dv = np.random.default_rng(8).normal(size=u.shape) * sc.grid.dx
    assert rel_linf(sub.newton_hvp(dv), oracle.hvp(sc, ref, u, dv)) <= 1e-4


def test_deterministic_mode_is_bitwise_reproducible(ctx, monkeypatch):
    """OSMPM_DETERMINISTIC=1: the gradient / Jacobi diagonal / HVP scatters store
    per-tile node blocks summed in a fixed tile order (hvp_sw.cuh k_det_gather) instead of RED-ing, so
    repeated evaluations and whole fixed-iteration solves are bitwise identical; parity unchanged."""
    from paper_2605_09097_b200 import osmpm
    monkeypatch.setenv("OSMPM_DETERMINISTIC", "1")
    sc = _scene("3d")
    d = sc.grid.dim
    ref = oracle.p2g(sc)
    u = random_u(ref.active, d, 2e-3 * sc.grid.dx, 7)
    dv = np.random.default_rng(8).normal(size=u.shape) * sc.grid.dx
    outs = []
    for rep in range(2):
        sub = make_sub(ctx, sc)
        sub.p2g()
        g, E = sub.newton_gradient(u)
        outs.append((g, E, sub.newton_diag(), sub.newton_hvp(dv), sub.newton_hvp(dv)))
    (g1, E1, d1, y1, y1b), (g2, E2, d2, y2, _) = outs
    assert np.array_equal(g1, g2) and E1 == E2 and np.array_equal(d1, d2)
    assert np.array_equal(y1, y1b) and np.array_equal(y1, y2)
    assert rel_linf(g1, oracle.gradient(sc, ref, u)) <= TOL
    assert rel_linf(d1, oracle.diag(sc, ref, u)) <= TOL
    assert rel_linf(y1, oracle.hvp(sc, ref, u, dv)) <= TOL
    vs = []
    for rep in range(2):
        sub = make_sub(ctx, sc)
        sub.p2g()
        sub.implicit_solve(osmpm.newton_settings(max_newton=3, max_cg=20, fixed_iters=1))
        vs.append(sub.read_grid_velocity())
    assert np.array_equal(vs[0], vs[1])


@pytest.mark.parametrize("n,nbits", [(0, 8), (1, 3), (4095, 8), (4097, 13), (100003, 22), (1 << 20, 22),
                                     (300000, 2), (70000, 32)])
def test_radix_sort_is_a_stable_sort(ctx, n, nbits):
    """a1: the hand-written radix sort equals numpy's stable argsort bit for bit (keys and the order of
    equal keys), on the low nbits bits, for empty / single / ragged / multi-tile sizes."""
    from paper_2605_09097_b200 import osmpm
    rng = np.random.default_rng(n + nbits)
    hi = min(1 << nbits, 1 << 32) if nbits < 32 else 1 << 32
    keys = rng.integers(0, hi, size=n, dtype=np.uint64).astype(np.uint32)
    if n > 10:
        keys[: n // 3] = keys[n // 3]  # many equal keys: stability matters
    vals = np.arange(n, dtype=np.int32)
    k, v = keys.copy(), vals.copy()
    osmpm.sort_pairs(ctx, k, v, nbits)
    masked = keys & np.uint32((1 << nbits) - 1 if nbits < 32 else 0xFFFFFFFF)
    order = np.argsort(masked, kind="stable")
    assert np.array_equal(v, vals[order]) and np.array_equal(k, keys[order])


@pytest.mark.parametrize("dim", [2, 3])
def test_psd_projected_solve_parity(ctx, dim):
    """R23: Newton-PCG with the PSD-projected tangent blocks (psd = 2) on an indefinite compressed state,
    against the oracle running the same projection: fixed 4 x 30 at 1e-8 (the converged-solve bar: the
    clamp of near-zero eigenvalues and the two Jacobi eigen-solvers' rounding enter every HVP of a badly
    conditioned system, measured 6e-9 in 2D), same counts (no negative curvature); and psd = 1 equals the
    exact-tangent solve there (no direction failed the descent check)."""
    from paper_2605_09097_b200 import osmpm
    sc = synth.random_fixture(dim=dim, cells=(4, 4, 1) if dim == 2 else (3, 3, 3), seed=59, F_sigma=0.0)
    sc.particles.F[:] = 0.3 * np.eye(dim)
    sc.dt = 1.0
    ref = oracle.p2g(sc)
    act = ref.active.astype(bool)
    for psd in (2, 1):
        kw = dict(max_newton=4, max_cg=30, fixed_iters=1, guess=1, psd=psd)
        u_ref, st_ref = oracle.implicit_solve(sc, ref, oracle.default_settings(**kw), raise_on_error=False)
        sub = make_sub(ctx, sc)
        sub.p2g()
        st = sub.implicit_solve(osmpm.newton_settings(**kw), raise_on_error=False)
        assert st.status == 0 and st_ref.status == 0
        assert st.psd_solves == st_ref.psd_solves and st.negcurv == st_ref.negcurv and st.cg_iters == st_ref.cg_iters
        assert rel_linf(sub.read_grid_velocity(), np.where(act[:, None], u_ref / sc.dt, 0.0)) <= 1e-8
        sub.close()


def test_solved_velocity_readable_until_next_p2g(ctx):
    """osmpm_read_grid_velocity after osmpm_g2p returns the velocity the particles moved with; after the
    next P2G there is no solved velocity until the next solve (STATE)."""
    from paper_2605_09097_b200 import osmpm
    sc = synth.random_fixture(dim=3, cells=(4, 4, 3), seed=141)
    sub = make_sub(ctx, sc)
    sub.p2g()
    sub.implicit_solve(osmpm.newton_settings(max_newton=2, max_cg=20, fixed_iters=1))
    v0 = sub.read_grid_velocity()
    assert np.abs(v0).max() > 0
    sub.g2p()
    np.testing.assert_array_equal(sub.read_grid_velocity(), v0)
    sub.p2g()
    with pytest.raises(osmpm.OsmpmError) as e:
        sub.read_grid_velocity()
    assert e.value.code == 11
    sub.close()
