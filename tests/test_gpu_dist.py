"""GPU parity of the slab decomposition.

The fine subdomain is split into G x-slabs ON ONE GPU (osmpm_ctx_set_local_slabs: the same slab
layout, ghost-plane halo exchange, owned-node reductions and particle migration as the multi-GPU
path, with device copies in place of NCCL).  Every kernel output must equal the oracle at the
per-kernel tolerance, and the decomposed solve / G2P / migration must reproduce the undecomposed
subdomain (only the fp atomic order differs).

Cases marked `nccl` join a one-rank NCCL communicator first (osmpm_ctx_init_comm with nranks = 1): the
subdomain then takes the multi-rank code path, so the all-reduces of the PCG scalars and of the
Newton / migration bounds, the all-gather of the halo records and the coupler's broadcast and
all-reduces run through NCCL on the GPU (neighbour exchanges find no neighbour)."""
import numpy as np
import pytest

import oracle
import synth
from gpu_helpers import random_u, rel_linf

pytestmark = pytest.mark.gpu

TOL = 1e-11
FIX = {
    # x-extents of several tile columns (3D tile edge 4 cells, 2D 16 cells) so that 2-4 slabs fit
    "3d": dict(dim=3, cells=(26, 7, 6), seed=301),
    "2d": dict(dim=2, cells=(70, 9, 1), seed=302),
    # 8 slabs (G = 8): 11 tile columns
    "3d8": dict(dim=3, cells=(44, 6, 5), seed=303),
}


def _ctx(slabs, nccl=False):
    from paper_2605_09097_b200 import osmpm
    c = osmpm.Context(0)
    if nccl:
        c.init_comm(0, 1, osmpm.comm_unique_id())
    if slabs > 1:
        c.set_local_slabs(slabs)
    return c


def _sub(ctx, sc, decompose=True):
    from paper_2605_09097_b200 import osmpm
    return osmpm.Subdomain(ctx, sc.grid, sc.dt, sc.particles, sc.materials, sc.gravity, decompose=decompose)


@pytest.mark.parametrize("name,slabs,nccl", [("3d", 2, False), ("3d", 3, False), ("2d", 2, False), ("2d", 4, False),
                                             ("3d8", 8, False), ("3d", 1, True), ("3d", 3, True), ("2d", 2, True)])
def test_decomposed_kernels_match_oracle(name, slabs, nccl):
    sc = synth.random_fixture(**FIX[name])
    d = sc.grid.dim
    ctx = _ctx(slabs, nccl)
    sub = _sub(ctx, sc)
    st, sl, fs, nl, cuts = sub.decomp()
    assert (st, sl, fs, nl) == (slabs, slabs, 0, sc.particles.n)
    assert len(cuts) == slabs - 1 and all(b > a for a, b in zip(cuts, cuts[1:]))
    ref = oracle.p2g(sc)
    sub.p2g()
    out = sub.read_grid()
    np.testing.assert_array_equal(out["active"], ref.active)
    for k in ("m", "p", "v", "fext", "fsig"):
        assert rel_linf(out[k], getattr(ref, k)) <= TOL, k
    u = random_u(ref.active, d, 2e-3 * sc.grid.dx, 7)
    g, E = sub.newton_gradient(u)
    assert rel_linf(g, oracle.gradient(sc, ref, u)) <= TOL
    E_ref, _ = oracle.energy(sc, ref, u)
    assert abs(E - E_ref) <= 1e-11 * max(abs(E_ref), 1.0)
    dv = np.random.default_rng(8).normal(size=u.shape)
    assert rel_linf(sub.newton_hvp(dv), oracle.hvp(sc, ref, u, dv)) <= TOL
    assert rel_linf(sub.newton_diag(), oracle.diag(sc, ref, u)) <= TOL
    sub.close()
    ctx.close()


@pytest.mark.parametrize("name,slabs,nccl", [("3d", 3, False), ("2d", 2, False), ("3d", 3, True), ("2d", 1, True)])
def test_decomposed_solve_matches_oracle_and_whole(name, slabs, nccl):
    from paper_2605_09097_b200 import osmpm
    sc = synth.random_fixture(**FIX[name])
    act = oracle.p2g(sc).active.astype(bool)
    kw = dict(newton_rtol=1e-12, cg_rtol=1e-12, max_cg=3000)
    # converged: against the oracle's Newton-PCG
    ctx = _ctx(slabs, nccl)
    sub = _sub(ctx, sc)
    sub.p2g()
    st = sub.implicit_solve(osmpm.newton_settings(**kw))
    v = sub.read_grid_velocity()
    u_ref, _ = oracle.implicit_solve(sc, oracle.p2g(sc), oracle.default_settings(**kw))
    assert rel_linf(v, np.where(act[:, None], u_ref / sc.dt, 0.0)) <= 1e-8
    # fixed iterations: against the undecomposed subdomain (same PCG, atomic order only)
    fixed = osmpm.newton_settings(max_newton=3, max_cg=40, fixed_iters=1)
    whole_ctx = _ctx(1)
    whole = _sub(whole_ctx, sc)
    res = []
    for s in (sub, whole):
        s.set_particles(x=sc.particles.x)
        s.p2g()
        s.implicit_solve(fixed)
        res.append(s.read_grid_velocity())
    assert rel_linf(res[0], res[1]) <= 1e-9
    assert st.newton_iters >= 1
    for s, c in ((sub, ctx), (whole, whole_ctx)):
        s.close()
        c.close()


@pytest.mark.parametrize("name,slabs,nccl", [("3d", 2, False), ("3d", 4, False), ("2d", 3, False), ("3d8", 8, False),
                                             ("3d", 2, True)])
def test_decomposed_single_reduction_pcg(name, slabs, nccl):
    """R22 over slabs: the single-reduction PCG (one reduction -- one all-reduce across ranks -- per
    iteration, curvature partials from every slab's HVP tiles) equals the oracle's single-reduction PCG
    (fixed 3 x 40 at 1e-9, converged at 1e-8) and the undecomposed subdomain."""
    from paper_2605_09097_b200 import osmpm
    sc = synth.random_fixture(**FIX[name])
    ref = oracle.p2g(sc)
    act = ref.active.astype(bool)
    for kw, tol in ((dict(max_newton=3, max_cg=40, fixed_iters=1), 1e-9),
                    (dict(newton_rtol=1e-12, cg_rtol=1e-12, max_cg=3000), 1e-8)):
        u_ref, st_ref = oracle.implicit_solve(sc, ref, oracle.default_settings(cg_variant=1, **kw))
        out = []
        for k in (slabs, 1):
            ctx = _ctx(k, nccl and k == slabs)
            sub = _sub(ctx, sc)
            sub.p2g()
            st = sub.implicit_solve(osmpm.newton_settings(cg_variant=1, **kw))
            assert st.status == 0
            if kw.get("fixed_iters"):
                assert st.cg_iters == st_ref.cg_iters == 120
            out.append(sub.read_grid_velocity())
            sub.close()
            ctx.close()
        v_ref = np.where(act[:, None], u_ref / sc.dt, 0.0)
        assert rel_linf(out[0], v_ref) <= tol and rel_linf(out[1], v_ref) <= tol
        assert rel_linf(out[0], out[1]) <= tol


@pytest.mark.parametrize("name,slabs,nccl", [("3d", 3, False), ("2d", 3, False), ("3d8", 8, False), ("3d", 3, True)])
def test_migration_conserves_and_matches_whole(name, slabs, nccl):
    """Advect every particle by ~1.3 cells along +x (uniform grid velocity) so that particles cross
    the cuts; particle count, mass and momentum are conserved exactly, states equal the whole
    subdomain's, and the next P2G is unchanged by the decomposition."""
    sc = synth.random_fixture(**dict(FIX[name], cells=tuple(FIX[name]["cells"])))
    d = sc.grid.dim
    n = sc.particles.n
    shift = 1.3 * sc.grid.dx
    outs = []
    for slabs_ in (slabs, 1):
        ctx = _ctx(slabs_, nccl and slabs_ == slabs)
        s = _sub(ctx, sc)
        s.p2g()
        nn = int(np.prod(sc.grid.dims[:d]))
        vel = np.zeros((nn, d))
        vel[:, 0] = shift / sc.dt
        s.set_grid_velocity(vel)
        s.g2p()
        s.sync()
        stt, _, _, nl, _ = s.decomp()
        assert nl == n
        parts = s.read_particles()
        s.p2g()
        grid = s.read_grid()
        outs.append((parts, grid))
        s.close()
        ctx.close()
    (pa, ga), (pb, gb) = outs
    for k in ("x", "v", "F", "B"):
        assert rel_linf(pa[k], pb[k]) <= 1e-13, k
    np.testing.assert_allclose(pa["x"][:, 0] - sc.particles.x[:, 0], shift, rtol=0, atol=1e-12)
    # conservation across the migration: total mass and momentum on the grid
    assert abs(ga["m"].sum() - sc.particles.m.sum()) <= 1e-12 * sc.particles.m.sum()
    assert rel_linf(ga["m"], gb["m"]) <= 1e-12
    assert rel_linf(ga["p"], gb["p"]) <= 1e-12
    np.testing.assert_array_equal(ga["active"], gb["active"])


def test_decomposed_projection_matches_whole():
    """Pi_{S->B} from a decomposed fine subdomain: every slab projects its owned
    nodes only, so the result equals the undecomposed projection."""
    from paper_2605_09097_b200 import osmpm
    sc = synth.random_fixture(**FIX["3d"])
    coarse_grid = synth.Grid(3, sc.grid.origin, sc.grid.dx * 4, tuple(max(3, (k + 3) // 4 + 1) for k in sc.grid.dims))
    cx = np.asarray(coarse_grid.origin) + coarse_grid.dx * np.array([[2.0, 2.0, 2.0]])
    cpart = synth.make_particles(cx, coarse_grid.dx ** 3, 1000.0)
    res = []
    for slabs in (3, 1):
        ctx = _ctx(slabs)
        f = _sub(ctx, sc)
        c = osmpm.Subdomain(ctx, coarse_grid, sc.dt, cpart, sc.materials, sc.gravity, decompose=False)
        f.p2g()
        c.p2g()
        res.append(osmpm.transmit(f, c, osmpm.FINE_TO_COARSE, alpha=0.0, eps_tol=1e-12))
        c.close()
        f.close()
        ctx.close()
    assert rel_linf(res[0], res[1]) <= 1e-12


@pytest.mark.parametrize("mode", ["fused", "pass", "loopback"])
@pytest.mark.parametrize("name,slabs", [("3d", 3), ("2d", 4), ("3d8", 8)])
def test_halo_modes(monkeypatch, mode, name, slabs):
    """R24: the HVP's fused halo (every slab RED-s the planes it shares with a neighbour into the
    neighbour's y too), the halo pass it replaces (OSMPM_FUSED_HALO=0), and the alternating-buffer /
    inbox-signal protocol of the multi-rank halo run between local slabs (OSMPM_HALO_LOOPBACK=1) give the
    oracle's HVP at 1e-11 and the oracle's fixed-iteration solves (both PCG variants) at 1e-9."""
    from paper_2605_09097_b200 import osmpm
    if mode == "pass":
        monkeypatch.setenv("OSMPM_FUSED_HALO", "0")
    if mode == "loopback":
        monkeypatch.setenv("OSMPM_HALO_LOOPBACK", "1")
    sc = synth.random_fixture(**FIX[name])
    d = sc.grid.dim
    ref = oracle.p2g(sc)
    act = ref.active.astype(bool)
    ctx = _ctx(slabs)
    sub = _sub(ctx, sc)
    sub.p2g()
    u = random_u(ref.active, d, 2e-3 * sc.grid.dx, 11)
    sub.newton_gradient(u)
    dv = np.random.default_rng(12).normal(size=u.shape)
    assert rel_linf(sub.newton_hvp(dv), oracle.hvp(sc, ref, u, dv)) <= TOL
    kw = dict(max_newton=3, max_cg=41, fixed_iters=1)  # odd: the alternating buffers end on y2
    for variant in (0, 1):
        u_ref, st_ref = oracle.implicit_solve(sc, ref, oracle.default_settings(cg_variant=variant, **kw))
        for rep in range(2):  # the second solve reuses the halo state (inbox counts, buffer identities)
            sub.set_particles(x=sc.particles.x)
            sub.p2g()
            st = sub.implicit_solve(osmpm.newton_settings(cg_variant=variant, **kw))
            assert st.status == 0 and st.cg_iters == st_ref.cg_iters
            v = sub.read_grid_velocity()
            assert rel_linf(v, np.where(act[:, None], u_ref / sc.dt, 0.0)) <= 1e-9, (variant, rep)
    sub.close()
    ctx.close()
