"""GPU parity of the Schwarz coupler (Alg. 1) against the oracle frame:
receiver sets, a full frame in parity mode (fixed K, tight Newton / PCG tolerances; fp64 bar 1e-8 on
displacements), exact translation, and the sub-step API contract."""
import numpy as np
import pytest

import oracle
import synth
from oracle import schwarz as OS
from gpu_helpers import make_sub, rel_linf

pytestmark = pytest.mark.gpu

TIGHT = dict(newton_rtol=1e-12, cg_rtol=1e-12, max_cg=20000, max_newton=50)


@pytest.fixture(scope="module")
def ctx():
    from paper_2605_09097_b200 import osmpm
    c = osmpm.Context(0)
    yield c
    c.close()


def _clamp(scene):
    xs, _ = OS.node_positions(scene.grid)
    sel = np.flatnonzero(xs[:, 0] <= 1e-12)
    return sel


def _gpu_frame(ctx, coarse, fine, M, K, clamp_fine=None):
    from paper_2605_09097_b200 import osmpm
    sb = make_sub(ctx, coarse)
    ss = make_sub(ctx, fine)
    if clamp_fine is not None and len(clamp_fine):
        ss.set_dirichlet(clamp_fine, np.full(len(clamp_fine), 3, np.uint8), np.zeros((len(clamp_fine), 2)))
    st = osmpm.schwarz_settings(M=M, parity_fixed_k=K, eps_tol=-1.0, coarse=osmpm.newton_settings(**TIGHT),
                                fine=osmpm.newton_settings(**TIGHT))
    cpl = osmpm.Coupler(sb, ss, st)
    rep = cpl.step()
    return sb, ss, rep, cpl


def test_cantilever_frame_parity(ctx):
    coarse, fine = synth.c1_cantilever()
    M, K = 4, 3
    sel = _clamp(fine)
    nn = oracle.n_nodes(fine.grid)
    mask = np.zeros((nn, 2), np.uint8)
    mask[sel] = 1
    ref = OS.schwarz_step(coarse, fine, M, parity_fixed_k=K, user_S=OS.UserBC(mask, np.zeros((nn, 2))),
                          newton_coarse=oracle.default_settings(**TIGHT), newton_fine=oracle.default_settings(**TIGHT))
    sb, ss, rep, _ = _gpu_frame(ctx, coarse, fine, M, K, clamp_fine=sel)
    assert rep.n_recv_B == ref.n_recv_B and rep.n_recv_S == ref.n_recv_S
    assert rep.iters == K and rep.fine_substeps == K * M
    fo = ss.read_particles()
    co = sb.read_particles()
    for out, r, x0 in ((fo, ref.fine_particles, fine.particles.x), (co, ref.coarse_particles, coarse.particles.x)):
        assert rel_linf(out["x"] - x0, r.x - x0) <= 1e-8
        assert rel_linf(out["v"], r.v) <= 1e-8
        assert rel_linf(out["F"], r.F) <= 1e-8
    np.testing.assert_allclose(np.array(rep.r_B[:K]), np.array(ref.r_B), rtol=1e-6, atol=1e-12)
    np.testing.assert_allclose(np.array(rep.r_S[:K]), np.array(ref.r_S), rtol=1e-6, atol=1e-12)


def test_translation_frame_exact(ctx):
    c = np.array([0.3, -0.2])
    coarse, fine = synth.c1_cantilever(g=0.0)
    for sc in (coarse, fine):
        sc.particles.v[:] = c
    fine.dt = coarse.dt / 4
    sb, ss, rep, _ = _gpu_frame(ctx, coarse, fine, 4, 2)
    for sub, sc in ((sb, coarse), (ss, fine)):
        out = sub.read_particles()
        np.testing.assert_allclose(out["v"], np.tile(c, (sc.particles.n, 1)), rtol=0, atol=1e-10)
        np.testing.assert_allclose(out["x"], sc.particles.x + coarse.dt * c, rtol=0, atol=1e-12)


def test_substep_contract(ctx):
    from paper_2605_09097_b200 import osmpm
    coarse, fine = synth.c1_cantilever()
    sb = make_sub(ctx, coarse)
    ss = make_sub(ctx, fine)
    cpl = osmpm.Coupler(sb, ss, osmpm.schwarz_settings(M=4))
    with pytest.raises(osmpm.OsmpmError):
        cpl.substep(1)          # before prepare
    cpl.prepare()
    with pytest.raises(osmpm.OsmpmError) as ei:
        cpl.substep(5)          # m > M
    assert ei.value.code == 1
    with pytest.raises(osmpm.OsmpmError):
        cpl.substep(1)          # the coarse solve of this iteration has not run yet
    sb.implicit_solve(osmpm.newton_settings(**TIGHT))
    for m in range(1, 5):
        st = cpl.substep(m)
        assert st.status == 0


@pytest.mark.parametrize("M", [2, 4])
def test_free_fall_is_the_converged_frame(ctx, M):
    """The GPU frame converges to backward-Euler free fall on both grids (the fixed point exists only
    with alpha = m / M in the temporal interpolation; tests/test_oracle_schwarz.py)."""
    from paper_2605_09097_b200 import osmpm
    import test_oracle_schwarz as TOS
    coarse, fine, c, g = TOS._falling_pair(M)
    sb = make_sub(ctx, coarse)
    ss = make_sub(ctx, fine)
    st = osmpm.schwarz_settings(M=M, eps_conv=1e-10, k_max=200, eps_tol=-1.0,
                                coarse=osmpm.newton_settings(**TIGHT), fine=osmpm.newton_settings(**TIGHT))
    rep = osmpm.Coupler(sb, ss, st).step()
    assert rep.iters < 60
    for sub, sc, n in ((ss, fine, M), (sb, coarse, 1)):
        out = sub.read_particles()
        x, v = TOS.free_fall_closed_form(sc.particles.x, c, g, sc.dt, n)
        np.testing.assert_allclose(out["v"], np.tile(v, (sc.particles.n, 1)), rtol=0, atol=1e-8)
        np.testing.assert_allclose(out["x"], x, rtol=0, atol=1e-10)
