"""Pins of oracle O4 (energy/gradient), O5 (HVP), O6 (Jacobi diagonal) and O7 (Newton-PCG)
against finite differences, exact completeness identities, brute force and special cases
(SURVEY.md §8(c).3 rows O4-O7)."""
import numpy as np
import pytest

import oracle
import synth


def _setup(dim, seed, cells=(3, 3, 2), u_scale=1e-3, **kw):
    sc = synth.random_fixture(dim=dim, seed=seed, cells=cells, **kw)
    gs = oracle.p2g(sc)
    rng = np.random.default_rng(seed + 100)
    act = gs.active.astype(bool)
    u = np.zeros_like(gs.v)
    u[act] = rng.normal(0.0, u_scale * sc.grid.dx, size=(act.sum(), dim))
    return sc, gs, u, act, rng


def _nodes(grid):
    d = grid.dim
    shp = oracle.node_shape(grid)
    k = np.stack(np.meshgrid(*[np.arange(s) for s in shp], indexing="ij"), -1).reshape(-1, d)
    return np.asarray(grid.origin[:d]) + k * grid.dx


@pytest.mark.parametrize("dim", [2, 3])
def test_gradient_is_energy_derivative(dim):
    sc, gs, u, act, rng = _setup(dim, 41)
    g = oracle.gradient(sc, gs, u)
    dvec = np.zeros_like(u)
    dvec[act] = rng.normal(size=(act.sum(), dim)) * sc.grid.dx
    an = (g * dvec).sum()
    errs = []
    for eps in (1e-4, 1e-5):
        ep, _ = oracle.energy(sc, gs, u + eps * dvec)
        em, _ = oracle.energy(sc, gs, u - eps * dvec)
        errs.append(abs((ep - em) / (2 * eps) / an - 1.0))
    # central differences converge as O(eps^2) to the analytic directional derivative
    assert errs[1] < 2e-7 and errs[1] < errs[0] / 50


@pytest.mark.parametrize("dim", [2, 3])
def test_hvp_is_gradient_derivative(dim):
    sc, gs, u, act, rng = _setup(dim, 42)
    dvec = np.zeros_like(u)
    dvec[act] = rng.normal(size=(act.sum(), dim)) * sc.grid.dx
    y = oracle.hvp(sc, gs, u, dvec)
    errs = []
    for eps in (1e-4, 1e-5):
        fd = (oracle.gradient(sc, gs, u + eps * dvec) - oracle.gradient(sc, gs, u - eps * dvec)) / (2 * eps)
        errs.append(np.abs(fd - y).max() / np.abs(y).max())
    # O(eps^2) convergence of the central difference
    assert errs[1] < 2e-8 and (errs[1] < errs[0] / 50 or errs[1] < 1e-11)


@pytest.mark.parametrize("dim", [2, 3])
def test_hvp_symmetry_and_positivity(dim):
    sc, gs, u, act, rng = _setup(dim, 43)
    a = np.zeros_like(u)
    b = np.zeros_like(u)
    a[act] = rng.normal(size=(act.sum(), dim))
    b[act] = rng.normal(size=(act.sum(), dim))
    ha = oracle.hvp(sc, gs, u, a)
    hb = oracle.hvp(sc, gs, u, b)
    assert (b * ha).sum() == pytest.approx((a * hb).sum(), rel=1e-13)
    assert (a * ha).sum() > 0


@pytest.mark.parametrize("dim", [2, 3])
def test_hvp_completeness_identities(dim):
    sc, gs, u, act, rng = _setup(dim, 44)
    d = dim
    xi = _nodes(sc.grid)
    pt = sc.particles
    mdt = gs.m[:, None] / sc.dt ** 2
    # (i) translations are in the null space of K; (ii) Σ_i (Kd)_i = 0 for any d
    c = rng.normal(size=d)
    K_c = oracle.hvp(sc, gs, u, np.tile(c, (xi.shape[0], 1))) - mdt * c
    dv = rng.normal(size=u.shape)
    y = oracle.hvp(sc, gs, u, dv)
    Kd = y - mdt * dv
    assert np.abs(K_c).max() <= 1e-12 * np.abs(Kd).max()
    assert np.abs(Kd.sum(axis=0)).max() <= 1e-12 * np.abs(Kd).max()
    # (iii) affine d_i = A x_i + c: dF_p = A F_p^n, Σ_i (Kd)_i x_i^T = Σ_p V0 dP(F_p(u); A F_p^n) F_p^nT
    A = rng.normal(size=(d, d))
    da = xi @ A.T + c
    Kda = oracle.hvp(sc, gs, u, da) - mdt * da
    lhs = Kda.T @ xi
    rhs = np.zeros((d, d))
    for p in range(pt.n):
        st = oracle.stencil(sc.grid, pt.x[p])
        idx, N, gN, xip = st
        Fu = (np.eye(d) + u[idx].T @ gN) @ pt.F[p]
        mu, lam = oracle.lame(*sc.materials[pt.mat[p]])
        rhs += pt.V0[p] * oracle.dP(Fu, A @ pt.F[p], mu, lam) @ pt.F[p].T
    np.testing.assert_allclose(lhs, rhs, rtol=1e-11, atol=1e-12 * np.abs(rhs).max())


@pytest.mark.parametrize("dim", [2, 3])
def test_hvp_rest_rotations(dim):
    # (iv) at rest (F^n = I, u = 0) infinitesimal rotations d_i = W x_i (W skew) give K d = 0
    sc = synth.random_fixture(dim=dim, seed=45, cells=(3, 3, 2), F_sigma=0.0)
    gs = oracle.p2g(sc)
    xi = _nodes(sc.grid)
    rng = np.random.default_rng(1)
    W = rng.normal(size=(dim, dim))
    W = W - W.T
    dv = xi @ W.T
    Kd = oracle.hvp(sc, gs, np.zeros_like(gs.v), dv) - gs.m[:, None] / sc.dt ** 2 * dv
    ref = oracle.hvp(sc, gs, np.zeros_like(gs.v), xi @ (W + W.T + np.eye(dim)).T)
    assert np.abs(Kd).max() <= 1e-12 * np.abs(ref).max()


def test_hvp_mass_only_when_no_stiffness():
    # mu = lam = 0 (E = 0) -> H d = (m / dt^2) d exactly
    sc = synth.random_fixture(dim=3, seed=46, cells=(3, 2, 2), materials=[(0.0, 0.3), (0.0, 0.3)])
    gs = oracle.p2g(sc)
    dv = np.random.default_rng(2).normal(size=gs.v.shape)
    y = oracle.hvp(sc, gs, np.zeros_like(gs.v), dv)
    np.testing.assert_array_equal(y, gs.m[:, None] / sc.dt ** 2 * dv)


@pytest.mark.parametrize("dim", [2, 3])
def test_diag_brute_force(dim):
    sc, gs, u, act, rng = _setup(dim, 47, cells=(2, 2, 2))
    dg = oracle.diag(sc, gs, u)
    d = dim
    nodes = np.flatnonzero(act)
    sel = rng.choice(nodes, size=min(25, nodes.size), replace=False)
    for i in sel:
        for a in range(d):
            e = np.zeros_like(u)
            e[i, a] = 1.0
            h = oracle.hvp(sc, gs, u, e)
            assert dg[i, a] == pytest.approx(h[i, a], rel=1e-13)


def _settings(**kw):
    base = dict(newton_rtol=1e-12, cg_rtol=1e-12, max_cg=2000, max_newton=50)
    base.update(kw)
    return oracle.default_settings(**base)


def test_newton_all_dirichlet():
    sc = synth.random_fixture(dim=2, seed=48, cells=(3, 3, 1))
    gs = oracle.p2g(sc)
    vD = np.random.default_rng(3).normal(size=gs.v.shape)
    u, st = oracle.implicit_solve(sc, gs, _settings(), dirichlet_mask=np.ones(gs.v.shape, np.uint8),
                                  dirichlet_v=vD)
    act = gs.active.astype(bool)
    np.testing.assert_array_equal(u[act], sc.dt * vD[act])
    assert st.cg_iters == 0


@pytest.mark.parametrize("dim", [2, 3])
def test_newton_free_fall_without_stiffness(dim):
    # no elasticity: the minimiser is xhat = xtilde + dt^2 g, i.e. v^{n+1} = v^n + dt g
    sc = synth.random_fixture(dim=dim, seed=49, cells=(2, 2, 2), materials=[(0.0, 0.3), (0.0, 0.3)])
    gs = oracle.p2g(sc)
    u, st = oracle.implicit_solve(sc, gs, _settings())
    act = gs.active.astype(bool)
    vnew = u / sc.dt
    np.testing.assert_allclose(vnew[act], gs.v[act] + sc.dt * np.asarray(sc.gravity[:dim]), rtol=0, atol=1e-12)


def test_newton_matches_brute_force_minimiser():
    # a few dozen unknowns: Newton-PCG + line search reaches the minimiser of E_h found by an
    # independent dense brute-force Newton whose Hessian is built column by column from central
    # differences of the gradient (no HVP, no PCG), with a dense direct solve.
    sc = synth.random_fixture(dim=2, seed=50, cells=(2, 2, 1), ppa=2, dt=5e-3, v_sigma=0.3)
    gs = oracle.p2g(sc)
    act = gs.active.astype(bool)
    nfree = act.sum() * 2
    assert nfree <= 60
    u_n, st = oracle.implicit_solve(sc, gs, _settings())
    assert st.status == 0

    def grad(z):
        u = np.zeros_like(gs.v)
        u[act] = z.reshape(-1, 2)
        return oracle.gradient(sc, gs, u)[act].ravel()

    def energy(z):
        u = np.zeros_like(gs.v)
        u[act] = z.reshape(-1, 2)
        return oracle.energy(sc, gs, u)[0]

    z = (sc.dt * gs.v[act]).ravel()
    h = 1e-7
    for _ in range(60):
        g = grad(z)
        if np.linalg.norm(g) < 1e-9 * st.grad_norm0:
            break
        H = np.zeros((z.size, z.size))
        for k in range(z.size):
            e = np.zeros_like(z)
            e[k] = h
            H[:, k] = (grad(z + e) - grad(z - e)) / (2 * h)
        step = np.linalg.solve(0.5 * (H + H.T), -g)
        a = 1.0
        while not energy(z + a * step) < energy(z) and a > 1e-6:
            a *= 0.5
        z = z + a * step
    scale = np.abs(u_n[act]).max()
    assert np.abs(z.reshape(-1, 2) - u_n[act]).max() <= 1e-8 * scale


@pytest.mark.parametrize("dim", [2, 3])
def test_newton_energy_decreases_and_converges(dim):
    sc = synth.random_fixture(dim=dim, seed=51, cells=(3, 3, 2), F_sigma=0.1, v_sigma=1.0)
    gs = oracle.p2g(sc)
    energies = []
    for k in range(1, 6):
        u, st = oracle.implicit_solve(sc, gs, _settings(max_newton=k), raise_on_error=False)
        energies.append(oracle.energy(sc, gs, u)[0])
    assert all(b <= a * (1 + 1e-13) + 1e-13 * abs(a) for a, b in zip(energies, energies[1:]))
    u, st = oracle.implicit_solve(sc, gs, _settings())
    assert st.status == 0
    g = oracle.gradient(sc, gs, u)
    act = gs.active.astype(bool)
    assert np.linalg.norm(g[act]) <= 1e-12 * st.grad_norm0 * 1.0001


def test_newton_fixed_iterations_runs_exact_count():
    sc = synth.random_fixture(dim=3, seed=52, cells=(2, 2, 2))
    gs = oracle.p2g(sc)
    st_set = oracle.default_settings(max_newton=3, max_cg=7, fixed_iters=1)
    u, st = oracle.implicit_solve(sc, gs, st_set)
    assert st.newton_iters == 3 and st.cg_iters == 21


def test_newton_accepts_the_energy_roundoff_floor():
    """R8: near the static limit (dt = 10 s, Dirichlet band, tiny load) the backtracking line search can
    no longer resolve a decrease of E_h; once |g| <= sqrt(rtol) * max(|g0|, f_s) the iterate is accepted as
    converged instead of failing with LINESEARCH_STAGNATION (this coarse solve of the quasi-static
    cantilever frame stalls at |g| / |g0| ~ 1.3e-6 with rtol = 1e-8)."""
    import os
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "scripts"))
    import eb_cantilever as eb
    from oracle import schwarz as OS
    D = eb.E * eb.H ** 3 / (12 * (1 - eb.NU ** 2))
    g = 0.05 * D / (eb.RHO * eb.H * eb.L ** 3)
    coarse, fine = synth.c1_cantilever(g=g)
    coarse.dt, fine.dt = 1.0, 0.25
    gsB, gsS = oracle.p2g(coarse), oracle.p2g(fine)
    hatB, _ = OS.receivers(coarse, fine, gsB, gsS, 1e-6)
    nn = gsB.m.shape[0]
    mask = np.zeros((nn, 2), np.uint8)
    mask[hatB] = 1
    st = oracle.default_settings(newton_rtol=1e-8, cg_rtol=1e-10, max_cg=20000, max_newton=40)
    u, s = oracle.implicit_solve(coarse, gsB, st, dirichlet_mask=mask, dirichlet_v=np.zeros((nn, 2)),
                                 raise_on_error=False)
    assert s.status == 0 and s.ls_halvings > 0
    assert s.grad_norm <= 1e-4 * s.grad_norm0 and s.grad_norm > 1e-8 * s.grad_norm0
    assert s.floor_accept == 1  # the loosened acceptance is reported, never silent
    # a solve that reaches newton_rtol does not raise the flag
    sc = synth.random_fixture(dim=2, seed=57, cells=(4, 3, 1))
    _, s2 = oracle.implicit_solve(sc, oracle.p2g(sc), oracle.default_settings(newton_rtol=1e-10, cg_rtol=1e-12))
    assert s2.status == 0 and s2.floor_accept == 0


def test_fixed_mode_line_search_failure_takes_zero_step():
    """R8 fixed-iteration policy: when no trial step decreases E_h (forced here by max_cg = 0, i.e. a
    zero Newton direction, and a negative noise tolerance, so that no trial is ever accepted), the
    solve neither errors nor moves: alpha = 0 is taken, every such iteration is counted, and u stays
    at the initial guess x^ = x~ (u = dt v^n on free DOFs)."""
    sc = synth.random_fixture(dim=3, seed=58, cells=(3, 2, 2))
    gs = oracle.p2g(sc)
    st = oracle.default_settings(max_newton=4, max_cg=0, fixed_iters=1, energy_noise_rtol=-1.0)
    u, s = oracle.implicit_solve(sc, gs, st)
    act = gs.active.astype(bool)
    assert s.status == 0 and s.ls_failures == 4 and s.newton_iters == 4 and s.ls_halvings == 4 * 21
    assert np.array_equal(u[act], sc.dt * gs.v[act])
    # the same settings in tolerance mode are a LINESEARCH_STAGNATION error
    _, s3 = oracle.implicit_solve(sc, gs, oracle.default_settings(max_cg=0, energy_noise_rtol=-1.0),
                                  raise_on_error=False)
    assert s3.status == oracle.LS_STAGNATION and s3.ls_failures == 0


def test_fixed_mode_negative_curvature_stops_pcg():
    """R7: p^T H p <= 0 stops PCG in both modes.  A strongly compressed state (F = 0.3 I, so that
    mu - lambda ln J > mu s^2) makes the neo-Hookean tangent indefinite for rotation-like modes; from
    u = 0 (guess 1) the Krylov directions meet it and the event is counted, in fixed mode as well, with
    the PCG iterations cut short (fewer than the 2 x 30 a fixed solve would otherwise run)."""
    sc = synth.random_fixture(dim=2, seed=59, cells=(4, 4, 1), F_sigma=0.0)
    sc.particles.F[:] = np.diag([0.3, 0.3])
    sc.dt = 1.0
    gs = oracle.p2g(sc)
    for fixed in (1, 0):
        u, s = oracle.implicit_solve(sc, gs, oracle.default_settings(max_newton=2, max_cg=30, fixed_iters=fixed,
                                                                     guess=1), raise_on_error=False)
        assert s.negcurv >= 1 and s.cg_iters < 60
        if fixed:
            assert s.status == 0 and s.newton_iters == 2


@pytest.mark.parametrize("dim", [2, 3])
def test_single_reduction_pcg_matches_standard_pcg(dim):
    """R22: the single-reduction PCG (Chronopoulos-Gear) produces the standard PCG's Krylov iterates
    (identical in exact arithmetic): fixed 3 x 20 solves agree to round-off, converged solves to the
    tolerance, and both report the same counts."""
    sc = synth.random_fixture(dim=dim, seed=61, cells=(4, 3, 3) if dim == 3 else (7, 5, 1))
    gs = oracle.p2g(sc)
    u0, s0 = oracle.implicit_solve(sc, gs, oracle.default_settings(max_newton=3, max_cg=20, fixed_iters=1))
    u1, s1 = oracle.implicit_solve(sc, gs, oracle.default_settings(max_newton=3, max_cg=20, fixed_iters=1,
                                                                   cg_variant=1))
    act = gs.active.astype(bool)
    scale = np.abs(u0[act]).max()
    assert np.abs(u1[act] - u0[act]).max() <= 1e-10 * scale
    assert s1.cg_iters == s0.cg_iters == 60 and s1.newton_iters == 3
    kw = dict(newton_rtol=1e-12, cg_rtol=1e-12, max_cg=4000)
    uc0, c0 = oracle.implicit_solve(sc, gs, oracle.default_settings(**kw))
    uc1, c1 = oracle.implicit_solve(sc, gs, oracle.default_settings(cg_variant=1, **kw))
    assert c0.status == c1.status == 0
    assert np.abs(uc1[act] - uc0[act]).max() <= 1e-9 * np.abs(uc0[act]).max()


def test_single_reduction_pcg_special_cases():
    """mu = lambda = 0: H = M / dt^2 is the Jacobi preconditioner itself, so one PCG iteration solves
    the Newton system exactly (free fall: v^{n+1} = v^n + dt g) -- in both variants; the
    indefinite tangent of test_fixed_mode_negative_curvature_stops_pcg stops both at the same point."""
    sc = synth.random_fixture(dim=2, seed=62, cells=(5, 4, 1))
    sc.materials = [(0.0, 0.3), (0.0, 0.3)]
    sc.gravity = (0.3, -9.81, 0.0)
    gs = oracle.p2g(sc)
    u, s = oracle.implicit_solve(sc, gs, oracle.default_settings(cg_variant=1, newton_rtol=1e-13, cg_rtol=1e-14))
    act = gs.active.astype(bool)
    v = u[act] / sc.dt
    np.testing.assert_allclose(v, gs.v[act] + sc.dt * np.array([0.3, -9.81]), rtol=0, atol=1e-12)
    sc2 = synth.random_fixture(dim=2, seed=59, cells=(4, 4, 1), F_sigma=0.0)
    sc2.particles.F[:] = np.diag([0.3, 0.3])
    sc2.dt = 1.0
    gs2 = oracle.p2g(sc2)
    out = []
    for var in (0, 1):
        _, st = oracle.implicit_solve(sc2, gs2, oracle.default_settings(max_newton=2, max_cg=30, fixed_iters=1,
                                                                        guess=1, cg_variant=var),
                                      raise_on_error=False)
        out.append((st.negcurv, st.cg_iters))
    assert out[0] == out[1] and out[0][0] >= 1


def _tangent_columns(F, E, nu):
    d = F.shape[0]
    mu, lam = oracle.lame(E, nu)
    T = np.zeros((d * d, d * d))
    for k in range(d * d):
        e = np.zeros(d * d)
        e[k] = 1.0
        T[:, k] = oracle.dP(F, e.reshape(d, d), mu, lam).reshape(-1)
    return T


@pytest.mark.parametrize("dim", [2, 3])
def test_psd_projection_of_the_tangent_block(dim):
    """R23: T+ is the nearest PSD matrix to the tangent block T = d^2 Psi / dF dF (whose
    columns come from the pinned oracle.dP): on a stretched state where T is positive definite T+ = T;
    on a strongly compressed, indefinite state T+ equals the eigen-clamp computed independently with
    numpy's symmetric eigensolver, and is PSD."""
    rng = np.random.default_rng(71 + dim)
    S = rng.normal(size=(dim, dim))
    F = 1.05 * np.eye(dim) + 0.005 * (S + S.T)
    T = _tangent_columns(F, 1e5, 0.3)
    assert np.linalg.eigvalsh(0.5 * (T + T.T)).min() > 0
    np.testing.assert_allclose(oracle.tangent_psd(F, 1e5, 0.3), T, rtol=0, atol=1e-10 * np.abs(T).max())
    F = 0.3 * np.eye(dim) + 0.01 * rng.normal(size=(dim, dim))
    T = _tangent_columns(F, 1e5, 0.3)
    w, V = np.linalg.eigh(0.5 * (T + T.T))
    assert w.min() < 0
    ref = (V * np.maximum(w, 0.0)) @ V.T
    Tp = oracle.tangent_psd(F, 1e5, 0.3)
    np.testing.assert_allclose(Tp, ref, rtol=0, atol=1e-12 * np.abs(ref).max())
    assert np.linalg.eigvalsh(Tp).min() >= -1e-12 * np.abs(w).max()


def test_psd_hvp_and_solve():
    """R23: on a stretched (convex) state the projected HVP equals the exact one; on the indefinite
    compressed state the projected operator is PSD above the mass term (d^T H d >= d^T M d / dt^2), PCG
    meets no negative curvature and Newton lowers E_h further than with the exact tangent; psd = 1
    (projection only when the first direction is not a descent direction) reproduces psd = 0 there,
    since a positive Jacobi diagonal keeps truncated PCG directions descent directions."""
    sc = synth.random_fixture(dim=2, seed=63, cells=(4, 4, 1), F_sigma=0.0)
    sc.particles.F[:] = 1.05 * np.eye(2)
    gs = oracle.p2g(sc)
    rng = np.random.default_rng(5)
    u = np.zeros_like(gs.v)
    act = gs.active.astype(bool)
    u[act] = rng.normal(0, 1e-4 * sc.grid.dx, size=(act.sum(), 2))
    dv = rng.normal(size=u.shape)
    h0, h1 = oracle.hvp(sc, gs, u, dv), oracle.hvp(sc, gs, u, dv, psd=True)
    np.testing.assert_allclose(h1, h0, rtol=0, atol=1e-9 * np.abs(h0).max())
    sc2 = synth.random_fixture(dim=2, seed=59, cells=(4, 4, 1), F_sigma=0.0)
    sc2.particles.F[:] = np.diag([0.3, 0.3])
    sc2.dt = 1.0
    gs2 = oracle.p2g(sc2)
    act2 = np.repeat(gs2.active.astype(bool)[:, None], 2, axis=1)
    for k in range(3):
        d = np.where(act2, rng.normal(size=gs2.v.shape), 0.0)
        Hd = oracle.hvp(sc2, gs2, np.zeros_like(gs2.v), d, psd=True)
        mass = (gs2.m[:, None] * d * d).sum() / sc2.dt ** 2
        assert (d * Hd).sum() >= mass * (1 - 1e-12)
    res = {}
    for psd in (0, 1, 2):
        u, s = oracle.implicit_solve(sc2, gs2, oracle.default_settings(max_newton=4, max_cg=30, fixed_iters=1,
                                                                       guess=1, psd=psd), raise_on_error=False)
        res[psd] = (u, s)
    assert res[2][1].negcurv == 0 and res[2][1].psd_solves == 4 and res[2][1].status == 0
    assert res[0][1].negcurv > 0 and res[0][1].psd_solves == 0
    assert res[2][1].energy < res[0][1].energy
    assert res[1][1].psd_solves == 0 and np.array_equal(res[1][0], res[0][0])
