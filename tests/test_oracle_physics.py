"""Physics pin of the oracle's whole single-subdomain implicit step against a closed form the paper
fixes: the static cantilever under gravity in the Euler-Bernoulli (small-deflection) limit of the
elastica, tip deflection = Gamma L / 8 with Gamma = q L^3 / D, D = E h^3 / (12 (1 - nu^2))
(§4.1; tests/golden/g6_euler_bernoulli.txt).  One backward-Euler step with a time
step large enough that the inertia term vanishes: Newton-PCG then finds the static equilibrium of the
MPM discretisation (APIC P2G, neo-Hookean energy, B-spline gradients, clamp at x <= 0, G2P).  A
dropped or mis-signed term anywhere in energy / gradient / Hessian / G2P moves the tip far outside
the bands below; the discretisation error must shrink at first order under refinement."""
import os
import sys

import numpy as np
import pytest

from conftest import read_golden

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "scripts"))
import eb_cantilever as eb  # noqa: E402


def test_golden_matches_closed_form():
    L, h, E, nu, rho, g, gamma, tip = read_golden("g6_euler_bernoulli.txt")[0]
    D = E * h ** 3 / (12 * (1 - nu ** 2))
    assert gamma == pytest.approx(rho * g * h * L ** 3 / D, rel=1e-3)
    assert tip == pytest.approx(gamma * L / 8, rel=1e-6)
    assert (eb.L, eb.H, eb.E, eb.NU, eb.RHO) == (L, h, E, nu, rho)


def test_oracle_cantilever_converges_to_euler_bernoulli():
    tips = {}
    for dx in (0.05, 0.025):
        tip, ref, st = eb.run_oracle(dx)
        assert st.status == 0
        tips[dx] = tip / ref
    # MPM is a few % too flexible at 4 cells through the thickness, first order in dx
    assert 1.0 < tips[0.05] < 1.10
    assert 1.0 < tips[0.025] < 1.05
    assert (tips[0.05] - 1) / (tips[0.025] - 1) > 1.8


def test_oracle_cantilever_quasi_static():
    # the inertia term m / dt^2 no longer matters at dt = 10 s: dt = 20 s moves the tip by < 1 %
    t10, _, _ = eb.run_oracle(0.05)
    sc, idx, ref = eb.scene(0.05, dt=20.0)
    import oracle
    gs = oracle.p2g(sc)
    dm = np.zeros((oracle.n_nodes(sc.grid), 2), np.uint8)
    dm[idx] = 1
    u, st = oracle.implicit_solve(sc, gs, oracle.default_settings(newton_rtol=1e-10, cg_rtol=1e-10, max_cg=20000,
                                                                   max_newton=30),
                                  dirichlet_mask=dm, dirichlet_v=np.zeros((oracle.n_nodes(sc.grid), 2)),
                                  raise_on_error=False)
    act = gs.active.astype(bool)
    t20 = eb.tip_deflection(sc.particles.x, oracle.g2p(sc, np.where(act[:, None], u / sc.dt, 0.0)).x)
    assert abs(t20 - t10) / t10 < 0.01


# --------------------------------------------------------------------------------------------------
# Hertz line contact (§4.2; tests/golden/g7_hertz.txt), scripts/hertz.py: a
# semi-circular cylinder on a rigid frictionless plane under a body load of resultant F, static
# single-domain MPM with unilateral gap contact at the plane nodes.  The paper reports that the
# profile converges to the Hertz semi-ellipse "with the error reducing approximately linearly with
# mesh element size"; the oracle must do the same and its Richardson extrapolation
# must land on the closed-form half-width and peak pressure.
import hertz as hz  # noqa: E402


def test_hertz_golden_matches_closed_form():
    R, E, nu, F, b, pmax = read_golden("g7_hertz.txt")[0]
    assert (hz.R, hz.E, hz.NU, hz.F_LINE) == (R, E, nu, F)
    bb, pp = hz.hertz(F)
    assert bb == pytest.approx(b, rel=1e-6) and pp == pytest.approx(pmax, rel=1e-6)


def test_oracle_hertz_contact_converges_to_closed_form():
    b_ref, p_ref = hz.hertz()
    res = {n: hz.run_oracle(n) for n in (32, 64)}
    for r in res.values():
        assert r["F"] == pytest.approx(hz.F_LINE, rel=1e-5)        # plane reactions balance the load
        assert r["stats"].status == 0
    err_b = {n: r["b"] / b_ref - 1 for n, r in res.items()}
    err_p = {n: r["p0"] / p_ref - 1 for n, r in res.items()}
    # too wide and too low (diffuse MPM boundary), first order in dx
    assert 0 < err_b[64] < err_b[32] < 0.6 and err_p[32] < err_p[64] < 0
    assert 1.8 < err_b[32] / err_b[64] < 2.6 and 1.8 < err_p[32] / err_p[64] < 2.3
    # Richardson extrapolation of the first-order sequence lands on Hertz
    assert (2 * res[64]["b"] - res[32]["b"]) / b_ref == pytest.approx(1, abs=0.06)
    assert (2 * res[64]["p0"] - res[32]["p0"]) / p_ref == pytest.approx(1, abs=0.02)


# --------------------------------------------------------------------------------------------------
# Eshelby misfit inclusion (§4.3; tests/golden/g8_eshelby.txt), scripts/eshelby.py:
# particles of a circular inclusion start at F0 = (1 - delta) I inside a traction-free matrix disk,
# static single-domain MPM (plane strain, two materials, mirror-symmetry constraints on the centre
# lines).  Reference: the paper's Lame solution, kept with the finite outer radius (the composite disk).
import eshelby as es  # noqa: E402


def test_eshelby_golden_and_reference_solution():
    for E_out, nu, ratio, delta, P in read_golden("g8_eshelby.txt"):
        assert (E_out, nu, delta) == (es.E_OUT, es.NU, es.DELTA)
        # the paper's compliances in E and nu: C_out = (1 + nu)/E_out, C_in = (1 - 2 nu)(1 + nu)/E_in
        assert P == pytest.approx(delta / ((1 + nu) / E_out + (1 - 2 * nu) * (1 + nu) / (E_out * ratio)), rel=1e-6)
        assert es.paper_pressure(ratio) == pytest.approx(P, rel=1e-6)
        # the finite composite disk: traction free at b, displacement and traction continuous at R ...
        A, B, C, (li, Gi, lo, Go) = es.lame_finite(ratio)
        srr, stt = es.reference_stress(ratio, [es.B_OUT, es.R_INC * (1 - 1e-12), es.R_INC])
        assert abs(srr[0]) < 1e-9 * P and srr[1] == pytest.approx(srr[2], rel=1e-9)
        assert A * es.R_INC == pytest.approx(B * es.R_INC + C / es.R_INC, rel=1e-12)
        # ... uniform hydrostatic inside, and the paper's unbounded solution as b -> infinity
        srr_u, stt_u = es.reference_stress(ratio, [0.5 * es.R_INC, 2 * es.R_INC, 3 * es.R_INC], b=1e5)
        np.testing.assert_allclose(srr_u, [-P, -P / 4, -P / 9], rtol=1e-6)
        np.testing.assert_allclose(stt_u, [-P, P / 4, P / 9], rtol=1e-6)


@pytest.mark.parametrize("ratio", [1.0, 5.0])
def test_oracle_eshelby_converges_to_lame(ratio):
    res = {n: es.run_oracle(n, ratio) for n in (32, 64, 128)}
    err_p = {n: abs(r["p_in"] / r["p_ref"] - 1) for n, r in res.items()}
    err_o = {n: r["err_out"] for n, r in res.items()}
    assert err_o[32] > err_o[64] > err_o[128]                       # monotone under refinement
    assert err_o[32] / err_o[64] > 1.5 and err_o[64] / err_o[128] > 1.5
    assert err_o[128] < (0.005 if ratio == 1 else 0.025)
    assert err_p[128] < (0.005 if ratio == 1 else 0.03)
    assert all(r["stats"].status == 0 for r in res.values())
