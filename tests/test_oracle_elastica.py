"""Pins of the elastica oracle (oracle/elastica.py; §4.1).

Against what mathematics fixes, not against the oracle's own formula:
  * regular perturbation in Gamma of the BVP (derived by hand): theta = G t1 + G^3 t3 + ...
    with t1 = (1 - (1-s)^3) / 6, giving
        y(1) = Gamma / 8 - Gamma^3 / 640 + O(Gamma^5),     x(1) = 1 - Gamma^2 / 112 + O(Gamma^4),
        theta'(0) = Gamma / 2 + O(Gamma^3)
    (the linear term is the Euler-Bernoulli tip deflection q L^4 / (8 D), golden G6);
  * the inextensible rod: x(1)^2 + y(1)^2 < 1, and the heavy-load limit of a hanging rod;
  * fourth-order convergence of the integrator (error ratio ~16 per halving);
  * the scratch shooting values quoted by SURVEY.md §8(c).3 O13 / §8(f) N2 (an independent computation).
"""
import math

import pytest

from oracle import elastica as EL


@pytest.mark.parametrize("gamma", [1e-3, 1e-2, 5e-2, 1e-1])
def test_small_load_perturbation_series(gamma):
    r = EL.solve(gamma)
    assert abs(r["y_tip"] - (gamma / 8 - gamma ** 3 / 640)) <= 0.01 * gamma ** 5 + 1e-13
    assert abs(r["x_tip"] - (1 - gamma ** 2 / 112)) <= 0.01 * gamma ** 4 + 1e-13
    assert abs(r["k0"] - gamma / 2) <= 0.1 * gamma ** 3 + 1e-13


def test_cubic_coefficient_is_resolved():
    # (y - G/8) / G^3 -> -1/640: a dropped cos-theta factor or a wrong sign in the load term fails here
    for g in (0.02, 0.04):
        r = EL.solve(g)
        assert (r["y_tip"] - g / 8) / g ** 3 == pytest.approx(-1 / 640, rel=2e-3)


def test_inextensible_and_monotone_master_curve():
    gammas = [0.03, 0.1, 0.3, 1.0, 3.0, 10.0, 26.8]
    hw = []
    for g in gammas:
        r = EL.solve(g)
        assert r["x_tip"] ** 2 + r["y_tip"] ** 2 < 1.0
        assert 0.0 < r["theta_tip"] < math.pi / 2
        hw.append(r["HW"])
    assert all(b > a for a, b in zip(hw, hw[1:]))  # H/W is a monotone function of Gamma


def test_heavy_load_hangs_down():
    r = EL.solve(2000.0, n=8000)
    assert r["y_tip"] > 0.9 and r["x_tip"] < 0.3 and r["theta_tip"] > 1.3


def test_rk4_is_fourth_order():
    g, k = 3.0, EL.solve(3.0)["k0"]
    ref = EL.integrate(g, k, 8000)[3]
    e1 = abs(EL.integrate(g, k, 50)[3] - ref)
    e2 = abs(EL.integrate(g, k, 100)[3] - ref)
    assert 12.0 < e1 / e2 < 20.0


def test_survey_cross_check_values():
    # "C1's stated Gamma = 26.8 (elastica tip y = 0.863 L, x = 0.369 L, by our
    # shooting)"; §8(c).3 O13: "Gamma = 0.231 -> 0.02886"
    r = EL.solve(26.8)
    assert r["y_tip"] == pytest.approx(0.863, abs=1.5e-3) and r["x_tip"] == pytest.approx(0.369, abs=1.5e-3)
    assert EL.solve(0.231)["y_tip"] == pytest.approx(0.02886, abs=1e-5)


def test_gamma_definition():
    # Gamma = rho A g L^3 / (D w), D = E h^3 / (12 (1 - nu^2)); golden G6 parameters
    g = EL.g_for_gamma(0.05, 1e5, 0.3, 1000.0, 1.0, 0.2)
    assert g == pytest.approx(0.018315, rel=1e-4)
    assert EL.gamma_of(1e5, 0.3, 1000.0, g, 1.0, 0.2) == pytest.approx(0.05, rel=1e-14)
