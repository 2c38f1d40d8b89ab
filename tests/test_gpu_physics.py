"""GPU: the static cantilever against Euler-Bernoulli (§4.1; G6) through the C ABI,
under refinement (first-order convergence of the MPM discretisation to the closed form), and equal to
the oracle's static solution at the coarsest resolution."""
import os
import sys

import numpy as np
import pytest

sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "scripts"))
import eb_cantilever as eb  # noqa: E402

pytestmark = pytest.mark.gpu


def test_gpu_cantilever_converges_to_euler_bernoulli():
    err = []
    for dx in (0.05, 0.025, 0.0125, 0.00625):
        tip, ref, st = eb.run_gpu(dx)
        assert st.status == 0
        err.append(tip / ref - 1)
    assert all(e > 0 for e in err)
    assert all(a / b > 1.8 for a, b in zip(err, err[1:]))  # first order in dx
    assert err[-1] < 0.01


def test_gpu_cantilever_equals_oracle():
    tg, _, _ = eb.run_gpu(0.05)
    to, _, _ = eb.run_oracle(0.05)
    assert tg == pytest.approx(to, rel=1e-8)


# Hertz line contact (§4.2; G7) through the C ABI: the same static unilateral-contact
# driver as the oracle pin (scripts/hertz.py), refined to dx = 1/256 (103k particles; the paper refines
# h_S to 5e-3).  Beyond that the nodal gap contact of DESIGN.md R19 breaks down (measured at 1/512: the
# gap at the contact edge exceeds a cell and the edge nodes carry only the tail of the B-spline
# support; the pressure profile oscillates there), which is a limit of that reading, not of the path.
import hertz as hz  # noqa: E402


def test_gpu_hertz_contact_converges_to_closed_form():
    b_ref, p_ref = hz.hertz()
    ns = (64, 128, 256)
    res = {n: hz.run_gpu(n) for n in ns}
    for r in res.values():
        assert r["F"] == pytest.approx(hz.F_LINE, rel=1e-5)
    eb_ = [res[n]["b"] / b_ref - 1 for n in ns]
    ep_ = [res[n]["p0"] / p_ref - 1 for n in ns]
    assert all(e > 0 for e in eb_) and all(e < 0 for e in ep_)
    assert all(1.8 < a / b < 2.5 for a, b in zip(eb_, eb_[1:]))     # first order in dx
    assert all(1.8 < a / b < 2.5 for a, b in zip(ep_, ep_[1:]))
    assert eb_[-1] < 0.06 and ep_[-1] > -0.04
    # Richardson extrapolation of the finest pair lands on Hertz
    assert (2 * res[256]["b"] - res[128]["b"]) / b_ref == pytest.approx(1, abs=0.01)
    assert (2 * res[256]["p0"] - res[128]["p0"]) / p_ref == pytest.approx(1, abs=0.01)


def test_gpu_hertz_equals_oracle():
    g = hz.run_gpu(64)
    o = hz.run_oracle(64)
    assert g["rounds"] == o["rounds"]
    np.testing.assert_array_equal(g["xc"], o["xc"])
    assert np.abs(g["p"] - o["p"]).max() <= 1e-7 * np.abs(o["p"]).max()
    assert g["b"] == pytest.approx(o["b"], rel=1e-8) and g["p0"] == pytest.approx(o["p0"], rel=1e-8)


# Eshelby misfit inclusion (§4.3; G8) through the C ABI, refined to dx = 1/512 (3.1 M
# particles in the matrix disk) for the paper's three stiffness ratios.
import eshelby as es  # noqa: E402


@pytest.mark.parametrize("ratio", [1.0, 2.0, 5.0])
def test_gpu_eshelby_converges_to_lame(ratio):
    ns = (64, 128, 256, 512)
    res = {n: es.run_gpu(n, ratio) for n in ns}
    err_o = [res[n]["err_out"] for n in ns]
    err_p = [abs(res[n]["p_in"] / res[n]["p_ref"] - 1) for n in ns]
    assert err_o[-1] < 0.006 and err_p[-1] < 0.007
    if ratio > 1:
        # first order in dx once the interface is resolved (ratio 1 reaches the O(delta) floor first)
        assert all(a > b for a, b in zip(err_o, err_o[1:]))
        assert all(a / b > 1.4 for a, b in zip(err_p[1:], err_p[2:]))


def test_gpu_eshelby_equals_oracle():
    g = es.run_gpu(64, 5.0)
    o = es.run_oracle(64, 5.0)
    assert np.abs(g["F"] - o["F"]).max() <= 1e-8 * np.abs(o["F"] - np.eye(2)).max()
    assert g["p_in"] == pytest.approx(o["p_in"], rel=1e-8) and g["err_out"] == pytest.approx(o["err_out"], rel=1e-6)
