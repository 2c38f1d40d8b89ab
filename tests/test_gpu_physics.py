"""GPU: the static cantilever against Euler-Bernoulli (§4.1; G6) through the C ABI,
under refinement (first-order convergence of the MPM discretisation to the closed form), and equal to
the oracle's static solution at the coarsest resolution."""
import os
import sys

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
