"""Diagnostic: the quasi-static dual-domain cantilever frame of dbg_dual_k.py run by the
ORACLE Schwarz driver, once with the paper's mass-weighted projection Pi and once with an
affine (weighted least-squares, linear-field-exact) variant of it, to test whether Pi's support-wide
average is what keeps the coupled fixed point at ~0.54 of Euler-Bernoulli.  Not part of the method."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
import synth  # noqa: E402
from oracle import schwarz as OS  # noqa: E402
import eb_cantilever as eb  # noqa: E402

D = eb.E * eb.H ** 3 / (12 * (1 - eb.NU ** 2))
G = 0.05 * D / (eb.RHO * eb.H * eb.L ** 3)
PAPER_PROJECT = OS.project


def affine_project(grid_s, gs_fine, grid_b, eps_tol=0.0, v_fine=None, m_fine=None, active_fine=None):
    """v_B,I = a from min sum_j m_j N_I(x_j) |v_j - a - B (x_j - x_I)|^2 over the active fine nodes in
    the support of coarse node I (2D); falls back to the weighted mean when the fit is singular."""
    vb, num, den = PAPER_PROJECT(grid_s, gs_fine, grid_b, eps_tol, v_fine, m_fine, active_fine)
    ms = gs_fine.m if m_fine is None else m_fine
    vs = gs_fine.v if v_fine is None else v_fine
    act = (gs_fine.active if active_fine is None else active_fine).astype(bool)
    xs, _ = OS.node_positions(grid_s)
    nb = oracle.n_nodes(grid_b)
    S0 = np.zeros(nb)
    S1 = np.zeros((nb, 2))
    S2 = np.zeros((nb, 2, 2))
    T0 = np.zeros((nb, 2))
    T1 = np.zeros((nb, 2, 2))
    for j in np.flatnonzero(act):
        st = oracle.stencil(grid_b, xs[j])
        if st is None:
            continue
        idx, N, _, xip = st          # xip = x_I - x_j
        w = ms[j] * N
        dxj = -xip                    # x_j - x_I
        np.add.at(S0, idx, w)
        np.add.at(S1, idx, w[:, None] * dxj)
        np.add.at(S2, idx, w[:, None, None] * dxj[:, :, None] * dxj[:, None, :])
        np.add.at(T0, idx, w[:, None] * vs[j][None, :])
        np.add.at(T1, idx, w[:, None, None] * dxj[:, :, None] * vs[j][None, None, :])
    out = vb.copy()
    for I in np.flatnonzero(S0 > 0):
        A = np.zeros((3, 3))
        A[0, 0] = S0[I]
        A[0, 1:] = A[1:, 0] = S1[I]
        A[1:, 1:] = S2[I]
        rhs = np.vstack([T0[I][None, :], T1[I]])
        if np.linalg.cond(A) < 1e10:
            out[I] = np.linalg.solve(A, rhs)[0]
    return out, num, den


def frame(project, K=300):
    OS.project = project
    coarse, fine = synth.c1_cantilever(g=G)
    coarse.dt, fine.dt = 10.0, 2.5
    xs, _ = OS.node_positions(fine.grid)
    nn = oracle.n_nodes(fine.grid)
    mask = np.zeros((nn, 2), np.uint8)
    mask[xs[:, 0] <= 1e-12] = 1
    st = oracle.default_settings(newton_rtol=1e-8, cg_rtol=1e-10, max_cg=20000, max_newton=40)
    res = OS.schwarz_step(coarse, fine, 4, parity_fixed_k=K, newton_coarse=st, newton_fine=st,
                          user_S=OS.UserBC(mask, np.zeros((nn, 2))))
    OS.project = PAPER_PROJECT
    x0 = coarse.particles.x
    tip = x0[:, 0] > eb.L - 0.06
    return -(res.coarse_particles.x[tip, 1] - x0[tip, 1]).mean() / (0.05 * eb.L / 8), res.r_B[-1]


if __name__ == "__main__":
    K = int(sys.argv[1]) if len(sys.argv) > 1 else 300
    for name, pj in (("paper Pi", PAPER_PROJECT), ("affine Pi", affine_project)):
        t, r = frame(pj, K)
        print(f"{name}: tip {t:.4f} of Euler-Bernoulli after K = {K} (r_B {r:.2e})", flush=True)
