"""Euler-Bernoulli check of the static cantilever (§4.1, linear limit of the elastica;
tests/golden/g6_euler_bernoulli.txt): single-domain MPM beam clamped at x = 0 under gravity with
Gamma = q L^3 / D = 0.05 (D = E h^3 / (12 (1 - nu^2)), q = rho g h), one backward-Euler step with a
time step so large that the inertia term vanishes (the Newton solve then finds the static
equilibrium), tip deflection from G2P vs Gamma L / 8.

  python scripts/eb_cantilever.py [--gpu] [--oracle] [--dx 0.05 0.025 ...]
"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

L, H, E, NU, RHO = 1.0, 0.2, 1.0e5, 0.3, 1000.0


def scene(dx, gamma=0.05, dt=10.0):
    D = E * H ** 3 / (12 * (1 - NU ** 2))
    g = gamma * D / (RHO * H * L ** 3)
    y0 = 1.0
    x, vol = synth.lattice((0.0, y0), (L, y0 + H), dx, 2)
    p = synth.make_particles(x, vol, RHO)
    grid = synth.grid_around(x, dx, 4, 2)
    sc = synth.Scene(grid, p, [(E, NU)], dt, (0.0, -g, 0.0), meta={"config": "E-B"})
    # clamp: every node at x <= 0 (R17)
    nx, ny = grid.dims[0], grid.dims[1]
    ix = np.arange(nx)
    xs = grid.origin[0] + ix * dx
    clamp_i = ix[xs <= 1e-12]
    idx = (clamp_i[:, None] * ny + np.arange(ny)[None, :]).reshape(-1).astype(np.int64)
    return sc, idx, gamma * L / 8


def tip_deflection(x0, x1):
    tip = x0[:, 0] > L - 0.06
    return -(x1[tip, 1] - x0[tip, 1]).mean()


def run_gpu(dx, max_cg=20000):
    from paper_2605_09097_b200 import osmpm
    sc, idx, ref = scene(dx)
    ctx = osmpm.Context(0)
    sub = osmpm.Subdomain(ctx, sc.grid, sc.dt, sc.particles, sc.materials, sc.gravity)
    sub.set_dirichlet(idx, np.full(idx.shape[0], 3, np.uint8), np.zeros((idx.shape[0], 2)))
    sub.p2g()
    st = sub.implicit_solve(osmpm.newton_settings(newton_rtol=1e-10, cg_rtol=1e-10, max_cg=max_cg, max_newton=30))
    sub.g2p()
    x1 = sub.read_particles()["x"]
    tip = tip_deflection(sc.particles.x, x1)
    sub.close()
    ctx.close()
    return tip, ref, st


def run_oracle(dx, max_cg=20000):
    import oracle
    sc, idx, ref = scene(dx)
    gs = oracle.p2g(sc)
    dm = np.zeros((oracle.n_nodes(sc.grid), 2), np.uint8)
    dm[idx] = 1
    u, st = oracle.implicit_solve(sc, gs, oracle.default_settings(newton_rtol=1e-10, cg_rtol=1e-10, max_cg=max_cg,
                                                                   max_newton=30),
                                  dirichlet_mask=dm, dirichlet_v=np.zeros((oracle.n_nodes(sc.grid), 2)))
    act = gs.active.astype(bool)
    pts = oracle.g2p(sc, np.where(act[:, None], u / sc.dt, 0.0))
    return tip_deflection(sc.particles.x, pts.x), ref, st


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpu", action="store_true")
    ap.add_argument("--oracle", action="store_true")
    ap.add_argument("--dx", type=float, nargs="+", default=[0.05, 0.025, 0.0125])
    a = ap.parse_args()
    for dx in a.dx:
        if a.gpu:
            tip, ref, st = run_gpu(dx)
            print(f"gpu    dx={dx:<7g} tip={tip:.6g} EB={ref:.6g} ratio={tip / ref:.4f} newton={st.newton_iters} "
                  f"cg={st.cg_iters}", flush=True)
        if a.oracle:
            tip, ref, st = run_oracle(dx)
            print(f"oracle dx={dx:<7g} tip={tip:.6g} EB={ref:.6g} ratio={tip / ref:.4f} newton={st.newton_iters} "
                  f"cg={st.cg_iters}", flush=True)

