"""Diagnostic (R21): one quasi-static Schwarz frame of the dual-domain cantilever
(dbg_dual_k.py) on the GPU with the paper's Pi and with OSMPM_PI=affine."""
import os
import sys
sys.path.insert(0, 'scripts')
sys.path.insert(0, '.')
import numpy as np
import synth
from oracle import schwarz as OS
import eb_cantilever as eb
from paper_2605_09097_b200 import osmpm

D = eb.E * eb.H ** 3 / (12 * (1 - eb.NU ** 2))
g = 0.05 * D / (eb.RHO * eb.H * eb.L ** 3)


def frame(K=200, M=4, dT=10.0):
    coarse, fine = synth.c1_cantilever(g=g)
    coarse.dt, fine.dt = dT, dT / M
    ctx = osmpm.Context(0)
    sb = osmpm.Subdomain(ctx, coarse.grid, coarse.dt, coarse.particles, coarse.materials, coarse.gravity)
    ss = osmpm.Subdomain(ctx, fine.grid, fine.dt, fine.particles, fine.materials, fine.gravity)
    xs, _ = OS.node_positions(fine.grid)
    clamp = np.flatnonzero(xs[:, 0] <= 1e-12)
    ss.set_dirichlet(clamp, np.full(clamp.size, 3, np.uint8), np.zeros((clamp.size, 2)))
    ns = osmpm.newton_settings(newton_rtol=1e-8, cg_rtol=1e-10, max_cg=40000, max_newton=40)
    cpl = osmpm.Coupler(sb, ss, osmpm.schwarz_settings(M=M, parity_fixed_k=K, coarse=ns, fine=ns))
    rep = cpl.step()
    x0 = coarse.particles.x
    tip = x0[:, 0] > eb.L - 0.06
    d = -(sb.read_particles()["x"][tip, 1] - x0[tip, 1]).mean()
    r = rep.r_B[min(K, 256) - 1]
    cpl.close()
    sb.close()
    ss.close()
    ctx.close()
    return d / (0.05 * eb.L / 8), r


if __name__ == "__main__":
    for mode in ("paper", "affine"):
        if mode == "affine":
            os.environ["OSMPM_PI"] = "affine"
        t, r = frame()
        print(f"{mode} Pi: tip {t:.4f} of Euler-Bernoulli (r_B {r:.2e})", flush=True)
