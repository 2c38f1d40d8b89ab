"""Diagnostic (N2): one quasi-static Schwarz frame (dT = 10 s, M = 4, fixed K) of the
dual-domain cantilever (C1 geometry: coarse x in [0.2, 1.0] at dx 0.05, fine x in [0, x_f] at 0.0125,
clamp at x = 0) under the Euler-Bernoulli load Gamma = 0.05: tip deflection against Gamma L / 8 as
the overlap [0.2, x_f] widens."""
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


def pair(x_f, dT=10.0, M=4):
    y0 = 1.0
    out = []
    for (lo, hi, dx, cut, dt) in ((0.2, 1.0, 0.05, 0.2, dT), (0.0, x_f, 0.0125, x_f, dT / M)):
        x, vol = synth.lattice((lo, y0), (hi, y0 + 0.2), dx, 2)
        bnd = (np.abs(x[:, 0] - cut) < dx).astype(np.uint8)
        p = synth.make_particles(x, vol, 1000.0, boundary=bnd)
        out.append(synth.Scene(synth.grid_around(x, dx, 4, 2), p, [(1.0e5, 0.3)], dt, (0.0, -g, 0.0)))
    return out


for x_f, K in ((0.3, 300), (0.4, 300), (0.5, 300), (0.6, 300)):
    coarse, fine = pair(x_f)
    ctx = osmpm.Context(0)
    sb = osmpm.Subdomain(ctx, coarse.grid, coarse.dt, coarse.particles, coarse.materials, coarse.gravity)
    ss = osmpm.Subdomain(ctx, fine.grid, fine.dt, fine.particles, fine.materials, fine.gravity)
    xs, _ = OS.node_positions(fine.grid)
    clamp = np.flatnonzero(xs[:, 0] <= 1e-12)
    ss.set_dirichlet(clamp, np.full(clamp.size, 3, np.uint8), np.zeros((clamp.size, 2)))
    ns = osmpm.newton_settings(newton_rtol=1e-8, cg_rtol=1e-10, max_cg=40000, max_newton=40)
    cpl = osmpm.Coupler(sb, ss, osmpm.schwarz_settings(M=4, parity_fixed_k=K, coarse=ns, fine=ns))
    rep = cpl.step()
    x0 = coarse.particles.x
    tip = x0[:, 0] > eb.L - 0.06
    cb = sb.read_particles()
    d = -(cb["x"][tip, 1] - x0[tip, 1]).mean()
    rb = np.array(rep.r_B[:min(K, 256)])
    print(f"x_f={x_f}: receivers B {rep.n_recv_B} S {rep.n_recv_S}, tip {d / (0.05 * eb.L / 8):.4f} of "
          f"Euler-Bernoulli, r_B {rb[-1]:.2e}", flush=True)
    cpl.close()
    sb.close()
    ss.close()
    ctx.close()
