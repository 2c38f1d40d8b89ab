"""Quasi-static dual-domain cantilever (§4.1, the C1 geometry of synth.c1_cantilever)
under the Euler-Bernoulli load Gamma = 0.05 (g = 0.0183 m/s^2, tests/golden/g6), relaxed frame by
frame (dT = 1 s, M = 4) until the l-inf particle velocity is below 1e-6 on both grids; tip deflection
of the coarse particles near x = L against Gamma L / 8 and against the single-domain static solve of
the coarse resolution (scripts/eb_cantilever.py).  Diagnostic driver.

  python scripts/dual_eb.py [--dT 1.0] [--max-frames 400]
"""
import argparse
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

import eb_cantilever as eb  # noqa: E402
import synth  # noqa: E402


def run(dT=1.0, M=4, max_frames=400, tol=1e-6):
    from paper_2605_09097_b200 import osmpm
    from oracle import schwarz as OS
    D = eb.E * eb.H ** 3 / (12 * (1 - eb.NU ** 2))
    g = 0.05 * D / (eb.RHO * eb.H * eb.L ** 3)
    coarse, fine = synth.c1_cantilever(g=g)
    coarse.dt, fine.dt = dT, dT / M
    ctx = osmpm.Context(0)
    sb = osmpm.Subdomain(ctx, coarse.grid, coarse.dt, coarse.particles, coarse.materials, coarse.gravity)
    ss = osmpm.Subdomain(ctx, fine.grid, fine.dt, fine.particles, fine.materials, fine.gravity)
    xs, _ = OS.node_positions(fine.grid)
    clamp = np.flatnonzero(xs[:, 0] <= 1e-12)
    ss.set_dirichlet(clamp, np.full(clamp.size, 3, np.uint8), np.zeros((clamp.size, 2)))
    ns = osmpm.newton_settings(newton_rtol=1e-8, newton_atol=1e-7, cg_rtol=1e-10, max_cg=20000, max_newton=40,
                               energy_noise_rtol=1e-12)
    cpl = osmpm.Coupler(sb, ss, osmpm.schwarz_settings(M=M, eps_conv=1e-6, k_max=500, coarse=ns, fine=ns))
    x0 = coarse.particles.x.copy()
    tip = x0[:, 0] > eb.L - 0.06
    hist = []
    for f in range(max_frames):
        rep = cpl.step()
        cb = sb.read_particles(fields=("x", "v"))
        vs = ss.read_particles(fields=("v",))["v"]
        defl = -(cb["x"][tip, 1] - x0[tip, 1]).mean()
        vmax = max(np.abs(cb["v"]).max(), np.abs(vs).max())
        hist.append((f + 1, rep.iters, defl, vmax))
        if vmax < tol:
            break
    cpl.close()
    sb.close()
    ss.close()
    ctx.close()
    return hist, 0.05 * eb.L / 8


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--dT", type=float, default=1.0)
    ap.add_argument("--max-frames", type=int, default=400)
    a = ap.parse_args()
    hist, ref = run(a.dT, max_frames=a.max_frames)
    for f, k, d, v in hist[:5] + hist[-5:]:
        print(f"frame {f:4d}: Schwarz {k:3d}, tip {d:.6g} ({d / ref:.4f} of EB), max|v| {v:.2e}")
