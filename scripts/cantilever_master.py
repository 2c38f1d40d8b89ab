"""Gravity-loaded cantilever master curve on the GPU (§4.1).

The beam (L x H, clamped at x = 0, the paper's material E = 100 kPa, nu = 0.4, rho = 1000, 3 x 3
particles per cell) is loaded progressively through a list of gravito-bending parameters Gamma
(g adjusted), one quasi-static frame per load level (backward Euler with a time step
dT so long that inertia is negligible; every frame starts from the previous equilibrium).  Two runs:

  single  one subdomain at dx (the paper's "single-domain")
  dual    OS-MPM: fine subdomain x in [0, 0.3] (dx_B / r, clamped) + coarse subdomain x in [0.2, L]
          (dx_B), coupled by the Schwarz frame of Alg. 1, eps_conv = 1e-5

The tip of the centre line gives W = x_tip / L and H = (y_root - y_tip) / L, compared with the planar
elastica (oracle/elastica.py: H / W, and the tip deflection y(1)).

  python scripts/cantilever_master.py --mode res    # Gamma = 0.05: dual vs single vs E-B over dx_B
  python scripts/cantilever_master.py --mode curve  # master curve H/W over log-spaced Gamma
Prints one JSON line per run.
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synth  # noqa: E402
from oracle import elastica as EL  # noqa: E402  (analytical reference only; never on the GPU path)

L, H, E, NU, RHO = 1.0, 0.2, 1.0e5, 0.4, 1000.0
Y0 = 1.0


PSD = 0
MAX_NEWTON = 100


def newton(guess=1, rtol=1e-8):
    """guess 1: u = 0 (a single load step from rest); guess 0: u = dt v^n, the previous frame's increment
    (progressive loading: each load level starts from the previous equilibrium's increment).  PSD (set by
    --psd): 1 projects the per-particle tangent blocks when a Newton direction fails the descent test,
    2 always (R23)."""
    from paper_2605_09097_b200 import osmpm
    return osmpm.newton_settings(newton_rtol=rtol, newton_atol=0.0, cg_rtol=1e-10, max_cg=40000, max_newton=MAX_NEWTON,
                                 guess=guess, energy_noise_rtol=1e-12, psd=PSD)


def tip_mask(x0, dx):
    return (x0[:, 0] > L - 0.75 * dx) & (np.abs(x0[:, 1] - (Y0 + H / 2)) < 0.75 * dx)


def measure(x0, x, dx):
    """(W, H) of the centre-line tip from the displacement of the particles nearest to it (the lattice
    puts them a fraction of a cell inside the beam end, so positions are not compared with L)."""
    t = tip_mask(x0, dx)
    ux, uy = (x[t, 0] - x0[t, 0]).mean(), (x[t, 1] - x0[t, 1]).mean()
    return 1.0 + ux / L, -uy / L


def clamp_nodes(grid):
    nx, ny = grid.dims[0], grid.dims[1]
    xs = grid.origin[0] + np.arange(nx) * grid.dx
    ci = np.flatnonzero(xs <= 1e-12)
    return (ci[:, None] * ny + np.arange(ny)[None, :]).reshape(-1).astype(np.int64)


def run_single(dx, gammas, dT=10.0, guess=1, rtol=1e-8):
    from paper_2605_09097_b200 import osmpm
    sc = synth.cantilever_single(dx, L=L, H=H, E=E, nu=NU, rho=RHO, dT=dT, y0=Y0)
    ctx = osmpm.Context(0)
    sub = osmpm.Subdomain(ctx, sc.grid, sc.dt, sc.particles, sc.materials, sc.gravity)
    cl = clamp_nodes(sc.grid)
    sub.set_dirichlet(cl, np.full(cl.size, 3, np.uint8), np.zeros((cl.size, 2)))
    out = []
    for G in gammas:
        g = EL.g_for_gamma(G, E, NU, RHO, L, H)
        sub.set_gravity((0.0, -g, 0.0))
        t0 = time.time()
        sub.p2g()
        try:
            st = sub.implicit_solve(newton(guess, rtol))
        except osmpm.OsmpmError as e:
            out.append({"gamma": G, "error": str(e)})
            break
        sub.g2p()
        x = sub.read_particles(fields=("x",))["x"]
        W, Hh = measure(sc.particles.x, x, dx)
        out.append({"gamma": G, "W": W, "H": Hh, "newton": st.newton_iters, "cg": st.cg_iters,
                    "floor_accept": st.floor_accept, "psd_solves": st.psd_solves, "s": round(time.time() - t0, 2)})
    sub.close()
    ctx.close()
    return out


def run_dual(dx_b, gammas, r=4, dT=10.0, M=1, k_max=2000, guess=1, rtol=1e-8):
    from paper_2605_09097_b200 import osmpm
    coarse, fine = synth.cantilever_pair(dx_b, r=r, L=L, H=H, E=E, nu=NU, rho=RHO, dT=dT, M=M, y0=Y0)
    ctx = osmpm.Context(0)
    sb = osmpm.Subdomain(ctx, coarse.grid, coarse.dt, coarse.particles, coarse.materials, coarse.gravity)
    ss = osmpm.Subdomain(ctx, fine.grid, fine.dt, fine.particles, fine.materials, fine.gravity)
    cl = clamp_nodes(fine.grid)
    ss.set_dirichlet(cl, np.full(cl.size, 3, np.uint8), np.zeros((cl.size, 2)))
    ns = newton(guess, rtol)
    cpl = osmpm.Coupler(sb, ss, osmpm.schwarz_settings(M=M, eps_conv=1e-5, k_max=k_max, coarse=ns, fine=ns))
    out = []
    for G in gammas:
        g = EL.g_for_gamma(G, E, NU, RHO, L, H)
        sb.set_gravity((0.0, -g, 0.0))
        ss.set_gravity((0.0, -g, 0.0))
        t0 = time.time()
        try:
            rep = cpl.step()
        except osmpm.OsmpmError as e:  # reported, and the sweep stops there
            out.append({"gamma": G, "error": str(e)})
            break
        x = sb.read_particles(fields=("x",))["x"]
        W, Hh = measure(coarse.particles.x, x, dx_b)
        out.append({"gamma": G, "W": W, "H": Hh, "schwarz": rep.iters, "converged": rep.converged,
                    "r_B": rep.r_B[max(rep.iters - 1, 0)], "r_S": rep.r_S[max(rep.iters - 1, 0)],
                    "s": round(time.time() - t0, 2)})
    cpl.close()
    sb.close()
    ss.close()
    ctx.close()
    return out


def elastica_row(G):
    e = EL.solve(G)
    return {"gamma": G, "W": e["x_tip"], "H": e["y_tip"], "HW": e["HW"]}


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--mode", default="res", choices=["res", "curve"])
    ap.add_argument("--dxb", type=float, nargs="+", default=[0.05, 0.025, 0.0125])
    ap.add_argument("--gammas", type=float, nargs="+", default=[0.03, 0.1, 0.3, 1.0, 3.0])
    ap.add_argument("--dT", type=float, default=10.0)
    ap.add_argument("--no-dual", action="store_true")
    ap.add_argument("--guess", type=int, default=1)
    ap.add_argument("--rtol", type=float, default=1e-8)
    ap.add_argument("--psd", type=int, default=0, choices=[0, 1, 2])
    ap.add_argument("--max-newton", type=int, default=100)
    ap.add_argument("--no-single", action="store_true")
    a = ap.parse_args()
    PSD = a.psd
    MAX_NEWTON = a.max_newton
    if a.mode == "res":
        G = [0.05]
        ref = elastica_row(0.05)
        for dxb in a.dxb:
            rs = run_single(dxb, G, a.dT)[0]
            rf = run_single(dxb / 4, G, a.dT)[0]
            line = {"mode": "res", "dx_B": dxb, "elastica": ref, "single_coarse": rs, "single_fine": rf}
            if not a.no_dual:
                line["dual"] = run_dual(dxb, G, dT=a.dT)[0]
            print(json.dumps(line), flush=True)
    else:
        for dxb in a.dxb:
            line = {"mode": "curve", "dx_B": dxb, "elastica": [elastica_row(G) for G in a.gammas],
                    "single": [] if a.no_single else run_single(dxb, a.gammas, a.dT, guess=a.guess, rtol=a.rtol)}
            print(json.dumps(line), flush=True)
            if not a.no_dual:
                line["dual"] = run_dual(dxb, a.gammas, dT=a.dT, guess=a.guess, rtol=a.rtol)
                print(json.dumps(line), flush=True)
