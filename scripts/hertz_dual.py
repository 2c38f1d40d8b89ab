"""Hertz line contact with OS-MPM on the GPU: the coarse grid fixed, the fine subdomain around the contact
refined (§4.2).

The cylinder, material, load and contact treatment are those of scripts/hertz.py (R = 0.5, E = 1 MPa,
nu = 0.3, body load of resultant F = 4315.37 N/m: b = 0.05, p_max = 54.9 kPa; unilateral contact on the
plane row y = 0 by the gap active set of DESIGN.md R19; symmetry v_x = 0 on x = 0).  Decomposition as
BASELINE.json configs[1]: fine Omega_S = the box [-0.2, 0.2] x [0, 0.2] at h_S, coarse Omega_B = the half
disk minus the box shrunk by `overlap` coarse cells at h_B = 1/64 (the paper: 1.56e-2), both 2 x 2
particles per cell; P^∂ within one own cell of each artificial cut.  The contact patch (b = 0.05) lies
inside Omega_S, so only the fine grid carries the contact constraints.

Every active-set round solves, from the initial state, `ramp` quasi-static Schwarz frames (dT = 10 s,
M = 1; eps_conv = 1e-5) with the load stepped up to its full value; the plane reactions are the fine Newton
gradient over all DOFs at the last frame's solved increment (osmpm_newton_gradient on the fine state
restored to the start of that frame).  Reports b (second moment), p(0) and the relative L2 distance of the
pressure profile to the semi-ellipse, against Hertz at the applied resultant and at the measured contact
force (the overlap's material is weighed by both subdomains).

  python scripts/hertz_dual.py [--inv-hs 64 128 256]
"""
import argparse
import json
import math
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))

import hertz as hz  # noqa: E402
import synth  # noqa: E402

BOX_W, BOX_H = 0.2, 0.2
INV_HB = 64


def scenes(inv_hs, overlap=2, dT=10.0):
    hS, hB = 1.0 / inv_hs, 1.0 / INV_HB
    c = np.array([0.0, hz.R])
    disk = lambda p: ((p - c) ** 2).sum(axis=1) < hz.R * hz.R  # noqa: E731
    # fine: the box around the contact
    xf, vf = synth.lattice((-BOX_W, 0.0), (BOX_W, BOX_H), hS, 2, inside=disk)
    bf = ((np.abs(xf[:, 0]) > BOX_W - hS) | (xf[:, 1] > BOX_H - hS)).astype(np.uint8)
    pf = synth.make_particles(xf, vf, hz.RHO, boundary=bf)
    # coarse: the half disk minus the box shrunk by `overlap` coarse cells
    wi, hi = BOX_W - overlap * hB, BOX_H - overlap * hB
    inside_box = lambda p: (np.abs(p[:, 0]) < wi) & (p[:, 1] < hi)  # noqa: E731
    xc, vc = synth.lattice((-hz.R, 0.0), (hz.R, hz.R), hB, 2, inside=lambda p: disk(p) & ~inside_box(p))
    bc = ((np.abs(xc[:, 0]) < wi + hB) & (xc[:, 1] < hi + hB)).astype(np.uint8)
    pc = synth.make_particles(xc, vc, hz.RHO, boundary=bc)
    g = hz.F_LINE / (hz.RHO * math.pi * hz.R ** 2 / 2)   # resultant F on the half disk
    fine = synth.Scene(synth.grid_around(xf, hS, 4, 2, align_origin=(0.0, 0.0)), pf, [(hz.E, hz.NU)], dT,
                       (0.0, -g, 0.0))
    coarse = synth.Scene(synth.grid_around(np.vstack([xf, xc]), hB, 4, 2, align_origin=(0.0, 0.0)), pc,
                         [(hz.E, hz.NU)], dT, (0.0, -g, 0.0))
    return coarse, fine


def nodes(grid):
    nx, ny = grid.dims[0], grid.dims[1]
    k = np.stack(np.meshgrid(np.arange(nx), np.arange(ny), indexing="ij"), -1).reshape(-1, 2)
    return np.asarray(grid.origin[:2]) + k * grid.dx


def run(inv_hs, max_rounds=30, ramp=1):
    from paper_2605_09097_b200 import osmpm
    coarse, fine = scenes(inv_hs)
    ctx = osmpm.Context(0)
    sb = osmpm.Subdomain(ctx, coarse.grid, coarse.dt, coarse.particles, coarse.materials, coarse.gravity)
    ss = osmpm.Subdomain(ctx, fine.grid, fine.dt, fine.particles, fine.materials, fine.gravity)
    xsB, xsS = nodes(coarse.grid), nodes(fine.grid)
    axisB = np.flatnonzero(np.abs(xsB[:, 0]) <= 1e-12)
    sb.set_dirichlet(axisB, np.full(axisB.size, 1, np.uint8), np.zeros((axisB.size, 2)))
    plane = np.flatnonzero(np.abs(xsS[:, 1]) <= 1e-12)
    axis = np.flatnonzero(np.abs(xsS[:, 0]) <= 1e-12)
    gap = np.zeros(xsS.shape[0])
    xp = np.minimum(np.abs(xsS[plane, 0]), hz.R)
    gap[plane] = hz.R - np.sqrt(hz.R * hz.R - xp * xp)
    # at 1/256 the relative 1e-8 sits below E_h's round-off floor (Newton stalls near 6e-5 of |g0|): the
    # fine solves stop at 1e-6 of |g0| there, far below the nodal reactions the pressure is read from
    fine_h = inv_hs >= 256
    ns = osmpm.newton_settings(newton_rtol=1e-6 if fine_h else 1e-8, cg_rtol=1e-10, max_cg=100000 if fine_h else 60000,
                               max_newton=200 if fine_h else 60, guess=1, energy_noise_rtol=1e-9 if fine_h else 1e-12)
    cpl = osmpm.Coupler(sb, ss, osmpm.schwarz_settings(M=1, eps_conv=1e-5, k_max=2000, coarse=ns, fine=ns))
    sb.checkpoint()
    ss.checkpoint()
    ss.p2g()
    act = ss.read_grid()["active"].astype(bool)
    t0 = time.time()
    iters = []

    g_full = fine.gravity[1]
    init = [(sub, {k: np.ascontiguousarray(getattr(sc.particles, k)) for k in ("x", "v", "F", "B")})
            for sub, sc in ((sb, coarse), (ss, fine))]

    def solve(sel, bits, vel):
        # from the initial state, `ramp` quasi-static frames with the load (and the prescribed contact gap
        # displacements) stepped up in equal parts, so that no frame takes the whole settlement at once;
        # the fine state before the last frame is kept for the reactions.  The active-set test needs the
        # total displacement of the plane nodes: ramp x the last increment (proportional loading)
        for sub, st0 in init:
            sub.set_particles(**st0)
        rep = None
        for k in range(1, ramp + 1):
            for sub in (sb, ss):
                sub.set_gravity((0.0, k / ramp * g_full, 0.0))
            ss.set_dirichlet(sel, bits, vel / ramp)
            if k == ramp:
                ss.checkpoint()
            rep = cpl.step()
            iters.append(rep.iters)
        return ss.read_grid_velocity() * fine.dt * ramp, rep

    def gradient(u):
        # reactions at the last frame: the fine Newton gradient over all DOFs at its solved increment
        ss.restore()
        ss.set_dirichlet(np.zeros(0, np.int64), np.zeros(0, np.uint8), np.zeros((0, 2)))
        ss.p2g()
        return ss.newton_gradient(u / ramp)[0]

    try:
        res = hz.active_set(solve, gradient, fine, xsS, plane, axis, gap, act, max_rounds=max_rounds)
    finally:
        cpl.close()
        sb.close()
        ss.close()
        ctx.close()
    b_ref, p_ref = hz.hertz()
    # the overlap's material is weighed by both subdomains, so the plane carries more than the applied
    # resultant; Hertz at the measured contact force F compares the profile's shape
    b_F, p_F = hz.hertz(res["F"])
    xc, pc = res["xc"], res["p"]
    ph = p_ref * np.sqrt(np.maximum(0.0, 1 - (xc / b_ref) ** 2))
    grid_x = np.arange(-2 * b_ref, 2 * b_ref + 1e-12, 1.0 / inv_hs)
    p_on = np.interp(grid_x, xc, pc, left=0.0, right=0.0)
    p_hz = p_ref * np.sqrt(np.maximum(0.0, 1 - (grid_x / b_ref) ** 2))
    return {"inv_hs": inv_hs, "inv_hb": INV_HB, "b": res["b"], "b_err": res["b"] / b_ref - 1, "p0": res["p0"],
            "p0_err": res["p0"] / p_ref - 1, "F": res["F"], "F_over_applied": res["F"] / hz.F_LINE,
            "b_err_at_F": res["b"] / b_F - 1, "p0_err_at_F": res["p0"] / p_F - 1, "ramp": ramp, "profile_L2_rel": float(np.linalg.norm(p_on - p_hz)
                                                                                      / np.linalg.norm(p_hz)),
            "rounds": res["rounds"], "schwarz_iters": iters, "seconds": round(time.time() - t0, 2),
            "particles_fine": int(fine.particles.n), "particles_coarse": int(coarse.particles.n),
            "profile": {"x": xc.tolist(), "p": pc.tolist(), "hertz": ph.tolist()}}


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--inv-hs", type=int, nargs="+", default=[64, 128, 256])
    ap.add_argument("--ramp", type=int, nargs="+", default=None, help="load steps per h_S (default 1, 1, 8)")
    a = ap.parse_args()
    ramps = a.ramp or [1 if n < 256 else 8 for n in a.inv_hs]
    for n, rp in zip(a.inv_hs, ramps):
        print(json.dumps(run(n, ramp=rp)), flush=True)
