"""Hertz line-contact check (§4.2; tests/golden/g7_hertz.txt): a compliant
semi-circular cylinder of radius R (the half disk below its centre (0, R)) pressed onto the rigid
frictionless plane y = 0 by a body load whose resultant is F per unit length, solved to static
equilibrium by single-domain MPM (one backward-Euler step with a time step so large that the inertia
term vanishes, as in the Euler-Bernoulli check), with unilateral contact at the plane by an active
set on the grid nodes of the row y = 0:

  * the gap between the cylinder and the plane above node x_i is Hertz's g(x_i) = R - sqrt(R^2 -
    x_i^2) (the undeformed surface); a node in the contact set C is held at u_y = -g(x_i) (Dirichlet
    velocity -g/dt), the others are free.  A grid node under the diffuse MPM boundary carries mass
    from particles up to 1.5 cells above it, so constraining every plane node that has mass (g = 0)
    would spread the contact over |x| < sqrt(3 R dx), which shrinks only as sqrt(dx);
  * symmetry v_x = 0 on the axis x = 0 (exact for the mirror-symmetric particle lattice; removes the
    horizontal rigid mode that a frictionless plane leaves);
  * C starts as the plane nodes within 2 cells of the axis; after each static solve the plane
    reactions r_i = g_{i,y}(u) (the gradient of E_h at the solution over all DOFs,
    osmpm_newton_gradient: zero on free DOFs, the constraint force on constrained ones; their sum
    is sum_p m_p g = F) are read; nodes pulling on the plane (r < 0) leave C, free plane nodes that
    moved through it (u_y < -g) join it; repeat until C is unchanged.

The contact pressure profile is p(x_i) = sum over the plane rows of r_i / dx at node column x_i.  It
is compared with the Hertz semi-ellipse p(x) = p_max sqrt(1 - (x/b)^2), b = 2 sqrt(F R (1-nu^2) /
(pi E)), p_max = 2F/(pi b) through
  * b_est = 2 sqrt(sum x^2 p / sum p) (the second moment of a semi-ellipse is b^2/4), and
  * p0 = p(0), the pressure at the centre node column.
The same driver runs on the GPU through the C ABI (`run_gpu`) and on the oracle (`run_oracle`).

  python scripts/hertz.py [--gpu] [--oracle] [--dx 64 128 256]     (cells per metre)
"""
import argparse
import math
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

R, E, NU, RHO = 0.5, 1.0e6, 0.3, 1000.0
F_LINE = 4315.3745          # N/m (G7): b = 0.05, p_max = 54,945 Pa


def hertz(F=F_LINE):
    b = 2.0 * math.sqrt(F * R * (1 - NU * NU) / (math.pi * E))
    return b, 2.0 * F / (math.pi * b)


def scene(inv_dx, dt=10.0, F=F_LINE):
    dx = 1.0 / inv_dx
    c = np.array([0.0, R])
    x, vol = synth.lattice((-R, 0.0), (R, R), dx, 2, inside=lambda p: ((p - c) ** 2).sum(axis=1) < R * R)
    p = synth.make_particles(x, vol, RHO)
    g = F / p.m.sum()                      # body load whose resultant is exactly F
    grid = synth.grid_around(x, dx, 4, 2)
    sc = synth.Scene(grid, p, [(E, NU)], dt, (0.0, -g, 0.0), meta={"config": "Hertz"})
    nx, ny = grid.dims[0], grid.dims[1]
    k = np.stack(np.meshgrid(np.arange(nx), np.arange(ny), indexing="ij"), -1).reshape(-1, 2)
    xs = np.asarray(grid.origin[:2]) + k * dx
    plane = np.flatnonzero(np.abs(xs[:, 1]) <= 1e-12)
    axis = np.flatnonzero(np.abs(xs[:, 0]) <= 1e-12)
    gap = np.zeros(xs.shape[0])
    xp = np.minimum(np.abs(xs[plane, 0]), R)
    gap[plane] = R - np.sqrt(R * R - xp * xp)
    return sc, xs, plane, axis, gap


def _dirichlet_lists(nn, plane_on, axis, gap, dt):
    """(node indices, component bits, velocities (n, 2)) of the symmetry and contact constraints"""
    bits = np.zeros(nn, np.uint8)
    bits[axis] |= 1
    bits[plane_on] |= 2
    sel = np.flatnonzero(bits)
    vel = np.zeros((sel.size, 2))
    vel[:, 1] = np.where(bits[sel] & 2, -gap[sel] / dt, 0.0)
    return sel, bits[sel], vel


def _profile(xs, plane, r, dx):
    cols = {}
    for i, ri in zip(plane, r):
        key = int(round(xs[i, 0] / dx))
        cols[key] = cols.get(key, 0.0) + ri
    kk = np.array(sorted(cols))
    pc = np.array([cols[k] for k in kk]) / dx
    return kk * dx, pc


def active_set(solve, gradient, sc, xs, plane, axis, gap, active_nodes, max_rounds=30):
    """The unilateral-contact loop of the module docstring; `solve(sel, bits, vel)` returns (u (nn, 2),
    stats), `gradient(u)` returns g (nn, 2) over all DOFs."""
    nn = xs.shape[0]
    on = np.zeros(nn, bool)
    in_plane = np.zeros(nn, bool)
    in_plane[plane] = True
    on[plane] = active_nodes[plane] & (np.abs(xs[plane, 0]) <= 2.5 * sc.grid.dx)
    rounds = 0
    while True:
        rounds += 1
        sel, bits, vel = _dirichlet_lists(nn, np.flatnonzero(on), axis, gap, sc.dt)
        u, st = solve(sel, bits, vel)
        g = gradient(u)
        r = g[:, 1]           # sum_i g_i = sum f_int - sum f_ext = +W at equilibrium: the plane's push
        release = on & (r < 0)
        add = (~on) & active_nodes & in_plane & (u[:, 1] < -gap - 1e-12 * sc.grid.dx)
        if os.environ.get("HERTZ_VERBOSE"):
            pen = (u[:, 1] + gap)[in_plane & active_nodes & ~on]
            print(f"   round {rounds}: |C| = {on.sum()}, release {release.sum()}, add {add.sum()}, "
                  f"min r = {r[on].min():.3e}, max r = {r[on].max():.3e}, min free clearance = "
                  f"{pen.min() if pen.size else 0:.3e}, newton {getattr(st, 'newton_iters', '-')}, "
                  f"cg {getattr(st, 'cg_iters', '-')}", flush=True)
        if not release.any() and not add.any():
            break
        if rounds >= max_rounds:
            raise RuntimeError("contact active set did not settle")
        on[release] = False
        on[add] = True
    pl = np.flatnonzero(on)
    xc, pc = _profile(xs, pl, r[pl], sc.grid.dx)
    Ftot = pc.sum() * sc.grid.dx
    b_est = 2.0 * math.sqrt((xc * xc * pc).sum() / pc.sum())
    p0 = float(pc[np.argmin(np.abs(xc))])
    if os.environ.get("HERTZ_VERBOSE"):
        b_ref, p_ref = hertz()
        for xx, pp in zip(xc, pc):
            print(f"      x = {xx:+.5f}  p = {pp:10.1f}  Hertz {p_ref * math.sqrt(max(0.0, 1 - (xx / b_ref) ** 2)):10.1f}")
    return dict(b=b_est, p0=p0, F=Ftot, rounds=rounds, xc=xc, p=pc, stats=st, u=u)


def run_gpu(inv_dx, max_cg=40000):
    from paper_2605_09097_b200 import osmpm
    sc, xs, plane, axis, gap = scene(inv_dx)
    ctx = osmpm.Context(0)
    sub = osmpm.Subdomain(ctx, sc.grid, sc.dt, sc.particles, sc.materials, sc.gravity)
    sub.p2g()
    act = sub.read_grid()["active"].astype(bool)
    settings = osmpm.newton_settings(newton_rtol=1e-9, cg_rtol=1e-10, max_cg=max_cg, max_newton=40)

    def solve(sel, bits, vel):
        sub.set_dirichlet(sel, bits, vel)
        sub.p2g()
        st = sub.implicit_solve(settings)
        return sub.read_grid_velocity() * sc.dt, st

    def gradient(u):
        sub.set_dirichlet(np.zeros(0, np.int64), np.zeros(0, np.uint8), np.zeros((0, 2)))
        return sub.newton_gradient(u)[0]

    try:
        return active_set(solve, gradient, sc, xs, plane, axis, gap, act)
    finally:
        sub.close()
        ctx.close()


def run_oracle(inv_dx, max_cg=40000):
    import oracle
    sc, xs, plane, axis, gap = scene(inv_dx)
    gs = oracle.p2g(sc)
    act = gs.active.astype(bool)
    nn = xs.shape[0]
    settings = oracle.default_settings(newton_rtol=1e-9, cg_rtol=1e-10, max_cg=max_cg, max_newton=40)

    def solve(sel, bits, vel):
        dm = np.zeros((nn, 2), np.uint8)
        dv = np.zeros((nn, 2))
        dm[sel, 0] = bits & 1
        dm[sel, 1] = (bits >> 1) & 1
        dv[sel] = vel
        return oracle.implicit_solve(sc, gs, settings, dirichlet_mask=dm, dirichlet_v=dv)

    def gradient(u):
        return oracle.gradient(sc, gs, u)

    return active_set(solve, gradient, sc, xs, plane, axis, gap, act)


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpu", action="store_true")
    ap.add_argument("--oracle", action="store_true")
    ap.add_argument("--dx", type=int, nargs="+", default=[64, 128, 256])
    a = ap.parse_args()
    b_ref, p_ref = hertz()
    import time
    for n in a.dx:
        for kind, fn in (("gpu", run_gpu), ("oracle", run_oracle)):
            if not getattr(a, kind):
                continue
            t = time.time()
            res = fn(n)
            print(f"{kind:6s} dx=1/{n:<5d} b={res['b']:.5f} (Hertz {b_ref:.5f}, {res['b'] / b_ref - 1:+.2%})  "
                  f"p0={res['p0']:.1f} (Hertz {p_ref:.1f}, {res['p0'] / p_ref - 1:+.2%})  F={res['F']:.2f} "
                  f"rounds={res['rounds']} newton={res['stats'].newton_iters} cg={res['stats'].cg_iters} "
                  f"{time.time() - t:.1f}s", flush=True)
