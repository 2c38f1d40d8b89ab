"""Eshelby inclusion check (§4.3; tests/golden/g8_eshelby.txt): a circular inclusion
of radius R whose particles start with the misfit deformation gradient F0 = (1 - delta) I
inside an elastic matrix, relaxed to static equilibrium by single-domain MPM (one backward-Euler step
with a time step so large that the inertia term vanishes, as in the Euler-Bernoulli and Hertz checks;
plane strain, neo-Hookean, 2x2 particles per cell), against the Lame solution of the paper:

  P = delta / (C_out + C_in),  C_out = 1 / (2 G_out),  C_in = (1 - 2 nu_in) / (2 G_in)
  r < R:  sigma_rr = sigma_tt = -P;   r >= R:  sigma_rr = -P (R/r)^2,  sigma_tt = P (R/r)^2

The paper's formulas hold for an unbounded matrix.  The matrix here is a disk of radius b (traction
free), so the reference is the same Lame construction with the outer boundary kept (`lame_finite`):
inclusion u = A r, matrix u = B r + C / r, plane-strain stresses sigma_rr = 2(lam + G) a - 2 G c / r^2,
sigma_tt = 2(lam + G) a + 2 G c / r^2 for u = a r + c / r, with (i) sigma_rr(b) = 0, (ii) u continuous
at R, (iii) sigma_rr continuous at R, the inclusion's elastic strain being A - delta (F_e = (I + grad u) F0
= (1 + A - delta) I to first order); b -> infinity gives back the paper's P (tests pin that limit).
Symmetry makes the centre lines exact mirror planes of the lattice: v_x = 0 on x = xc, v_y = 0 on
y = yc (removes the rigid modes of the traction-free problem).

Stresses are sampled at particles, sigma = P(F) F^T / J with the particles' F after G2P, and compared
with the reference: the inclusion's mean in-plane pressure over r < R - 2h, and the relative L2 error
of (sigma_rr, sigma_tt) over the matrix annulus 1.5 R < r < b - 3h.

  python scripts/eshelby.py [--gpu] [--oracle] [--ratio 1 2 5] [--dx 32 64 128]   (cells per metre)
"""
import argparse
import math
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import synth  # noqa: E402

E_OUT, NU, RHO = 1.0e5, 0.3, 1000.0   # PAPER.md:605 (E_out = 1.0e2 kPa, nu = 0.3)
R_INC, B_OUT = 0.1, 0.5
DELTA = float(os.environ.get("ESHELBY_DELTA", "0.001"))  # linear-strain regime
XC = YC = 0.5


def lame(E, nu):
    return E * nu / ((1 + nu) * (1 - 2 * nu)), E / (2 * (1 + nu))


def paper_pressure(ratio, delta=DELTA):
    """P = delta / (C_out + C_in), unbounded matrix."""
    _, Go = lame(E_OUT, NU)
    _, Gi = lame(E_OUT * ratio, NU)
    return delta / (1.0 / (2 * Go) + (1 - 2 * NU) / (2 * Gi))


def lame_finite(ratio, delta=DELTA, R=R_INC, b=B_OUT):
    """(A, B, C) of the composite disk: inclusion u = A r, matrix u = B r + C / r (module docstring)."""
    li, Gi = lame(E_OUT * ratio, NU)
    lo, Go = lame(E_OUT, NU)
    ki, ko = 2 * (li + Gi), 2 * (lo + Go)
    # unknowns (A, B, C):  ko B - 2 Go C / b^2 = 0 ;  A R - B R - C / R = 0 ;
    #                      ki (A - delta) - ko B + 2 Go C / R^2 = 0
    M = np.array([[0.0, ko, -2 * Go / b ** 2], [R, -R, -1.0 / R], [ki, -ko, 2 * Go / R ** 2]])
    rhs = np.array([0.0, 0.0, ki * delta])
    A, B, C = np.linalg.solve(M, rhs)
    return A, B, C, (li, Gi, lo, Go)


def reference_stress(ratio, r, delta=DELTA, R=R_INC, b=B_OUT):
    """(sigma_rr, sigma_tt) of the finite composite disk at radii r."""
    A, B, C, (li, Gi, lo, Go) = lame_finite(ratio, delta, R, b)
    r = np.maximum(np.asarray(r, dtype=np.float64), 1e-12)
    s_in = 2 * (li + Gi) * (A - delta)
    srr = np.where(r < R, s_in, 2 * (lo + Go) * B - 2 * Go * C / r ** 2)
    stt = np.where(r < R, s_in, 2 * (lo + Go) * B + 2 * Go * C / r ** 2)
    return srr, stt


def scene(inv_dx, ratio, delta=DELTA, dt=10.0):
    dx = 1.0 / inv_dx
    c = np.array([XC, YC])
    x, vol = synth.lattice((XC - B_OUT, YC - B_OUT), (XC + B_OUT, YC + B_OUT), dx, 2,
                           inside=lambda p: ((p - c) ** 2).sum(axis=1) < B_OUT * B_OUT)
    r = np.sqrt(((x - c) ** 2).sum(axis=1))
    inc = r < R_INC
    p = synth.make_particles(x, vol, RHO, mat=inc.astype(np.int32))
    p.F[inc] = (1.0 - delta) * np.eye(2)          # F0 = (1 - delta) I
    grid = synth.grid_around(x, dx, 4, 2)
    sc = synth.Scene(grid, p, [(E_OUT, NU), (E_OUT * ratio, NU)], dt, (0.0, 0.0, 0.0), meta={"config": "Eshelby"})
    nx, ny = grid.dims[0], grid.dims[1]
    k = np.stack(np.meshgrid(np.arange(nx), np.arange(ny), indexing="ij"), -1).reshape(-1, 2)
    xs = np.asarray(grid.origin[:2]) + k * dx
    bits = np.zeros(xs.shape[0], np.uint8)
    bits[np.abs(xs[:, 0] - XC) <= 1e-12] |= 1
    bits[np.abs(xs[:, 1] - YC) <= 1e-12] |= 2
    sel = np.flatnonzero(bits)
    return sc, sel, bits[sel]


def cauchy(F, mu, lam):
    """sigma = (mu / J)(F F^T - I) + (lam ln J / J) I, the Cauchy stress of the neo-Hookean P (R2)."""
    J = F[:, 0, 0] * F[:, 1, 1] - F[:, 0, 1] * F[:, 1, 0]
    FFt = np.einsum("nij,nkj->nik", F, F)
    s = (mu / J)[:, None, None] * (FFt - np.eye(2)) + (lam * np.log(J) / J)[:, None, None] * np.eye(2)
    return s


def measure(sc, ratio, x0, F, delta=DELTA):
    dx = sc.grid.dx
    mat = sc.particles.mat
    lo, Go = lame(E_OUT, NU)
    li, Gi = lame(E_OUT * ratio, NU)
    mu = np.where(mat == 1, Gi, Go)
    lam = np.where(mat == 1, li, lo)
    sig = cauchy(F, mu, lam)
    d = x0 - np.array([XC, YC])
    r = np.sqrt((d ** 2).sum(axis=1))
    er = d / np.maximum(r, 1e-300)[:, None]
    et = np.stack([-er[:, 1], er[:, 0]], axis=1)
    srr = np.einsum("ni,nij,nj->n", er, sig, er)
    stt = np.einsum("ni,nij,nj->n", et, sig, et)
    ref_rr, ref_tt = reference_stress(ratio, r, delta)
    inside = r < R_INC - 2 * dx
    ann = (r > 1.5 * R_INC) & (r < B_OUT - 3 * dx)
    p_in = -0.5 * (sig[inside, 0, 0] + sig[inside, 1, 1]).mean()
    num = np.sqrt(((srr[ann] - ref_rr[ann]) ** 2 + (stt[ann] - ref_tt[ann]) ** 2).sum())
    den = np.sqrt((ref_rr[ann] ** 2 + ref_tt[ann] ** 2).sum())
    return dict(p_in=p_in, p_ref=-reference_stress(ratio, [0.0], delta)[0][0], err_out=num / den)


def _settings(max_cg):
    # the static Newton reaches the energy's roundoff floor (R8 line search) near |g| ~ 1e-7 |g0| once
    # the inclusion is stiffer than the matrix; 1e-7 |g0| is ~1e-10 of the interface traction
    return dict(newton_rtol=1e-7, cg_rtol=1e-10, max_cg=max_cg, max_newton=40)


def run_gpu(inv_dx, ratio, max_cg=40000):
    from paper_2605_09097_b200 import osmpm
    sc, sel, bits = scene(inv_dx, ratio)
    ctx = osmpm.Context(0)
    sub = osmpm.Subdomain(ctx, sc.grid, sc.dt, sc.particles, sc.materials, sc.gravity)
    try:
        sub.set_dirichlet(sel, bits, np.zeros((sel.size, 2)))
        sub.p2g()
        st = sub.implicit_solve(osmpm.newton_settings(**_settings(max_cg)))
        sub.g2p()
        out = sub.read_particles()
        res = measure(sc, ratio, sc.particles.x, out["F"])
        res.update(stats=st, F=out["F"])
        return res
    finally:
        sub.close()
        ctx.close()


def run_oracle(inv_dx, ratio, max_cg=40000):
    import oracle
    sc, sel, bits = scene(inv_dx, ratio)
    gs = oracle.p2g(sc)
    nn = oracle.n_nodes(sc.grid)
    dm = np.zeros((nn, 2), np.uint8)
    dm[sel, 0] = bits & 1
    dm[sel, 1] = (bits >> 1) & 1
    u, st = oracle.implicit_solve(sc, gs, oracle.default_settings(**_settings(max_cg)), dirichlet_mask=dm,
                                  dirichlet_v=np.zeros((nn, 2)))
    act = gs.active.astype(bool)
    pts = oracle.g2p(sc, np.where(act[:, None], u / sc.dt, 0.0))
    res = measure(sc, ratio, sc.particles.x, pts.F)
    res.update(stats=st, F=pts.F)
    return res


if __name__ == "__main__":
    import time
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpu", action="store_true")
    ap.add_argument("--oracle", action="store_true")
    ap.add_argument("--ratio", type=float, nargs="+", default=[1.0, 2.0, 5.0])
    ap.add_argument("--dx", type=int, nargs="+", default=[32, 64, 128])
    a = ap.parse_args()
    for ratio in a.ratio:
        print(f"ratio {ratio:g}: P (paper, unbounded) = {paper_pressure(ratio):.3f}, "
              f"P (disk b = {B_OUT}) = {-reference_stress(ratio, [0.0])[0][0]:.3f}", flush=True)
        for n in a.dx:
            for kind, fn in (("gpu", run_gpu), ("oracle", run_oracle)):
                if not getattr(a, kind):
                    continue
                t = time.time()
                res = fn(n, ratio)
                print(f"  {kind:6s} dx=1/{n:<5d} p_in={res['p_in']:.3f} ({res['p_in'] / res['p_ref'] - 1:+.2%})  "
                      f"err_out={res['err_out']:.4f}  newton={res['stats'].newton_iters} cg={res['stats'].cg_iters} "
                      f"{time.time() - t:.1f}s", flush=True)
