"""Oracle O11-O12: boundary grid sets, overlap arbitration and the multiplicative Schwarz frame
(§3.2.1, §3.3-3.5, Alg. 1 at PAPER.md:436-481), written step by step in the paper's order
on top of the pinned C primitives (p2g, implicit_solve, g2p, project, interp).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Readings of the paper that this file takes are
DESIGN.md R10-R16 (= SURVEY.md Z13-Z26); each is cited where it is used.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import (boundary_mass, default_settings, g2p, implicit_solve, interp, median, node_shape, p2g, project)


def node_positions(grid):
    d = grid.dim
    shp = node_shape(grid)
    k = np.stack(np.meshgrid(*[np.arange(s) for s in shp], indexing="ij"), -1).reshape(-1, d)
    return np.asarray(grid.origin[:d]) + k * grid.dx, k


def gamma_set(scene, gs, tau_rel):
    """Gamma_alpha = {i active : sum_{p in P^∂} m_p N_i(x_p) > tau_Gamma} (Eq.
    boundary_grid_set); tau_Gamma = tau_rel * median particle mass (R11)."""
    tau = tau_rel * median(scene.particles.m)
    mb = boundary_mass(scene)
    return (gs.active.astype(bool) & (mb > tau)), tau


def coincident_coarse_index(grid_b, xs, tol):
    """Index of the coarse node at the same physical location as each fine node, or -1 (R12)."""
    d = grid_b.dim
    X = (xs - np.asarray(grid_b.origin[:d])) / grid_b.dx
    k = np.round(X).astype(np.int64)
    ok = np.all(np.abs(X - k) * grid_b.dx <= tol, axis=1)
    for a in range(d):
        ok &= (k[:, a] >= 0) & (k[:, a] < grid_b.dims[a])
    idx = np.full(xs.shape[0], -1, np.int64)
    if d == 3:
        idx[ok] = (k[ok, 0] * grid_b.dims[1] + k[ok, 1]) * grid_b.dims[2] + k[ok, 2]
    else:
        idx[ok] = k[ok, 0] * grid_b.dims[1] + k[ok, 1]
    return idx


def receivers(coarse, fine, gsB, gsS, tau_rel):
    """Gamma-hat_B, Gamma-hat_S after the mass arbitration of coincident boundary nodes
    (Eq. overlap_donor: donor = argmax nodal mass, tie -> B) and the eligibility
    filter of DESIGN.md R13.  Returns boolean masks over the dense node boxes."""
    gB, tauB = gamma_set(coarse, gsB, tau_rel)
    gS, tauS = gamma_set(fine, gsS, tau_rel)
    xs, _ = node_positions(fine.grid)
    tol = 1e-9 * min(coarse.grid.dx, fine.grid.dx)
    cidx = coincident_coarse_index(coarse.grid, xs, tol)
    hatB = gB.copy()
    hatS = gS.copy()
    for j in np.flatnonzero(gS & (cidx >= 0)):
        I = cidx[j]
        if not gB[I]:
            continue
        # ambiguous node: the donor keeps no Dirichlet condition there
        if gsB.m[I] >= gsS.m[j]:       # donor B (ties -> B): S receives, B is free
            hatB[I] = False
        else:                          # donor S: B receives, S is free
            hatS[j] = False
    # eligibility (R13): coarse receivers need fine support, fine receivers need active coarse support
    _, _, den = project(fine.grid, gsS, coarse.grid, 0.0)
    hatB &= den > tauB
    cb = coarse.grid
    for j in np.flatnonzero(hatS):
        X = (xs[j] - np.asarray(cb.origin[:cb.dim])) / cb.dx
        base = np.floor(X - 0.5).astype(np.int64)
        f = X - base
        ok = True
        for off in np.ndindex(*([3] * cb.dim)):
            w = 1.0
            for a in range(cb.dim):
                fa = f[a]
                wa = (0.5 * (1.5 - fa) ** 2, 0.75 - (fa - 1.0) ** 2, 0.5 * (fa - 0.5) ** 2)[off[a]]
                w *= wa
            if w <= 0.0:
                continue
            kk = base + np.asarray(off)
            if np.any(kk < 0) or np.any(kk >= np.asarray(cb.dims[:cb.dim])):
                ok = False
                break
            I = (kk[0] * cb.dims[1] + kk[1]) * cb.dims[2] + kk[2] if cb.dim == 3 else kk[0] * cb.dims[1] + kk[1]
            if not gsB.active[I]:
                ok = False
                break
        hatS[j] = ok
    return hatB, hatS


@dataclass
class UserBC:
    """Physical Dirichlet conditions of one subdomain (clamp / contact / driven), dense masks."""
    mask: np.ndarray = None   # (nn, d) uint8
    vel: np.ndarray = None    # (nn, d)


@dataclass
class SchwarzResult:
    coarse_particles: object
    fine_particles: object
    iters: int
    r_B: list = field(default_factory=list)
    r_S: list = field(default_factory=list)
    n_recv_B: int = 0
    n_recv_S: int = 0
    converged: bool = False


def _residual(new, old):
    """relative l2 change over all receivers and components (zero denominator ->
    absolute, R15)"""
    den = np.linalg.norm(new)
    num = np.linalg.norm(new - old)
    return num / den if den > 0 else num


def _dirichlet(nn, d, recv_mask, recv_vel, user: UserBC):
    m = np.zeros((nn, d), np.uint8)
    v = np.zeros((nn, d))
    if user is not None and user.mask is not None:
        m |= user.mask
        v = np.where(user.mask.astype(bool), user.vel, v)
    if recv_mask is not None:
        rm = recv_mask.astype(bool)
        m[rm] = 1
        v[rm] = recv_vel[rm]
    return m, v


def schwarz_step(coarse, fine, M, eps_conv=1e-5, eps_tol=None, tau_rel=1e-6, k_max=100, parity_fixed_k=0,
                 newton_coarse=None, newton_fine=None, user_B: UserBC = None, user_S: UserBC = None):
    """One global frame t_n -> t_{n+1} of Alg. 1.  `coarse.dt` is the coarse step
    dT and `fine.dt` the fine step dt = dT / M.  Returns the new particle sets."""
    d = fine.grid.dim
    ncB = newton_coarse or default_settings(newton_rtol=1e-12, cg_rtol=1e-12, max_cg=20000)
    ncS = newton_fine or default_settings(newton_rtol=1e-12, cg_rtol=1e-12, max_cg=20000)
    if eps_tol is None:
        eps_tol = 1e-12 * float(fine.particles.m.sum())   # DESIGN.md R14
    # ---- Step 0 ----------------------------------------------------------
    stored = fine.particles.copy()                                       # Eq. store_states
    gsB = p2g(coarse)
    gsS = p2g(fine, stored)
    hatB, hatS = receivers(coarse, fine, gsB, gsS, tau_rel)
    nnB = gsB.m.shape[0]
    nnS = gsS.m.shape[0]
    recvB = np.flatnonzero(hatB)
    recvS = np.flatnonzero(hatS)
    vGB, _, _ = project(fine.grid, gsS, coarse.grid, eps_tol)           # v_GammaB^(0) = Pi(v_S^n), R16
    vGB = vGB[recvB]
    vB_prev = gsB.v.copy()                                              # v_B^(0) := v_B^n (R15)
    res = SchwarzResult(coarse.particles, stored, 0, n_recv_B=len(recvB), n_recv_S=len(recvS))
    n_iter = parity_fixed_k if parity_fixed_k > 0 else k_max
    vB_new = None
    fine_pt = stored
    for k in range(n_iter):
        # ---- Step 1: coarse solve over dT with Dirichlet Gamma-hat_B <- v_GammaB^(k) (Eq. implicit_solve_coarse)
        rv = np.zeros((nnB, d))
        rv[recvB] = vGB
        mB, vB_bc = _dirichlet(nnB, d, hatB, rv, user_B)
        uB, _ = implicit_solve(coarse, gsB, ncB, dirichlet_mask=mB, dirichlet_v=vB_bc)
        vB_new = np.where(gsB.active[:, None].astype(bool), uB / coarse.dt, 0.0)
        # ---- Step 2: restore, P2G, endpoint interpolation (Eq. spatial_interp_n) -------------------
        fine_pt = stored.copy()                                          # Alg. 1
        vS_n = interp(coarse.grid, gsB.v, gsB.v, 0.0, fine.grid, recvS)     # I(v_B^n)
        vS_np1 = interp(coarse.grid, vB_new, vB_new, 0.0, fine.grid, recvS)  # I(v_B^(k+1))
        last = None
        for m in range(1, M + 1):
            gsm = p2g(fine, fine_pt)                                     # (re)P2G of the current state
            alpha = m / M                                                # Eq. temporal_interp
            vbc = (1.0 - alpha) * vS_n + alpha * vS_np1
            rv = np.zeros((nnS, d))
            rv[recvS] = vbc
            mS, vS_bc = _dirichlet(nnS, d, hatS, rv, user_S)            # Gamma-hat_S ∩ active (R14)
            uS, _ = implicit_solve(fine, gsm, ncS, dirichlet_mask=mS, dirichlet_v=vS_bc, particles=fine_pt)
            vS_sol = np.where(gsm.active[:, None].astype(bool), uS / fine.dt, 0.0)
            fine_pt = g2p(fine, vS_sol, particles=fine_pt)               # Eqs. g2p_*_substep, advect
            last = (gsm, vS_sol)
        # ---- Step 3: interface residuals (Eqs. convergence_residuals / criterion) ----------------
        gsm, vS_sol = last
        vGB_new, _, _ = project(fine.grid, gsm, coarse.grid, eps_tol, v_fine=vS_sol)   # R16
        vGB_new = vGB_new[recvB]
        rB = _residual(vGB_new, vGB)
        vS_old = interp(coarse.grid, vB_prev, vB_prev, 0.0, fine.grid, recvS)
        rS = _residual(vS_np1, vS_old)
        res.r_B.append(rB)
        res.r_S.append(rS)
        res.iters = k + 1
        vGB = vGB_new
        vB_prev = vB_new
        if rB <= eps_conv and rS <= eps_conv:
            res.converged = True
            if parity_fixed_k <= 0:
                break
    # ---- Step 4: post-convergence coarse G2P + advection ------------------------
    res.coarse_particles = g2p(coarse, vB_new)
    res.fine_particles = fine_pt
    return res
