"""ctypes front end of the fp64 CPU oracle (oracle/osmpm_oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs.  The product package never imports this module.

Every function here is argument marshalling around the C definition it names; the
arithmetic lives in osmpm_oracle.c (each C function cites its PAPER.md passage).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "osmpm_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

OK, OUT_OF_DOMAIN, INVERTED, NEWTON_NC, LS_STAGNATION = 0, 1, 2, 3, 4


class OrcGrid(C.Structure):
    _fields_ = [("d", C.c_int32), ("o", C.c_double * 3), ("dx", C.c_double), ("n", C.c_int64 * 3)]


class OrcNewtonSettings(C.Structure):
    _fields_ = [("max_newton", C.c_int32), ("max_cg", C.c_int32), ("fixed_iters", C.c_int32),
                ("guess", C.c_int32), ("newton_rtol", C.c_double), ("newton_atol", C.c_double),
                ("cg_rtol", C.c_double), ("ls_min_alpha", C.c_double),
                ("energy_noise_rtol", C.c_double), ("cg_variant", C.c_int32), ("psd", C.c_int32)]


class OrcSolveStats(C.Structure):
    _fields_ = [("newton_iters", C.c_int32), ("cg_iters", C.c_int32), ("ls_halvings", C.c_int32),
                ("status", C.c_int32), ("grad_norm0", C.c_double), ("grad_norm", C.c_double),
                ("energy", C.c_double), ("negcurv", C.c_int32), ("ls_failures", C.c_int32),
                ("floor_accept", C.c_int32), ("psd_solves", C.c_int32)]


def build(force: bool = False) -> str:
    """Compile the oracle with plain IEEE semantics (no FMA contraction, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        subprocess.check_call(["gcc", "-O2", "-ffp-contract=off", "-fno-fast-math", "-std=c99",
                               "-shared", "-fPIC", "-o", _LIB, _SRC, "-lm"])
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        _lib = C.CDLL(build())
        _lib.orc_psi.restype = C.c_double
        _lib.orc_median.restype = C.c_double
    return _lib


def _p(a, dtype=np.float64):
    assert a.dtype == dtype and a.flags.c_contiguous, (a.dtype, a.flags)
    return a.ctypes.data_as(C.c_void_p)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def grid_struct(grid) -> OrcGrid:
    g = OrcGrid()
    g.d = grid.dim
    for a in range(3):
        g.o[a] = grid.origin[a]
        g.n[a] = grid.dims[a] if a < grid.dim else 1
    g.dx = grid.dx
    return g


def node_shape(grid):
    return tuple(grid.dims[: grid.dim])


def n_nodes(grid):
    return int(np.prod(node_shape(grid)))


def mats_arrays(materials):
    E = np.array([m[0] for m in materials], dtype=np.float64)
    nu = np.array([m[1] for m in materials], dtype=np.float64)
    return E, nu


def check(rc, what):
    if rc != OK:
        raise RuntimeError(f"oracle {what} failed with status {rc}")


# --------------------------------------------------------------------------------------------
# O1 stencil, O3 constitutive
# --------------------------------------------------------------------------------------------

def bspline1(f, dx=1.0):
    w = np.zeros(3)
    dw = np.zeros(3)
    lib().orc_bspline1(C.c_double(f), C.c_double(dx), _p(w), _p(dw))
    return w, dw


def stencil(grid, x):
    """(node indices, N, grad N, x_i - x_p) of one point; None if outside the safe interior."""
    g = grid_struct(grid)
    d = grid.dim
    idx = np.zeros(27, np.int64)
    N = np.zeros(27)
    gN = np.zeros(81)
    xip = np.zeros(81)
    c = lib().orc_stencil(C.byref(g), _p(_f64(x)), _p(idx, np.int64), _p(N), _p(gN), _p(xip))
    if c < 0:
        return None
    return idx[:c], N[:c], gN[: c * d].reshape(c, d), xip[: c * d].reshape(c, d)


def lame(E, nu):
    mu = C.c_double()
    lam = C.c_double()
    lib().orc_lame(C.c_double(E), C.c_double(nu), C.byref(mu), C.byref(lam))
    return mu.value, lam.value


def psi(F, mu, lam):
    F = _f64(F)
    return lib().orc_psi(C.c_int(F.shape[0]), _p(F), C.c_double(mu), C.c_double(lam))


def P(F, mu, lam):
    F = _f64(F)
    out = np.zeros_like(F)
    lib().orc_P(C.c_int(F.shape[0]), _p(F), C.c_double(mu), C.c_double(lam), _p(out))
    return out


def dP(F, dF, mu, lam):
    F = _f64(F)
    dF = _f64(dF)
    out = np.zeros_like(F)
    lib().orc_dP(C.c_int(F.shape[0]), _p(F), _p(dF), C.c_double(mu), C.c_double(lam), _p(out))
    return out


def median(v):
    v = _f64(v)
    return lib().orc_median(C.c_int64(v.shape[0]), _p(v))


# --------------------------------------------------------------------------------------------
# O2 P2G, Γ mass
# --------------------------------------------------------------------------------------------

class GridState:
    """Dense node-box fields produced by P2G (shape (n_nodes,) / (n_nodes, d))."""

    def __init__(self, m, p, v, fext, fsig, active):
        self.m, self.p, self.v, self.fext, self.fsig, self.active = m, p, v, fext, fsig, active


def p2g(scene, particles=None) -> GridState:
    pt = scene.particles if particles is None else particles
    grid = scene.grid
    g = grid_struct(grid)
    d = grid.dim
    nn = n_nodes(grid)
    E, nu = mats_arrays(scene.materials)
    m = np.zeros(nn)
    p = np.zeros((nn, d))
    v = np.zeros((nn, d))
    fext = np.zeros((nn, d))
    fsig = np.zeros((nn, d))
    act = np.zeros(nn, np.uint8)
    bad = C.c_int64(-1)
    grav = _f64(np.array(scene.gravity[:3]))
    rc = lib().orc_p2g(C.byref(g), C.c_int64(pt.n), _p(_f64(pt.x)), _p(_f64(pt.v)), _p(_f64(pt.F)),
                       _p(_f64(pt.B)), _p(_f64(pt.m)), _p(_f64(pt.V0)), _p(pt.mat, np.int32),
                       _p(E), _p(nu), _p(grav), _p(m), _p(p), _p(v), _p(fext), _p(fsig),
                       _p(act, np.uint8), C.byref(bad))
    check(rc, f"p2g (particle {bad.value})")
    return GridState(m, p, v, fext, fsig, act)


def boundary_mass(scene, particles=None):
    pt = scene.particles if particles is None else particles
    g = grid_struct(scene.grid)
    mb = np.zeros(n_nodes(scene.grid))
    rc = lib().orc_boundary_mass(C.byref(g), C.c_int64(pt.n), _p(_f64(pt.x)), _p(_f64(pt.m)),
                                 _p(pt.boundary, np.uint8), _p(mb))
    check(rc, "boundary_mass")
    return mb


# --------------------------------------------------------------------------------------------
# O4-O7 Newton operators and solve
# --------------------------------------------------------------------------------------------

def _newton_args(scene, particles):
    pt = scene.particles if particles is None else particles
    E, nu = mats_arrays(scene.materials)
    return pt, (C.c_int64(pt.n), _p(_f64(pt.x)), _p(_f64(pt.F)), _p(_f64(pt.V0)),
                _p(pt.mat, np.int32), _p(E), _p(nu), C.c_double(scene.dt)), (E, nu)


def energy(scene, gs: GridState, u, particles=None):
    pt, args, keep = _newton_args(scene, particles)
    g = grid_struct(scene.grid)
    e = C.c_double()
    ea = C.c_double()
    u = _f64(u)
    rc = lib().orc_energy(C.byref(g), *args, _p(gs.m), _p(gs.v), _p(gs.fext), _p(u), C.byref(e), C.byref(ea))
    check(rc, "energy")
    return e.value, ea.value


def gradient(scene, gs: GridState, u, particles=None):
    pt, args, keep = _newton_args(scene, particles)
    g = grid_struct(scene.grid)
    u = _f64(u)
    out = np.zeros_like(u)
    rc = lib().orc_gradient(C.byref(g), *args, _p(gs.m), _p(gs.v), _p(gs.fext), _p(u), _p(out))
    check(rc, "gradient")
    return out


def hvp(scene, gs: GridState, u, dvec, node_mask=None, particles=None, psd=False):
    """psd: per-particle tangent blocks projected to PSD (R23)."""
    pt, args, keep = _newton_args(scene, particles)
    g = grid_struct(scene.grid)
    u = _f64(u)
    dvec = _f64(dvec)
    out = np.zeros_like(u)
    nm = None if node_mask is None else np.ascontiguousarray(node_mask, dtype=np.uint8)
    rc = lib().orc_hvp_ex(C.byref(g), *args, _p(gs.m), _p(u), _p(dvec),
                          None if nm is None else _p(nm, np.uint8), _p(out), C.c_int(1 if psd else 0))
    check(rc, "hvp")
    return out


def diag(scene, gs: GridState, u, particles=None, psd=False):
    pt, args, keep = _newton_args(scene, particles)
    g = grid_struct(scene.grid)
    u = _f64(u)
    out = np.zeros_like(u)
    rc = lib().orc_diag_ex(C.byref(g), *args, _p(gs.m), _p(u), _p(out), C.c_int(1 if psd else 0))
    check(rc, "diag")
    return out


def tangent_psd(F, E, nu):
    """The PSD projection T+ of one particle's tangent block d^2 Psi / dF dF (d^2 x d^2, row-major vec)."""
    F = _f64(F)
    d = F.shape[0]
    mu, lam = lame(E, nu)
    out = np.zeros((d * d, d * d))
    lib().orc_tangent_psd(C.c_int(d), _p(np.ascontiguousarray(F)), C.c_double(mu), C.c_double(lam), _p(out))
    return out


def default_settings(**kw) -> OrcNewtonSettings:
    s = OrcNewtonSettings()
    s.max_newton = kw.get("max_newton", 50)
    s.max_cg = kw.get("max_cg", 1000)
    s.fixed_iters = kw.get("fixed_iters", 0)
    s.guess = kw.get("guess", 0)
    s.newton_rtol = kw.get("newton_rtol", 1e-8)
    s.newton_atol = kw.get("newton_atol", 0.0)
    s.cg_rtol = kw.get("cg_rtol", 1e-8)
    s.ls_min_alpha = kw.get("ls_min_alpha", 2.0 ** -20)
    s.energy_noise_rtol = kw.get("energy_noise_rtol", 1e-13)
    s.cg_variant = kw.get("cg_variant", 0)
    s.psd = kw.get("psd", 0)
    return s


def free_mask(gs: GridState, d, dirichlet_mask=None):
    """free DOF = active node and not a Dirichlet component."""
    fm = np.repeat(gs.active[:, None], d, axis=1).astype(np.uint8)
    if dirichlet_mask is not None:
        fm &= (1 - np.asarray(dirichlet_mask, np.uint8).reshape(fm.shape))
    return np.ascontiguousarray(fm)


def implicit_solve(scene, gs: GridState, settings=None, dirichlet_mask=None, dirichlet_v=None,
                   particles=None, u0=None, raise_on_error=True):
    """Returns (u, stats).  Dirichlet DOFs take u = dt * v_D; inactive DOFs u = 0."""
    pt, args, keep = _newton_args(scene, particles)
    g = grid_struct(scene.grid)
    d = scene.grid.dim
    st = settings or default_settings()
    fm = free_mask(gs, d, dirichlet_mask)
    u = np.zeros_like(gs.v) if u0 is None else np.array(u0, dtype=np.float64, copy=True)
    if dirichlet_mask is not None:
        dm = np.asarray(dirichlet_mask, np.uint8).reshape(u.shape).astype(bool)
        act = np.repeat(gs.active[:, None].astype(bool), d, axis=1)
        u[dm & act] = scene.dt * np.asarray(dirichlet_v, np.float64).reshape(u.shape)[dm & act]
    u[~np.repeat(gs.active[:, None].astype(bool), d, axis=1)] = 0.0
    u = np.ascontiguousarray(u)
    stats = OrcSolveStats()
    rc = lib().orc_implicit_solve(C.byref(g), *args, _p(gs.m), _p(gs.v), _p(gs.fext), _p(fm, np.uint8),
                                  C.byref(st), _p(u), C.byref(stats))
    if raise_on_error:
        check(rc, "implicit_solve")
    return u, stats


# --------------------------------------------------------------------------------------------
# O8 G2P, O9 Π, O10 I+T
# --------------------------------------------------------------------------------------------

def g2p(scene, vgrid, particles=None, dt=None):
    """Returns the updated particle set (a copy)."""
    pt = (scene.particles if particles is None else particles).copy()
    g = grid_struct(scene.grid)
    bad = C.c_int64(-1)
    vgrid = _f64(vgrid)
    rc = lib().orc_g2p(C.byref(g), C.c_int64(pt.n), _p(pt.x), _p(pt.v), _p(pt.F), _p(pt.B), _p(vgrid),
                       C.c_double(scene.dt if dt is None else dt), C.byref(bad))
    check(rc, f"g2p (particle {bad.value})")
    return pt


def project(grid_s, gs_fine: GridState, grid_b, eps_tol=0.0, v_fine=None, m_fine=None, active_fine=None):
    gS = grid_struct(grid_s)
    gB = grid_struct(grid_b)
    d = grid_s.dim
    nnb = n_nodes(grid_b)
    num = np.zeros((nnb, d))
    den = np.zeros(nnb)
    vb = np.zeros((nnb, d))
    ms = _f64(gs_fine.m if m_fine is None else m_fine)
    vs = _f64(gs_fine.v if v_fine is None else v_fine)
    act = np.ascontiguousarray(gs_fine.active if active_fine is None else active_fine, dtype=np.uint8)
    rc = lib().orc_project(C.byref(gS), _p(ms), _p(vs), _p(act, np.uint8), C.byref(gB),
                           C.c_double(eps_tol), _p(num), _p(den), _p(vb))
    check(rc, "project")
    return vb, num, den


def interp(grid_b, vb0, vb1, alpha, grid_s, targets):
    gB = grid_struct(grid_b)
    gS = grid_struct(grid_s)
    d = grid_b.dim
    t = np.ascontiguousarray(targets, dtype=np.int64)
    out = np.zeros((t.shape[0], d))
    rc = lib().orc_interp(C.byref(gB), _p(_f64(vb0)), _p(_f64(vb1)), C.c_double(alpha), C.byref(gS),
                          C.c_int64(t.shape[0]), _p(t, np.int64), _p(out))
    check(rc, "interp")
    return out
