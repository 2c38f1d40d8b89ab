"""Seeded synthetic inputs shared by the oracle tests, the GPU tests and bench.py.

This module holds NO arithmetic of the method (no shape functions, no transfers,
no constitutive law, no solver).  It only lays particles on lattices, draws
seeded random states and packages grid descriptors, exactly as DESIGN.md §3
("input recipe") states.  Both `oracle/` and the CUDA path consume the very
same arrays, so no cross-language RNG is needed.

Shapes follow BASELINE.json `configs` (C1..C5) with the resolutions fixed in
SURVEY.md App. A (A1-A13); random-state fixtures follow SURVEY.md §8(d)
("Parity fixtures").
"""
from __future__ import annotations

from dataclasses import dataclass, field
import math
import numpy as np


@dataclass
class Grid:
    """Node box: x_i = origin + dx * i, i in [0, dims)  (§2.2.2)."""
    dim: int
    origin: tuple
    dx: float
    dims: tuple  # always 3 entries; dims[2] == 1 in 2D

    @property
    def n_nodes(self) -> int:
        return int(np.prod(self.dims[: self.dim]))


@dataclass
class Particles:
    """Particle SoA in creation order (§2.2.4)."""
    x: np.ndarray          # (n, d) float64
    v: np.ndarray          # (n, d)
    F: np.ndarray          # (n, d, d) row-major
    B: np.ndarray          # (n, d, d)
    m: np.ndarray          # (n,)
    V0: np.ndarray         # (n,)
    mat: np.ndarray        # (n,) int32
    boundary: np.ndarray   # (n,) uint8  (P^∂ markers)

    @property
    def n(self) -> int:
        return self.x.shape[0]

    @property
    def dim(self) -> int:
        return self.x.shape[1]

    def copy(self) -> "Particles":
        return Particles(*(np.array(a, copy=True) for a in (
            self.x, self.v, self.F, self.B, self.m, self.V0, self.mat, self.boundary)))

    def subset(self, idx) -> "Particles":
        return Particles(*(np.ascontiguousarray(a[idx]) for a in (
            self.x, self.v, self.F, self.B, self.m, self.V0, self.mat, self.boundary)))


@dataclass
class Scene:
    grid: Grid
    particles: Particles
    materials: list            # [(E, nu), ...]
    dt: float
    gravity: tuple = (0.0, 0.0, 0.0)
    meta: dict = field(default_factory=dict)


# --------------------------------------------------------------------------------------------
# lattices
# --------------------------------------------------------------------------------------------

def lattice(lo, hi, dx, ppa, rng=None, jitter=0.0, inside=None):
    """Particles on a regular ppa^d lattice per cell of the cell lattice covering [lo, hi].

    Offsets inside a cell are (j + 1/2)/ppa * dx (e.g. ppa = 2 -> 1/4, 3/4).  With
    `jitter` > 0 each coordinate is perturbed by U(-jitter, jitter) * (dx / ppa)
    (BASELINE.json C1: "jittered by U(-0.1, 0.1)·spacing").
    `inside(x)` (vectorised) keeps only the particles it returns True for.
    Returns (n, d) float64 and the per-particle volume dx^d / ppa^d.
    """
    lo = np.asarray(lo, dtype=np.float64)
    hi = np.asarray(hi, dtype=np.float64)
    d = lo.shape[0]
    ncell = np.maximum(np.round((hi - lo) / dx).astype(np.int64), 1)
    axes = []
    for a in range(d):
        k = np.arange(ncell[a], dtype=np.float64)
        j = (np.arange(ppa, dtype=np.float64) + 0.5) / ppa
        axes.append((lo[a] + (k[:, None] + j[None, :]) * dx).reshape(-1))
    mesh = np.meshgrid(*axes, indexing="ij")
    x = np.stack([m.reshape(-1) for m in mesh], axis=1)
    if inside is not None:
        x = x[inside(x)]
    if jitter > 0.0:
        assert rng is not None
        x = x + rng.uniform(-jitter, jitter, size=x.shape) * (dx / ppa)
    vol = dx ** d / ppa ** d
    return np.ascontiguousarray(x), vol


def grid_around(x, dx, pad_cells, dim, align_origin=None):
    """A node box covering the particles plus `pad_cells` cells on every side.

    The origin is snapped to the lattice `align_origin + dx * k` (default 0), so that two
    grids with commensurate spacings share coincident nodes."""
    base = np.zeros(dim) if align_origin is None else np.asarray(align_origin, dtype=np.float64)
    lo = x.min(axis=0)
    hi = x.max(axis=0)
    klo = np.floor((lo - base) / dx).astype(np.int64) - pad_cells
    khi = np.ceil((hi - base) / dx).astype(np.int64) + pad_cells
    origin = base + klo * dx
    dims = (khi - klo + 1).astype(np.int64)
    o3 = [0.0, 0.0, 0.0]
    d3 = [1, 1, 1]
    for a in range(dim):
        o3[a] = float(origin[a])
        d3[a] = int(dims[a])
    return Grid(dim, tuple(o3), float(dx), tuple(d3))


def make_particles(x, vol, rho, rng=None, v_sigma=0.0, F_sigma=0.0, B_scale=0.0, dx=None,
                   mat=None, boundary=None, rho_range=None):
    """Particle states: m = rho*V0, v ~ N(0, v_sigma), F = I + N(0, F_sigma),
    B = (dx^2/4) * C with C ~ N(0, B_scale) (SURVEY.md §8(d) parity fixtures)."""
    n, d = x.shape
    V0 = np.full(n, vol, dtype=np.float64)
    if rho_range is not None:
        rhop = rng.uniform(rho_range[0], rho_range[1], size=n)
    else:
        rhop = np.full(n, rho, dtype=np.float64)
    m = rhop * V0
    v = rng.normal(0.0, v_sigma, size=(n, d)) if v_sigma > 0 else np.zeros((n, d))
    F = np.broadcast_to(np.eye(d), (n, d, d)).copy()
    if F_sigma > 0:
        F += rng.normal(0.0, F_sigma, size=(n, d, d))
    B = np.zeros((n, d, d))
    if B_scale > 0:
        B = rng.normal(0.0, B_scale, size=(n, d, d)) * (dx * dx / 4.0)
    mat = np.zeros(n, dtype=np.int32) if mat is None else np.asarray(mat, dtype=np.int32)
    boundary = np.zeros(n, dtype=np.uint8) if boundary is None else np.asarray(boundary, dtype=np.uint8)
    return Particles(np.ascontiguousarray(x, dtype=np.float64), v, F, B, m, V0, mat, boundary)


# --------------------------------------------------------------------------------------------
# random parity fixtures
# --------------------------------------------------------------------------------------------

def random_fixture(dim=3, cells=(6, 5, 4), ppa=2, seed=1, dx=0.1, F_sigma=0.05, B_scale=1.0,
                   v_sigma=0.3, jitter=0.45, pad=3, n_mats=2, boundary_frac=0.2, dt=1e-2,
                   gravity=(0.3, -9.81, 0.2), materials=None, rho=1000.0):
    """A jittered block of particles in random states (random F near I, random B, random v),
    two materials, random P^∂ flags: exercises every term the configs leave at zero."""
    rng = np.random.default_rng(seed)
    lo = np.full(dim, 0.35)
    hi = lo + np.asarray(cells[:dim], dtype=np.float64) * dx
    x, vol = lattice(lo, hi, dx, ppa, rng=rng, jitter=jitter)
    n = x.shape[0]
    mat = rng.integers(0, n_mats, size=n).astype(np.int32)
    bnd = (rng.uniform(size=n) < boundary_frac).astype(np.uint8)
    p = make_particles(x, vol, rho, rng=rng, v_sigma=v_sigma, F_sigma=F_sigma, B_scale=B_scale,
                       dx=dx, mat=mat, boundary=bnd, rho_range=(0.5 * rho, 1.5 * rho))
    grid = grid_around(x, dx, pad, dim)
    if materials is None:
        materials = [(1.0e5, 0.3), (3.0e5, 0.4)][:n_mats]
    g = tuple(list(gravity[:dim]) + [0.0] * (3 - dim))
    return Scene(grid, p, materials, dt, g, meta={"kind": "random_fixture", "seed": seed})


# --------------------------------------------------------------------------------------------
# BASELINE.json configs
# --------------------------------------------------------------------------------------------

def c1_cantilever(seed_fine=1000, seed_coarse=1001, g=9.81):
    """C1: 2D cantilever 1.0 x 0.2, clamped at x = 0, E = 1e5, nu = 0.3, rho = 1000.
    Fine Omega_S = x in [0, 0.3] at dx = 0.0125, coarse Omega_B = x in [0.2, 1.0] at dx = 0.05
    (SURVEY.md A1), 2x2 ppc, jitter U(-0.1, 0.1) * spacing.  Returns (coarse, fine) scenes.
    P^∂: particles within one own cell of the artificial cut."""
    y0 = 1.0
    out = []
    for (lo_x, hi_x, dx, seed, cut) in ((0.2, 1.0, 0.05, seed_coarse, 0.2),
                                         (0.0, 0.3, 0.0125, seed_fine, 0.3)):
        rng = np.random.default_rng(seed)
        x, vol = lattice((lo_x, y0), (hi_x, y0 + 0.2), dx, 2, rng=rng, jitter=0.1)
        bnd = (np.abs(x[:, 0] - cut) < dx).astype(np.uint8)
        p = make_particles(x, vol, 1000.0, rng=rng, boundary=bnd)
        grid = grid_around(x, dx, 4, 2)
        out.append(Scene(grid, p, [(1.0e5, 0.3)], 1e-2 if dx == 0.05 else 2.5e-3,
                         (0.0, -g, 0.0), meta={"config": "C1", "M": 4}))
    return out[0], out[1]


def c2_hertz(seed_fine=2000, seed_coarse=2001, ppa_fine=2):
    """C2: disk R = 0.5 centred (0, 0.5) on the plane y = 0; E = 1e6, nu = 0.3, rho = 1000.
    Fine box [-0.2, 0.2] x [0, 0.2] at 1/256, coarse = disk minus the box shrunk by 2 coarse
    cells at 1/32."""
    R = 0.5
    c = np.array([0.0, 0.5])

    def disk(x):
        return ((x - c) ** 2).sum(axis=1) < R * R

    rng = np.random.default_rng(seed_fine)
    dxs = 1.0 / 256
    xs, vs = lattice((-0.2, 0.0), (0.2, 0.2), dxs, ppa_fine, rng=rng, jitter=0.1,
                     inside=lambda x: disk(x) & (x[:, 1] > 0.0))
    bnd_s = ((np.abs(np.abs(xs[:, 0]) - 0.2) < dxs) | (np.abs(xs[:, 1] - 0.2) < dxs)).astype(np.uint8)
    ps = make_particles(xs, vs, 1000.0, rng=rng, boundary=bnd_s)
    rng = np.random.default_rng(seed_coarse)
    dxb = 1.0 / 32
    shrink = 2 * dxb
    xb, vb = lattice((-0.5, 0.0), (0.5, 1.0), dxb, 2, rng=rng, jitter=0.1,
                     inside=lambda x: disk(x) & ~((np.abs(x[:, 0]) < 0.2 - shrink) & (x[:, 1] < 0.2 - shrink)))
    inner = (np.abs(xb[:, 0]) < 0.2 - shrink + dxb) & (xb[:, 1] < 0.2 - shrink + dxb)
    pb = make_particles(xb, vb, 1000.0, rng=rng, boundary=inner.astype(np.uint8))
    gb = grid_around(xb, dxb, 4, 2)
    gs = grid_around(xs, dxs, 4, 2)
    mats = [(1.0e6, 0.3)]
    return (Scene(gb, pb, mats, 1e-2, (0.0, 0.0, 0.0), meta={"config": "C2", "M": 4}),
            Scene(gs, ps, mats, 2.5e-3, (0.0, 0.0, 0.0), meta={"config": "C2", "M": 4}))


def c3_inclusion(level=256, seed_fine=None, seed_coarse=3100):
    """C3: unit-square matrix (E = 1e5) with a centred inclusion r = 0.1 (E = 1e7), nu = 0.3.
    Fine [0.35, 0.65]^2 at dx = 1/level, 3x3 ppc; coarse = square minus [0.38125, 0.61875]^2
    at 1/64.  material id 1 inside the inclusion."""
    seed_fine = 3000 + level if seed_fine is None else seed_fine
    rng = np.random.default_rng(seed_fine)
    dxs = 1.0 / level
    xs, vs = lattice((0.35, 0.35), (0.65, 0.65), dxs, 3, rng=rng, jitter=0.1)
    mat_s = (((xs - 0.5) ** 2).sum(axis=1) < 0.01).astype(np.int32)
    bnd_s = (np.max(np.abs(xs - 0.5), axis=1) > 0.15 - dxs).astype(np.uint8)
    ps = make_particles(xs, vs, 1000.0, rng=rng, mat=mat_s, boundary=bnd_s)
    rng = np.random.default_rng(seed_coarse)
    dxb = 1.0 / 64
    xb, vb = lattice((0.0, 0.0), (1.0, 1.0), dxb, 3, rng=rng, jitter=0.1,
                     inside=lambda x: np.max(np.abs(x - 0.5), axis=1) > 0.11875)
    bnd_b = (np.max(np.abs(xb - 0.5), axis=1) < 0.11875 + dxb).astype(np.uint8)
    pb = make_particles(xb, vb, 1000.0, rng=rng, mat=np.zeros(xb.shape[0], np.int32), boundary=bnd_b)
    mats = [(1.0e5, 0.3), (1.0e7, 0.3)]
    M = level // 128
    return (Scene(grid_around(xb, dxb, 4, 2), pb, mats, 1e-2, (0.0, 0.0, 0.0), meta={"config": "C3", "M": M}),
            Scene(grid_around(xs, dxs, 4, 2), ps, mats, 1e-2 / M, (0.0, 0.0, 0.0), meta={"config": "C3", "M": M}))


def c4_fold(seed_fine=4000, seed_coarse=4001, y_extent=0.5):
    """C4: plate [0,1] x [0,0.5] x [0,0.04], E = 5e5, nu = 0.4; fine crease band
    x in [0.425, 0.575] at 1/256 (2x2x2 ppc), coarse plate minus x in [0.45625, 0.54375] at 1/64
    (A7).  `y_extent` < 0.5 gives the reduced band used for parity."""
    rng = np.random.default_rng(seed_fine)
    dxs = 1.0 / 256
    xs, vs = lattice((0.425, 0.0, 0.0), (0.575, y_extent, 0.04), dxs, 2)
    bnd_s = (np.abs(np.abs(xs[:, 0] - 0.5) - 0.075) < dxs).astype(np.uint8)
    ps = make_particles(xs, vs, 1000.0, rng=rng, boundary=bnd_s)
    rng = np.random.default_rng(seed_coarse)
    dxb = 1.0 / 64
    xb, vb = lattice((0.0, 0.0, 0.0), (1.0, y_extent, 0.04), dxb, 2,
                     inside=lambda x: np.abs(x[:, 0] - 0.5) > 0.04375)
    bnd_b = (np.abs(np.abs(xb[:, 0] - 0.5) - 0.04375) < dxb).astype(np.uint8)
    pb = make_particles(xb, vb, 1000.0, rng=rng, boundary=bnd_b)
    mats = [(5.0e5, 0.4)]
    return (Scene(grid_around(xb, dxb, 4, 3), pb, mats, 1e-2, (0.0, 0.0, -9.81), meta={"config": "C4", "M": 4}),
            Scene(grid_around(xs, dxs, 4, 3), ps, mats, 2.5e-3, (0.0, 0.0, -9.81), meta={"config": "C4", "M": 4}))


def c5_stress(n_cells=128, seed=5000, dx=1.0 / 512, full_box=True, pad=3):
    """C5: a random-density neo-Hookean cube of n_cells^3 cells at dx = 1/512 centred at
    (0.5, 0.5, 0.5) inside the 512^3 region, 8 ppc (2x2x2), rho ~ U(500, 1500),
    v ~ N(0, 0.1), F = I + N(0, 1e-3), B = 0, E = 1e5, nu = 0.3, dt = 1e-3.
    n_cells = 128 -> 16,777,216 particles; smaller n_cells give the oracle-sized cube."""
    rng = np.random.default_rng(seed)
    side = n_cells * dx
    lo = np.full(3, 0.5 - side / 2)
    # lattice() is vectorised; for 16.7M particles build it axis by axis to bound memory
    k = np.arange(n_cells, dtype=np.float64)
    off = np.array([0.25, 0.75])
    ax = (lo[0] + (k[:, None] + off[None, :]) * dx).reshape(-1)
    n1 = ax.shape[0]
    x = np.empty((n1 ** 3, 3), dtype=np.float64)
    x[:, 0] = np.repeat(ax, n1 * n1)
    x[:, 1] = np.tile(np.repeat(ax, n1), n1)
    x[:, 2] = np.tile(ax, n1 * n1)
    vol = dx ** 3 / 8.0
    n = x.shape[0]
    V0 = np.full(n, vol)
    m = rng.uniform(500.0, 1500.0, size=n) * vol
    v = rng.normal(0.0, 0.1, size=(n, 3))
    F = np.empty((n, 3, 3))
    F[:] = np.eye(3)
    F += rng.normal(0.0, 1e-3, size=(n, 3, 3))
    B = np.zeros((n, 3, 3))
    p = Particles(x, v, F, B, m, V0, np.zeros(n, np.int32), np.zeros(n, np.uint8))
    if full_box:
        grid = Grid(3, (0.0, 0.0, 0.0), dx, (513, 513, 513))
    else:
        grid = grid_around(x, dx, pad, 3)
    return Scene(grid, p, [(1.0e5, 0.3)], 1e-3, (0.0, 0.0, 0.0),
                 meta={"config": "C5", "n_cells": n_cells})


def c5_coarse_field(grid_fine: Grid, n_cells=128, seed=5001, dx_coarse=1.0 / 128, n_modes=8, amp=0.1):
    """Passive coarse overlap grid for C5: dx = 1/128 over the cube +- 2 coarse
    cells, with a smooth random velocity field = sum of `n_modes` random Fourier modes."""
    rng = np.random.default_rng(seed)
    side = n_cells * grid_fine.dx
    lo = 0.5 - side / 2 - 2 * dx_coarse
    k0 = int(math.floor(lo / dx_coarse + 1e-9))
    nn = int(round(side / dx_coarse)) + 5
    grid = Grid(3, (k0 * dx_coarse,) * 3, dx_coarse, (nn, nn, nn))
    idx = np.stack(np.meshgrid(*(np.arange(nn),) * 3, indexing="ij"), axis=-1).reshape(-1, 3)
    xn = np.asarray(grid.origin) + idx * dx_coarse
    v = np.zeros((xn.shape[0], 3))
    for _ in range(n_modes):
        kv = rng.normal(0.0, 2.0 * math.pi * 2.0, size=3)
        ph = rng.uniform(0, 2 * math.pi)
        a = rng.normal(0.0, amp, size=3)
        v += np.cos(xn @ kv + ph)[:, None] * a[None, :]
    return grid, v.reshape(nn, nn, nn, 3)


def c5_bench_workload(cells=128, full_box=True, pad=3):
    """The timed C5 workload of bench.py: the fine cube of c5_stress, a passive coarse
    subdomain of one particle per coarse cell carrying the smooth field of c5_coarse_field (its P2G
    gives v_B^n; bench.py sets v_B^{n+1} = 1.01 v_B^n), and the fine receivers: the fine nodes of the
    cube's footprint outside the cube shrunk by 2 cells, as linear indices of the fine node box.
    Returns (fine Scene, coarse Scene, receivers int64[])."""
    fine = c5_stress(n_cells=cells, full_box=full_box, pad=pad)
    cgrid, cvel = c5_coarse_field(fine.grid, n_cells=cells)
    side = cells * fine.grid.dx
    lo = 0.5 - side / 2
    xb, vol = lattice([lo] * 3, [lo + side] * 3, cgrid.dx, 1)
    cpart = make_particles(xb, vol, 1000.0)
    idx = np.clip(np.round((xb - np.asarray(cgrid.origin)) / cgrid.dx).astype(int), 0, cgrid.dims[0] - 1)
    cpart.v = np.ascontiguousarray(cvel[idx[:, 0], idx[:, 1], idx[:, 2]])
    coarse = Scene(cgrid, cpart, [(1.0e5, 0.3)], 4e-3, (0.0, 0.0, 0.0))
    # footprint nodes k0-1 .. k0+cells+1 (absolute node indices of the 1/512 lattice) minus the
    # cube shrunk by 2 cells, as indices of this fine grid's box
    dx = fine.grid.dx
    k0 = int(round(lo / dx))
    kk = np.arange(k0 - 1, k0 + cells + 2)
    K = np.stack(np.meshgrid(kk, kk, kk, indexing="ij"), -1).reshape(-1, 3)
    inner = np.all((K >= k0 + 2) & (K <= k0 + cells - 2), axis=1)
    R = K[~inner] - np.round(np.asarray(fine.grid.origin) / dx).astype(np.int64)[None, :]
    gd = fine.grid.dims
    assert (R >= 0).all() and (R < np.asarray(gd)[None, :3]).all()
    recv = (R[:, 0] * gd[1] + R[:, 1]) * gd[2] + R[:, 2]
    return fine, coarse, np.ascontiguousarray(recv.astype(np.int64))


def cantilever_pair(dx_coarse, r=4, ppa=3, L=1.0, H=0.2, x_fine=(0.0, 0.3), x_coarse=(0.2, 1.0), E=1.0e5, nu=0.4,
                    rho=1000.0, g=0.0, dT=10.0, M=1, y0=1.0, seed=1100):
    """The dual-domain cantilever of PAPER.md:511-549 (§4.1) at a chosen resolution: beam L x H clamped at
    x = 0, split longitudinally into a fine subdomain x in x_fine (dx = dx_coarse / r) and a coarse one
    x in x_coarse (dx_coarse), ppa x ppa particles per cell on the regular lattice (the paper: 9 per cell),
    material E, nu, rho (the paper: 100 kPa, 0.4, 1000), gravity g downward.  P^∂: particles within one own
    cell of each artificial cut (R10).  Returns (coarse, fine) scenes; dt = dT (coarse) and
    dT / M (fine)."""
    out = []
    for (lo_x, hi_x, dx, cut) in ((x_coarse[0], x_coarse[1], dx_coarse, x_coarse[0]),
                                  (x_fine[0], x_fine[1], dx_coarse / r, x_fine[1])):
        x, vol = lattice((lo_x, y0), (hi_x, y0 + H), dx, ppa)
        bnd = (np.abs(x[:, 0] - cut) < dx).astype(np.uint8)
        p = make_particles(x, vol, rho, boundary=bnd)
        grid = grid_around(np.vstack([x, [[lo_x - 0.3 * L, y0 - L], [hi_x + 0.1 * L, y0 + H + 0.1 * L]]]), dx, 4, 2)
        out.append(Scene(grid, p, [(E, nu)], dT if dx == dx_coarse else dT / M, (0.0, -g, 0.0),
                         meta={"config": "cantilever", "M": M}))
    return out[0], out[1]


def cantilever_single(dx, ppa=3, L=1.0, H=0.2, E=1.0e5, nu=0.4, rho=1000.0, g=0.0, dT=10.0, y0=1.0):
    """The single-domain cantilever of the same geometry ("single-domain")."""
    x, vol = lattice((0.0, y0), (L, y0 + H), dx, ppa)
    p = make_particles(x, vol, rho)
    grid = grid_around(np.vstack([x, [[0.0, y0 - L], [L, y0 + H + 0.1 * L]]]), dx, 4, 2)
    return Scene(grid, p, [(E, nu)], dT, (0.0, -g, 0.0), meta={"config": "cantilever"})  # the tip curls inward
