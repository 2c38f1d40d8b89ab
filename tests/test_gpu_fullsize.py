"""Full-size parity at the benchmark's workload and launch configuration (BASELINE.json configs[4],
C5: 16,777,216 particles in the 513^3 node box, the kernels bench.py times).

The GPU runs P2G, the Newton gradient, the HVP and G2P on the WHOLE C5 particle set through the C
ABI.  The oracle cannot, so outputs are SAMPLED: a node's P2G / gradient / HVP value depends only on
the particles whose quadratic stencil covers it (base node within two cells below it on every
axis), and a particle's G2P result only on the grid values of its own stencil.  For each sampled
node (interior, faces, edges, corners of the cube) the oracle evaluates exactly those particles on
a cropped node box; for each sampled particle it runs G2P on that particle alone.  Node vectors u,
d and the grid velocity are closed-form fields of the node index, generated independently on both
sides.  Tolerance: rel L-inf <= 1e-11 over the samples (fp64 per-kernel bar, north_star)."""
import numpy as np
import pytest

import oracle
import synth
from gpu_helpers import rel_linf

pytestmark = pytest.mark.gpu

TOL = 1e-11
N_CELLS = int(__import__("os").environ.get("OSMPM_FULLSIZE_CELLS", "128"))


def field_np(k, scale, phase):
    """closed-form node field: scale * sin(0.7 k0 + 1.3 k1 + 2.1 k2 + phase + a), a = component"""
    base = 0.7 * k[:, 0] + 1.3 * k[:, 1] + 2.1 * k[:, 2] + phase
    return scale * np.sin(base[:, None] + np.arange(3)[None, :])


def field_torch(dims, scale, phase, dev):
    import torch
    idx = torch.arange(dims[0] * dims[1] * dims[2], device=dev, dtype=torch.int64)
    k2 = idx % dims[2]
    k1 = (idx // dims[2]) % dims[1]
    k0 = idx // (dims[1] * dims[2])
    base = 0.7 * k0.double() + 1.3 * k1.double() + 2.1 * k2.double() + phase
    out = scale * torch.sin(base[:, None] + torch.arange(3, device=dev, dtype=torch.float64)[None, :])
    return out.contiguous()


@pytest.fixture(scope="module")
def c5():
    sc = synth.c5_stress(n_cells=N_CELLS)
    x = sc.particles.x
    base = np.floor((x - np.asarray(sc.grid.origin)) / sc.grid.dx - 0.5).astype(np.int64)
    return sc, base


def _sample_nodes(base, rng):
    lo, hi = base.min(axis=0), base.max(axis=0) + 2  # node range touched by the particles
    mid = [rng.integers(lo + 3, hi - 3) for _ in range(24)]
    edge = []
    for _ in range(24):  # on faces / edges / corners (ragged: partially covered stencils)
        k = rng.integers(lo, hi + 1)
        for a in rng.choice(3, size=rng.integers(1, 4), replace=False):
            k[a] = rng.choice([lo[a], lo[a] + 1, hi[a] - 1, hi[a]])
        edge.append(k)
    return np.array(mid + edge)


def _crop_scene(sc, sel):
    """the particles `sel` on a node box aligned with the C5 grid covering the whole cube"""
    pt = sc.particles.subset(sel)
    x = sc.particles.x
    ext = np.stack([x.min(axis=0), x.max(axis=0)])
    grid = synth.grid_around(ext, sc.grid.dx, 4, 3, align_origin=np.asarray(sc.grid.origin))
    shift = np.round((np.asarray(grid.origin) - np.asarray(sc.grid.origin)) / sc.grid.dx).astype(np.int64)
    return synth.Scene(grid, pt, sc.materials, sc.dt, sc.gravity), shift


def test_fullsize_p2g_gradient_hvp_g2p_sampled(c5):
    import torch
    from paper_2605_09097_b200 import osmpm
    sc, base = c5
    dev = torch.device("cuda", 0)
    dims = sc.grid.dims
    dx, dt = sc.grid.dx, sc.dt
    rng = np.random.default_rng(2024)
    ctx = osmpm.Context(0, torch.cuda.current_stream(dev).cuda_stream)
    sub = osmpm.Subdomain(ctx, sc.grid, sc.dt, sc.particles, sc.materials, sc.gravity)
    assert sub.n == 8 * N_CELLS ** 3

    # ---- GPU at full size --------------------------------------------------------------------
    sub.p2g()
    grid = sub.read_grid(device=dev)
    u = field_torch(dims, 1e-3 * dx, 0.3, dev)
    dvec = field_torch(dims, 1.0, 1.1, dev)
    g_gpu, E_gpu = sub.newton_gradient(u)
    y_gpu = sub.newton_hvp(dvec)
    del u, dvec

    # ---- sampled nodes: the oracle on their contributing particles ------------------------------
    nodes = _sample_nodes(base, rng)
    contrib = np.zeros(base.shape[0], dtype=bool)
    for k in nodes:
        contrib |= np.all((base >= k - 2) & (base <= k), axis=1)
    sel = np.nonzero(contrib)[0]
    sub_sc, shift = _crop_scene(sc, sel)
    cd = sub_sc.grid.dims
    kk = np.stack(np.meshgrid(*(np.arange(c) for c in cd), indexing="ij"), -1).reshape(-1, 3) + shift
    ref = oracle.p2g(sub_sc)
    u_c = field_np(kk, 1e-3 * dx, 0.3)
    d_c = field_np(kk, 1.0, 1.1)
    g_ref = oracle.gradient(sub_sc, ref, u_c)
    y_ref = oracle.hvp(sub_sc, ref, u_c, d_c)

    gi = (nodes[:, 0] * dims[1] + nodes[:, 1]) * dims[2] + nodes[:, 2]
    loc = nodes - shift
    ci = (loc[:, 0] * cd[1] + loc[:, 1]) * cd[2] + loc[:, 2]
    gi_t = torch.from_numpy(gi).to(dev)
    take = lambda t: t[gi_t].cpu().numpy()  # noqa: E731
    assert ref.active[ci].all()
    assert rel_linf(take(grid["m"]), ref.m[ci]) <= TOL
    assert rel_linf(take(grid["p"]), ref.p[ci]) <= TOL
    assert rel_linf(take(grid["v"]), ref.v[ci]) <= TOL
    assert rel_linf(take(grid["fsig"]), ref.fsig[ci]) <= TOL
    assert rel_linf(take(g_gpu), g_ref[ci]) <= TOL
    assert rel_linf(take(y_gpu), y_ref[ci]) <= TOL
    assert np.isfinite(E_gpu)
    del grid, g_gpu, y_gpu

    # ---- G2P at full size, sampled particles -----------------------------------------------------
    vg = field_torch(dims, 0.05, 2.0, dev)
    sub.set_grid_velocity(vg)
    del vg
    sub.g2p()
    sub.sync()
    out = sub.read_particles(device=dev)
    ps = np.sort(rng.choice(sc.particles.n, size=256, replace=False))
    ps = np.concatenate([ps, [0, sc.particles.n - 1]])
    psc, shift = _crop_scene(sc, ps)
    cd = psc.grid.dims
    kk = np.stack(np.meshgrid(*(np.arange(c) for c in cd), indexing="ij"), -1).reshape(-1, 3) + shift
    pref = oracle.g2p(psc, field_np(kk, 0.05, 2.0))
    ps_t = torch.from_numpy(ps).to(dev)
    for k in ("x", "v", "F", "B"):
        assert rel_linf(out[k][ps_t].cpu().numpy(), getattr(pref, k)) <= TOL, k
    sub.close()
    ctx.close()
