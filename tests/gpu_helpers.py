"""Shared helpers of the GPU parity tests (marshalling + the error metric of DESIGN.md R15)."""
import numpy as np


def rel_linf(a, b):
    """max|a - b| / max|b| over all entries."""
    a = np.asarray(a, dtype=np.float64)
    b = np.asarray(b, dtype=np.float64)
    den = np.abs(b).max()
    if den == 0:
        return np.abs(a).max()
    return np.abs(a - b).max() / den


def make_sub(ctx, scene, precision=0):
    from paper_2605_09097_b200 import osmpm
    return osmpm.Subdomain(ctx, scene.grid, scene.dt, scene.particles, scene.materials, scene.gravity,
                           precision=precision)


def random_u(gs_active, d, scale, seed):
    rng = np.random.default_rng(seed)
    u = np.zeros((gs_active.shape[0], d))
    act = gs_active.astype(bool)
    u[act] = rng.normal(0.0, scale, size=(act.sum(), d))
    return u
