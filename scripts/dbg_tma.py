"""HVP tensor-map prefetch debugging: c5_stress scenes of growing size, one HVP each."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2605_09097_b200 import osmpm  # noqa: E402

dev = torch.device("cuda", 0)
for n in [int(a) for a in sys.argv[1:]] or [8, 16, 24, 32, 48, 64, 96, 128]:
    sc = synth.c5_stress(n_cells=n)
    ctx = osmpm.Context(0, torch.cuda.current_stream(dev).cuda_stream)
    sub = osmpm.Subdomain(ctx, sc.grid, sc.dt, sc.particles, sc.materials, sc.gravity)
    sub.p2g()
    dims = sc.grid.dims
    nn = dims[0] * dims[1] * dims[2]
    u = torch.full((nn, 3), 1e-7, device=dev, dtype=torch.float64)
    d = torch.ones((nn, 3), device=dev, dtype=torch.float64)
    try:
        sub.newton_gradient(u)
        y = sub.newton_hvp(d)
        sub.sync()
        print(n, sub.n, "ok", float(y.abs().sum()), flush=True)
    except Exception as e:  # noqa: BLE001
        print(n, sub.n, "FAIL", e, flush=True)
        break
    sub.close()
    ctx.close()
