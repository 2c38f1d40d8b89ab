import sys; sys.path.insert(0,'tests'); sys.path.insert(0,'.')
import numpy as np, test_gpu_configs as T
from paper_2605_09097_b200 import osmpm
ctx = osmpm.Context(0)
coarse, fine, ref, rep, co, fo = T._frame(ctx, "c4", precision=osmpm.F32)
eps32 = float(np.finfo(np.float32).eps)
for nm, out, r, sc in (("fine", fo, ref.fine_particles, fine), ("coarse", co, ref.coarse_particles, coarse)):
    x0 = sc.particles.x
    for k, a0, rr in (("x", x0, r.x), ("v", 0*r.v, r.v), ("F", np.eye(3), r.F)):
        e = np.abs(out[k] - rr)
        print(nm, k, "max abs err", e.max(), "max|val-a0|", np.abs(rr - a0).max(), "rel", e.max()/np.abs(rr - a0).max(), "eps-bound", 9*eps32*np.abs(rr).max())
ctx.close()
