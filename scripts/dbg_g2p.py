import sys, numpy as np, torch
sys.path.insert(0, '.'); sys.path.insert(0, 'tests')
import synth
from test_gpu_fullsize import field_torch
from paper_2605_09097_b200 import osmpm
ncell = int(sys.argv[1]) if len(sys.argv) > 1 else 128
sc = synth.c5_stress(n_cells=ncell)
dev = torch.device("cuda", 0)
ctx = osmpm.Context(0, torch.cuda.current_stream(dev).cuda_stream)
sub = osmpm.Subdomain(ctx, sc.grid, sc.dt, sc.particles, sc.materials, sc.gravity)
x0 = torch.from_numpy(sc.particles.x).to(dev)
def chk(tag):
    out = sub.read_particles(device=dev, fields=("x", "F"))
    torch.cuda.synchronize()
    x = out["x"]; F = out["F"]
    print(tag, "max|x-x0|", (x - x0).abs().max().item(), "det min", torch.linalg.det(F).min().item(), flush=True)
dims = sc.grid.dims
chk("created")
sub.p2g(); chk("p2g")
grid = sub.read_grid(device=dev); chk("read_grid")
u = field_torch(dims, 1e-3 * sc.grid.dx, 0.3, dev)
g, E = sub.newton_gradient(u); chk("grad")
print("E", E)
d = field_torch(dims, 1.0, 1.1, dev)
y = sub.newton_hvp(d); chk("hvp")
del u, d, g, y, grid
vg = field_torch(dims, 0.05, 2.0, dev)
print("vg finite", torch.isfinite(vg).all().item(), vg.abs().max().item())
sub.set_grid_velocity(vg); chk("setv")
vr = sub.read_grid_velocity(device=dev)
print("vnew vs vg max diff on box", (vr - vg).abs().max().item())
sub.g2p()
try:
    sub.sync(); print("g2p sync ok")
except Exception as e: print("ERR", e)
chk("g2p")
