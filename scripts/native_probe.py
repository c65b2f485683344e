import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2103_13744_b200 as gf
from paper_2103_13744_b200 import render as R, _native as N, _device as D
aabb = gf.Aabb((-1.0,)*3, (1.0,)*3)
grid = gf.init_network_grid(aabb, (16,16,16), seed=0)
z = np.load('tests/golden/toy_occupancy_256.npz')
occ = gf.OccupancyGrid(aabb, z['res'], z['bits'].copy())
cfg = gf.RenderConfig()
cam = gf.sphere_cameras(aabb, 1, 800, seed=0)[0]
n = 640000
out = torch.empty((n, 3), device='cuda'); st = torch.zeros(4, dtype=torch.int64, device='cuda')
ws = torch.empty(R._render_ws_bytes(grid, cfg.native(0), n), dtype=torch.uint8, device='cuda')
for _ in range(5): R.render_rays_device(grid, occ, cfg, 0, cam=cam, out=out, stats=st, ws=ws)
torch.cuda.synchronize()
p = grid.resolved_precision(None, render=True); packed = grid.device_params(p)
args = (grid.native_arch(), grid.native_geom(), N.ptr(packed), N.PRECISION[p], occ.native_geom(), N.ptr(occ.device_bits()), cfg.native(0),
        N.make_camera(cam), None, None, 0, 1, n, N.ptr(out), N.ptr(st), None, 0, None, N.ptr(ws), ws.numel(), D.stream_handle())
lib = N.lib()
def tm(f, reps=50):
    torch.cuda.synchronize(); a = time.perf_counter()
    for _ in range(reps): f()
    b = time.perf_counter(); torch.cuda.synchronize()
    return (b - a) / reps * 1e6
print("native gf_render_rays host us", tm(lambda: lib.gf_render_rays(*args)))
print("render_rays_device host us", tm(lambda: R.render_rays_device(grid, occ, cfg, 0, cam=cam, out=out, stats=st, ws=ws)))
