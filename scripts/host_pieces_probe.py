import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2103_13744_b200 as gf
from paper_2103_13744_b200 import render as R, _native as N
aabb = gf.Aabb((-1.0,)*3, (1.0,)*3)
grid = gf.init_network_grid(aabb, (16,16,16), seed=0)
z = np.load('tests/golden/toy_occupancy_256.npz')
occ = gf.OccupancyGrid(aabb, z['res'], z['bits'].copy())
cfg = gf.RenderConfig()
cam = gf.sphere_cameras(aabb, 1, 8, seed=0)[0]
def tm(f, n=200):
    for _ in range(5): f()
    t0 = time.perf_counter()
    for _ in range(n): f()
    return (time.perf_counter() - t0) / n * 1e6
print("resolved_precision", tm(lambda: grid.resolved_precision(None, render=True)))
p = grid.resolved_precision(None, render=True)
print("device_params", tm(lambda: grid.device_params(p)))
print("params.fingerprint", tm(lambda: grid.params.fingerprint()))
print("make_camera", tm(lambda: N.make_camera(cam)))
print("cfg.native", tm(lambda: cfg.native(0)))
print("occ.native_geom+bits", tm(lambda: (occ.native_geom(), occ.device_bits())))
print("native_arch+geom", tm(lambda: (grid.native_arch(), grid.native_geom())))
print("_render_ws_bytes", tm(lambda: R._render_ws_bytes(grid, cfg.native(0), 64)))
print("stream_handle", tm(lambda: gf._device.stream_handle() if hasattr(gf, '_device') else None))
