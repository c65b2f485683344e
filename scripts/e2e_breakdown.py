"""Where render_image's end-to-end time goes beyond the device frame (GPU box)."""
import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2103_13744_b200 as gf
from paper_2103_13744_b200 import render as R
aabb = gf.Aabb((-1.0,)*3, (1.0,)*3)
grid = gf.init_network_grid(aabb, (16,16,16), seed=0)
z = np.load('tests/golden/toy_occupancy_256.npz')
occ = gf.OccupancyGrid(aabb, z['res'], z['bits'].copy())
cfg = gf.RenderConfig()
cam = gf.sphere_cameras(aabb, 1, 800, seed=0)[0]
n = 640000
for _ in range(10): gf.render_image(grid, occ, cam, cfg, seed=0)
T = {k: [] for k in ("prep", "enqueue", "alloc", "copy_enq", "sync", "stats", "total")}
for _ in range(30):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    t = gf._device.require_cuda() if hasattr(gf, "_device") else torch
    ncfg = cfg.native(0)
    ws_bytes = R._render_ws_bytes(grid, ncfg, n)
    c = R._render_context(n, ws_bytes)
    c["stats"].zero_()
    t1 = time.perf_counter()
    rgb = torch.empty((n, 3), device="cuda") if "rgb" not in c else c["rgb"]
    out_rgb, st, _ = R.render_rays_device(grid, occ, cfg, 0, cam=cam, out=rgb, stats=c["stats"], ws=c["ws"])
    t2 = time.perf_counter()
    host = torch.empty(out_rgb.shape, dtype=torch.float32, pin_memory=True)
    t3 = time.perf_counter()
    host.copy_(out_rgb, non_blocking=True)
    c["host_stats"].copy_(st, non_blocking=True)
    t4 = time.perf_counter()
    torch.cuda.current_stream().synchronize()
    t5 = time.perf_counter()
    stats = R._stats_from(c["host_stats"])
    img = host.numpy().reshape(cam.height, cam.width, 3)
    t6 = time.perf_counter()
    for k, a, b in (("prep", t0, t1), ("enqueue", t1, t2), ("alloc", t2, t3), ("copy_enq", t3, t4), ("sync", t4, t5),
                    ("stats", t5, t6), ("total", t0, t6)):
        T[k].append((b - a) * 1e3)
print({k: round(float(np.median(v)), 4) for k, v in T.items()})
tt = []
for _ in range(30):
    torch.cuda.synchronize(); a = time.perf_counter(); gf.render_image(grid, occ, cam, cfg, seed=0); tt.append(time.perf_counter() - a)
print("render_image", round(float(np.median(tt)) * 1e3, 4))
