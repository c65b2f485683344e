"""Where the fixed per-call cost of render_image goes (run on the GPU box):
device time of the frame (events), the native call + sync, and the whole API."""
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
for size in (8, 800):
    cam = gf.sphere_cameras(aabb, 1, size, seed=0)[0]
    n = size * size
    out = torch.empty((n, 3), device='cuda'); st = torch.zeros(4, dtype=torch.int64, device='cuda')
    ws = torch.empty(R._render_ws_bytes(grid, cfg.native(0), n), dtype=torch.uint8, device='cuda')
    for _ in range(5): gf.render_image(grid, occ, cam, cfg, seed=0)
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(); e0.record()
    for _ in range(20): R.render_rays_device(grid, occ, cfg, 0, cam=cam, out=out, stats=st, ws=ws)
    e1.record(); torch.cuda.synchronize(); dev = e0.elapsed_time(e1) / 20
    t = []
    for _ in range(20):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        R.render_rays_device(grid, occ, cfg, 0, cam=cam, out=out, stats=st, ws=ws); torch.cuda.synchronize()
        t.append(time.perf_counter() - t0)
    call = np.median(t) * 1e3
    t = []
    for _ in range(20):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        R.render_rays_device(grid, occ, cfg, 0, cam=cam, out=out, stats=st, ws=ws)
        t.append(time.perf_counter() - t0)
    torch.cuda.synchronize()
    host_only = np.median(t) * 1e3
    t = []
    for _ in range(20):
        torch.cuda.synchronize(); t0 = time.perf_counter(); gf.render_image(grid, occ, cam, cfg, seed=0); t.append(time.perf_counter() - t0)
    api = np.median(t) * 1e3
    print(f"{size}x{size}: device {dev:.3f} ms (events, back-to-back)  call+sync {call:.3f}  host enqueue {host_only:.3f}  render_image {api:.3f}")
# host-mapped output vs device output + copy, through render_rays_device
cam = gf.sphere_cameras(aabb, 1, 800, seed=0)[0]
n = 800 * 800
st = torch.zeros(4, dtype=torch.int64, device='cuda')
ws = torch.empty(R._render_ws_bytes(grid, cfg.native(0), n), dtype=torch.uint8, device='cuda')
dev = torch.empty((n, 3), device='cuda')
host = torch.empty((n, 3), pin_memory=True)
for name, fn in (("device out + D2H", lambda: (R.render_rays_device(grid, occ, cfg, 0, cam=cam, out=dev, stats=st, ws=ws),
                                                host.copy_(dev, non_blocking=True))),
                 ("host-mapped out", lambda: R.render_rays_device(grid, occ, cfg, 0, cam=cam, out=host, stats=st, ws=ws))):
    for _ in range(5): fn()
    t = []
    for _ in range(30):
        torch.cuda.synchronize(); t0 = time.perf_counter(); fn(); torch.cuda.synchronize(); t.append(time.perf_counter() - t0)
    print(f"{name}: {np.median(t)*1e3:.3f} ms")
