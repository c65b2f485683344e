import sys, time
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2103_13744_b200 as gf
aabb = gf.Aabb((-1.0,)*3, (1.0,)*3)
grid = gf.init_network_grid(aabb, (16,16,16), seed=0, precision="fp16")
z = np.load('tests/golden/toy_occupancy_256.npz')
occ = gf.OccupancyGrid(aabb, z['res'], z['bits'].copy())
for size in (8, 800):
    cam = gf.sphere_cameras(aabb, 1, size, seed=0)[0]
    cfg = gf.RenderConfig()
    for _ in range(5): gf.render_image(grid, occ, cam, cfg, seed=0)
    t=[]
    for _ in range(20):
        torch.cuda.synchronize(); t0=time.perf_counter(); gf.render_image(grid, occ, cam, cfg, seed=0); t.append(time.perf_counter()-t0)
    print(size, "median ms", 1e3*np.median(t))
x = torch.empty(800*800*3, device='cuda'); h = torch.empty(800*800*3, pin_memory=True)
for _ in range(3): h.copy_(x, non_blocking=True); torch.cuda.synchronize()
e0=torch.cuda.Event(enable_timing=True); e1=torch.cuda.Event(enable_timing=True)
e0.record(); 
for _ in range(20): h.copy_(x, non_blocking=True)
e1.record(); torch.cuda.synchronize(); ms=e0.elapsed_time(e1)/20
print("D2H 7.68 MB pinned: %.3f ms = %.1f GB/s" % (ms, 7.68e6/ms/1e6))
