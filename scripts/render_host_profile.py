import sys, time, cProfile, pstats
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2103_13744_b200 as gf
aabb = gf.Aabb((-1.0,)*3, (1.0,)*3)
grid = gf.init_network_grid(aabb, (16,16,16), seed=0, precision="fp16")
z = np.load('tests/golden/toy_occupancy_256.npz')
occ = gf.OccupancyGrid(aabb, z['res'], z['bits'].copy())
cam = gf.sphere_cameras(aabb, 1, int(sys.argv[1]) if len(sys.argv) > 1 else 800, seed=0)[0]
cfg = gf.RenderConfig()
for _ in range(5): gf.render_image(grid, occ, cam, cfg, seed=0)
pr = cProfile.Profile(); pr.enable()
for _ in range(50): gf.render_image(grid, occ, cam, cfg, seed=0)
pr.disable()
pstats.Stats(pr).sort_stats('tottime').print_stats(18)
