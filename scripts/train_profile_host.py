import sys, time, cProfile, pstats
sys.path.insert(0, '.')
import numpy as np, torch
import paper_2103_13744_b200 as gf
from paper_2103_13744_b200 import train
aabb = gf.Aabb((-1.0,)*3, (1.0,)*3)
grid = gf.init_network_grid(aabb, (16,16,16), seed=0)
z = np.load('tests/golden/toy_occupancy_256.npz')
occ = gf.OccupancyGrid(aabb, z['res'], z['bits'])
cfg = train.TrainConfig()
cam = gf.sphere_cameras(aabb, 1, 800, seed=0)[0]
o, d = gf.render.generate_rays(cam)
rng = np.random.default_rng(0)
pix = rng.choice(len(o), size=cfg.batch_size_pixels, replace=False)
smp = train.prepare_ray_samples(o[pix], d[pix], aabb, cfg.k_train, True, rng, occ=occ)
gt = rng.random((len(pix), 3)).astype(np.float32)
state = train.AdamState.for_params(grid.params)
for i in range(2):
    loss, grads = train.photometric_loss_and_grads(grid, smp, gt, cfg.background)
    train.adam_update(grid.params, grads, state, 5e-4, cfg)
torch.cuda.synchronize()
pr = cProfile.Profile(); pr.enable()
for i in range(3):
    t0=time.perf_counter()
    loss, grads = train.photometric_loss_and_grads(grid, smp, gt, cfg.background)
    torch.cuda.synchronize(); t1=time.perf_counter()
    train.adam_update(grid.params, grads, state, 5e-4, cfg)
    torch.cuda.synchronize(); t2=time.perf_counter()
    print(f"loss+grads {1e3*(t1-t0):.1f} ms  adam {1e3*(t2-t1):.1f} ms")
pr.disable()
pstats.Stats(pr).sort_stats('cumulative').print_stats(25)
