"""Device timing of one photometric training step at the reference's default
scale (TrainConfig(): 8192-pixel batch, k_train=384, 16^3 lattice of 32-wide
MLPs, toy-scene occupancy 256^3).  Prints one JSON line with per-stage CUDA-
event times.  Diagnostic, not the driver's bench line."""

import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))

import paper_2103_13744_b200 as gf  # noqa: E402
from paper_2103_13744_b200 import _device as D  # noqa: E402
from paper_2103_13744_b200 import train  # noqa: E402
from paper_2103_13744_b200.batched import grouped_backward_device, grouped_forward_device  # noqa: E402


def ev():
    e = torch.cuda.Event(enable_timing=True)
    e.record()
    return e


def main():
    aabb = gf.Aabb((-1.0,) * 3, (1.0,) * 3)
    grid = gf.init_network_grid(aabb, (16, 16, 16), seed=0)
    z = np.load(ROOT / "tests" / "golden" / "toy_occupancy_256.npz")
    occ = gf.OccupancyGrid(aabb, z["res"], z["bits"])
    cfg = train.TrainConfig()
    cam = gf.sphere_cameras(aabb, 1, 800, seed=0)[0]
    o, d = gf.render.generate_rays(cam)
    rng = np.random.default_rng(0)
    pix = rng.choice(len(o), size=cfg.batch_size_pixels, replace=False)
    t0 = time.perf_counter()
    smp = train.prepare_ray_samples(o[pix], d[pix], aabb, cfg.k_train, True, rng, occ=occ)
    t_prep = time.perf_counter() - t0
    gt = rng.random((len(pix), 3)).astype(np.float32)
    q = len(smp.positions)
    out = {"queries": q, "rays": len(pix), "k": cfg.k_train, "prepare_s_host": t_prep}
    for it in range(4):
        torch.cuda.synchronize()
        w0 = time.perf_counter()
        e0 = ev()
        layout = gf.group_by_network(gf.QueryBatch(smp.positions, smp.directions, grid.cell_index(smp.positions)),
                                     grid.n_cells)
        e1 = ev()
        cache = grouped_forward_device(grid, layout)
        e2 = ev()
        loss, grads = train.photometric_loss_and_grads(grid, smp, gt, cfg.background)
        e3 = ev()
        t = D.require_cuda()
        dc = t.zeros((q, 3), device="cuda")
        ds = t.ones((q,), device="cuda")
        e4 = ev()
        gw, gb = grouped_backward_device(grid, layout, cache, dc, ds)
        e5 = ev()
        torch.cuda.synchronize()
        wall = time.perf_counter() - w0
        if it:
            out.update(group_ms=e0.elapsed_time(e1), forward_ms=e1.elapsed_time(e2),
                       loss_and_grads_total_ms=e2.elapsed_time(e3), backward_kernel_ms=e4.elapsed_time(e5),
                       wall_s=wall, loss=loss)
    out["backward_rows_per_s"] = q / (out["backward_kernel_ms"] * 1e-3)
    print(json.dumps(out))


if __name__ == "__main__":
    main()
