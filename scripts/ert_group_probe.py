"""Frame time of the C2 view with density bias 20 (ERT-heavy: ~100k rays
terminate) for the current GF_GROUP setting: the cost of speculative rounds.
Diagnostic only."""
import json, sys, time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import paper_2103_13744_b200 as gf  # noqa: E402

aabb = gf.Aabb((-1.0,) * 3, (1.0,) * 3)
grid = gf.init_network_grid(aabb, (16, 16, 16), seed=0, precision="fp16")
grid.params.biases["density"][:] = 20.0
z = np.load(ROOT / "tests" / "golden" / "toy_occupancy_256.npz")
occ = gf.OccupancyGrid(aabb, z["res"], z["bits"].copy())
cam = gf.sphere_cameras(aabb, 64, 800, seed=0)[0]
cfg = gf.RenderConfig()
for _ in range(3):
    img, st = gf.render_image(grid, occ, cam, cfg, seed=0)
torch.cuda.synchronize()
t = []
for _ in range(10):
    t0 = time.perf_counter()
    img, st = gf.render_image(grid, occ, cam, cfg, seed=0)
    t.append(time.perf_counter() - t0)
print(json.dumps({"e2e_ms_median": 1e3 * float(np.median(t)), "queries": st.total_queries,
                  "ert": st.ert_terminated_rays, "checksum": float(img.sum())}))
