import sys, time, os
sys.path.insert(0, '.')
import torch, bench, paper_2103_13744_b200 as gf
from paper_2103_13744_b200.render import render_rays_device
from paper_2103_13744_b200 import _native as N
aabb, grid, occ, cams = bench.build_inputs(gf)
cfg = gf.RenderConfig(); cam = cams[0]
n = cam.width * cam.height
out = torch.empty((n, 3), dtype=torch.float32, device="cuda"); st = torch.zeros(4, dtype=torch.int64, device="cuda")
ws = torch.empty(N.lib().gf_render_workspace_bytes(grid.native_arch(), grid.native_geom(), cfg.native(0), n), dtype=torch.uint8, device="cuda")
for i in range(int(os.environ.get("NF", "30"))):
    st.zero_(); render_rays_device(grid, occ, cfg, 0, cam=cam, out=out, stats=st, ws=ws)
    torch.cuda.synchronize()
    if i % 10 == 0: print("frame", i, flush=True)
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record()
for i in range(20):
    st.zero_(); render_rays_device(grid, occ, cfg, 0, cam=cam, out=out, stats=st, ws=ws)
e1.record(); torch.cuda.synchronize()
print("ms/frame", e0.elapsed_time(e1) / 20, st.tolist(), flush=True)
