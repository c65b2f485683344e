"""Diagnostics: exact-path candidate count of the C2 frame (GF_COUNT_CANDIDATES=1)."""
import os, sys
os.environ["GF_COUNT_CANDIDATES"] = "1"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench, torch
import paper_2103_13744_b200 as gf
aabb, grid, occ, cams = bench.build_inputs(gf)
grid.precision = "fp16"
for name, bias in (("random", None), ("bias20", 20.0)):
    if bias is not None:
        grid.params.biases["density"][:] = bias
    img, st = gf.render_image(grid, occ, cams[0], gf.RenderConfig(), seed=0)
    print(name, "candidates", st.n_rays - 640000, "queries", st.total_queries, "ess", st.ess_skipped, "ert", st.ert_terminated_rays)
