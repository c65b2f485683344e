"""BASELINE configs 4 and 5 on the device, checked against the oracle.

* 64-wide networks (config 4's architecture): golden query + traced render on
  an 8^3 lattice (fixtures from the reference, tests/golden/make_golden.py),
  and the full config 4 (32^3 lattice, 1920x1080) through size-independent
  properties: exact per-block RenderStats and colours of sampled 4096-ray
  blocks against the oracle, and bit-identity of a block rendered alone vs
  inside the full frame.
* Bulk query (config 5): the reference's input recipe at 2^14 points against
  the golden vector, and the full 2^26 points with a sampled oracle check.
"""

import numpy as np
import pytest

from conftest import golden, have_gpu
from oracle import gridfield_oracle as O

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not have_gpu(), reason="needs a CUDA device")]

UNIT_MIN, UNIT_MAX = np.full(3, -1.0), np.ones(3)
QUERY_TOL = {"fp32": 2e-6, "fp16": 2e-3}   # as test_gpu_parity.test_query_points_vs_golden
IMG_TOL = {"fp32": 2e-5, "fp16": 1e-3}


@pytest.fixture(scope="module")
def gf():
    import paper_2103_13744_b200 as m

    return m


@pytest.mark.parametrize("precision", ["fp32", "fp16"])
def test_query_64_wide_vs_golden(gf, precision):
    z = golden("query_w64")
    g = gf.init_network_grid(gf.Aabb(UNIT_MIN, UNIT_MAX), (8, 8, 8), seed=4,
                             arch=gf.MlpArchitecture(hidden_width=64))
    rgb, sig = g.query_points(z["pts"], z["dirs"], precision=precision)
    tol = QUERY_TOL[precision]
    assert np.max(np.abs(rgb - z["rgb"])) <= tol
    assert np.max(np.abs(sig - z["sigma"])) <= tol


@pytest.mark.parametrize("precision", ["fp32", "fp16"])
def test_bulk_query_recipe_vs_golden(gf, precision):
    z = golden("query_c5")
    g = gf.init_network_grid(gf.Aabb(UNIT_MIN, UNIT_MAX), (16, 16, 16), seed=0)
    rgb, sig = g.query_points(z["pts"], z["dirs"], precision=precision)
    tol = QUERY_TOL[precision]
    assert np.max(np.abs(rgb - z["rgb"])) <= tol
    assert np.max(np.abs(sig - z["sigma"])) <= tol


def test_bulk_query_full_size(gf):
    """Config 5 at its full 2^26 points (tensor-core path): a seeded sample of
    results against the oracle, output ranges everywhere, and the result of a
    point independent of the batch it arrives in."""
    import torch

    n = 1 << 26
    g = gf.init_network_grid(gf.Aabb(UNIT_MIN, UNIT_MAX), (16, 16, 16), seed=0)
    pts, dirs = O.bulk_query_inputs(UNIT_MIN, UNIT_MAX, n, seed=0)
    p_d, d_d = torch.from_numpy(pts).cuda(), torch.from_numpy(dirs).cuda()
    rgb, sig = g.query_points(p_d, d_d, precision="fp16")
    assert rgb.shape == (n, 3) and sig.shape == (n,)
    assert bool(torch.isfinite(rgb).all()) and bool(((rgb >= 0) & (rgb <= 1)).all()) and bool((sig >= 0).all())
    idx = np.sort(np.random.default_rng(7).choice(n, 1 << 14, replace=False))
    lat = O.init_lattice(UNIT_MIN, UNIT_MAX, (16, 16, 16), seed=0)
    rc, rs = O.query_points(lat, pts[idx], dirs[idx])
    assert np.max(np.abs(rgb[idx].cpu().numpy() - rc)) <= QUERY_TOL["fp16"]
    assert np.max(np.abs(sig[idx].cpu().numpy() - rs)) <= QUERY_TOL["fp16"]
    sub_rgb, sub_sig = g.query_points(p_d[idx], d_d[idx], precision="fp16")
    assert torch.equal(sub_rgb, rgb[idx]) and torch.equal(sub_sig, sig[idx])


@pytest.fixture(scope="module")
def c4(gf):
    import bench

    return bench.build_c4(gf)


@pytest.mark.parametrize("precision", ["fp16", "fp32"])
def test_config4_full_size_sampled_blocks(gf, c4, precision):
    """Config 4 (32^3 lattice of 64-wide MLPs, 1920x1080): the device frame's
    sampled 4096-ray blocks against the oracle -- counts exact, colours within
    tolerance -- and bit-identical to the same blocks rendered on their own."""
    import torch

    aabb, grid, occ, cam = c4
    cfg = gf.RenderConfig()
    n = cam.width * cam.height
    full, st_full, _ = gf.render.render_rays_device(grid, occ, cfg, 0, cam=cam, precision=precision)
    full = full.cpu().numpy()
    assert int(st_full[3]) == n and np.all((full >= 0) & (full <= 1))
    lat = O.lattice_from_grid(grid)
    occ_o = O.Occupancy(UNIT_MIN, UNIT_MAX, np.asarray(occ.resolution), np.asarray(occ.bits))
    o, d = O.pixel_rays(cam.width, cam.height, cam.fx, cam.fy, cam.cx, cam.cy, cam.c2w)
    q = lambda p, dd: O.query_points(lat, p, dd)  # noqa: E731
    n_blocks = (n + O.RAY_BLOCK - 1) // O.RAY_BLOCK
    for b in (n_blocks // 2 - 3, n_blocks // 2 + 20):  # centre blocks: the object fills them
        s, e = b * O.RAY_BLOCK, min((b + 1) * O.RAY_BLOCK, n)
        gen = np.random.default_rng(np.random.SeedSequence([0, s]))
        ref, _, ctr = O.march_block(q, lat.b_min, lat.b_max, occ_o, o[s:e].astype(np.float64),
                                    d[s:e].astype(np.float64), O.MarchConfig(), gen)
        blk, st, _ = gf.render.render_rays_device(grid, occ, cfg, 0, cam=cam, ray_offset=s, n_rays=e - s,
                                                  precision=precision)
        st = [int(v) for v in st.cpu()]
        assert ctr.total_queries > 0
        assert st == [ctr.total_queries, ctr.ess_skipped, ctr.ert_terminated_rays, e - s]
        blk = blk.cpu().numpy()
        assert np.max(np.abs(blk - ref)) <= IMG_TOL[precision]
        assert np.array_equal(blk, full[s:e])
    torch.cuda.empty_cache()
