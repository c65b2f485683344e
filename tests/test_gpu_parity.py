"""CUDA path vs the CPU oracle / golden vectors, through the C-ABI.

Bars (stated per test): bit-exact for sample placement, cell indices, counts,
ordering and index work; float tolerance for MLP outputs and images
(numpy's float32 sin/cos/exp/expm1 are not correctly rounded, so absolute
values cannot be bit-identical — see DESIGN.md §parity).
"""

import numpy as np
import pytest

from conftest import golden, golden_camera, have_gpu, toy_occupancy_bits
from oracle import gridfield_oracle as O
from test_oracle_golden import RENDER_CASES, LATTICES, case_config, case_inputs

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not have_gpu(), reason="needs a CUDA device")]

UNIT = (np.full(3, -1.0), np.ones(3))
FP32_IMG_TOL = 2e-5      # fp32 SIMT MLP vs numpy/OpenBLAS: reassociation + 1-2 ulp transcendentals
FP16_IMG_TOL = 1e-3      # north-star bound for tensor-core MMA (fp16 operands, fp32 accumulate)
PRECISIONS = [("fp32", FP32_IMG_TOL), ("fp16", FP16_IMG_TOL)]


@pytest.fixture(scope="module")
def gf():
    import paper_2103_13744_b200 as m

    return m


def unit(gf):
    return gf.Aabb(*UNIT)


def device_grid(gf, name):
    gname, oname = LATTICES[name]
    aabb = unit(gf)
    if gname == "g2":
        g = gf.init_network_grid(aabb, (2, 3, 4), seed=9)
        g.params.biases["density"][:] = 5.0
    elif gname == "gw":
        g = gf.init_network_grid(aabb, (8, 8, 8), seed=4, arch=gf.MlpArchitecture(hidden_width=64))
        g.params.biases["density"][:] = 20.0
    else:
        g = gf.init_network_grid(aabb, (16, 16, 16), seed=0)
        if gname == "gb":
            g.params.biases["density"][:] = 20.0
    if oname == "solid":
        occ = gf.OccupancyGrid.solid(aabb, (256, 256, 256))
    elif oname == "toy":
        res, bits = toy_occupancy_bits()
        occ = gf.OccupancyGrid(aabb, res, bits.copy())
    elif oname == "empty":
        occ = gf.OccupancyGrid.solid(aabb, (8, 8, 8), value=False)
    else:
        occ = None
    return g, occ


def device_camera(gf, z, suffix=""):
    c = golden_camera(z, suffix)
    return gf.Camera(c.width, c.height, c.fx, c.fy, c.cx, c.cy, c.c2w)


def precision_available(gf, precision):
    g = gf.init_network_grid(unit(gf), (1, 1, 1), seed=0)
    try:
        g.query_points(np.zeros((1, 3), np.float32), np.array([[0, 0, 1]], np.float32), precision=precision)
        return True
    except Exception as e:  # noqa: BLE001
        if "no MLP kernel" in str(e) or "no fp16 device layout" in str(e) or "has no" in str(e):
            return False
        raise


# ---------------------------------------------------------------------------
# rays, pointwise primitives
# ---------------------------------------------------------------------------
def test_generate_rays_bit_exact(gf):
    z = golden("rays")
    for i in range(int(z["n"])):
        o, d = gf.render.generate_rays(device_camera(gf, z, f"_{i}"))
        assert np.array_equal(o, z[f"o_{i}"])
        assert np.array_equal(d, z[f"d_{i}"]), f"camera {i}"


def test_pointwise_primitives(gf):
    z = golden("pointwise")
    aabb = unit(gf)
    # binning and clipping: bit-exact
    for key, res in (("bin16", (16,) * 3), ("bin256", (256,) * 3), ("bin_5_7_3", (5, 7, 3))):
        flat = gf.core.flatten_cell_index(gf.bin_point(z["bin_pts"], aabb, res), res)
        assert np.array_equal(flat, z[key]), key
    assert np.array_equal(gf.clip_into(z["clip_in"], aabb), z["clip_out"])
    # encoding / alpha: numpy float32 sin/cos/expm1 are within ~2 ulp of CUDA's
    enc = gf.positional_encode(z["enc_in"], 10)
    assert enc.dtype == np.float32 and enc.shape == (256, 63)
    assert np.max(np.abs(enc - z["enc_x"])) <= 4e-7
    assert np.max(np.abs(gf.positional_encode(z["enc_d_in"], 4) - z["enc_d"])) <= 4e-7
    a = gf.density_to_alpha(z["alpha_sigma"], z["alpha_delta"])
    assert np.max(np.abs(a - z["alpha"]) / np.maximum(np.abs(z["alpha"]), 1e-30)) <= 3e-7
    # reference known answers (test_core.py)
    assert np.array_equal(gf.bin_point(np.zeros(3), gf.Aabb((0, 0, 0), (1, 1, 1)), (16,) * 3), [0, 0, 0])
    assert np.array_equal(gf.bin_point(np.array([0.999, 0.5, 0.25]), gf.Aabb((0, 0, 0), (1, 1, 1)), (16,) * 3),
                          [15, 8, 4])
    assert np.array_equal(gf.bin_point(np.ones(3), gf.Aabb((0, 0, 0), (1, 1, 1)), (16,) * 3), [15, 15, 15])
    with pytest.raises(ValueError, match="component 1"):
        gf.bin_point(np.array([0.5, 1.5, 0.5]), gf.Aabb((0, 0, 0), (1, 1, 1)), (16,) * 3)
    assert np.allclose(gf.positional_encode(np.zeros(3), 1), [0, 0, 0, 0, 0, 0, 1, 1, 1])
    assert gf.density_to_alpha(10.0, 0.01) == pytest.approx(1 - np.exp(-0.1), rel=1e-12)
    assert gf.density_to_alpha(0.0, 0.1) == 0.0


def test_composite_known_answers(gf):
    rgb, t = gf.composite(np.array([[1.0, 0, 0]]), np.array([1.0]))
    assert np.allclose(rgb, [1, 0, 0]) and t == 0.0
    rgb, t = gf.composite(np.array([[1.0, 0, 0], [0, 1.0, 0]]), np.array([0.5, 1.0]))
    assert np.allclose(rgb, [0.5, 0.5, 0.0]) and t == 0.0
    rgb, t = gf.composite(np.zeros((0, 3)), np.zeros(0))
    assert np.allclose(rgb, 0) and t == 1.0
    rng = np.random.default_rng(0)
    c = rng.random((64, 20, 3)).astype(np.float32)
    a = rng.random((64, 20)).astype(np.float32)
    rgb, t = gf.composite(c, a)
    r2, t2 = O.composite(c, a)
    assert np.array_equal(rgb, r2) and np.array_equal(t, t2)  # same op order, float32: bit-exact
    c64, a64 = c.astype(np.float64), a.astype(np.float64)
    rgb, t = gf.composite(c64, a64)
    r2, t2 = O.composite(c64, a64)
    assert np.array_equal(rgb, r2) and np.array_equal(t, t2)


def test_occupied_at(gf):
    res, bits = toy_occupancy_bits()
    occ = gf.OccupancyGrid(unit(gf), res, bits.copy())
    occ_o = O.Occupancy(*UNIT, res, bits)
    pts = np.random.default_rng(3).uniform(-1, 1, (50_000, 3)).astype(np.float32)
    assert np.array_equal(occ.occupied_at(pts), occ_o.lookup(pts))
    with pytest.raises(ValueError, match="outside bounds"):
        occ.occupied_at(np.array([[2.0, 0.5, 0.5]], np.float32))


# ---------------------------------------------------------------------------
# network queries
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("precision,tol", [("fp32", 2e-6), ("fp16", 2e-3)])
def test_query_points_vs_golden(gf, precision, tol):
    if not precision_available(gf, precision):
        pytest.skip(f"{precision} MLP kernel not built")
    z = golden("query16")
    g = gf.init_network_grid(unit(gf), (16, 16, 16), seed=3)
    rgb, sig = g.query_points(z["pts"], z["dirs"], precision=precision)
    assert rgb.shape == (len(z["pts"]), 3) and sig.shape == (len(z["pts"]),)
    assert np.max(np.abs(rgb - z["rgb"])) <= tol
    assert np.max(np.abs(sig - z["sigma"])) <= tol
    # shuffle invariance (test_batched.py:97-106) is exact on the device
    perm = np.random.default_rng(1).permutation(len(z["pts"]))
    rgb2, sig2 = g.query_points(z["pts"][perm], z["dirs"][perm], precision=precision)
    assert np.array_equal(rgb2, rgb[perm]) and np.array_equal(sig2, sig[perm])


@pytest.mark.parametrize("precision", ["fp32", "fp16"])
def test_tagged_density_bias_known_answer(gf, precision):
    """test_grid.py:214-229: zero weights + per-cell density bias = cell index,
    so sigma reveals the device's cell assignment exactly."""
    if not precision_available(gf, precision):
        pytest.skip(f"{precision} MLP kernel not built")
    g = gf.init_network_grid(unit(gf), (16, 16, 16), seed=5)
    for k in g.params.weights:
        g.params.weights[k][:] = 0
        g.params.biases[k][:] = 0
    g.params.biases["density"][:, 0] = np.arange(g.n_cells, dtype=np.float32)
    z = golden("query16")
    rgb, sig = g.query_points(z["pts"], z["dirs"], precision=precision)
    assert np.array_equal(sig, z["keys"].astype(np.float32))
    assert np.all(rgb == 0.5)


def test_query_out_of_bounds_message(gf):
    g = gf.init_network_grid(unit(gf), (4, 4, 4), seed=11)
    pts = np.zeros((10, 3), np.float32)
    pts[7, 1] = 1.5
    with pytest.raises(ValueError, match="component 1"):
        g.query_points(pts, np.tile(np.float32([0, 0, 1]), (10, 1)))
    with pytest.raises(ValueError, match="outside bounds"):
        gf.query_field(g, np.array([3.0, 0.0, 0.0]), np.array([0.0, 0.0, 1.0]))


def test_group_by_network_bit_exact(gf):
    z = golden("query16")
    b = gf.QueryBatch(z["pts"], z["dirs"], z["keys"])
    lay = gf.group_by_network(b, 4096)
    assert np.array_equal(lay.order, z["order"])
    assert np.array_equal(lay.inverse, z["inverse"])
    assert np.array_equal(lay.offsets, z["offsets"])
    # ragged + empty + single-network cases against the oracle's stable sort
    rng = np.random.default_rng(7)
    for n, nk in ((0, 8), (1, 1), (300, 1), (5000, 32), (100_000, 4096)):
        keys = rng.integers(0, nk, n)
        lay = gf.group_by_network(gf.QueryBatch(np.zeros((n, 3), np.float32), np.zeros((n, 3), np.float32), keys), nk)
        ref = O.group(keys, nk)
        assert np.array_equal(lay.order, ref.order) and np.array_equal(lay.offsets, ref.offsets)
        assert np.array_equal(lay.inverse, ref.inverse)
    with pytest.raises(ValueError, match="out of range"):
        gf.group_by_network(gf.QueryBatch(np.zeros((4, 3)), np.zeros((4, 3)), np.array([0, 1, 2, 3])), 2)


@pytest.mark.parametrize("precision,tol", [("fp32", 2e-6), ("fp16", 2e-3)])
def test_grouped_forward_matches_sequential_oracle(gf, precision, tol):
    """test_batched.py:72-95: random per-cell batch sizes 0..50 on a 4^3 grid."""
    if not precision_available(gf, precision):
        pytest.skip(f"{precision} MLP kernel not built")
    rng = np.random.default_rng(42)
    g = gf.init_network_grid(unit(gf), (4, 4, 4), seed=1)
    lat = O.init_lattice(*UNIT, (4, 4, 4), seed=1)
    sizes = rng.integers(0, 51, g.n_cells)
    cell = 2.0 / 4
    pts, dirs, idx = [], [], []
    for flat, count in enumerate(sizes):
        lo = -1.0 + np.array([flat % 4, (flat // 4) % 4, flat // 16]) * cell
        pts.append(lo + rng.random((count, 3)) * cell)
        d = rng.normal(size=(count, 3))
        dirs.append(d / np.linalg.norm(d, axis=-1, keepdims=True))
        idx.append(np.full(count, flat))
    b = gf.QueryBatch(np.concatenate(pts).astype(np.float32), np.concatenate(dirs).astype(np.float32),
                      np.concatenate(idx))
    lay = gf.group_by_network(b, g.n_cells)
    c, s = gf.grouped_forward(g, lay, precision=precision)
    rc, rs = O.grouped_eval(lat, lay.positions, lay.directions, O.Groups(lay.order, lay.inverse, lay.offsets))
    assert np.max(np.abs(c - rc)) <= tol and np.max(np.abs(s - rs)) <= tol


# ---------------------------------------------------------------------------
# rendering
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("name", RENDER_CASES)
@pytest.mark.parametrize("precision,tol", PRECISIONS)
def test_render_matches_golden(gf, name, precision, tol):
    if not precision_available(gf, precision):
        pytest.skip(f"{precision} MLP kernel not built")
    z = golden(name)
    g, occ = device_grid(gf, name)
    cam = device_camera(gf, z)
    cfg = case_config(z)
    cfg = gf.RenderConfig(k=cfg.k, epsilon=cfg.epsilon, background=cfg.background, ert_chunk=cfg.ert_chunk,
                          stratified=cfg.stratified)
    img, st = gf.render_image(g, occ, cam, cfg, seed=int(z["seed"]), precision=precision)
    assert st.total_queries == int(z["total_queries"])
    assert st.ess_skipped == int(z["ess_skipped"])
    assert st.ert_terminated_rays == int(z["ert_terminated_rays"])
    assert st.n_rays == int(z["n_rays"])
    assert img.shape == z["image"].shape and img.dtype == np.float32
    err = float(np.max(np.abs(img - z["image"])))
    assert err <= tol, err
    if name == "render_empty":
        assert np.array_equal(img, np.broadcast_to(np.array(cfg.background, np.float32), img.shape))


@pytest.mark.parametrize("name", ["render_s32_trace", "render_toy96_bias20", "render_inside_chunk7", "render_axis",
                                  "render_s32_k50", "render_two_blocks", "render_w64_bias20"])
def test_render_trace_bit_exact(gf, name):
    """Every queried sample: same ray, same slot, same float32 position, same
    network cell as the oracle (itself pinned to the reference's trace)."""
    z = golden(name)
    g, occ = device_grid(gf, name)
    lat, occ_o = case_inputs(name)
    cam = device_camera(gf, z)
    c = case_config(z)
    cfg = gf.RenderConfig(k=c.k, epsilon=c.epsilon, background=c.background, ert_chunk=c.ert_chunk,
                          stratified=c.stratified)
    _, ctr = O.render_image(lat, occ_o, golden_camera(z), c, seed=int(z["seed"]), trace=True)
    rgb, st, tr = gf.render.render_rays_device(g, occ, cfg, int(z["seed"]), cam=cam, precision="fp32",
                                               trace_capacity=int(z["total_queries"]) + 16)
    ray = np.concatenate([r[1] for r in ctr.rounds])
    slot = np.concatenate([r[2] for r in ctr.rounds])
    pos = np.concatenate([r[3] for r in ctr.rounds])
    cells = O.bin_cells(pos, lat.b_min, lat.b_max, lat.res)
    assert len(tr) == len(ray) == int(z["total_queries"])
    o_ref = np.lexsort((slot, ray))
    o_dev = np.lexsort((tr["slot"], tr["ray"]))
    assert np.array_equal(tr["ray"][o_dev], ray[o_ref])
    assert np.array_equal(tr["slot"][o_dev], slot[o_ref])
    dev_pos = np.stack([tr["x"], tr["y"], tr["z"]], axis=-1)[o_dev]
    assert np.array_equal(dev_pos, pos[o_ref])
    assert np.array_equal(tr["cell"][o_dev].astype(np.int64), cells[o_ref])


def test_render_rays_api_and_sharding_bit_identical(gf):
    """render_rays on explicit rays == render_image; any split of the ray set
    at any offset reproduces the full image bit for bit (multi-GPU contract)."""
    z = golden("render_two_blocks")
    g, occ = device_grid(gf, "render_two_blocks")
    cam = device_camera(gf, z)
    cfg = gf.RenderConfig(k=64)
    img, st = gf.render_image(g, occ, cam, cfg, seed=11)
    o, d = gf.render.generate_rays(cam)
    rgb, st2 = gf.render_rays(g, occ, o, d, cfg, seed=11)
    assert np.array_equal(rgb.reshape(img.shape), img) and st2.total_queries == st.total_queries
    n = cam.width * cam.height
    for cut in (1, 4095, 4096, 5000):
        a, sa, _ = gf.render.render_rays_device(g, occ, cfg, 11, cam=cam, ray_offset=0, n_rays=cut)
        b, sb, _ = gf.render.render_rays_device(g, occ, cfg, 11, cam=cam, ray_offset=cut, n_rays=n - cut)
        full = np.concatenate([a.cpu().numpy(), b.cpu().numpy()]).reshape(img.shape)
        assert np.array_equal(full, img)
        assert int(sa[0] + sb[0]) == st.total_queries


def test_weight_cache_invalidated_by_in_place_edit(gf):
    """test_grid.py:188-191 pattern: mutate params in place, query again."""
    g = gf.init_network_grid(unit(gf), (2, 2, 2), seed=3)
    x = np.array([[-0.5, -0.5, -0.5]], np.float32)
    d = np.array([[0, 0, 1]], np.float32)
    _, s0 = g.query_points(x, d)
    g.params.biases["density"][:] = 7.0
    _, s1 = g.query_points(x, d)
    assert s1[0] != s0[0]
    for k in g.params.weights:
        g.params.weights[k][0] = 0
        g.params.biases[k][0] = 0
    c, s = gf.query_field(g, np.array([-0.5, -0.5, -0.5]), np.array([0.0, 0.0, 1.0]))
    assert np.allclose(c, 0.5) and s == 0.0


def test_deterministic_across_runs(gf):
    g, occ = device_grid(gf, "render_toy96_bias20")
    cam = gf.sphere_cameras(unit(gf), 1, 128, seed=9)[0]
    a, sa = gf.render_image(g, occ, cam, gf.RenderConfig(), seed=7)
    b, sb = gf.render_image(g, occ, cam, gf.RenderConfig(), seed=7, workers=8)
    assert np.array_equal(a, b) and sa.total_queries == sb.total_queries
    c, _ = gf.render_image(g, occ, cam, gf.RenderConfig(), seed=8)
    assert not np.array_equal(a, c)


def test_graph_reuse_across_views_bit_identical(gf, monkeypatch):
    """Views, seeds and output buffers change between calls while the cached
    CUDA graph is updated in place (cudaGraphExecUpdate): every frame must be
    bit-identical to an eager (uncaptured) render of the same call."""
    aabb = unit(gf)
    g = gf.init_network_grid(aabb, (16, 16, 16), seed=0)
    g.params.biases["density"][:] = 20.0
    from conftest import toy_occupancy_bits

    res, bits = toy_occupancy_bits()
    occ = gf.OccupancyGrid(aabb, res, bits.copy())
    cams = gf.sphere_cameras(aabb, 3, 40, seed=4)
    cfg = gf.RenderConfig(k=96)
    got = [gf.render_image(g, occ, cams[i % 3], cfg, seed=i, precision="fp16") for i in range(6)]
    monkeypatch.setenv("GF_NO_GRAPH", "1")
    for i in range(6):
        img, st = gf.render_image(g, occ, cams[i % 3], cfg, seed=i, precision="fp16")
        assert np.array_equal(img, got[i][0])
        assert st.to_dict() | {"wall_ms": 0} == got[i][1].to_dict() | {"wall_ms": 0}


@pytest.mark.gpu
@pytest.mark.skipif(not have_gpu(), reason="needs CUDA")
@pytest.mark.parametrize("precision", ["fp16", "fp32"])
def test_grouped_rounds_bit_identical(precision, monkeypatch):
    """Rounds run in groups (GF_GROUP, default 2) with speculative placement
    and per-round ERT at compositing: images and every RenderStats counter
    must be bit-identical to one round at a time, on an ERT-heavy frame."""
    import paper_2103_13744_b200 as gf

    aabb = gf.Aabb((-1.0,) * 3, (1.0,) * 3)
    grid = gf.init_network_grid(aabb, (16, 16, 16), seed=0, precision=precision)
    grid.params.biases["density"][:] = 20.0
    res, bits = toy_occupancy_bits()
    occ = gf.OccupancyGrid(aabb, res, bits.copy())
    cam = gf.sphere_cameras(aabb, 1, 96, seed=3)[0]
    out = {}
    for mode in ("1", "2", "3", "4", "2-nofuse"):
        monkeypatch.setenv("GF_GROUP", mode[0])
        monkeypatch.setenv("GF_NO_FUSE", "1" if mode.endswith("nofuse") else "0")
        for cfg in (gf.RenderConfig(), gf.RenderConfig(k=200, ert_chunk=24)):
            img, st = gf.render_image(grid, occ, cam, cfg, seed=7)
            out.setdefault(cfg.k, []).append((mode, img, (st.total_queries, st.ess_skipped, st.ert_terminated_rays)))
    for k, runs in out.items():
        _, img0, st0 = runs[0]
        assert st0[2] > 0  # the frame really terminates rays early
        for mode, img, st in runs[1:]:
            assert st == st0, (k, mode, st, st0)
            assert np.array_equal(img, img0), (k, mode)


@pytest.mark.parametrize("w,h", [(37, 23), (130, 9), (16, 8), (17, 9)])
def test_ragged_image_shapes_match_oracle(gf, w, h):
    """Images whose sides are not multiples of the marcher's 16x8-pixel CTA
    tiles (partial tiles at the right and bottom edges), on the toy 256^3
    occupancy (occupancy bricks, specialised marcher): counts exact, colours
    within the fp16 / fp32 bounds of the oracle."""
    from oracle import gridfield_oracle as O

    aabb = unit(gf)
    g = gf.init_network_grid(aabb, (16, 16, 16), seed=0)
    g.params.biases["density"][:] = 8.0
    res, bits = toy_occupancy_bits()
    occ = gf.OccupancyGrid(aabb, res, bits.copy())
    c = gf.sphere_cameras(aabb, 1, 64, seed=7)[0]
    cam = gf.Camera(w, h, c.fx * w / 64, c.fy * h / 64, w / 2, h / 2, c.c2w)
    lat = O.init_lattice(aabb.b_min, aabb.b_max, (16, 16, 16), seed=0)
    lat.biases["density"][:] = 8.0
    occ_o = O.Occupancy(aabb.b_min, aabb.b_max, np.asarray(res), np.asarray(bits))
    ref_img, ref = O.render_image(lat, occ_o, cam, O.MarchConfig(), seed=0)
    for precision, tol in (("fp16", 1e-3), ("fp32", 2e-5)):
        img, st = gf.render_image(g, occ, cam, gf.RenderConfig(), seed=0, precision=precision)
        assert (st.total_queries, st.ess_skipped, st.ert_terminated_rays) == \
            (ref.total_queries, ref.ess_skipped, ref.ert_terminated_rays), (w, h, precision)
        assert float(np.abs(img - ref_img).max()) <= tol, (w, h, precision)


FUZZ = [  # (k, ert_chunk, epsilon, stratified, density bias, occupancy, grid res, image, seed)
    (37, 5, 0.01, True, 12.0, "toy", (16, 16, 16), (20, 13), 1),
    (96, 32, 0.2, True, 20.0, "toy", (4, 4, 4), (24, 24), 2),
    (64, 17, 0.0, True, 3.0, "solid", (2, 3, 4), (11, 31), 3),
    (50, 64, 0.05, True, 25.0, "toy", (16, 16, 16), (16, 16), 4),
    (128, 32, 0.01, False, 20.0, "toy", (8, 8, 8), (19, 17), 5),
    (33, 1, 0.3, True, 30.0, None, (16, 16, 16), (9, 7), 6),
    (200, 24, 0.001, True, 15.0, "toy", (16, 16, 16), (32, 8), 7),
]


@pytest.mark.parametrize("case", FUZZ, ids=[f"k{c[0]}c{c[1]}e{c[2]}" for c in FUZZ])
def test_config_fuzz_matches_oracle(gf, case):
    """Assorted RenderConfig / lattice / occupancy / image combinations (chunk
    sizes that are not 32, chunks longer than 32 (sequential marcher), k not
    a multiple of the chunk, no ERT, unstratified, no occupancy, ragged
    images) against the oracle: counts exact, colours within the fp16 / fp32
    bounds."""
    from oracle import gridfield_oracle as O

    k, chunk, eps, strat, bias, oname, gres, (w, h), seed = case
    aabb = unit(gf)
    g = gf.init_network_grid(aabb, gres, seed=seed)
    g.params.biases["density"][:] = bias
    lat = O.init_lattice(aabb.b_min, aabb.b_max, gres, seed=seed)
    lat.biases["density"][:] = bias
    occ = occ_o = None
    if oname == "toy":
        res, bits = toy_occupancy_bits()
    elif oname == "solid":
        res, bits = np.array([128] * 3), np.asarray(gf.OccupancyGrid.solid(aabb, (128, 128, 128)).bits)
    if oname is not None:
        occ = gf.OccupancyGrid(aabb, res, np.asarray(bits).copy())
        occ_o = O.Occupancy(aabb.b_min, aabb.b_max, np.asarray(res), np.asarray(bits))
    c = gf.sphere_cameras(aabb, 1, 64, seed=seed + 10)[0]
    cam = gf.Camera(w, h, c.fx * w / 64, c.fy * h / 64, w / 2, h / 2, c.c2w)
    cfg = gf.RenderConfig(k=k, ert_chunk=chunk, epsilon=eps, stratified=strat)
    ref_img, ref = O.render_image(lat, occ_o, cam, O.MarchConfig(k=k, ert_chunk=chunk, epsilon=eps,
                                                                   stratified=strat), seed=seed)
    for precision, tol in (("fp16", 1e-3), ("fp32", 2e-5)):
        img, st = gf.render_image(g, occ, cam, cfg, seed=seed, precision=precision)
        assert (st.total_queries, st.ess_skipped, st.ert_terminated_rays, st.n_rays) == \
            (ref.total_queries, ref.ess_skipped, ref.ert_terminated_rays, w * h), (case, precision)
        assert float(np.abs(img - ref_img).max()) <= tol, (case, precision)
