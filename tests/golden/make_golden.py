"""Generate golden vectors from the reference package itself.

Run in the authoring container (the GPU box has no /root/reference):

    python tests/golden/make_golden.py

It imports ``gridfield`` read-only from /root/reference/pkg/src, drives the
reference's own public API on small seeded inputs, and writes compressed .npz
fixtures next to this script.  Tests pin the oracle (oracle/) against these
files and then check the CUDA path against the oracle.
"""

from __future__ import annotations

import os
import sys
import time
from pathlib import Path

import numpy as np

REF = Path(os.environ.get("GRIDFIELD_REFERENCE", "/root/reference/pkg/src"))
OUT = Path(__file__).resolve().parent
sys.path.insert(0, str(REF))

import gridfield  # noqa: E402  (the reference)
from gridfield import core, grid as ggrid, mlp, occupancy, render, scene, batched  # noqa: E402


def save(name, **arrays):
    np.savez_compressed(OUT / f"{name}.npz", **arrays)
    print(f"wrote {name}.npz  ({(OUT / f'{name}.npz').stat().st_size / 1024:.1f} KiB)")


def cam_arrays(cam):
    return dict(
        cam_w=np.int64(cam.width), cam_h=np.int64(cam.height),
        cam_f=np.array([cam.fx, cam.fy, cam.cx, cam.cy], np.float64),
        cam_c2w=np.asarray(cam.c2w, np.float64),
    )


class Tracer:
    """Wraps NetworkGrid.query_points to record the positions of every field
    query in call order (one call per block-round)."""

    def __init__(self, g):
        self.g = g
        self.aabb = g.aabb
        self.calls = []

    def query_points(self, p, d):
        self.calls.append((np.array(p, np.float32), np.array(d, np.float32)))
        return self.g.query_points(p, d)


def unit():
    return core.Aabb((-1.0, -1.0, -1.0), (1.0, 1.0, 1.0))


def gen_rays():
    out = {}
    cams = scene.sphere_cameras(unit(), 3, 96, seed=0)
    odd = render.Camera(37, 23, 31.5, 29.0, 17.25, 12.75, render.look_at_pose(np.array([0.3, -2.5, 0.7]), np.zeros(3)))
    ident = render.Camera(16, 16, 16.0, 16.0, 8.0, 8.0, np.eye(4))
    for i, cam in enumerate(cams + [odd, ident]):
        o, d = render.generate_rays(cam)
        for k, v in cam_arrays(cam).items():
            out[f"{k}_{i}"] = v
        out[f"o_{i}"], out[f"d_{i}"] = o, d
    out["n"] = np.int64(len(cams) + 2)
    save("rays", **out)


def gen_pcg():
    ents = np.array([[0, 0], [0, 4096], [7, 12288], [3, 4096 * 156], [2**33 + 5, 4096 * 7], [123456789, 0]], dtype=np.uint64)
    st = np.zeros((len(ents), 4), np.uint64)
    draws = np.zeros((len(ents), 64), np.float32)
    for i, (a, b) in enumerate(ents):
        s = np.random.PCG64(np.random.SeedSequence([int(a), int(b)])).state["state"]
        st[i] = [s["state"] >> 64, s["state"] & (2**64 - 1), s["inc"] >> 64, s["inc"] & (2**64 - 1)]
        draws[i] = np.random.default_rng(np.random.SeedSequence([int(a), int(b)])).random(64, dtype=np.float32)
    save("pcg64", entropy=ents, state=st, draws=draws)


def gen_pointwise():
    rng = np.random.default_rng(5)
    v = rng.uniform(-1, 1, (256, 3)).astype(np.float32)
    v[:4] = [[0, 0, 0], [1, 1, 1], [-1, -1, -1], [0.5, -0.25, 0.125]]
    d = rng.normal(size=(256, 3)).astype(np.float32)
    d /= np.linalg.norm(d, axis=-1, keepdims=True)
    aabb = unit()
    pts = rng.uniform(-1, 1, (4096, 3)).astype(np.float32)
    pts[:6] = [[-1, -1, -1], [1, 1, 1], [0, 0, 0], [0.999, 0.5, 0.25], [-0.875, 0.125, 0.9999999], [np.float32(0.125), -0.5, 1]]
    far = rng.uniform(-1.2, 1.2, (2048, 3)).astype(np.float32)
    sig = np.concatenate([rng.uniform(0, 50, 1000), [0, 1e-6, 1e6, 10.0]]).astype(np.float32)
    dl = np.concatenate([rng.uniform(0, 0.02, 1000), [0.1, 0.5, 0.1, 0.01]]).astype(np.float32)
    save(
        "pointwise",
        enc_in=v, enc_x=core.positional_encode(v, 10), enc_d_in=d, enc_d=core.positional_encode(d, 4),
        bin_pts=pts,
        bin16=core.flatten_cell_index(core.bin_point(pts, aabb, (16, 16, 16)), (16, 16, 16)),
        bin256=core.flatten_cell_index(core.bin_point(pts, aabb, (256, 256, 256)), (256, 256, 256)),
        bin_5_7_3=core.flatten_cell_index(core.bin_point(pts, aabb, (5, 7, 3)), (5, 7, 3)),
        clip_in=far, clip_out=core.clip_into(far, aabb),
        alpha_sigma=sig, alpha_delta=dl, alpha=core.density_to_alpha(sig, dl),
    )


def gen_query():
    aabb = unit()
    g = ggrid.init_network_grid(aabb, (16, 16, 16), seed=3)
    rng = np.random.default_rng(0)
    n = 20000
    pts = rng.uniform(-1, 1, (n, 3)).astype(np.float32)
    dirs = rng.normal(size=(n, 3)).astype(np.float32)
    dirs /= np.linalg.norm(dirs, axis=-1, keepdims=True)
    c, s = g.query_points(pts, dirs)
    keys = g.cell_index(pts)
    lay = batched.group_by_network(batched.QueryBatch(pts, dirs, keys), g.n_cells)
    # small grid with tagged density bias (test_grid.py:214-229 style)
    g4 = ggrid.init_network_grid(aabb, (4, 4, 4), seed=5)
    for k in g4.params.weights:
        g4.params.weights[k][:] = 0
        g4.params.biases[k][:] = 0
    g4.params.biases["density"][:, 0] = np.arange(g4.n_cells, dtype=np.float32)
    _, s4 = g4.query_points(pts[:2000], dirs[:2000])
    save(
        "query16",
        pts=pts, dirs=dirs, rgb=c, sigma=s, keys=keys,
        order=lay.order, inverse=lay.inverse, offsets=lay.offsets,
        tag_sigma=s4,
        w0_checksum=np.float64(g.params.weights["trunk0"].astype(np.float64).sum()),
    )


def toy_occ(res=256):
    path = OUT / f"toy_occupancy_{res}.npz"
    if path.exists():
        z = np.load(path)
        return occupancy.OccupancyGrid(unit(), z["res"], z["bits"])
    t = time.time()
    sc = scene.standard_toy_scene()
    occ = occupancy.extract_occupancy(sc.density_at, sc.aabb, (res,) * 3, tau=10.0, workers=os.cpu_count())
    print(f"toy occupancy {res}^3 in {time.time() - t:.1f}s, {occ.occupied_fraction():.4f} occupied")
    np.savez_compressed(path, res=occ.resolution, bits=occ.bits)
    return occ


def render_case(name, g, occ, cam, cfg, seed=0, keep_trace=True):
    tr = Tracer(g)
    img, st = render.render_image(tr, occ, cam, cfg, seed=seed, workers=1)
    pos = np.concatenate([c[0] for c in tr.calls]) if tr.calls else np.zeros((0, 3), np.float32)
    counts = np.array([len(c[0]) for c in tr.calls], np.int64)
    cells = g.cell_index(pos) if len(pos) else np.zeros(0, np.int64)
    arr = dict(
        image=img, total_queries=np.int64(st.total_queries), ess_skipped=np.int64(st.ess_skipped),
        ert_terminated_rays=np.int64(st.ert_terminated_rays), n_rays=np.int64(st.n_rays),
        k=np.int64(cfg.k), epsilon=np.float64(cfg.epsilon), background=np.array(cfg.background, np.float64),
        ert_chunk=np.int64(cfg.ert_chunk), stratified=np.bool_(cfg.stratified), seed=np.int64(seed),
        call_counts=counts, cell_hist=np.bincount(cells, minlength=g.n_cells).astype(np.int64),
        pos_checksum=np.float64(pos.astype(np.float64).sum()),
        **cam_arrays(cam),
    )
    if keep_trace:
        arr["trace_pos"] = pos
    save(name, **arr)
    print(f"  {name}: Q={st.total_queries} ess={st.ess_skipped} ert={st.ert_terminated_rays}")


def gen_render():
    aabb = unit()
    cam64 = scene.sphere_cameras(aabb, 1, 64, seed=0)[0]
    g0 = ggrid.init_network_grid(aabb, (16, 16, 16), seed=0)
    solid = occupancy.OccupancyGrid.solid(aabb, (256, 256, 256))
    # C1: the BASELINE oracle configuration
    render_case("render_c1", g0, solid, cam64, render.RenderConfig(k=128), keep_trace=False)
    gb = ggrid.init_network_grid(aabb, (16, 16, 16), seed=0)
    gb.params.biases["density"][:] = 20.0
    render_case("render_c1_bias20", gb, solid, cam64, render.RenderConfig(k=128), keep_trace=False)
    occ = toy_occ(256)
    cam96 = scene.sphere_cameras(aabb, 1, 96, seed=0)[0]
    render_case("render_toy96", g0, occ, cam96, render.RenderConfig(), keep_trace=False)
    render_case("render_toy96_bias20", gb, occ, cam96, render.RenderConfig(), keep_trace=False)
    # small cases with full per-query traces and edge configurations
    cam32 = scene.sphere_cameras(aabb, 1, 32, seed=2)[0]
    render_case("render_s32_trace", gb, occ, cam32, render.RenderConfig(k=96), seed=5)
    render_case("render_s32_k50", gb, occ, cam32, render.RenderConfig(k=50, ert_chunk=32, background=(0.2, 0.4, 0.6)), seed=1)
    render_case("render_s32_nostrat", gb, None, cam32, render.RenderConfig(k=64, stratified=False, epsilon=0.0), seed=0)
    g2 = ggrid.init_network_grid(aabb, (2, 3, 4), seed=9)
    g2.params.biases["density"][:] = 5.0
    inside = render.Camera(24, 20, 12.0, 12.0, 12.0, 10.0, render.look_at_pose(np.array([0.2, 0.1, -0.3]), np.array([0.5, 0.9, 0.4])))
    render_case("render_inside_chunk7", g2, None, inside, render.RenderConfig(k=40, ert_chunk=7, epsilon=0.05), seed=3)
    axis = render.Camera(16, 16, 16.0, 16.0, 8.0, 8.0, render.look_at_pose(np.array([0.0, 0.0, -3.0]), np.zeros(3)))
    render_case("render_axis", gb, occ, axis, render.RenderConfig(k=64), seed=0)
    empty = occupancy.OccupancyGrid.solid(aabb, (8, 8, 8), value=False)
    render_case("render_empty", g0, empty, cam32, render.RenderConfig(k=32, background=(1.0, 0.5, 0.25)), seed=0)
    # multi-block ray set (2 blocks + ragged tail) through render_rays
    cam80 = scene.sphere_cameras(aabb, 1, 80, seed=6)[0]  # 6400 rays = 1 full block + 2304
    render_case("render_two_blocks", gb, occ, cam80, render.RenderConfig(k=64), seed=11, keep_trace=False)


def w64_grid(res=(8, 8, 8), seed=4):
    """The C4 architecture (64-wide tiny MLPs) on a small lattice."""
    return ggrid.init_network_grid(unit(), res, seed=seed, arch=mlp.MlpArchitecture(hidden_width=64))


def gen_wide():
    """64-wide networks (BASELINE config 4's architecture): a query and a
    traced render on an 8^3 lattice."""
    aabb = unit()
    g = w64_grid()
    rng = np.random.default_rng(2)
    n = 8000
    pts = rng.uniform(-1, 1, (n, 3)).astype(np.float32)
    dirs = rng.normal(size=(n, 3)).astype(np.float32)
    dirs /= np.linalg.norm(dirs, axis=-1, keepdims=True)
    c, s = g.query_points(pts, dirs)
    save("query_w64", pts=pts, dirs=dirs, rgb=c, sigma=s,
         w0_checksum=np.float64(g.params.weights["trunk0"].astype(np.float64).sum()))
    gb = w64_grid()
    gb.params.biases["density"][:] = 20.0
    occ = toy_occ(256)
    cam = scene.sphere_cameras(aabb, 1, 40, seed=7)[0]
    render_case("render_w64_bias20", gb, occ, cam, render.RenderConfig(k=128), seed=2)


def gen_bulk():
    """BASELINE config 5's input recipe (bench.py:108-112 of the reference:
    uniform positions in the box, normalised normal directions, default_rng(0))
    at 2^14 points through the 16^3 seed-0 lattice."""
    g = ggrid.init_network_grid(unit(), (16, 16, 16), seed=0)
    rng = np.random.default_rng(0)
    n = 1 << 14
    span = (g.aabb.b_max - g.aabb.b_min).astype(np.float32)
    pts = g.aabb.b_min.astype(np.float32) + rng.random((n, 3), dtype=np.float32) * span
    dirs = rng.normal(size=(n, 3)).astype(np.float32)
    dirs /= np.linalg.norm(dirs, axis=-1, keepdims=True)
    c, s = g.query_points(pts, dirs)
    save("query_c5", pts=pts, dirs=dirs, rgb=c, sigma=s, keys=g.cell_index(pts))


def gen_scene():
    """Analytic scenes (scene.py) through the reference's
    render_image: dense / ESS / ERT renders and field queries."""
    sc = scene.standard_toy_scene()
    aabb = sc.aabb
    cam48 = scene.sphere_cameras(aabb, 1, 48, seed=3)[0]
    cfg = render.RenderConfig(k=128, stratified=False)
    for name, c, occ in (("render_scene_ert", cfg, None), ("render_scene_dense", cfg.replace(epsilon=0.0), None)):
        img, st = render.render_image(sc, occ, cam48, c, seed=0)
        save(name, image=img, total_queries=np.int64(st.total_queries), ess_skipped=np.int64(st.ess_skipped),
             ert_terminated_rays=np.int64(st.ert_terminated_rays), n_rays=np.int64(st.n_rays), k=np.int64(c.k),
             epsilon=np.float64(c.epsilon), background=np.array(c.background, np.float64),
             ert_chunk=np.int64(c.ert_chunk), stratified=np.bool_(c.stratified), seed=np.int64(0), **cam_arrays(cam48))
    occ = occupancy.extract_occupancy(sc.density_at, aabb, (32, 32, 32), tau=0.0)
    cam_b = scene.sphere_cameras(aabb, 1, 48, seed=4)[0]
    c = cfg.replace(epsilon=0.0)
    img, st = render.render_image(sc, occ, cam_b, c, seed=0)
    save("render_scene_ess", image=img, total_queries=np.int64(st.total_queries), ess_skipped=np.int64(st.ess_skipped),
         ert_terminated_rays=np.int64(st.ert_terminated_rays), n_rays=np.int64(st.n_rays), k=np.int64(c.k),
         epsilon=np.float64(c.epsilon), background=np.array(c.background, np.float64), ert_chunk=np.int64(c.ert_chunk),
         stratified=np.bool_(c.stratified), seed=np.int64(0), occ_res=occ.resolution, occ_bits=occ.bits,
         **cam_arrays(cam_b))
    sp = scene.specular_toy_scene()
    cam32 = scene.sphere_cameras(aabb, 1, 32, seed=5)[0]
    c = render.RenderConfig(k=96)
    img, st = render.render_image(sp, None, cam32, c, seed=5)
    save("render_scene_specular", image=img, total_queries=np.int64(st.total_queries),
         ess_skipped=np.int64(st.ess_skipped), ert_terminated_rays=np.int64(st.ert_terminated_rays),
         n_rays=np.int64(st.n_rays), k=np.int64(c.k), epsilon=np.float64(c.epsilon),
         background=np.array(c.background, np.float64), ert_chunk=np.int64(c.ert_chunk),
         stratified=np.bool_(c.stratified), seed=np.int64(5), **cam_arrays(cam32))
    rng = np.random.default_rng(8)
    n = 8192
    pts = rng.uniform(-1, 1, (n, 3)).astype(np.float32)
    dirs = rng.normal(size=(n, 3)).astype(np.float32)
    dirs /= np.linalg.norm(dirs, axis=-1, keepdims=True)
    out = {}
    for tag, s_ in (("std", sc), ("spec", sp), ("rand", scene.random_toy_scene(4, 7))):
        c_, s2 = s_.query_points(pts, dirs)
        out[f"{tag}_rgb"], out[f"{tag}_sigma"] = c_, s2
    save("query_scene", pts=pts, dirs=dirs, **out)


def gen_extract():
    """occupancy.extract_occupancy (occupancy.py:94-128) through
    the reference: analytic scenes (bit-exact targets) at cubic, ragged and
    non-power-of-two boxes, and a density_probe of a random-init lattice
    (tolerance target: cells with a probe within `margin` of tau are marked)."""
    from gridfield import train

    out = {}
    sc, sp, rnd = scene.standard_toy_scene(), scene.specular_toy_scene(), scene.random_toy_scene(11, 6)
    cases = [
        ("toy64", sc, sc.aabb, (64, 64, 64), 10.0),
        ("rand48", rnd, rnd.aabb, (48, 40, 36), 10.0),
        ("spec_box", sp, core.Aabb((-0.9, -1.0, -0.7), (1.0, 0.8, 1.0)), (40, 24, 33), 0.0),
        ("toy_tau_f64", sc, sc.aabb, (30, 30, 30), np.float64(20.000001)),
    ]
    for tag, s_, box, res, tau in cases:
        occ = occupancy.extract_occupancy(s_.density_at, box, res, tau=tau)
        out[f"{tag}_bits"] = occ.bits
        out[f"{tag}_res"] = np.asarray(res, np.int64)
        out[f"{tag}_box"] = np.stack([box.b_min, box.b_max])
        out[f"{tag}_tau"] = np.float64(tau)
        out[f"{tag}_tau_is_f64"] = np.bool_(isinstance(tau, np.float64))
        print(tag, occ.occupied_fraction())
    print("random scene boxes:", len(rnd.boxes), "spheres:", len(rnd.spheres))
    # network density probe: random-init 4^3 lattice with per-cell density biases
    aabb = unit()
    g = ggrid.init_network_grid(aabb, (4, 4, 4), seed=3)
    rng = np.random.default_rng(21)
    g.params.biases["density"][:] = rng.uniform(-0.5, 2.0, g.params.biases["density"].shape).astype(np.float32)
    field = train.density_probe(g)
    res = (24, 20, 16)
    box = core.Aabb((-1.0, -0.75, -1.0), (0.9, 1.0, 0.6))
    lo = occupancy.extract_occupancy(field, box, res, tau=0.0)
    # tau at the median per-cell max density, and a margin mask for the tolerance check
    n = int(np.prod(res))
    cell = box.cell_size(res)
    flat = np.arange(n)
    lows = box.b_min + np.stack([flat % res[0], (flat // res[0]) % res[1], flat // (res[0] * res[1])], -1) * cell
    pts = (lows[:, None, :] + occupancy._PROBE_OFFSETS[None] * cell).astype(np.float32)
    sig = field(core.clip_into(pts.reshape(-1, 3), box)).reshape(n, 27)
    tau = float(np.round(np.median(sig.max(1)), 4))
    occ = occupancy.extract_occupancy(field, box, res, tau=tau)
    near = (np.abs(sig - np.float32(tau)) < 5e-3).any(1)
    out.update(net_bits=occ.bits, net_res=np.asarray(res, np.int64), net_box=np.stack([box.b_min, box.b_max]),
               net_tau=np.float64(tau), net_near=np.packbits(near, bitorder="little"), net_tau0_bits=lo.bits,
               net_near0=np.packbits((np.abs(sig) < 5e-3).any(1), bitorder="little"),
               net_bias=np.asarray(g.params.biases["density"]), net_seed=np.int64(3), net_grid_res=np.array([4, 4, 4]))
    print("net", occ.occupied_fraction(), "near", near.mean(), "tau", tau)
    try:  # extraction box leaving the network's box: the reference's message
        occupancy.extract_occupancy(field, core.Aabb((-1.0, -1.0, -1.0), (1.0, 1.25, 1.0)), (8, 8, 8), tau=1.0)
        raise AssertionError("expected an out-of-bounds error")
    except ValueError as e:
        out["net_oob_message"] = np.array(str(e))
        print("oob:", e)
    save("extract", **out)


def _fixed_batch(grid, n_rays, k, seed, occ=None):
    """test_train.py:92-103 fixed_batch."""
    from gridfield import train

    rng = np.random.default_rng(seed)
    origins = np.tile(np.array([[-2.0, 0.0, 0.0]], np.float32), (n_rays, 1))
    offsets = rng.uniform(-0.6, 0.6, (n_rays, 2)).astype(np.float32)
    targets = np.concatenate([np.zeros((n_rays, 1), np.float32), offsets], axis=1)
    dirs = targets - origins
    dirs /= np.linalg.norm(dirs, axis=-1, keepdims=True)
    samples = train.prepare_ray_samples(origins, dirs, grid.aabb, k, True, rng, occ=occ)
    gt = rng.random((n_rays, 3)).astype(np.float32)
    return origins, dirs, samples, gt


def _grads_dict(prefix, g):
    out = {}
    for k_, v in g.weights.items():
        out[f"{prefix}w_{k_}"] = np.asarray(v)
    for k_, v in g.biases.items():
        out[f"{prefix}b_{k_}"] = np.asarray(v)
    return out


def gen_train():
    """Training kernels through the reference: grouped_backward
    on random upstream gradients (32- and 64-wide), photometric_loss_and_grads
    on test_train.py's fixed batch (with and without regularisation / density
    noise), adam_update, and one distill_step."""
    from gridfield import train

    out = {}
    aabb = core.Aabb((0.0, 0.0, 0.0), (1.0, 1.0, 1.0))
    # grouped_backward, 32-wide (3,2,2) lattice with density biases around 0
    for tag, res, arch, n in (("g32", (3, 2, 2), None, 3000), ("g64", (2, 1, 1), mlp.MlpArchitecture(hidden_width=64), 700)):
        g = ggrid.init_network_grid(aabb, res, seed=11, arch=arch)
        rng = np.random.default_rng(12)
        for k_ in g.params.biases:
            g.params.biases[k_][:] = rng.normal(0, 0.3, g.params.biases[k_].shape).astype(np.float32)
        pts = rng.uniform(0, 1, (n, 3)).astype(np.float32)
        pts[:7] = np.float32(1.0)  # upper faces
        dirs = rng.normal(size=(n, 3)).astype(np.float32)
        dirs /= np.linalg.norm(dirs, axis=-1, keepdims=True)
        dcol = rng.normal(size=(n, 3)).astype(np.float32)
        dsig = rng.normal(size=n).astype(np.float32)
        layout = batched.group_by_network(batched.QueryBatch(pts, dirs, g.cell_index(pts)), g.n_cells)
        caches = []
        batched.grouped_forward(g, layout, caches=caches)
        grads = batched.grouped_backward(g, layout, caches, dcol, dsig)
        out.update({f"{tag}_pts": pts, f"{tag}_dirs": dirs, f"{tag}_dcol": dcol, f"{tag}_dsig": dsig,
                    f"{tag}_res": np.array(res), f"{tag}_biases": np.concatenate([np.asarray(v).ravel() for v in g.params.biases.values()])})
        out.update(_grads_dict(f"{tag}_", grads))
    # photometric loss + grads on the reference test's fixed batch
    g = ggrid.init_network_grid(aabb, (2, 2, 2), seed=5)
    g.params.biases["density"][:] = 1.5
    _, _, smp, gt = _fixed_batch(g, 64, 32, 1)
    noise = np.random.default_rng(13).normal(0, 0.5, len(smp.positions)).astype(np.float32)
    out.update(ph_pos=smp.positions, ph_dirs=smp.directions, ph_ray=smp.ray_index, ph_slot=smp.slot,
               ph_deltas=smp.deltas, ph_nrays=np.int64(smp.n_rays), ph_k=np.int64(smp.k), ph_gt=gt, ph_noise=noise)
    for tag, kw in (("ph0", {}), ("ph_reg", {"reg_weight": 1e-3}), ("ph_noise", {"sigma_noise": noise})):
        loss, grads = train.photometric_loss_and_grads(g, smp, gt, (1.0, 1.0, 1.0), **kw)
        out[f"{tag}_loss"] = np.float64(loss)
        out.update(_grads_dict(f"{tag}_", grads))
    # adam: two steps with the ph0 gradients
    cfg = train.TrainConfig()
    _, grads = train.photometric_loss_and_grads(g, smp, gt, (1.0, 1.0, 1.0))
    st = train.AdamState.for_params(g.params)
    p = g.params.copy()
    train.adam_update(p, grads, st, 5e-4, cfg)
    train.adam_update(p, grads, st, 3e-4, cfg)
    out.update(_grads_dict("adam_p_", p))
    out.update(_grads_dict("adam_m_", st.m))
    out.update(_grads_dict("adam_v_", st.v))
    # one distill step (test_train.py:255-270 setup)
    enc = core.PositionalEncoding()
    dcfg = train.TrainConfig(distill_points_per_cell=8, teacher_hidden_layers=4, teacher_hidden_width=32,
                             teacher_direction_width=32, teacher_skip_layer=None)
    teacher = ggrid.init_network_grid(aabb, (1, 1, 1), seed=6, arch=dcfg.teacher_architecture(enc), encoding=enc)
    student = ggrid.init_network_grid(aabb, (2, 2, 2), seed=7)
    st = train.AdamState.for_params(student.params)
    losses = [train.distill_step(student, teacher, dcfg, st, np.random.default_rng(3), delta_ref=0.01)]
    out["ds_loss"] = np.array(losses)
    out.update(_grads_dict("ds_p_", student.params))
    # prepare_ray_samples: occupancy-filtered, a Generator holding a buffered
    # half (odd number of float32 draws before), and non-stratified
    occ4 = occupancy.OccupancyGrid.from_bool_array(aabb, (4, 1, 1), np.array([False, False, False, True]))
    for tag, pre, strat, occ_ in (("prep_occ", 0, True, occ4), ("prep_odd", 3, True, None), ("prep_mid", 0, False, None)):
        rng = np.random.default_rng(17)
        if pre:
            rng.random(pre, dtype=np.float32)
        n_r, k_ = 24, 40
        origins = np.tile(np.array([[-2.0, 0.0, 0.0]], np.float32), (n_r, 1))
        offs = rng.uniform(-0.6, 0.6, (n_r, 2)).astype(np.float32)
        dirs = np.concatenate([np.zeros((n_r, 1), np.float32), offs], axis=1) - origins
        dirs /= np.linalg.norm(dirs, axis=-1, keepdims=True)
        smp = train.prepare_ray_samples(origins, dirs, aabb, k_, strat, rng, occ=occ_)
        after = rng.random(5, dtype=np.float32)  # pins the Generator state left behind
        out.update({f"{tag}_o": origins, f"{tag}_d": dirs, f"{tag}_pos": smp.positions, f"{tag}_dirs": smp.directions,
                    f"{tag}_ray": smp.ray_index, f"{tag}_slot": smp.slot, f"{tag}_deltas": smp.deltas,
                    f"{tag}_after": after, f"{tag}_k": np.int64(k_), f"{tag}_pre": np.int64(pre)})
    # three photometric_step calls on a tiny duck-typed dataset (test_train.py:183-197 shape)
    class DS:
        def __init__(self, aabb, cams, images):
            self.aabb, self.cameras, self.images = aabb, cams, images

        def indices(self, split):
            return [0, 1, 2] if split == "train" else [1]

    cams = scene.sphere_cameras(aabb, 3, 16, seed=1)
    imgs = np.random.default_rng(31).random((3, 16, 16, 3)).astype(np.float32)
    ds = DS(aabb, cams, imgs)
    g = ggrid.init_network_grid(aabb, (2, 2, 2), seed=8)
    g.params.biases["density"][:] = 0.8
    pcfg = train.TrainConfig(batch_size_pixels=32, k_train=16)
    st = train.AdamState.for_params(g.params)
    rng = np.random.default_rng(9)
    out["step_losses"] = np.array([train.photometric_step(g, ds, pcfg, st, rng, lr=5e-4, noise_std=0.1 * i)
                                   for i in range(3)])
    out["step_after"] = rng.random(4)
    out["step_images"] = imgs
    out.update(_grads_dict("step_p_", g.params))
    out["free_space"] = np.float64(train.mean_free_space_density(g, np.arange(0, 8, 3)))
    save("train", **out)
    print("ph0 loss", out["ph0_loss"], "distill", losses, "steps", out["step_losses"])


def gen_ckpt():
    """A checkpoint written by the reference's io.save_checkpoint (io.py:150-175):
    (2,3,4) lattice, seed 9, density bias 5, with a 8^3 occupancy bitmap."""
    from gridfield import io as gio

    aabb = unit()
    g = ggrid.init_network_grid(aabb, (2, 3, 4), seed=9)
    g.params.biases["density"][:] = 5.0
    occ = occupancy.OccupancyGrid.from_bool_array(aabb, (8, 8, 8), np.arange(512) % 3 != 0)
    gio.save_checkpoint(OUT / "ckpt_small.gfckpt", g, occ)
    print("wrote ckpt_small.gfckpt", (OUT / "ckpt_small.gfckpt").stat().st_size)


C2_BLOCKS = (0, 40, 62, 70, 74, 76, 77, 78, 79, 80, 82, 84, 88, 96, 120, 156)


def gen_c2():
    """The benchmarked C2 frame (800x800, 16^3 random init seed 0, toy
    occupancy 256^3, RenderConfig() defaults, seed 0), as random init and
    with density bias 20 (ERT-heavy): full-frame RenderStats from
    render_image, and colours + counters of sampled 4096-ray blocks (centre
    blocks plus the ragged last one) from the reference's own _march_block
    with the block's SeedSequence([seed, block_start]) stream."""
    aabb = unit()
    cam = scene.sphere_cameras(aabb, 64, 800, seed=0)[0]
    occ = toy_occ(256)
    cfg = render.RenderConfig()
    o, d = render.generate_rays(cam)
    o64, d64 = o.astype(np.float64), d.astype(np.float64)
    out = dict(blocks=np.array(C2_BLOCKS, np.int64), **cam_arrays(cam))
    for tag, bias in (("rand", None), ("bias20", 20.0)):
        g = ggrid.init_network_grid(aabb, (16, 16, 16), seed=0)
        if bias is not None:
            g.params.biases["density"][:] = bias
        t = time.time()
        _, st = render.render_image(g, occ, cam, cfg, seed=0, workers=os.cpu_count())
        print(f"  c2 {tag}: full frame {time.time() - t:.1f}s Q={st.total_queries} ess={st.ess_skipped} "
              f"ert={st.ert_terminated_rays}")
        out[f"{tag}_stats"] = np.array([st.total_queries, st.ess_skipped, st.ert_terminated_rays, st.n_rays], np.int64)
        cols, bst = [], []
        for b in C2_BLOCKS:
            s0 = b * render.RAY_BLOCK
            sl = slice(s0, min(s0 + render.RAY_BLOCK, len(o)))
            rng = np.random.default_rng(np.random.SeedSequence([0, s0]))
            c, _, bs = render._march_block(g, occ, o64[sl], d64[sl], cfg, rng)
            cols.append(c.astype(np.float32))
            bst.append([bs.total_queries, bs.ess_skipped, bs.ert_terminated_rays, bs.n_rays])
        out[f"{tag}_block_rgb"] = np.concatenate(cols)
        out[f"{tag}_block_stats"] = np.array(bst, np.int64)
    save("render_c2", **out)


def gen_generic():
    """Manifests the fused tiny-MLP kernels do not cover (mlp.py:30-109),
    through the reference: the default teacher (10 x 256, skip 5, view 128)
    and the desk preset's teacher (6 x 96, skip 2, view 64) queried on random
    points; a traced render of a (2,2,2) lattice of 5 x 48 skip-2 networks
    with 6/3 octaves; and one distill_step with TrainConfig's default
    teacher (train.py:341-390)."""
    from gridfield import train

    out = {}
    aabb = unit()
    enc = core.PositionalEncoding()
    rng = np.random.default_rng(21)
    for tag, arch, res, n in (("teach", mlp.teacher_architecture(), (1, 1, 1), 384),
                              ("desk", train.TrainConfig.desk_preset().teacher_architecture(enc), (2, 1, 1), 300)):
        g = ggrid.init_network_grid(aabb, res, seed=23, arch=arch, encoding=enc)
        for k_ in g.params.biases:
            g.params.biases[k_][:] = rng.normal(0, 0.2, g.params.biases[k_].shape).astype(np.float32)
        pts = rng.uniform(-1, 1, (n, 3)).astype(np.float32)
        dirs = rng.normal(size=(n, 3)).astype(np.float32)
        dirs /= np.linalg.norm(dirs, axis=-1, keepdims=True)
        rgb, sig = g.query_points(pts, dirs)
        out.update({f"{tag}_pts": pts, f"{tag}_dirs": dirs, f"{tag}_rgb": rgb, f"{tag}_sigma": sig,
                    f"{tag}_res": np.array(res), f"{tag}_biases": np.concatenate([np.asarray(v).ravel() for v in g.params.biases.values()])})
    # traced render through a skip-layer lattice with non-default octaves
    enc63 = core.PositionalEncoding(num_freqs_position=6, num_freqs_direction=3)
    arch = mlp.MlpArchitecture(hidden_layers=5, hidden_width=48, position_input_dim=enc63.position_dim,
                               direction_input_dim=enc63.direction_dim, direction_layer_width=40, skip_layer=2)
    g = ggrid.init_network_grid(aabb, (2, 2, 2), seed=24, arch=arch, encoding=enc63)
    g.params.biases["density"][:] = 4.0
    cam = scene.sphere_cameras(aabb, 1, 24, seed=2)[0]
    cfg = render.RenderConfig(k=64)
    img, st = render.render_image(g, None, cam, cfg, seed=0)
    out.update(rimg=img, rstats=np.array([st.total_queries, st.ess_skipped, st.ert_terminated_rays, st.n_rays], np.int64))
    out.update(cam_arrays(cam))
    # one distill_step with the default teacher
    dcfg = train.TrainConfig(distill_points_per_cell=4)
    teacher = ggrid.init_network_grid(aabb, (1, 1, 1), seed=25, arch=dcfg.teacher_architecture(enc), encoding=enc)
    student = ggrid.init_network_grid(aabb, (2, 2, 2), seed=26)
    stt = train.AdamState.for_params(student.params)
    out["ds_loss"] = np.array([train.distill_step(student, teacher, dcfg, stt, np.random.default_rng(27), delta_ref=0.01)])
    out.update(_grads_dict("ds_p_", student.params))
    # render_rays on float64 rays that float32 cannot represent (render.py:368:
    # the slab test sees them, the samples their float32 roundings)
    g16 = ggrid.init_network_grid(aabb, (16, 16, 16), seed=0)
    g16.params.biases["density"][:] = 5.0
    rng64 = np.random.default_rng(31)
    n64 = 3000
    o64 = rng64.uniform(-3, 3, (n64, 3))
    o64[:, 0] = -3.0 + rng64.uniform(0, 1e-9, n64)  # a float32-invisible offset
    tgt = rng64.uniform(-0.9, 0.9, (n64, 3))
    d64 = tgt - o64
    d64 /= np.linalg.norm(d64, axis=-1, keepdims=True)
    d64[:40, 1:] = 0.0  # axis-parallel rays
    d64[:40, 0] = 1.0
    o64[:40, 1:] = rng64.uniform(-1.2, 1.2, (40, 2))
    rgb64, st64 = render.render_rays(g16, None, o64, d64, render.RenderConfig(k=64), seed=3)
    out.update(f64_o=o64, f64_d=d64, f64_rgb=rgb64,
               f64_stats=np.array([st64.total_queries, st64.ess_skipped, st64.ert_terminated_rays, st64.n_rays], np.int64))
    save("generic", **out)
    print("  distill loss", out["ds_loss"], "render Q", st.total_queries)


def gen_brute():
    """scene.render_brute_force (scene.py:214-252) and analytically_empty_cells
    (scene.py:186-211) through the reference."""
    out = {}
    for tag, sc, size, ns, seed in (("toy", scene.standard_toy_scene(), 24, 96, 3),
                                    ("spec", scene.specular_toy_scene(), 20, 64, 4),
                                    ("rand", scene.random_toy_scene(7), 16, 40, 5)):
        cam = scene.sphere_cameras(sc.aabb, 1, size, seed=seed)[0]
        out[f"{tag}_img"] = scene.render_brute_force(sc, cam, ns, background=(1.0, 0.5, 0.25))
        out.update({f"{k}_{tag}": v for k, v in cam_arrays(cam).items()})
        out[f"{tag}_ns"] = np.int64(ns)
    for tag, sc, res in (("toy", scene.standard_toy_scene(), (16, 16, 16)), ("rand", scene.random_toy_scene(7), (8, 5, 7))):
        out[f"empty_{tag}"] = scene.analytically_empty_cells(sc, res)
        out[f"empty_{tag}_res"] = np.array(res)
    save("brute", **out)


def main():
    what = sys.argv[1:] or ["rays", "pcg", "pointwise", "query", "render", "wide", "bulk", "scene", "ckpt", "extract",
                            "train", "c2", "generic", "brute"]
    for w in what:
        t = time.time()
        globals()[f"gen_{w}"]()
        print(f"[{w}] {time.time() - t:.1f}s")


if __name__ == "__main__":
    main()
