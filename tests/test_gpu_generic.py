"""Manifests beyond the fused tiny-MLP kernels (mlp.py:30-109) on the device:
the generic fp32 kernel (csrc/gf_mlp_generic.cu) against the reference.

Fixtures: tests/golden/generic.npz (tests/golden/make_golden.py gen_generic),
written by the reference: the default teacher (10 x 256, skip layer 5,
direction width 128) and the desk preset's teacher (6 x 96, skip 2, width
64) queried on random points, a traced-stats render of a (2,2,2) lattice of
5 x 48 skip-2 networks with 6/3 octaves, and one distill_step with
TrainConfig's default teacher (train.py:341-390).

Tolerances: float32; numpy's sgemm associates the 256-term dot products
differently from the device's sequential FMA chain, so outputs agree to
~1e-5 relative (bound: 2e-5 * max|ref| + 1e-4 * |ref|); render counts are
exact; one distill step moves parameters by at most ~lr, compared within
2e-6 absolute like tests/test_gpu_train.py.
"""

import numpy as np
import pytest

from conftest import golden, golden_camera, have_gpu

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not have_gpu(), reason="needs CUDA")]

LAYERS = ("trunk0", "trunk1", "density", "feature", "direction", "color")


def _gf():
    import paper_2103_13744_b200 as gf

    return gf


def _set_biases(g, flat):
    o = 0
    for k in g.params.biases:
        n = g.params.biases[k].size
        g.params.biases[k][...] = flat[o : o + n].reshape(g.params.biases[k].shape)
        o += n


def _close(got, ref, what, rel=1e-4, scale=2e-5):
    got, ref = np.asarray(got, np.float64), np.asarray(ref, np.float64)
    tol = scale * max(float(np.abs(ref).max()), 1e-30) + rel * np.abs(ref)
    err = np.abs(got - ref)
    assert np.all(err <= tol), f"{what}: max err {err.max():.3e}, max |ref| {np.abs(ref).max():.3e}"


@pytest.mark.parametrize("tag", ["teach", "desk"])
def test_teacher_query_matches_reference(tag):
    gf = _gf()
    from paper_2103_13744_b200 import train

    z = golden("generic")
    aabb = gf.Aabb((-1.0,) * 3, (1.0,) * 3)
    enc = gf.PositionalEncoding()
    arch = gf.teacher_architecture() if tag == "teach" else train.TrainConfig.desk_preset().teacher_architecture(enc)
    g = gf.init_network_grid(aabb, tuple(int(v) for v in z[f"{tag}_res"]), seed=23, arch=arch, encoding=enc)
    _set_biases(g, z[f"{tag}_biases"])
    assert not g.tensor_core_arch()
    rgb, sig = g.query_points(z[f"{tag}_pts"], z[f"{tag}_dirs"])
    _close(rgb, z[f"{tag}_rgb"], f"{tag} rgb")
    _close(sig, z[f"{tag}_sigma"], f"{tag} sigma")


def test_skip_layer_render_matches_reference():
    gf = _gf()
    z = golden("generic")
    aabb = gf.Aabb((-1.0,) * 3, (1.0,) * 3)
    enc = gf.PositionalEncoding(num_freqs_position=6, num_freqs_direction=3)
    arch = gf.MlpArchitecture(hidden_layers=5, hidden_width=48, position_input_dim=enc.position_dim,
                              direction_input_dim=enc.direction_dim, direction_layer_width=40, skip_layer=2)
    g = gf.init_network_grid(aabb, (2, 2, 2), seed=24, arch=arch, encoding=enc)
    g.params.biases["density"][:] = 4.0
    cam = golden_camera(z)
    img, st = gf.render_image(g, None, gf.Camera(cam.width, cam.height, cam.fx, cam.fy, cam.cx, cam.cy, cam.c2w),
                              gf.RenderConfig(k=64), seed=0)
    assert [st.total_queries, st.ess_skipped, st.ert_terminated_rays, st.n_rays] == list(z["rstats"])
    err = float(np.abs(img - z["rimg"]).max())
    assert err <= 2e-5, err


def test_distill_step_default_teacher_matches_reference():
    gf = _gf()
    from paper_2103_13744_b200 import train

    z = golden("generic")
    aabb = gf.Aabb((-1.0,) * 3, (1.0,) * 3)
    enc = gf.PositionalEncoding()
    cfg = train.TrainConfig(distill_points_per_cell=4)
    teacher = gf.init_network_grid(aabb, (1, 1, 1), seed=25, arch=cfg.teacher_architecture(enc), encoding=enc)
    student = gf.init_network_grid(aabb, (2, 2, 2), seed=26)
    st = train.AdamState.for_params(student.params)
    loss = train.distill_step(student, teacher, cfg, st, np.random.default_rng(27), delta_ref=0.01)
    assert abs(loss - float(z["ds_loss"][0])) <= 1e-4 * float(z["ds_loss"][0])
    for name in LAYERS:
        assert np.abs(student.params.weights[name] - z[f"ds_p_w_{name}"]).max() <= 2e-6, name
        assert np.abs(student.params.biases[name] - z[f"ds_p_b_{name}"]).max() <= 2e-6, name


def test_generic_grouped_backward_matches_reference_math():
    """grouped_backward of a skip-layer grid (no fused backward kernel) runs
    the dense device kernels per cell; the reference's batched.grouped_backward
    is mlp.backward per cell on the grouped rows (batched.py:154-187), checked
    here against the float64 device mlp.backward of the same rows."""
    gf = _gf()
    from paper_2103_13744_b200 import batched, mlp

    aabb = gf.Aabb((-1.0,) * 3, (1.0,) * 3)
    g = gf.init_network_grid(aabb, (2, 1, 1), seed=1, arch=gf.teacher_architecture(hidden_layers=5, hidden_width=64))
    rng = np.random.default_rng(2)
    pts = rng.uniform(-1, 1, (50, 3)).astype(np.float32)
    dirs = rng.normal(size=(50, 3)).astype(np.float32)
    dirs /= np.linalg.norm(dirs, axis=-1, keepdims=True)
    dc = rng.normal(size=(50, 3)).astype(np.float32)
    ds = rng.normal(size=50).astype(np.float32)
    layout = batched.group_by_network(batched.QueryBatch(pts, dirs, g.cell_index(pts)), g.n_cells)
    caches = []
    batched.grouped_forward(g, layout, caches=caches)
    grads = batched.grouped_backward(g, layout, caches, dc, ds)
    cells = g.cell_index(pts)
    for c in range(g.n_cells):
        m = cells == c
        x = g.encoding.encode_position(pts[m].astype(np.float64))
        d = g.encoding.encode_direction(dirs[m].astype(np.float64))
        ref = mlp.backward(g.params.at(c).astype(np.float64), x, d, dc[m].astype(np.float64), ds[m].astype(np.float64))
        for name in ref.weights:
            _close(grads.weights[name][c], ref.weights[name], f"cell {c} w {name}", rel=1e-3, scale=1e-4)
            _close(grads.biases[name][c], ref.biases[name], f"cell {c} b {name}", rel=1e-3, scale=1e-4)


def test_render_rays_float64_rays_match_reference():
    """render_rays with float64 rays float32 cannot represent (render.py:368):
    the device slab test runs on the float64 values, the samples on their
    float32 roundings, exactly as the reference (counts exact)."""
    gf = _gf()
    z = golden("generic")
    aabb = gf.Aabb((-1.0,) * 3, (1.0,) * 3)
    g = gf.init_network_grid(aabb, (16, 16, 16), seed=0)
    g.params.biases["density"][:] = 5.0
    o, d = z["f64_o"], z["f64_d"]
    assert not np.array_equal(o.astype(np.float32).astype(np.float64), o)
    rgb, st = gf.render_rays(g, None, o, d, gf.RenderConfig(k=64), seed=3, precision="fp32")
    assert [st.total_queries, st.ess_skipped, st.ert_terminated_rays, st.n_rays] == list(z["f64_stats"])
    assert float(np.abs(rgb - z["f64_rgb"]).max()) <= 2e-5
