"""Training kernels on the device against the reference.

Fixtures: tests/golden/train.npz, written by the reference itself
(tests/golden/make_golden.py gen_train): batched.grouped_backward on random
upstream gradients (32- and 64-wide lattices), train.photometric_loss_and_grads
on the reference test's fixed batch (plain / L2-regularised / density noise),
two adam_update steps, and one distill_step.

Tolerances (float32 throughout; numpy's sgemm and pairwise sums associate
differently from the device's fixed-order sums):
* gradients: |got - ref| <= 2e-4 * max|ref| + 1e-4 * |ref|, per layer;
* losses: relative 1e-5;
* Adam on the reference's own gradients: bit-exact (elementwise float32 in
  numpy's operation order);
* one distill step: parameters within 2e-6 absolute (lr = 5e-4 moves each by
  at most ~lr).
"""

import numpy as np
import pytest

from conftest import golden, have_gpu

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not have_gpu(), reason="needs CUDA")]

LAYERS = ("trunk0", "trunk1", "density", "feature", "direction", "color")


def _gf():
    import paper_2103_13744_b200 as gf

    return gf


def _close(got, ref, what, rel=1e-4, scale=2e-4):
    got, ref = np.asarray(got, np.float64), np.asarray(ref, np.float64)
    tol = scale * max(float(np.abs(ref).max()), 1e-30) + rel * np.abs(ref)
    err = np.abs(got - ref)
    assert np.all(err <= tol), f"{what}: max err {err.max():.3e}, max |ref| {np.abs(ref).max():.3e}"


def _check_grads(grads, z, prefix):
    for name in LAYERS:
        _close(grads.weights[name], z[f"{prefix}w_{name}"], f"{prefix}w_{name}")
        _close(grads.biases[name], z[f"{prefix}b_{name}"], f"{prefix}b_{name}")


@pytest.mark.parametrize("tag,width", [("g32", 32), ("g64", 64)])
def test_grouped_backward_matches_reference(tag, width):
    gf = _gf()
    z = golden("train")
    aabb = gf.Aabb((0.0,) * 3, (1.0,) * 3)
    arch = None if width == 32 else gf.MlpArchitecture(hidden_width=64)
    g = gf.init_network_grid(aabb, tuple(z[f"{tag}_res"]), seed=11, arch=arch)
    flat = z[f"{tag}_biases"]
    o = 0
    for k in g.params.biases:
        n = g.params.biases[k].size
        g.params.biases[k][...] = flat[o : o + n].reshape(g.params.biases[k].shape)
        o += n
    pts, dirs = z[f"{tag}_pts"], z[f"{tag}_dirs"]
    layout = gf.group_by_network(gf.QueryBatch(pts, dirs, g.cell_index(pts)), g.n_cells)
    caches = []
    gf.grouped_forward(g, layout, caches=caches)
    grads = gf.batched.grouped_backward(g, layout, caches, z[f"{tag}_dcol"], z[f"{tag}_dsig"])
    _check_grads(grads, z, f"{tag}_")


def _photo_setup(gf, z):
    from paper_2103_13744_b200 import train

    aabb = gf.Aabb((0.0,) * 3, (1.0,) * 3)
    g = gf.init_network_grid(aabb, (2, 2, 2), seed=5)
    g.params.biases["density"][:] = 1.5
    smp = train.RaySamples(z["ph_pos"], z["ph_dirs"], z["ph_ray"], z["ph_slot"], z["ph_deltas"], int(z["ph_nrays"]),
                           int(z["ph_k"]))
    return train, g, smp


@pytest.mark.parametrize("tag", ["ph0", "ph_reg", "ph_noise"])
def test_photometric_loss_and_grads_match_reference(tag):
    gf = _gf()
    z = golden("train")
    train, g, smp = _photo_setup(gf, z)
    kw = {"ph_reg": {"reg_weight": 1e-3}, "ph_noise": {"sigma_noise": z["ph_noise"]}}.get(tag, {})
    loss, grads = train.photometric_loss_and_grads(g, smp, z["ph_gt"], (1.0, 1.0, 1.0), **kw)
    assert abs(loss - float(z[f"{tag}_loss"])) <= 1e-5 * abs(float(z[f"{tag}_loss"]))
    _check_grads(grads, z, f"{tag}_")
    loss2, none = train.photometric_loss_and_grads(g, smp, z["ph_gt"], (1.0, 1.0, 1.0), want_grads=False, **kw)
    assert none is None and loss2 == loss


def test_adam_update_bit_exact_on_reference_gradients():
    gf = _gf()
    z = golden("train")
    train, g, _ = _photo_setup(gf, z)
    grads = gf.mlp.MlpParams(g.arch, {k: z[f"ph0_w_{k}"] for k in LAYERS}, {k: z[f"ph0_b_{k}"] for k in LAYERS})
    st = train.AdamState.for_params(g.params)
    p = g.params.copy()
    cfg = train.TrainConfig()
    train.adam_update(p, grads, st, 5e-4, cfg)
    train.adam_update(p, grads, st, 3e-4, cfg)
    for name in LAYERS:
        for pre, obj in (("adam_p_", p), ("adam_m_", st.m), ("adam_v_", st.v)):
            assert np.array_equal(obj.weights[name], z[f"{pre}w_{name}"]), (pre, name)
            assert np.array_equal(obj.biases[name], z[f"{pre}b_{name}"]), (pre, name)


def test_distill_step_matches_reference():
    gf = _gf()
    from paper_2103_13744_b200 import train

    z = golden("train")
    aabb = gf.Aabb((0.0,) * 3, (1.0,) * 3)
    enc = gf.PositionalEncoding()
    cfg = train.TrainConfig(distill_points_per_cell=8, teacher_hidden_layers=4, teacher_hidden_width=32,
                            teacher_direction_width=32, teacher_skip_layer=None)
    teacher = gf.init_network_grid(aabb, (1, 1, 1), seed=6, arch=cfg.teacher_architecture(enc), encoding=enc)
    student = gf.init_network_grid(aabb, (2, 2, 2), seed=7)
    st = train.AdamState.for_params(student.params)
    loss = train.distill_step(student, teacher, cfg, st, np.random.default_rng(3), delta_ref=0.01)
    assert abs(loss - float(z["ds_loss"][0])) <= 1e-5 * float(z["ds_loss"][0])
    for name in LAYERS:
        assert np.abs(student.params.weights[name] - z[f"ds_p_w_{name}"]).max() <= 2e-6, name
        assert np.abs(student.params.biases[name] - z[f"ds_p_b_{name}"]).max() <= 2e-6, name


def test_reference_training_semantics():
    """test_train.py: zero model -> loss 0 on background ground truth; the
    regulariser alone; gradients only reach cells that were sampled; the
    device path is deterministic."""
    gf = _gf()
    from paper_2103_13744_b200 import train

    z = golden("train")
    _, g, smp = _photo_setup(gf, z)
    for k in g.params.weights:
        g.params.weights[k][:] = 0
        g.params.biases[k][:] = 0
    gt = np.ones((int(z["ph_nrays"]), 3), np.float32)
    loss, grads = train.photometric_loss_and_grads(g, smp, gt, (1.0, 1.0, 1.0))
    assert loss == 0.0
    g.params.weights["color"][:] = 0.01
    reg, _ = train.regularization_term(g.params, 1e-6)
    loss2, _ = train.photometric_loss_and_grads(g, smp, gt, (1.0, 1.0, 1.0), reg_weight=1e-6)
    assert loss2 == pytest.approx(reg)
    # gradients land only in sampled cells
    _, g2, smp2 = _photo_setup(gf, z)
    cells = set(np.unique(g2.cell_index(smp2.positions)).tolist())
    _, gr = train.photometric_loss_and_grads(g2, smp2, z["ph_gt"], (1.0, 1.0, 1.0))
    for c in range(g2.n_cells):
        if c not in cells:
            assert not np.any(gr.weights["trunk0"][c])
    _, gr2 = train.photometric_loss_and_grads(g2, smp2, z["ph_gt"], (1.0, 1.0, 1.0))
    for name in LAYERS:
        assert np.array_equal(gr.weights[name], gr2.weights[name])


def test_overfit_fixed_batch_loss_drops():
    """test_train.py:123-135 on the device path."""
    gf = _gf()
    from paper_2103_13744_b200 import train

    z = golden("train")
    _, g, smp = _photo_setup(gf, z)
    state = train.AdamState.for_params(g.params)
    cfg = train.TrainConfig()
    losses = []
    for _ in range(50):
        loss, grads = train.photometric_loss_and_grads(g, smp, z["ph_gt"], (1, 1, 1))
        train.adam_update(g.params, grads, state, 5e-4, cfg)
        losses.append(loss)
    assert losses[-1] < losses[0]
    for i in range(0, 40, 10):
        assert losses[i + 10] < losses[i]


@pytest.mark.parametrize("tag", ["ph", "prep_occ", "prep_odd", "prep_mid"])
def test_prepare_ray_samples_bit_exact(tag):
    """train.prepare_ray_samples on the device: samples, order, deltas and the
    Generator state left behind are the reference's exactly."""
    gf = _gf()
    from paper_2103_13744_b200 import train

    z = golden("train")
    aabb = gf.Aabb((0.0,) * 3, (1.0,) * 3)
    if tag == "ph":  # test_train.py fixed_batch: rng draws the ray offsets, the jitter, then gt
        rng = np.random.default_rng(1)
        n = int(z["ph_nrays"])
        origins = np.tile(np.array([[-2.0, 0.0, 0.0]], np.float32), (n, 1))
        offs = rng.uniform(-0.6, 0.6, (n, 2)).astype(np.float32)
        dirs = np.concatenate([np.zeros((n, 1), np.float32), offs], axis=1) - origins
        dirs /= np.linalg.norm(dirs, axis=-1, keepdims=True)
        smp = train.prepare_ray_samples(origins, dirs, aabb, int(z["ph_k"]), True, rng)
        assert np.array_equal(rng.random((n, 3)).astype(np.float32), z["ph_gt"])
        ref = dict(pos=z["ph_pos"], dirs=z["ph_dirs"], ray=z["ph_ray"], slot=z["ph_slot"], deltas=z["ph_deltas"])
    else:
        rng = np.random.default_rng(17)
        if int(z[f"{tag}_pre"]):
            rng.random(int(z[f"{tag}_pre"]), dtype=np.float32)
        rng.uniform(-0.6, 0.6, (len(z[f"{tag}_o"]), 2))  # the offsets the fixture drew
        occ = None
        if tag == "prep_occ":
            occ = gf.OccupancyGrid.from_bool_array(aabb, (4, 1, 1), np.array([False, False, False, True]))
        smp = train.prepare_ray_samples(z[f"{tag}_o"], z[f"{tag}_d"], aabb, int(z[f"{tag}_k"]), tag != "prep_mid",
                                        rng, occ=occ)
        assert np.array_equal(rng.random(5, dtype=np.float32), z[f"{tag}_after"])
        ref = {key: z[f"{tag}_{key}"] for key in ("pos", "dirs", "ray", "slot", "deltas")}
    assert smp.positions.dtype == np.float64 and np.array_equal(smp.positions, ref["pos"])
    assert np.array_equal(smp.directions, ref["dirs"])
    assert np.array_equal(smp.ray_index, ref["ray"]) and np.array_equal(smp.slot, ref["slot"])
    assert np.array_equal(smp.deltas, ref["deltas"])


def test_photometric_step_matches_reference():
    """train.py:291-332 through the device: three steps on a tiny dataset with
    the caller's Generator driving view, pixels, jitter and density noise."""
    gf = _gf()
    from paper_2103_13744_b200 import train

    z = golden("train")
    aabb = gf.Aabb((0.0,) * 3, (1.0,) * 3)

    class DS:
        def __init__(self):
            self.aabb, self.cameras, self.images = aabb, gf.sphere_cameras(aabb, 3, 16, seed=1), z["step_images"]

        def indices(self, split):
            return [0, 1, 2] if split == "train" else [1]

    g = gf.init_network_grid(aabb, (2, 2, 2), seed=8)
    g.params.biases["density"][:] = 0.8
    cfg = train.TrainConfig(batch_size_pixels=32, k_train=16)
    st = train.AdamState.for_params(g.params)
    rng = np.random.default_rng(9)
    losses = [train.photometric_step(g, DS(), cfg, st, rng, lr=5e-4, noise_std=0.1 * i) for i in range(3)]
    np.testing.assert_allclose(losses, z["step_losses"], rtol=1e-5)
    assert np.array_equal(rng.random(4), z["step_after"])  # same draws consumed as the reference
    for name in LAYERS:
        assert np.abs(g.params.weights[name] - z[f"step_p_w_{name}"]).max() <= 5e-6, name
        assert np.abs(g.params.biases[name] - z[f"step_p_b_{name}"]).max() <= 5e-6, name
    assert train.mean_free_space_density(g, np.arange(0, 8, 3)) == pytest.approx(float(z["free_space"]), rel=1e-5)


@pytest.mark.parametrize("width", [32, 64])
def test_grouped_backward_chunking_edge_cases(width):
    """Cells with no rows (zero gradients); a crowded cell of 2316 rows = ten
    256-row chunks whose last tile holds 12 rows (more than 8 chunks: its
    chunk sums are split over parameter blocks; on the tensor-core path a
    tile of <= 16 rows has no second K sub-tile); a cell of 600 rows = three
    chunks; single-chunk cells of 1..40 rows (written in place); against the
    training oracle (batched.py:154-187, mlp.py:269-316)."""
    from oracle import gridfield_oracle as O
    from oracle import train_oracle as T

    gf = _gf()
    rng = np.random.default_rng(7)
    res = (4, 4, 4)
    aabb = gf.Aabb((0.0,) * 3, (1.0,) * 3)
    arch = None if width == 32 else gf.MlpArchitecture(hidden_width=64)
    g = gf.init_network_grid(aabb, res, seed=3, arch=arch)
    for k in g.params.biases:
        g.params.biases[k][...] = rng.normal(0.0, 0.3, g.params.biases[k].shape).astype(np.float32)
    pts = [rng.uniform(0.0, 0.25, (2316, 3)), rng.uniform(0.75, 1.0, (600, 3))]  # cells 0 and 63
    for c in range(1, 63, 3):  # every third cell; the rest stay empty
        ix, iy, iz = c % 4, (c // 4) % 4, c // 16
        n = 1 + (c * 7) % 40
        pts.append((np.array([ix, iy, iz]) + rng.uniform(0.05, 0.95, (n, 3))) / 4.0)
    pts = np.concatenate(pts).astype(np.float32)
    perm = rng.permutation(len(pts))
    pts = pts[perm]
    dirs = rng.normal(size=pts.shape).astype(np.float32)
    dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
    dcol = rng.normal(0.0, 1e-2, (len(pts), 3)).astype(np.float32)
    dsig = rng.normal(0.0, 1e-2, len(pts)).astype(np.float32)
    layout = gf.group_by_network(gf.QueryBatch(pts, dirs, g.cell_index(pts)), g.n_cells)
    caches = []
    gf.grouped_forward(g, layout, caches=caches)
    grads = gf.batched.grouped_backward(g, layout, caches, dcol, dsig)
    lat = O.init_lattice(np.zeros(3), np.ones(3), res, seed=3, width=width)
    for k in lat.weights:
        lat.weights[k][...] = g.params.weights[k]
        lat.biases[k][...] = g.params.biases[k]
    _, _, gw, gb = T.grouped_forward_backward(lat, pts, dirs, dcol, dsig)
    counts = np.bincount(g.cell_index(pts), minlength=g.n_cells)
    assert counts[0] == 2316 and counts[63] == 600 and (counts == 0).sum() > 30
    for name in LAYERS:
        _close(grads.weights[name], gw[name], name)
        _close(grads.biases[name], gb[name], name)
        assert not np.asarray(grads.weights[name])[counts == 0].any(), name


def test_backward_from_kept_activations_bit_identical():
    """The training forward's kept activations (gf_grouped_forward_act) feed
    the backward instead of its fp32 recompute: same operation order, so the
    gradients are bit-identical to the recomputing path, and the forward's
    colours / densities are those of the plain forward."""
    import dataclasses

    from paper_2103_13744_b200.batched import grouped_backward_device, grouped_forward_device

    gf = _gf()
    rng = np.random.default_rng(5)
    aabb = gf.Aabb((0.0,) * 3, (1.0,) * 3)
    g = gf.init_network_grid(aabb, (4, 4, 4), seed=9)
    for k in g.params.biases:
        g.params.biases[k][...] = rng.normal(0.0, 0.3, g.params.biases[k].shape).astype(np.float32)
    pts = rng.uniform(0.0, 1.0, (5000, 3)).astype(np.float32)
    pts[:700] *= 0.25  # one crowded cell: several chunks
    dirs = rng.normal(size=pts.shape).astype(np.float32)
    dirs /= np.linalg.norm(dirs, axis=1, keepdims=True)
    dcol = rng.normal(0.0, 1e-2, (len(pts), 3)).astype(np.float32)
    dsig = rng.normal(0.0, 1e-2, len(pts)).astype(np.float32)
    layout = gf.group_by_network(gf.QueryBatch(pts, dirs, g.cell_index(pts)), g.n_cells)
    kept = grouped_forward_device(g, layout, keep_activations=True)
    plain = grouped_forward_device(g, layout)
    assert kept.act is not None and plain.act is None
    assert np.array_equal(kept.rgb.cpu().numpy(), plain.rgb.cpu().numpy())
    assert np.array_equal(kept.sigma.cpu().numpy(), plain.sigma.cpu().numpy())
    _, _, f_act = grouped_backward_device(g, layout, kept, dcol, dsig)
    _, _, f_rec = grouped_backward_device(g, layout, dataclasses.replace(kept, act=None), dcol, dsig)
    assert np.array_equal(f_act.cpu().numpy(), f_rec.cpu().numpy())
