"""The training oracle (oracle/train_oracle.py) against the reference's own
outputs (tests/golden/train.npz): grouped_backward gradients, the photometric
loss and its gradients (plain / L2 / density noise), and Adam.  CPU only."""

import numpy as np
import pytest

from conftest import golden
from oracle import gridfield_oracle as O
from oracle import train_oracle as T

LAYERS = ("trunk0", "trunk1", "density", "feature", "direction", "color")


def _lattice(z, tag, res, width):
    lat = O.init_lattice(np.zeros(3), np.ones(3), res, seed=11, width=width)
    flat = z[f"{tag}_biases"]
    o = 0
    for k in lat.biases:
        n = lat.biases[k].size
        lat.biases[k][...] = flat[o : o + n].reshape(lat.biases[k].shape)
        o += n
    return lat


def _close(got, ref, rel=2e-5):
    ref = np.asarray(ref, np.float64)
    assert np.abs(np.asarray(got, np.float64) - ref).max() <= rel * max(np.abs(ref).max(), 1e-30)


@pytest.mark.parametrize("tag,width", [("g32", 32), ("g64", 64)])
def test_oracle_grouped_backward(tag, width):
    z = golden("train")
    lat = _lattice(z, tag, tuple(z[f"{tag}_res"]), width)
    _, _, gw, gb = T.grouped_forward_backward(lat, z[f"{tag}_pts"], z[f"{tag}_dirs"], z[f"{tag}_dcol"],
                                              z[f"{tag}_dsig"])
    for k in LAYERS:
        _close(gw[k], z[f"{tag}_w_{k}"])
        _close(gb[k], z[f"{tag}_b_{k}"])


def _photo_lattice():
    lat = O.init_lattice(np.zeros(3), np.ones(3), (2, 2, 2), seed=5)
    lat.biases["density"][:] = 1.5
    return lat


@pytest.mark.parametrize("tag", ["ph0", "ph_reg", "ph_noise"])
def test_oracle_photometric(tag):
    z = golden("train")
    kw = {"ph_reg": {"reg_weight": 1e-3}, "ph_noise": {"sigma_noise": z["ph_noise"]}}.get(tag, {})
    loss, gw, gb = T.photometric_loss_and_grads(_photo_lattice(), z["ph_pos"], z["ph_dirs"], z["ph_ray"],
                                                z["ph_slot"], z["ph_deltas"], int(z["ph_nrays"]), int(z["ph_k"]),
                                                z["ph_gt"], (1.0, 1.0, 1.0), **kw)
    assert loss == pytest.approx(float(z[f"{tag}_loss"]), rel=1e-9)
    for k in LAYERS:
        _close(gw[k], z[f"{tag}_w_{k}"])
        _close(gb[k], z[f"{tag}_b_{k}"])


def test_oracle_adam_bit_exact():
    z = golden("train")
    lat = _photo_lattice()
    arrays, grads = [], []
    for k in LAYERS:
        arrays += [lat.weights[k].copy(), lat.biases[k].copy()]
        grads += [z[f"ph0_w_{k}"], z[f"ph0_b_{k}"]]
    m = [np.zeros_like(a) for a in arrays]
    v = [np.zeros_like(a) for a in arrays]
    step = T.adam_update(arrays, grads, m, v, 0, 5e-4)
    T.adam_update(arrays, grads, m, v, step, 3e-4)
    for i, k in enumerate(LAYERS):
        assert np.array_equal(arrays[2 * i], z[f"adam_p_w_{k}"]) and np.array_equal(arrays[2 * i + 1], z[f"adam_p_b_{k}"])
        assert np.array_equal(m[2 * i], z[f"adam_m_w_{k}"]) and np.array_equal(v[2 * i], z[f"adam_v_w_{k}"])
