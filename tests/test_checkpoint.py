"""Checkpoints: the reference's own file format, byte for
byte, and the device packer fed straight from the file's payload.

Fixture: tests/golden/ckpt_small.gfckpt, written by the reference's
io.save_checkpoint (make_golden.py gen_ckpt).
"""

from pathlib import Path

import numpy as np
import pytest

from conftest import have_gpu
from oracle import gridfield_oracle as O

FIX = Path(__file__).resolve().parent / "golden" / "ckpt_small.gfckpt"
UNIT_MIN, UNIT_MAX = np.full(3, -1.0), np.ones(3)


def test_load_reference_checkpoint_and_resave_byte_identical(tmp_path):
    from paper_2103_13744_b200 import io

    grid, occ = io.load_checkpoint(FIX)
    lat = O.init_lattice(UNIT_MIN, UNIT_MAX, (2, 3, 4), seed=9)
    lat.biases["density"][:] = 5.0
    for name in lat.weights:
        assert np.array_equal(np.asarray(grid.params.weights[name]), lat.weights[name])
        assert np.array_equal(np.asarray(grid.params.biases[name]), lat.biases[name])
    assert np.array_equal(occ.to_bool_array(), np.arange(512) % 3 != 0)
    out = tmp_path / "again.gfckpt"
    io.save_checkpoint(out, grid, occ)
    assert out.read_bytes() == FIX.read_bytes()


def test_checkpoint_errors(tmp_path):
    from paper_2103_13744_b200 import io

    bad = tmp_path / "bad.gfckpt"
    bad.write_bytes(b"NOTACKPT" + FIX.read_bytes()[8:])
    with pytest.raises(ValueError, match="bad magic"):
        io.load_checkpoint(bad)
    short = tmp_path / "short.gfckpt"
    short.write_bytes(FIX.read_bytes()[:-7])
    with pytest.raises(ValueError, match="payload length"):
        io.load_checkpoint(short)


@pytest.mark.gpu
@pytest.mark.skipif(not have_gpu(), reason="needs a CUDA device")
@pytest.mark.parametrize("precision", ["fp16", "fp32"])
def test_payload_packing_matches_layer_packing(precision):
    """gf_pack_weights_flat over the file's parameter block == the per-layer
    packer; an in-place edit afterwards falls back to the per-layer path."""
    import torch

    from paper_2103_13744_b200 import io

    grid, occ = io.load_checkpoint(FIX)
    from_file = grid.device_params(precision).clone()
    grid._payload = None
    grid._cache.clear()
    from_layers = grid.device_params(precision)
    assert torch.equal(from_file, from_layers)
    grid2, _ = io.load_checkpoint(FIX)
    grid2.params.biases["density"][:] = 7.0  # tracked in-place edit: payload is stale now
    p2 = grid2.device_params(precision)
    assert not torch.equal(p2, from_layers)
    cam = __import__("paper_2103_13744_b200").sphere_cameras(grid.aabb, 1, 24, seed=1)[0]
    import paper_2103_13744_b200 as gf

    a, sa = gf.render_image(grid, occ, cam, gf.RenderConfig(k=48), precision=precision)
    g3, o3 = io.load_checkpoint(FIX)
    b, sb = gf.render_image(g3, o3, cam, gf.RenderConfig(k=48), precision=precision)
    assert np.array_equal(a, b) and sa.total_queries == sb.total_queries
