"""CPU-side checks of the C-ABI library: it loads, exports every symbol the
header declares, and its host-only helpers agree with numpy / the oracle."""

import re
from pathlib import Path

import numpy as np
import pytest

from conftest import ROOT, golden
from oracle import seedseq

HEADER = ROOT / "include" / "gridfield_b200.h"


def declared_symbols():
    text = HEADER.read_text()
    return sorted(set(re.findall(r"^GF_API\s+[\w\s\*]+?\b(gf_\w+)\s*\(", text, flags=re.M)))


@pytest.fixture(scope="module")
def native():
    from paper_2103_13744_b200 import _native as N

    if not N.LIB_PATH.exists():
        pytest.fail(f"{N.LIB_PATH} missing: run __graft_entry__.build()")
    return N


def test_library_exports_every_declared_symbol(native):
    lib = native.lib()
    syms = declared_symbols()
    assert len(syms) >= 20
    missing = [s for s in syms if not hasattr(lib, s)]
    assert not missing, missing
    # and the Python binding covers exactly the declared surface
    assert sorted(native.EXPORTED) == syms


def test_abi_version(native):
    assert native.lib().gf_abi_version() == native.ABI_VERSION == 2


def test_pcg64_block_state_matches_numpy_golden(native):
    z = golden("pcg64")
    for (a, b), st in zip(z["entropy"], z["state"]):
        state, inc = native.pcg64_block_state(int(a), int(b))
        assert state == (int(st[0]) << 64) | int(st[1])
        assert inc == (int(st[2]) << 64) | int(st[3])
        assert (state, inc) == seedseq.pcg64_seed([int(a), int(b)])


def test_param_count_and_packed_sizes(native):
    import paper_2103_13744_b200 as gf

    for width in (32, 64):
        arch = gf.MlpArchitecture(hidden_width=width)
        a = native.make_arch(arch, gf.PositionalEncoding())
        assert native.lib().gf_param_count(a) == arch.parameter_count()
        assert native.lib().gf_packed_bytes(a, 4096, 0) >= 4 * arch.parameter_count() * 4096


def test_workspace_sizes_are_positive(native):
    import paper_2103_13744_b200 as gf

    g = native.make_geom(gf.Aabb((-1,) * 3, (1,) * 3), (16, 16, 16))
    a = native.make_arch(gf.MlpArchitecture(), gf.PositionalEncoding())
    cfg = gf.RenderConfig().native(0)
    assert native.lib().gf_render_workspace_bytes(a, g, cfg, 640_000) > 640_000 * 32 * 32
    assert native.lib().gf_query_workspace_bytes(a, g, 1 << 20) > (1 << 20) * 8
    assert native.lib().gf_group_workspace_bytes(100_000, 4096) > 0


def test_invalid_arguments_fail_loudly(native):
    import paper_2103_13744_b200 as gf

    bad = native.make_arch(gf.MlpArchitecture(), gf.PositionalEncoding())
    bad.hidden_layers = 2
    st = native.lib().gf_pack_weights(bad, 1, None, None, None, 0, None)
    assert st == native.GF_ERR_INVALID
    assert b"architecture" in native.lib().gf_last_error()


def test_render_config_native_eps_semantics():
    import paper_2103_13744_b200 as gf

    assert gf.RenderConfig().native(0).eps_compare_f64 == 0  # Python float -> float32 compare (NEP 50)
    assert gf.RenderConfig(epsilon=np.float64(0.01)).native(0).eps_compare_f64 == 1
    with pytest.raises(ValueError):
        gf.RenderConfig(k=0)
    with pytest.raises(ValueError):
        gf.RenderConfig(epsilon=1.0)


def test_host_value_types_match_reference_contracts():
    import paper_2103_13744_b200 as gf

    with pytest.raises(ValueError, match="orthonormal"):
        bad = np.eye(4)
        bad[0, 0] = 1.5
        gf.Camera(8, 8, 8, 8, 4, 4, bad)
    with pytest.raises(ValueError):
        gf.Aabb((0, 0, 0), (1, 0.5, 0))
    assert gf.count_flops(gf.MlpArchitecture()) == 12392
    assert gf.MlpArchitecture().parameter_count() == 6212


def test_tracked_params_bump_version_on_in_place_edit():
    import paper_2103_13744_b200 as gf

    grid = gf.init_network_grid(gf.Aabb((-1,) * 3, (1,) * 3), (2, 2, 2), seed=0)
    fp0 = grid.params.fingerprint()
    grid.params.biases["density"][:] = 20.0
    fp1 = grid.params.fingerprint()
    assert fp0 != fp1
    grid.params.weights["trunk0"][0] *= 2
    assert grid.params.fingerprint() != fp1
    single = grid.params.at(0).copy()
    for k in grid.params.weights:
        grid.params.weights[k][:] = single.weights[k]
    assert grid.params.fingerprint() != fp1


def test_init_params_identical_to_oracle():
    import paper_2103_13744_b200 as gf
    from oracle import gridfield_oracle as O

    grid = gf.init_network_grid(gf.Aabb((-1,) * 3, (1,) * 3), (16, 16, 16), seed=3)
    lat = O.init_lattice(np.full(3, -1.0), np.ones(3), (16, 16, 16), seed=3)
    for k in lat.weights:
        assert np.array_equal(np.asarray(grid.params.weights[k]), lat.weights[k])
    assert float(np.asarray(grid.params.weights["trunk0"], np.float64).sum()) == float(golden("query16")["w0_checksum"])


def test_sphere_cameras_match_golden():
    import paper_2103_13744_b200 as gf

    z = golden("rays")
    cams = gf.sphere_cameras(gf.Aabb((-1,) * 3, (1,) * 3), 3, 96, seed=0)
    for i, c in enumerate(cams):
        assert np.array_equal(c.c2w, z[f"cam_c2w_{i}"])
        assert np.array_equal([c.fx, c.fy, c.cx, c.cy], z[f"cam_f_{i}"])


def test_no_oracle_import_in_product():
    pkg = ROOT / "paper_2103_13744_b200"
    for f in pkg.rglob("*.py"):
        text = f.read_text()
        assert "import oracle" not in text and "from oracle" not in text, f


@pytest.mark.parametrize("pre,draws", [(0, 0), (0, 1), (0, 7), (1, 6), (3, 1000), (2, 3073)])
def test_generator_advance_matches_numpy(pre, draws):
    """train._advance_float32_draws leaves a numpy PCG64 Generator exactly
    where rng.random(draws, float32) would (buffered 32-bit half included):
    the host half of the device sample preparation (train.py:186)."""
    from paper_2103_13744_b200 import train

    a, b = np.random.default_rng(5), np.random.default_rng(5)
    for r in (a, b):
        r.random(pre, dtype=np.float32)
    a.random(draws, dtype=np.float32)
    bg, st = train._pcg_state(b)
    train._advance_float32_draws(bg, st, draws)
    assert a.bit_generator.state == b.bit_generator.state
    assert np.array_equal(a.random(9, dtype=np.float32), b.random(9, dtype=np.float32))
    assert a.random() == b.random()


def test_pcg_output_function_matches_numpy():
    """train._xsl_rr is numpy's PCG64 output: one raw 64-bit draw."""
    from paper_2103_13744_b200 import train

    rng = np.random.default_rng(11)
    st = rng.bit_generator.state["state"]
    s, inc = st["state"], st["inc"]
    mult = 0x2360ED051FC65DA44385DF649FCCF645
    s1 = (s * mult + inc) % (1 << 128)
    assert train._xsl_rr(s1) == int(rng.integers(0, 2**64, dtype=np.uint64, endpoint=False))
