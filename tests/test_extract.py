"""Occupancy extraction (occupancy.py:94-128).

CPU: the oracle restatement reproduces the reference's bitmaps
(tests/golden/extract.npz, made by tests/golden/make_golden.py gen_extract) and
numpy's threshold semantics.  GPU: gf_extract_occupancy_analytic is bit-exact
against the reference (including the 256^3 toy-scene bitmap the C2 bench uses),
gf_extract_occupancy_network matches outside the cells whose probes sit within
the stated margin of tau, and the out-of-bounds error carries the reference's
message.
"""

import numpy as np
import pytest

from conftest import golden, have_gpu, toy_occupancy_bits
from oracle import analytic as OA
from oracle import gridfield_oracle as O

CASES = ("toy64", "rand48", "spec_box", "toy_tau_f64")
MARGIN = 5e-3  # |sigma - tau| below which a network-probe cell may flip (fp16 query tolerance 2e-3)


def _tau(z, tag):
    t = float(z[f"{tag}_tau"])
    return np.float64(t) if bool(z[f"{tag}_tau_is_f64"]) else t


def _oracle_scene(tag):
    return {"toy64": OA.standard_scene, "toy_tau_f64": OA.standard_scene, "spec_box": OA.specular_scene,
            "rand48": lambda: OA.random_scene(11, 6)}[tag]()


def _unpack(bits, n):
    return np.unpackbits(np.asarray(bits), count=n, bitorder="little").astype(bool)


@pytest.mark.parametrize("tag", CASES)
def test_oracle_extract_analytic_matches_reference(tag):
    z = golden("extract")
    sc = _oracle_scene(tag)
    box, res = z[f"{tag}_box"], z[f"{tag}_res"]
    bits = O.extract_occupancy(lambda p: OA.scene_query(sc, p, np.zeros_like(p))[1], box[0], box[1], res,
                               _tau(z, tag))
    assert np.array_equal(bits, z[f"{tag}_bits"])


def test_oracle_extract_network_matches_reference():
    z = golden("extract")
    lat = O.init_lattice(np.full(3, -1.0), np.full(3, 1.0), tuple(z["net_grid_res"]), seed=int(z["net_seed"]))
    lat.biases["density"][:] = z["net_bias"]
    res, box = z["net_res"], z["net_box"]
    n = int(np.prod(res))

    def field(p):
        return O.query_points(lat, p, np.broadcast_to(np.float32([0, 0, 1]), p.shape))[1]

    for key, near_key, tau in (("net_bits", "net_near", float(z["net_tau"])), ("net_tau0_bits", "net_near0", 0.0)):
        got = _unpack(O.extract_occupancy(field, box[0], box[1], res, tau), n)
        ref, near = _unpack(z[key], n), _unpack(z[near_key], n)
        assert np.array_equal(got[~near], ref[~near])


def test_density_threshold_semantics():
    from paper_2103_13744_b200.occupancy import density_threshold

    s = np.float32(10.000000953674316)
    # numpy: float32 densities vs a Python float compare in float32 (NEP 50) ...
    assert not (np.array([s]) > 10.0000009)[0]
    assert not float(s) > density_threshold(10.0000009)
    # ... and vs a float64 scalar in float64
    assert (np.array([s]) > np.float64(10.0000009))[0]
    assert float(s) > density_threshold(np.float64(10.0000009))
    assert density_threshold(10) == 10.0 and density_threshold(np.float32(0.1)) == float(np.float32(0.1))


def test_probe_points_layout():
    pts = O.probe_points([0.0, 0.0, 0.0], [1.0, 1.0, 1.0], (2, 2, 2))
    assert pts.shape == (8 * 27, 3) and pts.dtype == np.float32
    # cell 1 = (ix=1, iy=0, iz=0); probe 9a+3b+c has offsets (o[a], o[b], o[c])
    assert np.array_equal(pts[27 * 1 + 9 * 2 + 3 * 1 + 0], np.float32([1.0, 0.25, 0.0]))


# ----------------------------------------------------------------------------- GPU


def _gf():
    import paper_2103_13744_b200 as gf

    return gf


def _scene(gf, tag):
    if tag in ("toy64", "toy_tau_f64"):
        return gf.standard_toy_scene()
    if tag == "spec_box":
        return gf.specular_toy_scene()
    return gf.random_toy_scene(11, 6)


@pytest.mark.gpu
@pytest.mark.skipif(not have_gpu(), reason="needs CUDA")
@pytest.mark.parametrize("tag", CASES)
def test_device_extract_analytic_bit_exact(tag):
    gf = _gf()
    z = golden("extract")
    box = z[f"{tag}_box"]
    sc = _scene(gf, tag)
    occ = gf.extract_occupancy(sc.density_at, gf.Aabb(tuple(box[0]), tuple(box[1])), z[f"{tag}_res"], tau=_tau(z, tag))
    assert np.array_equal(np.asarray(occ.bits), z[f"{tag}_bits"])


@pytest.mark.gpu
@pytest.mark.skipif(not have_gpu(), reason="needs CUDA")
def test_device_extract_toy_256_bit_exact_and_renders():
    """The C2 bench bitmap (reference: 453 M probes, 6.7 s on 8 cores) on the device."""
    gf = _gf()
    res, bits = toy_occupancy_bits()
    sc = gf.standard_toy_scene()
    occ = gf.extract_occupancy(sc.density_at, sc.aabb, tuple(res), tau=10.0)
    assert np.array_equal(np.asarray(occ.bits), bits)
    # the extracted bitmap is adopted by the device cache and renders like the fixture's
    grid = gf.init_network_grid(sc.aabb, (16, 16, 16), seed=0)
    cam = gf.sphere_cameras(sc.aabb, 1, 40, seed=1)[0]
    a, sa = gf.render_image(grid, occ, cam, gf.RenderConfig(k=96), seed=0)
    b, sb = gf.render_image(grid, gf.OccupancyGrid(sc.aabb, res, bits.copy()), cam, gf.RenderConfig(k=96), seed=0)
    assert np.array_equal(a, b)
    assert (sa.total_queries, sa.ess_skipped, sa.ert_terminated_rays) == (sb.total_queries, sb.ess_skipped,
                                                                          sb.ert_terminated_rays)
    assert sa.total_queries > 0


def _net_grid(gf, z, precision):
    g = gf.init_network_grid(gf.Aabb((-1.0,) * 3, (1.0,) * 3), tuple(z["net_grid_res"]), seed=int(z["net_seed"]),
                             precision=precision)
    g.params.biases["density"][:] = z["net_bias"]
    return g


@pytest.mark.gpu
@pytest.mark.skipif(not have_gpu(), reason="needs CUDA")
@pytest.mark.parametrize("precision", ["fp32", "fp16"])
def test_device_extract_network_probe(precision):
    from paper_2103_13744_b200 import train

    gf = _gf()
    z = golden("extract")
    g = _net_grid(gf, z, precision)
    res, box = z["net_res"], z["net_box"]
    n = int(np.prod(res))
    aabb = gf.Aabb(tuple(box[0]), tuple(box[1]))
    for key, near_key, tau in (("net_bits", "net_near", float(z["net_tau"])), ("net_tau0_bits", "net_near0", 0.0)):
        occ = gf.extract_occupancy(train.density_probe(g), aabb, res, tau=tau)
        got, ref, near = _unpack(occ.bits, n), _unpack(z[key], n), _unpack(z[near_key], n)
        assert np.array_equal(got[~near], ref[~near]), (precision, key, int((got != ref)[~near].sum()))
    # a generic callable (host chunks through query_points) gives the same bitmap
    probe = train.density_probe(g)
    via_host = gf.extract_occupancy(lambda p: probe(p), aabb, res, tau=float(z["net_tau"]))
    dev = gf.extract_occupancy(probe, aabb, res, tau=float(z["net_tau"]))
    assert np.array_equal(np.asarray(via_host.bits), np.asarray(dev.bits))


@pytest.mark.gpu
@pytest.mark.skipif(not have_gpu(), reason="needs CUDA")
def test_device_extract_network_out_of_bounds_message():
    from paper_2103_13744_b200 import train

    gf = _gf()
    z = golden("extract")
    g = _net_grid(gf, z, "fp32")
    with pytest.raises(ValueError) as e:
        gf.extract_occupancy(train.density_probe(g), gf.Aabb((-1.0, -1.0, -1.0), (1.0, 1.25, 1.0)), (8, 8, 8), tau=1.0)
    assert str(e.value) == str(z["net_oob_message"])


@pytest.mark.gpu
@pytest.mark.skipif(not have_gpu(), reason="needs CUDA")
def test_device_extract_reference_edge_cases():
    """test_occupancy.py:20-57 through the device field: strict threshold,
    all-empty / all-occupied, tau validation, resolution cap."""
    gf = _gf()
    unit = gf.Aabb((0.0,) * 3, (1.0,) * 3)
    flat = gf.AnalyticScene(unit, boxes=[gf.Box((-1.0,) * 3, (2.0,) * 3, (1.0, 1.0, 1.0), 10.0, feather=0.0)])
    assert not gf.extract_occupancy(flat.density_at, unit, (4, 4, 4), tau=10.0).to_bool_array().any()
    assert gf.extract_occupancy(flat.density_at, unit, (4, 5, 3), tau=9.5).to_bool_array().all()
    empty = gf.AnalyticScene(unit)
    assert not gf.extract_occupancy(empty.density_at, unit, (7, 3, 5), tau=0.0).to_bool_array().any()
    with pytest.raises(ValueError, match="non-negative"):
        gf.extract_occupancy(flat.density_at, unit, (4, 4, 4), tau=-1.0)
    with pytest.raises(ValueError, match="capped"):
        gf.extract_occupancy(flat.density_at, unit, (257, 4, 4), tau=1.0)
