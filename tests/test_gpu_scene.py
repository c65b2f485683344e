"""Analytic scenes on the device against the reference's own
fixtures (tests/golden/make_golden.py gen_scene) and the reference's
acceptance criteria (test_acceptance.py:140-171, test_render.py:237-255).

Bars: densities and every sample count bit-exact (the field is float32
arithmetic evaluated in numpy's order); colours within 1e-6 (the texture uses
sinf vs numpy's SIMD sin, the view tint a 3-term dot vs BLAS); images 1e-5.
"""

import numpy as np
import pytest

from conftest import golden, golden_camera, have_gpu

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not have_gpu(), reason="needs a CUDA device")]


@pytest.fixture(scope="module")
def gf():
    import paper_2103_13744_b200 as m

    return m


def _camera(gf, z):
    c = golden_camera(z)
    return gf.Camera(c.width, c.height, c.fx, c.fy, c.cx, c.cy, c.c2w)


def _cfg(gf, z):
    return gf.RenderConfig(k=int(z["k"]), epsilon=float(z["epsilon"]), background=tuple(z["background"]),
                           ert_chunk=int(z["ert_chunk"]), stratified=bool(z["stratified"]))


def test_scene_query_vs_reference(gf):
    z = golden("query_scene")
    for tag, sc in (("std", gf.standard_toy_scene()), ("spec", gf.specular_toy_scene()),
                    ("rand", gf.random_toy_scene(4, 7))):
        rgb, sig = sc.query_points(z["pts"], z["dirs"])
        assert np.array_equal(sig, z[f"{tag}_sigma"]), tag  # bit-exact densities
        assert np.max(np.abs(rgb - z[f"{tag}_rgb"])) <= 1e-6, tag


@pytest.mark.parametrize("name", ["render_scene_ert", "render_scene_dense", "render_scene_ess", "render_scene_specular"])
def test_scene_render_vs_reference(gf, name):
    z = golden(name)
    sc = gf.specular_toy_scene() if "specular" in name else gf.standard_toy_scene()
    occ = gf.OccupancyGrid(sc.aabb, z["occ_res"], z["occ_bits"].copy()) if "occ_bits" in z else None
    img, st = gf.render_image(sc, occ, _camera(gf, z), _cfg(gf, z), seed=int(z["seed"]))
    assert st.total_queries == int(z["total_queries"])
    assert st.ess_skipped == int(z["ess_skipped"])
    assert st.ert_terminated_rays == int(z["ert_terminated_rays"])
    assert np.max(np.abs(img - z["image"])) <= 1e-5


def test_occupancy_extraction_of_scene_matches_reference(gf):
    """extract_occupancy(scene.density_at, ...) with the device field gives
    the reference's bitmap exactly (occupancy.py:94-128, tau = 0)."""
    z = golden("render_scene_ess")
    sc = gf.standard_toy_scene()
    occ = gf.extract_occupancy(sc.density_at, sc.aabb, (32, 32, 32), tau=0.0)
    assert np.array_equal(np.asarray(occ.bits), z["occ_bits"])


def test_ess_exactness_acceptance(gf):
    """test_acceptance.py:157-171 criterion (dev <= 1e-5) at 128x128, K=384:
    on the device, skipped samples have zero density, so dense and skipped
    renders agree bit for bit while the skipped render queries less."""
    sc = gf.standard_toy_scene()
    occ = gf.extract_occupancy(sc.density_at, sc.aabb, (64, 64, 64), tau=0.0)
    cam = gf.sphere_cameras(sc.aabb, 1, 128, seed=4)[0]
    cfg = gf.RenderConfig(k=384, epsilon=0.0, stratified=False)
    dense, s_dense = gf.render_image(sc, None, cam, cfg)
    skipped, s_skip = gf.render_image(sc, occ, cam, cfg)
    assert np.array_equal(dense, skipped)
    assert s_skip.total_queries < s_dense.total_queries and s_skip.ess_skipped > 0


def test_ert_bound_acceptance(gf):
    """test_acceptance.py:141-154 criterion: epsilon = 0.01 moves no pixel by
    more than 0.01 relative to no termination, and rays do terminate."""
    sc = gf.standard_toy_scene()
    occ = gf.extract_occupancy(sc.density_at, sc.aabb, (64, 64, 64), tau=10.0)
    cam = gf.sphere_cameras(sc.aabb, 1, 128, seed=3)[0]
    cfg = gf.RenderConfig(k=384, stratified=False)
    off, _ = gf.render_image(sc, occ, cam, cfg.replace(epsilon=0.0))
    on, st = gf.render_image(sc, occ, cam, cfg.replace(epsilon=0.01))
    assert float(np.abs(on - off).max()) <= 0.01
    assert st.ert_terminated_rays > 0


def test_scene_render_shards_bit_identical(gf):
    """Analytic scenes keep the marcher's shard invariance."""
    sc = gf.specular_toy_scene()
    cam = gf.sphere_cameras(sc.aabb, 1, 80, seed=6)[0]
    cfg = gf.RenderConfig(k=64)
    full, st, _ = gf.render.render_rays_device(sc, None, cfg, 3, cam=cam)
    n = cam.width * cam.height
    a, sa, _ = gf.render.render_rays_device(sc, None, cfg, 3, cam=cam, ray_offset=0, n_rays=4096)
    b, sb, _ = gf.render.render_rays_device(sc, None, cfg, 3, cam=cam, ray_offset=4096, n_rays=n - 4096)
    import torch

    assert torch.equal(torch.cat([a, b]), full)
    assert int(sa[0] + sb[0]) == int(st[0])


class _DuckField:
    """A caller-evaluated field (render.py:361-364 protocol: aabb +
    query_points) wrapping an AnalyticScene: the device marches, the field is
    called once per round group (gf_render_rays_field)."""

    def __init__(self, scene):
        self.scene = scene
        self.aabb = scene.aabb
        self.calls = 0

    def query_points(self, positions, directions):
        self.calls += 1
        return self.scene.query_points(positions, directions)


@pytest.mark.parametrize("stratified,eps", [(True, 0.01), (False, 0.0)])
def test_caller_evaluated_field_matches_builtin(gf, stratified, eps):
    """Any field object renders through the device marcher: same samples,
    counters and (the field being the same function) the same image as the
    built-in AnalyticScene path."""
    sc = gf.standard_toy_scene()
    occ = gf.extract_occupancy(sc.density_at, sc.aabb, (32, 32, 32), tau=10.0)
    cam = gf.sphere_cameras(sc.aabb, 1, 40, seed=3)[0]
    cfg = gf.RenderConfig(k=96, epsilon=eps, stratified=stratified)
    ref, st_ref = gf.render_image(sc, occ, cam, cfg, seed=5)
    duck = _DuckField(sc)
    img, st = gf.render_image(duck, occ, cam, cfg, seed=5)
    assert duck.calls > 0
    assert (st.total_queries, st.ess_skipped, st.ert_terminated_rays) == (
        st_ref.total_queries, st_ref.ess_skipped, st_ref.ert_terminated_rays)
    assert np.array_equal(img, ref)


def test_caller_field_errors_propagate(gf):
    class Bad:
        aabb = gf.Aabb((-1.0,) * 3, (1.0,) * 3)

        def query_points(self, p, d):
            raise RuntimeError("field exploded")

    cam = gf.sphere_cameras(Bad.aabb, 1, 8, seed=0)[0]
    with pytest.raises(RuntimeError, match="field exploded"):
        gf.render_image(Bad(), None, cam, gf.RenderConfig(k=16))


@pytest.mark.parametrize("tag,which", [("toy", "standard"), ("spec", "specular"), ("rand", "random")])
def test_brute_force_quadrature_matches_reference(gf, tag, which):
    """scene.render_brute_force (scene.py:214-252) on the device against the
    reference's own images (tests/golden/brute.npz): float64 placement,
    float32 field and Simpson depth, sequential compositing; the field's
    colours are ~1 ulp from numpy's SIMD sin, so images agree to 2e-6."""
    from paper_2103_13744_b200 import scene as S

    z = golden("brute")
    sc = {"standard": gf.standard_toy_scene, "specular": gf.specular_toy_scene,
          "random": lambda: gf.random_toy_scene(7)}[which]()
    cam = golden_camera(z, f"_{tag}")
    cam = gf.Camera(cam.width, cam.height, cam.fx, cam.fy, cam.cx, cam.cy, cam.c2w)
    img = S.render_brute_force(sc, cam, int(z[f"{tag}_ns"]), background=(1.0, 0.5, 0.25))
    err = float(np.abs(img - z[f"{tag}_img"]).max())
    assert err <= 2e-6, err


def test_analytically_empty_cells_match_reference(gf):
    from paper_2103_13744_b200 import scene as S

    z = golden("brute")
    for tag, sc in (("toy", gf.standard_toy_scene()), ("rand", gf.random_toy_scene(7))):
        got = S.analytically_empty_cells(sc, tuple(int(v) for v in z[f"empty_{tag}_res"]))
        assert np.array_equal(got, z[f"empty_{tag}"]), tag


def test_brute_force_quadrature_converges(gf):
    """test_scene_io.py:87-92 (the reference's own criterion): 4x384 and
    8x384 segments agree within 1e-3 on a 64x64 view."""
    from paper_2103_13744_b200 import scene as S

    sc = gf.standard_toy_scene()
    cam = gf.sphere_cameras(sc.aabb, 1, 64, seed=3)[0]
    a = S.render_brute_force(sc, cam, 4 * 384)
    b = S.render_brute_force(sc, cam, 8 * 384)
    assert float(np.abs(a - b).max()) <= 1e-3
