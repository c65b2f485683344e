"""Analytic test scenes on the device and synthetic camera rigs (mirror of
gridfield.scene, /root/reference/pkg/src/gridfield/scene.py).

``AnalyticScene`` keeps the reference's dataclass surface; its density and
colour are evaluated by the library (gf_query_analytic, csrc/gf_analytic.cu)
and ``render_image(scene, ...)`` marches it on the device
(gf_render_rays_analytic) -- SURVEY §8f item f1.  Toy dataset generation and
the brute-force quadrature renderer stay out of scope.
"""

from __future__ import annotations

from dataclasses import dataclass, field as dataclass_field

import numpy as np

from . import _device as D
from . import _native as N
from .core import Aabb
from .render import Camera, look_at_pose


@dataclass(frozen=True)
class Sphere:
    """scene.py:27-53: constant-colour ball, density feathered to zero at ``radius``."""

    center: tuple
    radius: float
    color: tuple
    density: float
    feather: float = 0.14


@dataclass(frozen=True)
class Box:
    """scene.py:56-74: axis-aligned slab with the same feathered edge."""

    lo: tuple
    hi: tuple
    color: tuple
    density: float
    feather: float = 0.14


@dataclass
class AnalyticScene:
    """scene.py:77-135: closed-form density/colour with compact support."""

    aabb: Aabb
    spheres: list = dataclass_field(default_factory=list)
    boxes: list = dataclass_field(default_factory=list)
    view_tint: float = 0.0
    tint_axis: tuple = (0.0, 0.0, 1.0)
    texture_freq: float = 0.0
    texture_amp: float = 0.3

    def __post_init__(self):
        for s in self.spheres:
            if s.density < 0 or s.radius <= 0:
                raise ValueError("spheres need positive radius and non-negative density")
        for b in self.boxes:
            if b.density < 0:
                raise ValueError("box density must be non-negative")

    def native(self) -> N.Analytic:
        """gf_analytic_t: spheres then boxes (the reference's iteration order)."""
        prims = [(0, p.center, (0.0, 0.0, 0.0), p.color, p.radius, p.density, p.feather) for p in self.spheres]
        prims += [(1, p.lo, p.hi, p.color, 0.0, p.density, p.feather) for p in self.boxes]
        if len(prims) > N.MAX_PRIMS:
            raise ValueError(f"the device scene holds at most {N.MAX_PRIMS} primitives")
        a = N.Analytic()
        for i in range(3):
            a.b_min[i] = float(self.aabb.b_min[i])
            a.b_max[i] = float(self.aabb.b_max[i])
            a.tint_axis[i] = float(self.tint_axis[i])
        a.n_prims = len(prims)
        for k, (kind, pa, pb, col, rad, dens, fea) in enumerate(prims):
            q = a.prims[k]
            q.kind = kind
            for i in range(3):
                q.a[i], q.b[i], q.color[i] = float(pa[i]), float(pb[i]), float(col[i])
            q.radius, q.density, q.feather = float(rad), float(dens), float(fea)
        a.texture_freq, a.texture_amp, a.view_tint = float(self.texture_freq), float(self.texture_amp), float(self.view_tint)
        return a

    def query_points(self, positions, directions):
        """scene.py:115-135 on the device; float32 in, (rgb (N,3), sigma (N,)) out
        (numpy in -> numpy out, CUDA tensors in -> tensors out)."""
        t = D.require_cuda()
        on_device = D.is_tensor(positions)
        p = D.to_device(positions, t.float32).reshape(-1, 3).contiguous()
        d = D.to_device(directions, t.float32).reshape(-1, 3).contiguous()
        if d.shape[0] != p.shape[0]:
            raise ValueError("positions and directions differ in length")
        rgb = D.empty((p.shape[0], 3), t.float32)
        sig = D.empty((p.shape[0],), t.float32)
        N.check(N.lib().gf_query_analytic(self.native(), N.ptr(p), N.ptr(d), int(p.shape[0]), N.ptr(rgb), N.ptr(sig),
                                          D.stream_handle()), "query_analytic")
        if on_device:
            return rgb, sig
        return rgb.cpu().numpy(), sig.cpu().numpy()

    def density_at(self, positions):
        """scene.py:108-113 (density is view-independent)."""
        x = np.asarray(positions, dtype=np.float32).reshape(-1, 3)
        return self.query_points(x, np.broadcast_to(np.array([0.0, 0.0, 1.0], np.float32), x.shape))[1]


def standard_toy_scene() -> AnalyticScene:
    """scene.py:138-160: the fixed three-sphere benchmark scene."""
    aabb = Aabb((-1.0, -1.0, -1.0), (1.0, 1.0, 1.0))
    return AnalyticScene(
        aabb=aabb,
        spheres=[
            Sphere(center=(-0.45, -0.38, -0.2), radius=0.48, color=(0.85, 0.18, 0.14), density=40.0, feather=0.067),
            Sphere(center=(0.5, -0.12, 0.14), radius=0.42, color=(0.16, 0.5, 0.85), density=40.0, feather=0.067),
            Sphere(center=(-0.02, 0.56, 0.38), radius=0.36, color=(0.9, 0.76, 0.18), density=40.0, feather=0.067),
        ],
        texture_freq=9.0,
    )


def specular_toy_scene() -> AnalyticScene:
    """scene.py:163-167: standard scene plus a view-dependent tint."""
    scene = standard_toy_scene()
    scene.view_tint = 0.3
    return scene


def random_toy_scene(seed: int, n_primitives: int = 5) -> AnalyticScene:
    """scene.py:170-186: seeded sphere/box union (identical draws)."""
    if not (3 <= n_primitives <= 8):
        raise ValueError("toy scene family uses 3..8 primitives")
    rng = np.random.default_rng(seed)
    aabb = Aabb((-1.0, -1.0, -1.0), (1.0, 1.0, 1.0))
    spheres, boxes = [], []
    for _ in range(n_primitives):
        center = rng.uniform(-0.55, 0.55, 3)
        color = tuple(rng.uniform(0.1, 0.95, 3))
        if rng.random() < 0.7:
            spheres.append(Sphere(tuple(center), float(rng.uniform(0.15, 0.4)), color, 40.0))
        else:
            half = rng.uniform(0.1, 0.3, 3)
            boxes.append(Box(tuple(center - half), tuple(center + half), color, 40.0))
    return AnalyticScene(aabb=aabb, spheres=spheres, boxes=boxes)


def sphere_cameras(aabb: Aabb, n_views: int, image_size: int, seed: int, radius_scale: float = 1.1,
                   fov_margin: float = 0.8) -> list:
    """scene.py:283-320: cameras on a sphere around the box centre, looking at it."""
    rng = np.random.default_rng(seed)
    center = aabb.center
    bound_r = 0.5 * aabb.diagonal
    orbit_r = radius_scale * aabb.diagonal
    half_tan = fov_margin * bound_r / np.sqrt(max(orbit_r**2 - bound_r**2, 1e-9))
    focal = 0.5 * image_size / half_tan
    cams = []
    for _ in range(n_views):
        v = rng.normal(size=3)
        v /= np.linalg.norm(v)
        pose = look_at_pose(center + orbit_r * v, center)
        cams.append(Camera(image_size, image_size, focal, focal, image_size / 2.0, image_size / 2.0, pose))
    return cams


def analytically_empty_cells(scene: AnalyticScene, resolution) -> np.ndarray:
    """scene.py:186-211: flat indices of the grid cells no primitive touches
    (sphere: clamped distance to the cell box within the radius; box:
    interval overlap), decided per cell on the device in float64."""
    res = np.asarray(resolution, dtype=np.int64).reshape(3)
    t = D.require_cuda()
    out = D.empty((int(np.prod(res)),), t.uint8)
    r3 = (N.C.c_int32 * 3)(*[int(v) for v in res])
    N.check(N.lib().gf_analytic_empty_cells(scene.native(), r3, N.ptr(out), D.stream_handle()),
            "analytically_empty_cells")
    return np.flatnonzero(out.cpu().numpy())


def render_brute_force(scene, cam: Camera, n_samples: int, background=(1.0, 1.0, 1.0), chunk_rays: int = 128) -> np.ndarray:
    """scene.py:214-252: ground-truth quadrature (no occupancy, no
    termination, no networks) on the device: every ray's box interval in
    ``n_samples`` segments with a Simpson optical depth from both ends and
    the midpoint, the midpoint's colour, composited in sample order.  Rays
    are independent, so ``chunk_rays`` (kept for the reference signature)
    does not change the result; the device works in chunks sized to its
    workspace."""
    if n_samples < 1:
        raise ValueError("n_samples must be >= 1")
    t = D.require_cuda()
    n = cam.width * cam.height
    chunk = int(max(1, min(n, (256 << 20) // (16 * int(n_samples)))))
    out = D.empty((n, 3), t.float32)
    bg = (N.C.c_float * 3)(*[float(np.float32(b)) for b in background])
    ws = D.workspace(N.lib().gf_brute_force_workspace_bytes(int(n_samples), chunk))
    sc, cc = scene.native(), N.make_camera(cam)
    for r0 in range(0, n, chunk):
        nr = min(chunk, n - r0)
        N.check(N.lib().gf_render_brute_force(sc, cc, int(n_samples), bg, r0, nr, N.ptr(out[r0:]), N.ptr(ws),
                                              ws.numel(), D.stream_handle()), "render_brute_force")
    return out.cpu().numpy().reshape(cam.height, cam.width, 3)
