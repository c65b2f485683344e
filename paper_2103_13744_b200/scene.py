"""Synthetic camera rigs (subset of gridfield.scene,
/root/reference/pkg/src/gridfield/scene.py:283-320).  Analytic density scenes
and dataset generation stay out of scope for the device build."""

from __future__ import annotations

import numpy as np

from .core import Aabb
from .render import Camera, look_at_pose


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
