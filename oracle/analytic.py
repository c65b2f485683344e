"""CPU oracle (test infrastructure only) for the analytic scene field.

numpy restatement of /root/reference/pkg/src/gridfield/scene.py:
_smoothstep (:21-24), Sphere.density_at (:40-53), Box.density_at (:65-74),
AnalyticScene.query_points (:115-135), standard/specular/random toy scenes
(:138-186).  Primitives are plain tuples here; evaluation follows the
reference's float32 arithmetic with NEP 50 weak Python scalars.  Pinned by
tests/test_oracle_golden.py against fixtures made by the reference itself.
Imported only by tests/, never by the product path.
"""

from __future__ import annotations

import numpy as np

SPHERE, BOX = 0, 1


def _smooth(u):
    u = np.clip(u, 0.0, 1.0)
    return u * u * (3.0 - 2.0 * u)


def prim_density(prim, x):
    """One primitive's density at float32 points x (N, 3)."""
    kind, a, b, _color, radius, density, feather = prim
    if kind == SPHERE:
        d2 = np.square(x[:, 0] - np.float32(a[0]))
        d2 += np.square(x[:, 1] - np.float32(a[1]))
        d2 += np.square(x[:, 2] - np.float32(a[2]))
        out = np.zeros_like(d2)
        inside = d2 < radius * radius
        if inside.any():
            if feather <= 0.0:
                out[inside] = density
            else:
                out[inside] = density * _smooth((radius - np.sqrt(d2[inside])) / feather)
        return out
    depth = np.minimum(x - np.asarray(a, np.float32), np.asarray(b, np.float32) - x).min(axis=-1)
    out = np.zeros_like(depth)
    inside = depth > 0.0
    if inside.any():
        out[inside] = density if feather <= 0.0 else density * _smooth(depth[inside] / feather)
    return out


def scene_query(scene, x, d):
    """(rgb, sigma) of the scene dict at float32 points x with directions d."""
    x = np.asarray(x, np.float32).reshape(-1, 3)
    sigma = np.zeros(len(x), np.float32)
    rgb = np.zeros((len(x), 3), np.float32)
    for prim in scene["prims"]:
        s = prim_density(prim, x)
        wins = (s > 0) & (s >= sigma)
        np.maximum(sigma, s, out=sigma)
        rgb[wins] = np.asarray(prim[3], np.float32)
    f = scene["texture_freq"]
    if f > 0.0:
        f32 = np.float32(f)
        amp = scene["texture_amp"]
        wave = 0.5 + 0.5 * np.sin(f32 * x[:, 0]) * np.sin(f32 * x[:, 1] + 1.3) * np.sin(f32 * x[:, 2] + 2.1)
        rgb *= ((1.0 - amp) + amp * wave)[:, None].astype(np.float32)
    tint = scene["view_tint"]
    if tint != 0.0:
        dd = np.asarray(d, np.float32).reshape(-1, 3)
        shift = (tint * 0.5) * (dd @ np.asarray(scene["tint_axis"], np.float32))
        rgb += shift[:, None] * (sigma > 0)[:, None]
        np.clip(rgb, 0.0, 1.0, out=rgb)
    return rgb, sigma


def _sphere(center, radius, color, density, feather=0.14):
    return (SPHERE, tuple(center), (0.0, 0.0, 0.0), tuple(color), float(radius), float(density), float(feather))


def _box(lo, hi, color, density, feather=0.14):
    return (BOX, tuple(lo), tuple(hi), tuple(color), 0.0, float(density), float(feather))


def standard_scene():
    return {
        "prims": [
            _sphere((-0.45, -0.38, -0.2), 0.48, (0.85, 0.18, 0.14), 40.0, 0.067),
            _sphere((0.5, -0.12, 0.14), 0.42, (0.16, 0.5, 0.85), 40.0, 0.067),
            _sphere((-0.02, 0.56, 0.38), 0.36, (0.9, 0.76, 0.18), 40.0, 0.067),
        ],
        "texture_freq": 9.0, "texture_amp": 0.3, "view_tint": 0.0, "tint_axis": (0.0, 0.0, 1.0),
    }


def specular_scene():
    s = standard_scene()
    s["view_tint"] = 0.3
    return s


def random_scene(seed, n_primitives=5):
    """scene.py:170-186 draws (spheres first, then boxes, as iterated there)."""
    rng = np.random.default_rng(seed)
    spheres, boxes = [], []
    for _ in range(n_primitives):
        center = rng.uniform(-0.55, 0.55, 3)
        color = tuple(rng.uniform(0.1, 0.95, 3))
        if rng.random() < 0.7:
            spheres.append(_sphere(center, float(rng.uniform(0.15, 0.4)), color, 40.0))
        else:
            half = rng.uniform(0.1, 0.3, 3)
            boxes.append(_box(center - half, center + half, color, 40.0))
    return {"prims": spheres + boxes, "texture_freq": 0.0, "texture_amp": 0.3, "view_tint": 0.0,
            "tint_axis": (0.0, 0.0, 1.0)}
