"""Spatial primitives (mirror of gridfield.core, /root/reference/pkg/src/gridfield/core.py).

Host-side value types (``Aabb``, ``PositionalEncoding``) are plain Python;
the array primitives on the render path (clip, binning, encoding, alpha) run
as CUDA kernels in libgridfield_b200.so and accept/return numpy arrays like
the originals.  float32 and float64 inputs are computed in their own dtype as
numpy does.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _device as D
from . import _native as N


@dataclass(frozen=True)
class Aabb:
    """Axis-aligned box (core.py:16-49)."""

    b_min: np.ndarray
    b_max: np.ndarray

    def __post_init__(self):
        lo = np.asarray(self.b_min, dtype=np.float64).reshape(3)
        hi = np.asarray(self.b_max, dtype=np.float64).reshape(3)
        if not np.all(lo < hi):
            raise ValueError(f"degenerate bounds: b_min={lo} must be < b_max={hi}")
        object.__setattr__(self, "b_min", lo)
        object.__setattr__(self, "b_max", hi)

    @property
    def extent(self) -> np.ndarray:
        return self.b_max - self.b_min

    @property
    def center(self) -> np.ndarray:
        return 0.5 * (self.b_min + self.b_max)

    @property
    def diagonal(self) -> float:
        return float(np.linalg.norm(self.extent))

    def contains(self, x: np.ndarray) -> np.ndarray:
        x = np.asarray(x)
        return np.all((x >= self.b_min) & (x <= self.b_max), axis=-1)

    def cell_size(self, resolution) -> np.ndarray:
        return self.extent / np.asarray(resolution, dtype=np.float64)


def validate_resolution(resolution) -> np.ndarray:
    """core.py:71-76."""
    r = np.asarray(resolution, dtype=np.int64).reshape(3)
    if np.any(r < 1):
        raise ValueError(f"grid resolution must be >= 1 per axis, got {r}")
    return r


def _bounds_error(x: np.ndarray, flat_component: int, aabb: Aabb) -> ValueError:
    """Rebuild the reference's message for the first offending component
    (core.py:94-101) from the device's error slot."""
    pts = x.reshape(-1, 3)
    i, axis = divmod(int(flat_component), 3)
    value = pts[i, axis]
    bound = aabb.b_min[axis] if value < aabb.b_min[axis] else aabb.b_max[axis]
    return ValueError(f"point outside bounds: component {axis} is {value!r}, bound {bound!r}")


def raise_if_out_of_bounds(err_tensor, x: np.ndarray, aabb: Aabb):
    e = int(err_tensor.item())
    if e != N.INT64_MAX:
        raise _bounds_error(np.asarray(x), e, aabb)


def _as_points32(x):
    x = np.asarray(x)
    if x.shape[-1:] != (3,):
        raise ValueError(f"points must have a trailing axis of 3, got {x.shape}")
    return x


def clip_into(x: np.ndarray, aabb: Aabb) -> np.ndarray:
    """core.py:52-68 (device for float32 points; float64 points cannot round
    out of the box, so the f64 clamp is exact)."""
    x = _as_points32(x)
    if x.dtype != np.float32:
        return np.clip(x, aabb.b_min, aabb.b_max).astype(x.dtype)
    t = D.require_cuda()
    xd = D.to_device(x.reshape(-1, 3), t.float32)
    out = D.empty(xd.shape, t.float32)
    lo = (N.C.c_double * 3)(*aabb.b_min)
    hi = (N.C.c_double * 3)(*aabb.b_max)
    N.check(N.lib().gf_clip_into(lo, hi, N.ptr(xd), xd.shape[0], N.ptr(out), D.stream_handle()), "clip_into")
    return out.cpu().numpy().reshape(x.shape)


def bin_point(x: np.ndarray, aabb: Aabb, resolution) -> np.ndarray:
    """core.py:79-104: integer cell indices (…, 3); raises on out-of-bounds."""
    r = validate_resolution(resolution)
    flat = _flat_cells(x, aabb, r)
    return np.stack([flat % r[0], (flat // r[0]) % r[1], flat // (r[0] * r[1])], axis=-1)


def _float_points(x):
    """(…,3) float32 / float64 points as a contiguous device tensor (other
    dtypes are promoted like numpy promotes them against the f64 bounds)."""
    t = D.require_cuda()
    x = np.asarray(x)
    f64 = x.dtype != np.float32
    pts = x.reshape(-1, 3)
    return D.to_device(pts, t.float64 if f64 else t.float32), int(f64), pts.shape[0]


def _flat_cells(x, aabb: Aabb, r) -> np.ndarray:
    """Device binning + x-major flatten (core.py:79-112) for (…,3) points."""
    x = np.asarray(x)
    t = D.require_cuda()
    xd, f64, n = _float_points(x)
    flat = D.empty((n,), t.int64)
    err = D.err_slot()
    N.check(N.lib().gf_bin_points(N.make_geom(aabb, r), N.ptr(xd), f64, n, N.ptr(flat), N.ptr(err),
                                  D.stream_handle()), "bin_point")
    raise_if_out_of_bounds(err, x, aabb)
    return flat.cpu().numpy().reshape(x.shape[:-1])


def flatten_cell_index(idx: np.ndarray, resolution) -> np.ndarray:
    """core.py:107-112 (x-major; the checkpoint contract)."""
    r = validate_resolution(resolution)
    idx = np.asarray(idx)
    return idx[..., 0] + r[0] * (idx[..., 1] + r[1] * idx[..., 2])


def unflatten_cell_index(flat: np.ndarray, resolution) -> np.ndarray:
    r = validate_resolution(resolution)
    flat = np.asarray(flat)
    return np.stack([flat % r[0], (flat // r[0]) % r[1], flat // (r[0] * r[1])], axis=-1)


def cell_bounds(idx: np.ndarray, aabb: Aabb, resolution):
    r = validate_resolution(resolution)
    lo = aabb.b_min + np.asarray(idx) * aabb.cell_size(r)
    return lo, lo + aabb.cell_size(r)


def positional_encode(v: np.ndarray, num_freqs: int, include_raw: bool = True) -> np.ndarray:
    """core.py:132-152 on the device: [v, sin(v f_0), cos(v f_0), …] with
    f_k = 2^k pi rounded to the input dtype (float32 or float64)."""
    v = np.asarray(v)
    if v.dtype not in (np.float32, np.float64):
        v = v.astype(np.float64)
    dim = v.shape[-1]
    t = D.require_cuda()
    f64 = v.dtype == np.float64
    flat = v.reshape(-1, dim)
    width = dim * (int(bool(include_raw)) + 2 * num_freqs)
    tdt = t.float64 if f64 else t.float32
    vd = D.to_device(flat, tdt)
    out = D.empty((flat.shape[0], width), tdt)
    N.check(N.lib().gf_positional_encode(N.ptr(vd), int(f64), flat.shape[0], dim, num_freqs, int(bool(include_raw)),
                                         N.ptr(out), D.stream_handle()), "positional_encode")
    return out.cpu().numpy().reshape(*v.shape[:-1], width)


@dataclass(frozen=True)
class PositionalEncoding:
    """core.py:155-184."""

    num_freqs_position: int = 10
    num_freqs_direction: int = 4
    include_raw_input: bool = True

    def __post_init__(self):
        if self.num_freqs_position < 0 or self.num_freqs_direction < 0:
            raise ValueError("frequency counts must be non-negative")

    @property
    def position_dim(self) -> int:
        return 3 * (int(self.include_raw_input) + 2 * self.num_freqs_position)

    @property
    def direction_dim(self) -> int:
        return 3 * (int(self.include_raw_input) + 2 * self.num_freqs_direction)

    def encode_position(self, x: np.ndarray) -> np.ndarray:
        return positional_encode(x, self.num_freqs_position, self.include_raw_input)

    def encode_direction(self, d: np.ndarray) -> np.ndarray:
        return positional_encode(d, self.num_freqs_direction, self.include_raw_input)


def density_to_alpha(sigma, delta):
    """core.py:187-194 on the device: -expm1(-sigma*delta) in the promoted
    dtype (float32 when both are float32, else float64)."""
    s = np.asarray(sigma)
    d = np.asarray(delta)
    dtype = np.float32 if (s.dtype == np.float32 and d.dtype == np.float32) else np.float64
    s, d = np.broadcast_arrays(s.astype(dtype), d.astype(dtype))
    t = D.require_cuda()
    tdt = t.float32 if dtype == np.float32 else t.float64
    sd = D.to_device(np.ascontiguousarray(s).reshape(-1), tdt)
    dd = D.to_device(np.ascontiguousarray(d).reshape(-1), tdt)
    out = D.empty(sd.shape, tdt)
    N.check(N.lib().gf_density_to_alpha(N.ptr(sd), N.ptr(dd), int(dtype == np.float64), sd.shape[0], N.ptr(out),
                                        D.stream_handle()), "density_to_alpha")
    res = out.cpu().numpy().reshape(s.shape)
    return res[()] if res.ndim == 0 else res
