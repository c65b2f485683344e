"""Cameras, rays, compositing and the device ray marcher (mirror of
gridfield.render, /root/reference/pkg/src/gridfield/render.py).

``render_rays`` / ``render_image`` run the whole march on the GPU: one call
into ``gf_render_rays`` generates (or takes) the rays, places the stratified
samples bit-exactly like the numpy reference (same PCG64 streams per 4096-ray
block), skips empty space, buckets the survivors by cell, evaluates the
per-cell MLPs, composites front to back and applies chunk-granular ERT.  The
host only transfers the camera in and the image + 4 counters out.
"""

from __future__ import annotations

import threading
import os
import time
from dataclasses import dataclass

import numpy as np

from . import _device as D
from . import _native as N
from .core import Aabb

RAY_BLOCK = 4096  # render.py:22


@dataclass(frozen=True)
class Camera:
    """render.py:25-76 (pinhole; +x right, +y down, +z forward)."""

    width: int
    height: int
    fx: float
    fy: float
    cx: float
    cy: float
    c2w: np.ndarray

    def __post_init__(self):
        if self.width < 1 or self.height < 1:
            raise ValueError("image dimensions must be positive")
        c2w = np.asarray(self.c2w, dtype=np.float64).reshape(4, 4)
        r = c2w[:3, :3]
        err = np.linalg.norm(r.T @ r - np.eye(3))
        if err > 1e-5:
            raise ValueError(f"pose rotation block not orthonormal (|R^T R - I| = {err:.2e})")
        object.__setattr__(self, "c2w", c2w)

    @property
    def center(self) -> np.ndarray:
        return self.c2w[:3, 3]

    @property
    def rotation(self) -> np.ndarray:
        return self.c2w[:3, :3]

    def scaled(self, focal_scale: float = 1.0, width: int | None = None, height: int | None = None) -> "Camera":
        w = width or self.width
        h = height or self.height
        sx, sy = w / self.width, h / self.height
        return Camera(w, h, self.fx * sx * focal_scale, self.fy * sy * focal_scale, self.cx * sx, self.cy * sy,
                      self.c2w)


def look_at_pose(eye, target, up=(0.0, 0.0, 1.0)) -> np.ndarray:
    """render.py:79-100."""
    eye = np.asarray(eye, dtype=np.float64)
    fwd = np.asarray(target, dtype=np.float64) - eye
    norm = np.linalg.norm(fwd)
    if norm == 0:
        raise ValueError("eye and target coincide")
    z = fwd / norm
    x = np.cross(z, np.asarray(up, dtype=np.float64))
    if np.linalg.norm(x) < 1e-8:
        x = np.cross(z, np.array([0.0, 1.0, 0.0]))
    x /= np.linalg.norm(x)
    y = np.cross(z, x)
    c2w = np.eye(4)
    c2w[:3, 0], c2w[:3, 1], c2w[:3, 2], c2w[:3, 3] = x, y, z, eye
    return c2w


@dataclass(frozen=True)
class Ray:
    """render.py:103-123."""

    origin: np.ndarray
    direction: np.ndarray
    t_near: float | None = None
    t_far: float | None = None

    def __post_init__(self):
        d = np.asarray(self.direction, dtype=np.float64)
        if abs(np.linalg.norm(d) - 1.0) > 1e-6:
            raise ValueError("ray direction must be unit length")
        object.__setattr__(self, "origin", np.asarray(self.origin, dtype=np.float64))
        object.__setattr__(self, "direction", d)

    @classmethod
    def clipped(cls, origin, direction, aabb: Aabb) -> "Ray":
        t0, t1 = intersect_aabb(np.asarray(origin)[None], np.asarray(direction)[None], aabb)
        return cls(origin, direction, t_near=float(t0[0]), t_far=float(t1[0]))


def generate_ray(cam: Camera, px) -> Ray:
    """render.py:126-136 (single ray through continuous pixel coords)."""
    u, v = float(px[0]), float(px[1])
    d = cam.rotation @ np.array([(u - cam.cx) / cam.fx, (v - cam.cy) / cam.fy, 1.0])
    return Ray(cam.center, d / np.linalg.norm(d))


def generate_rays(cam: Camera):
    """render.py:139-148 on the device: float32 origins and unit directions,
    row-major, bit-identical to the numpy reference."""
    t = D.require_cuda()
    n = cam.width * cam.height
    o = D.empty((n, 3), t.float32)
    d = D.empty((n, 3), t.float32)
    N.check(N.lib().gf_generate_rays(N.make_camera(cam), N.ptr(o), N.ptr(d), D.stream_handle()), "generate_rays")
    return o.cpu().numpy(), d.cpu().numpy()


def intersect_aabb(origins, directions, aabb: Aabb):
    """render.py:151-171 slab test in float64 on the device (gf_intersect_aabb;
    the marcher runs the same arithmetic inside k_ray_init)."""
    o = np.asarray(origins, dtype=np.float64)
    d = np.asarray(directions, dtype=np.float64)
    shape = np.broadcast_shapes(o.shape, d.shape)[:-1]
    o2 = np.ascontiguousarray(np.broadcast_to(o, shape + (3,))).reshape(-1, 3)
    d2 = np.ascontiguousarray(np.broadcast_to(d, shape + (3,))).reshape(-1, 3)
    t = D.require_cuda()
    od, dd = D.to_device(o2, t.float64), D.to_device(d2, t.float64)
    t0, t1 = D.empty((o2.shape[0],), t.float64), D.empty((o2.shape[0],), t.float64)
    lo = (N.C.c_double * 3)(*aabb.b_min)
    hi = (N.C.c_double * 3)(*aabb.b_max)
    N.check(N.lib().gf_intersect_aabb(N.ptr(od), N.ptr(dd), o2.shape[0], lo, hi, N.ptr(t0), N.ptr(t1),
                                      D.stream_handle()), "intersect_aabb")
    return t0.cpu().numpy().reshape(shape), t1.cpu().numpy().reshape(shape)


@dataclass
class RenderConfig:
    """render.py:174-207."""

    k: int = 384
    epsilon: float = 0.01
    background: tuple = (1.0, 1.0, 1.0)
    ert_chunk: int = 32
    stratified: bool = True

    def __post_init__(self):
        if self.k < 1:
            raise ValueError("k must be >= 1")
        if not (0.0 <= self.epsilon < 1.0):
            raise ValueError("epsilon must lie in [0, 1)")
        if self.ert_chunk < 1:
            raise ValueError("ert_chunk must be >= 1")

    def replace(self, **kw) -> "RenderConfig":
        merged = dict(k=self.k, epsilon=self.epsilon, background=self.background, ert_chunk=self.ert_chunk,
                      stratified=self.stratified)
        merged.update(kw)
        return RenderConfig(**merged)

    def native(self, seed: int) -> N.MarchCfg:
        c = N.MarchCfg()
        c.k, c.ert_chunk, c.stratified = int(self.k), int(self.ert_chunk), int(bool(self.stratified))
        # numpy compares float32 transmittance with a Python float as float32
        # (NEP 50); a float64 scalar forces a float64 comparison
        c.eps_compare_f64 = int(isinstance(self.epsilon, np.floating) and np.dtype(type(self.epsilon)) == np.float64)
        c.epsilon = float(self.epsilon)
        for a in range(3):
            c.background[a] = float(np.float32(self.background[a]))
        if int(seed) < 0:
            raise ValueError("seed must be non-negative")
        c.seed = int(seed)
        return c


@dataclass
class RenderStats:
    """render.py:210-231."""

    wall_ms: float = 0.0
    total_queries: int = 0
    ess_skipped: int = 0
    ert_terminated_rays: int = 0
    n_rays: int = 0

    def merge(self, other: "RenderStats"):
        self.total_queries += other.total_queries
        self.ess_skipped += other.ess_skipped
        self.ert_terminated_rays += other.ert_terminated_rays
        self.n_rays += other.n_rays

    def to_dict(self) -> dict:
        return {"wall_ms": self.wall_ms, "total_queries": self.total_queries, "ess_skipped": self.ess_skipped,
                "ert_terminated_rays": self.ert_terminated_rays, "n_rays": self.n_rays}


def sample_ray(ray: Ray, aabb: Aabb, occ=None, cfg: RenderConfig | None = None, rng=None):
    """render.py:234-266: one ray's k jittered samples minus unoccupied ones.
    The jitter comes from the caller's Generator on the host, exactly as in
    the reference; the slab test, the float64 placement, clip_into and the
    occupancy test run on the device."""
    from .core import clip_into

    cfg = cfg or RenderConfig()
    t0, t1 = intersect_aabb(ray.origin[None], ray.direction[None], aabb)
    t0, t1 = float(t0[0]), float(t1[0])
    if t1 <= t0:
        return np.zeros((0, 3), dtype=np.float32), np.zeros(0, dtype=np.float32)
    seg = (t1 - t0) / cfg.k
    jitter = (rng or np.random.default_rng()).random(cfg.k) if cfg.stratified else np.full(cfg.k, 0.5)
    t = D.require_cuda()
    jd = D.to_device(np.asarray(jitter, np.float64), t.float64)
    pts = D.empty((cfg.k, 3), t.float32)
    o3 = (N.C.c_double * 3)(*np.asarray(ray.origin, np.float64))
    d3 = (N.C.c_double * 3)(*np.asarray(ray.direction, np.float64))
    N.check(N.lib().gf_ray_samples(o3, d3, t0, seg, N.ptr(jd), cfg.k, N.ptr(pts), D.stream_handle()), "sample_ray")
    pts = clip_into(pts.cpu().numpy(), aabb)
    if occ is not None:
        pts = pts[occ.occupied_at(pts)]
    return pts, np.full(len(pts), seg, dtype=np.float32)


def composite(colors, alphas):
    """render.py:269-284 on the device (float32 or float64, batch dims)."""
    colors = np.asarray(colors)
    alphas = np.asarray(alphas)
    dtype = np.result_type(colors.dtype, alphas.dtype)
    if dtype not in (np.float32, np.float64):
        dtype = np.float64
    lead = alphas.shape[:-1]
    ns = alphas.shape[-1]
    nr = int(np.prod(lead)) if lead else 1
    if colors.shape[-2] == 0:
        return np.zeros((*lead, 3), dtype=colors.dtype), np.ones(lead, dtype=colors.dtype)
    t = D.require_cuda()
    tdt = t.float64 if dtype == np.float64 else t.float32
    cd = D.to_device(np.broadcast_to(colors, (*lead, ns, 3)).reshape(nr, ns, 3), tdt)
    ad = D.to_device(alphas.reshape(nr, ns), tdt)
    rgb = D.empty((nr, 3), tdt)
    tr = D.empty((nr,), tdt)
    fn = N.lib().gf_composite_f64 if dtype == np.float64 else N.lib().gf_composite
    N.check(fn(N.ptr(cd), N.ptr(ad), nr, ns, N.ptr(rgb), N.ptr(tr), D.stream_handle()), "composite")
    rgb_h = rgb.cpu().numpy().reshape(*lead, 3)
    tr_h = tr.cpu().numpy().reshape(lead)
    return rgb_h, (tr_h if lead else tr_h[()])


# ---------------------------------------------------------------------------
# the marcher
# ---------------------------------------------------------------------------
def _field_grid(field):
    """render.py:361-364 field protocol: NetworkGrid (per-cell MLPs) and
    AnalyticScene (closed-form field) are evaluated on the device; any other
    object with ``aabb`` and ``query_points(positions, directions)`` is a
    caller-evaluated field: the device still marches, places and composites,
    and hands the field each round group's samples (gf_render_rays_field)."""
    from .grid import NetworkGrid
    from .scene import AnalyticScene

    if isinstance(field, (NetworkGrid, AnalyticScene)):
        return field
    if hasattr(field, "aabb") and callable(getattr(field, "query_points", None)):
        return field
    raise TypeError(f"a field needs .aabb and .query_points(positions, directions); got {type(field).__name__}")


def _is_analytic(field) -> bool:
    from .scene import AnalyticScene

    return isinstance(field, AnalyticScene)


def _is_caller_field(field) -> bool:
    from .grid import NetworkGrid
    from .scene import AnalyticScene

    return not isinstance(field, (NetworkGrid, AnalyticScene))


def _box_geom(aabb):
    return N.make_geom(aabb, (1, 1, 1))


_WS_CACHE: dict = {}


def _render_ws_bytes(field, ncfg, n: int) -> int:
    if _is_analytic(field):
        return N.lib().gf_render_analytic_workspace_bytes(field.native(), ncfg, n)
    if _is_caller_field(field):
        return N.lib().gf_render_field_workspace_bytes(_box_geom(field.aabb), ncfg, n)
    # cached per (architecture, resolution, k, chunk, rays, GF_GROUP): one
    # native call and two struct builds saved on every render_image
    key = (field.params.arch, tuple(int(r) for r in field.resolution), ncfg.k, ncfg.ert_chunk, int(n),
           os.environ.get("GF_GROUP"))
    b = _WS_CACHE.get(key)
    if b is None:
        b = N.lib().gf_render_workspace_bytes(field.native_arch(), field.native_geom(), ncfg, n)
        if len(_WS_CACHE) > 256:
            _WS_CACHE.clear()
        _WS_CACHE[key] = b
    return b


def _field_callback(field, errors: list):
    """ctypes callback for gf_render_rays_field: gather the group's samples
    into (n, 3) arrays, evaluate the caller's field, scatter the results."""
    t = D.torch()

    def cb(user, srec, n, ray_dir, shift, stride, res, stream):
        try:
            pos = D.empty((n, 3), t.float32)
            dirs = D.empty((n, 3), t.float32)
            N.check(N.lib().gf_field_gather(srec, n, ray_dir, shift, stride, N.ptr(pos), N.ptr(dirs), stream),
                    "field gather")
            rgb, sigma = field.query_points(pos.cpu().numpy(), dirs.cpu().numpy())
            rgb_d = D.to_device(np.asarray(rgb, np.float32).reshape(n, 3), t.float32)
            sig_d = D.to_device(np.asarray(sigma, np.float32).reshape(n), t.float32)
            N.check(N.lib().gf_field_scatter(srec, n, N.ptr(rgb_d), N.ptr(sig_d), res, stream), "field scatter")
            t.cuda.current_stream().synchronize()  # rgb_d / sig_d live until the scatter ran
            return 0
        except BaseException as e:  # re-raised by the caller after the library returns
            errors.append(e)
            return 1

    return N.FIELD_FN(cb)


def shard_rays(n_rays: int, rank: int, world: int) -> tuple[int, int, int]:
    """Balanced multi-GPU partition of a ray set: rank r takes the 4096-ray
    jitter blocks r, r+world, r+2*world, ... (image content is centre-heavy,
    so contiguous bands would not balance).  Returns (ray_offset,
    block_stride, n_local_rays) for ``render_rays_device``."""
    if not (0 <= rank < world):
        raise ValueError("rank must lie in [0, world)")
    n_blocks = (n_rays + RAY_BLOCK - 1) // RAY_BLOCK
    mine = list(range(rank, n_blocks, world))
    n_local = sum(min(RAY_BLOCK, n_rays - b * RAY_BLOCK) for b in mine)
    return rank * RAY_BLOCK, world, n_local


def unshard_index(n_rays: int, world: int) -> np.ndarray:
    """For the all-gathered, per-rank padded shard buffers (world, cap, 3)
    flattened to (world*cap, 3), the row of each global ray in image order."""
    n_blocks = (n_rays + RAY_BLOCK - 1) // RAY_BLOCK
    cap = ((n_blocks + world - 1) // world) * RAY_BLOCK
    g = np.arange(n_rays)
    b, w = g // RAY_BLOCK, g % RAY_BLOCK
    return (b % world) * cap + (b // world) * RAY_BLOCK + w


_ctx = threading.local()


def _render_context(n: int, ws_bytes: int):
    """Per-thread persistent device buffers for a frame shape, so repeated
    calls present identical pointers to the library (its CUDA-graph cache is
    keyed on every kernel argument) and avoid allocator churn."""
    t = D.require_cuda()
    cache = getattr(_ctx, "bufs", None)
    if cache is None:
        cache = _ctx.bufs = {}
    key = (t.cuda.current_device(), n)
    c = cache.get(key)
    if c is None or c["ws"].numel() < ws_bytes:
        c = {"ws": D.workspace(ws_bytes), "rgb": D.empty((n, 3), t.float32),
             "stats": t.zeros(4, dtype=t.int64, device=D.device()),
             "host_stats": t.empty(4, dtype=t.int64, pin_memory=True)}
        cache[key] = c
    return c


def render_rays_device(grid, occupancy, cfg: RenderConfig, seed=0, *, cam: Camera | None = None, origins=None,
                       directions=None, ray_offset: int = 0, n_rays: int | None = None, block_stride: int = 1,
                       precision=None, out=None, stats=None, trace_capacity: int = 0, ws=None):
    """Device-resident core of render_rays / render_image.  Returns
    (rgb (n,3) float32 CUDA tensor, stats int64[4] CUDA tensor, trace or None).
    ``origins``/``directions`` may be CUDA tensors; ``cam`` generates rays
    for pixels [ray_offset, ray_offset + n_rays), or for the interleaved
    blocks of ``shard_rays`` when ``block_stride`` > 1."""
    t = D.require_cuda()
    analytic = _is_analytic(grid)
    caller = _is_caller_field(grid)
    if not analytic and not caller:
        p = grid.resolved_precision(precision, render=True)
        packed = grid.device_params(p)
    if cam is not None:
        total = cam.width * cam.height
        n = total - ray_offset if n_rays is None else int(n_rays)
        o_d = d_d = None
        ccam = N.make_camera(cam)
    else:
        f64 = getattr(origins, "dtype", None) in (np.float64, t.float64) or \
            getattr(directions, "dtype", None) in (np.float64, t.float64)
        rdt = t.float64 if f64 else t.float32
        o_d = D.to_device(origins, rdt).reshape(-1, 3)
        d_d = D.to_device(directions, rdt).reshape(-1, 3)
        n = o_d.shape[0]
        ccam = None
    ncfg = cfg.native(seed)
    if cam is None:
        ncfg.rays_f64 = int(o_d.dtype == t.float64)
    if occupancy is not None:
        occ_geom, occ_bits = occupancy.native_geom(), occupancy.device_bits()
    else:
        occ_geom, occ_bits = None, None
    rgb = out if out is not None else D.empty((n, 3), t.float32)
    st = stats if stats is not None else t.zeros(4, dtype=t.int64, device=rgb.device)
    trace = tcount = None
    if trace_capacity:
        trace = D.empty((trace_capacity * N.TRACE_DTYPE.itemsize,), t.uint8)
        tcount = t.zeros(1, dtype=t.int64, device=rgb.device)
    if ws is None:
        ws = D.workspace(_render_ws_bytes(grid, ncfg, n))
    if caller:
        errors = []
        fn = _field_callback(grid, errors)
        status = N.lib().gf_render_rays_field(
            fn, None, _box_geom(grid.aabb), occ_geom, N.ptr(occ_bits), ncfg, ccam, N.ptr(o_d), N.ptr(d_d),
            int(ray_offset), int(block_stride), int(n), N.ptr(rgb), N.ptr(st), N.ptr(trace), int(trace_capacity),
            N.ptr(tcount), N.ptr(ws), ws.numel(), D.stream_handle())
        if errors:
            raise errors[0]
        N.check(status, "render_rays")
    elif analytic:
        N.check(N.lib().gf_render_rays_analytic(
            grid.native(), occ_geom, N.ptr(occ_bits), ncfg, ccam, N.ptr(o_d), N.ptr(d_d), int(ray_offset),
            int(block_stride), int(n), N.ptr(rgb), N.ptr(st), N.ptr(trace), int(trace_capacity), N.ptr(tcount),
            N.ptr(ws), ws.numel(), D.stream_handle()), "render_rays")
    else:
        N.check(N.lib().gf_render_rays(
            grid.native_arch(), grid.native_geom(), N.ptr(packed), N.PRECISION[p], occ_geom, N.ptr(occ_bits), ncfg,
            ccam, N.ptr(o_d), N.ptr(d_d), int(ray_offset), int(block_stride), int(n), N.ptr(rgb), N.ptr(st),
            N.ptr(trace), int(trace_capacity), N.ptr(tcount), N.ptr(ws), ws.numel(), D.stream_handle()), "render_rays")
    tr = None
    if trace_capacity:
        cnt = int(tcount.item())
        if cnt > trace_capacity:
            raise RuntimeError(f"trace capacity {trace_capacity} too small for {cnt} samples")
        tr = np.frombuffer(trace[: cnt * N.TRACE_DTYPE.itemsize].cpu().numpy().tobytes(), dtype=N.TRACE_DTYPE)
    return rgb, st, tr


def _stats_from(st) -> RenderStats:
    v = [int(x) for x in st.cpu().tolist()]
    return RenderStats(total_queries=v[0], ess_skipped=v[1], ert_terminated_rays=v[2], n_rays=v[3])


def render_rays(field, occupancy, origins, directions, cfg: RenderConfig, seed: int = 0, workers: int = 1,
                precision=None):
    """render.py:351-384.  ``workers`` is accepted for API compatibility; the
    device result is identical for any value (ray blocks keep their own
    jitter streams)."""
    grid = _field_grid(field)
    o = np.asarray(origins)
    d = np.asarray(directions)
    # render.py:368-369 upcasts to float64: the slab test runs on those values
    # and the samples on their float32 roundings (render.py:304-306).
    # float32 rays go as they are (their float64 upcast is exact); anything
    # else goes as float64.
    f32 = o.dtype == np.float32 and d.dtype == np.float32
    dt = np.float32 if f32 else np.float64
    o = np.ascontiguousarray(o, dtype=dt).reshape(-1, 3)
    d = np.ascontiguousarray(d, dtype=dt).reshape(-1, 3)
    rgb, st, _ = render_rays_device(grid, occupancy, cfg, seed, origins=o, directions=d, precision=precision)
    return rgb.cpu().numpy(), _stats_from(st)


def render_image(field, occupancy, cam: Camera, cfg: RenderConfig, seed: int = 0, workers: int = 1,
                 precision=None):
    """render.py:387-400: full frame; stats.wall_ms covers ray generation
    through the image landing in host memory."""
    t_start = time.perf_counter()
    grid = _field_grid(field)
    t = D.require_cuda()
    n = cam.width * cam.height
    ncfg = cfg.native(seed)
    ws_bytes = _render_ws_bytes(grid, ncfg, n)
    c = _render_context(n, ws_bytes)
    if not c.get("stats_zero"):  # normally zeroed at the end of the previous call, off the critical path
        c["stats"].zero_()
    c["stats_zero"] = False
    rgb, st, _ = render_rays_device(grid, occupancy, cfg, seed, cam=cam, precision=precision, out=c["rgb"],
                                    stats=c["stats"], ws=c["ws"])
    # fresh pinned block per call (torch's caching host allocator recycles it
    # once the returned array is dropped), so the result needs no extra copy
    host = t.empty(rgb.shape, dtype=t.float32, pin_memory=True)
    host.copy_(rgb, non_blocking=True)
    c["host_stats"].copy_(st, non_blocking=True)
    c["stats"].zero_()  # stream-ordered after the copy: ready for the next call
    t.cuda.current_stream().synchronize()
    c["stats_zero"] = True
    stats = _stats_from(c["host_stats"])
    stats.wall_ms = (time.perf_counter() - t_start) * 1000.0
    return host.numpy().reshape(cam.height, cam.width, 3), stats


def shard_capacity(n_rays: int, world: int) -> int:
    """Rows of each rank's padded shard buffer (whole 4096-ray blocks)."""
    n_blocks = (n_rays + RAY_BLOCK - 1) // RAY_BLOCK
    return ((n_blocks + world - 1) // world) * RAY_BLOCK


class ShardedFrame:
    """Buffers of one rank's part of a multi-GPU frame of ``n_rays`` rays.

    Rank r renders the interleaved 4096-ray blocks of ``shard_rays`` into
    ``local[:n_local]`` (each block keeps its own jitter stream, render.py:
    371-375, so any split reproduces the single-GPU image bit for bit);
    ``gather`` all-gathers the padded shards, restores image order
    (``unshard_index``) into ``image`` and sums the 4 ``RenderStats``
    counters across ranks.  The collective is the only exchange (SURVEY
    §8e).  Works on CUDA tensors over NCCL and on CPU tensors over gloo."""

    def __init__(self, n_rays: int, rank: int, world: int, device=None, channels: int = 3):
        import torch

        self.n_rays, self.rank, self.world = int(n_rays), int(rank), int(world)
        self.offset, self.stride, self.n_local = shard_rays(self.n_rays, self.rank, self.world)
        self.cap = shard_capacity(self.n_rays, self.world)
        dev = device if device is not None else torch.device("cpu")
        self.local = torch.zeros((self.cap, channels), dtype=torch.float32, device=dev)
        self.gathered = torch.empty((self.world * self.cap, channels), dtype=torch.float32, device=dev)
        self.image = torch.empty((self.n_rays, channels), dtype=torch.float32, device=dev)
        self.index = torch.from_numpy(unshard_index(self.n_rays, self.world)).to(dev)
        self.stats = torch.zeros(4, dtype=torch.int64, device=dev)

    def gather(self, group=None):
        """All-gather the shards and assemble the frame (``image``, ``stats``)."""
        import torch
        import torch.distributed as dist

        if dist.get_backend(group) == "nccl":
            dist.all_gather_into_tensor(self.gathered, self.local, group=group)
        else:
            dist.all_gather(list(self.gathered.view(self.world, self.cap, -1).unbind(0)), self.local, group=group)
        torch.index_select(self.gathered, 0, self.index, out=self.image)
        dist.all_reduce(self.stats, group=group)
        return self.image, self.stats


_dist_ctx = threading.local()


def render_image_distributed(field, occupancy, cam: Camera, cfg: RenderConfig, seed: int = 0, group=None,
                             precision=None, frame: ShardedFrame | None = None, ws=None):
    """Multi-GPU render_image (one process per GPU, torch.distributed/NCCL).

    Each rank marches its interleaved 4096-ray blocks (``shard_rays``) with the
    blocks' own jitter streams, so the assembled image is bit-identical to the
    single-GPU render; the only exchange is one all-gather of the shards
    (float32 RGB) plus a 4-counter all-reduce (``ShardedFrame.gather``).
    Returns the (H, W, 3) image as a CUDA tensor on every rank and the global
    RenderStats."""
    import torch.distributed as dist

    D.require_cuda()
    grid = _field_grid(field)
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    n = cam.width * cam.height
    if frame is None:
        cache = getattr(_dist_ctx, "frames", None)
        if cache is None:
            cache = _dist_ctx.frames = {}
        key = (D.torch().cuda.current_device(), n, rank, world)
        frame = cache.get(key)
        if frame is None:
            frame = cache[key] = ShardedFrame(n, rank, world, D.device())
    frame.stats.zero_()
    if frame.n_local:
        if ws is None:
            ws_bytes = _render_ws_bytes(grid, cfg.native(seed), frame.n_local)
            ws = getattr(frame, "ws", None)
            if ws is None or ws.numel() < ws_bytes:
                ws = frame.ws = D.workspace(ws_bytes)
        render_rays_device(grid, occupancy, cfg, seed, cam=cam, ray_offset=frame.offset, n_rays=frame.n_local,
                           block_stride=frame.stride, precision=precision, out=frame.local[: frame.n_local],
                           stats=frame.stats, ws=ws)
    img, st = frame.gather(group)
    return img.view(cam.height, cam.width, 3), _stats_from(st)


def compute_psnr(a, b) -> float:
    """render.py:403-413."""
    a, b = np.asarray(a), np.asarray(b)
    if a.shape != b.shape:
        raise ValueError(f"image shapes differ: {a.shape} vs {b.shape}")
    mse = float(np.mean((a.astype(np.float64) - b.astype(np.float64)) ** 2))
    return float("inf") if mse == 0.0 else 10.0 * np.log10(1.0 / mse)
