"""CPU oracle for the KiloNeRF render / network-query hot path.

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
module, and only as the checker or the timed CPU baseline.  The product
(``paper_2103_13744_b200``) never calls into it.

This is a numpy restatement of the reference package ``gridfield``
(/root/reference/pkg/src/gridfield), written stage by stage so each device
kernel has a CPU twin to compare against.  Every function cites the reference
lines whose arithmetic it reproduces, including the numpy type-promotion rules
that decide which operations happen in float64 versus float32.  It is pinned
against golden vectors produced by the reference itself
(tests/golden/make_golden.py -> tests/golden/*.npz; tests/test_oracle_golden.py).

Third-party arithmetic: numpy 2.3.5 (float32 SIMD sin/cos/exp/expm1) and the
OpenBLAS sgemm behind ``np.matmul``; the grouped evaluation keeps the
reference's power-of-two segment stacking so the matmul shapes, and therefore
the sgemm results, are the same as the reference's.
"""

from __future__ import annotations

from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass, field

import numpy as np

RAY_BLOCK = 4096  # render.py:22

LAYER_ORDER = ("trunk", "density", "feature", "direction", "color")


# --------------------------------------------------------------------------
# lattice parameters (mlp.py:30-87, 198-219; grid.py:80-99)
# --------------------------------------------------------------------------


def layer_manifest(hidden_layers=4, width=32, pos_dim=63, dir_dim=27, view_width=None, skip_layer=None):
    """(name, in, out) list; mlp.py:73-84."""
    v = view_width or width
    out = [("trunk0", pos_dim, width)]
    for k in range(1, hidden_layers - 2):
        out.append((f"trunk{k}", width + pos_dim if k == skip_layer else width, width))
    out += [("density", width, 1), ("feature", width, width), ("direction", width + dir_dim, v), ("color", v, 3)]
    return out


@dataclass
class Lattice:
    """Everything the oracle needs to answer field queries for a NetworkGrid."""

    b_min: np.ndarray
    b_max: np.ndarray
    res: np.ndarray
    manifest: list
    weights: dict
    biases: dict
    pos_freqs: int = 10
    dir_freqs: int = 4
    include_raw: bool = True
    skip_layer: int | None = None

    @property
    def n_cells(self) -> int:
        return int(np.prod(self.res))

    @property
    def trunk_layers(self) -> int:
        return sum(1 for n, _, _ in self.manifest if n.startswith("trunk"))


def init_lattice(b_min, b_max, res, seed, hidden_layers=4, width=32, dtype=np.float32) -> Lattice:
    """mlp.py:198-219: U(+-1/sqrt(fan_in)) per layer in manifest order, zero biases."""
    res = np.asarray(res, dtype=np.int64).reshape(3)
    n = int(np.prod(res))
    gen = np.random.default_rng(seed)
    manifest = layer_manifest(hidden_layers, width)
    w, b = {}, {}
    for name, fan_in, fan_out in manifest:
        lim = 1.0 / np.sqrt(fan_in)
        w[name] = gen.uniform(-lim, lim, size=(n, fan_out, fan_in)).astype(dtype)
        b[name] = np.zeros((n, fan_out), dtype=dtype)
    return Lattice(np.asarray(b_min, np.float64), np.asarray(b_max, np.float64), res, manifest, w, b)


def lattice_from_grid(grid) -> Lattice:
    """Adapter for any object shaped like gridfield.NetworkGrid."""
    arch = grid.arch
    manifest = [(s.name, s.in_dim, s.out_dim) for s in arch.layers()]
    enc = grid.encoding
    return Lattice(
        np.asarray(grid.aabb.b_min, np.float64),
        np.asarray(grid.aabb.b_max, np.float64),
        np.asarray(grid.resolution, np.int64),
        manifest,
        dict(grid.params.weights),
        dict(grid.params.biases),
        enc.num_freqs_position,
        enc.num_freqs_direction,
        enc.include_raw_input,
        arch.skip_layer,
    )


# --------------------------------------------------------------------------
# pointwise primitives (core.py)
# --------------------------------------------------------------------------


def clamp_into_box(p, b_min, b_max):
    """core.py:52-68.  np.clip promotes float32 points against float64 bounds,
    so the clamp happens in f64 and is cast back; one nextafter step inward
    repairs a cast that rounded outside the box."""
    p = np.asarray(p)
    c = np.clip(p, b_min, b_max).astype(p.dtype)
    over = c > b_max
    if over.any():
        c[over] = np.nextafter(c[over], p.dtype.type(-np.inf))
    under = c < b_min
    if under.any():
        c[under] = np.nextafter(c[under], p.dtype.type(np.inf))
    return c


class OutOfBounds(ValueError):
    pass


def bin_cells(x, b_min, b_max, res):
    """core.py:79-104 (+ the flatten at 107-112).  Returns the flat x-major cell
    index; float64 divide by the f64 cell size, floor, clamp to r-1."""
    res = np.asarray(res, dtype=np.int64)
    x = np.asarray(x)
    bad = (x < b_min) | (x > b_max)
    if bad.any():
        first = np.argwhere(bad)[0]
        axis = int(first[-1])
        val = x[tuple(first)]
        bound = b_min[axis] if val < b_min[axis] else b_max[axis]
        raise OutOfBounds(f"point outside bounds: component {axis} is {val!r}, bound {bound!r}")
    step = (b_max - b_min) / res.astype(np.float64)
    ijk = np.minimum(np.floor((x - b_min) / step).astype(np.int64), res - 1)
    return ijk[..., 0] + res[0] * (ijk[..., 1] + res[1] * ijk[..., 2])


def encode(v, n_freqs, include_raw=True):
    """core.py:132-152: [v, sin(v*f_0), cos(v*f_0), ..., sin(v*f_L-1), cos(..)]
    with f_k = float(2**k * pi) cast to the input dtype (float32 product)."""
    v = np.asarray(v)
    parts = [v] if include_raw else []
    if n_freqs:
        f = ((2.0 ** np.arange(n_freqs)) * np.pi)[:, None].astype(v.dtype)
        a = v[..., None, :] * f
        sc = np.stack([np.sin(a), np.cos(a)], axis=-2)
        parts.append(sc.reshape(*v.shape[:-1], 2 * n_freqs * v.shape[-1]))
    return np.concatenate(parts, axis=-1).astype(v.dtype)


def alpha_of(sigma, delta):
    """core.py:187-194."""
    return -np.expm1(-np.asarray(sigma) * np.asarray(delta))


# --------------------------------------------------------------------------
# per-cell network (mlp.py:222-266)
# --------------------------------------------------------------------------


def _dense(w, b, x):
    return np.matmul(x, np.swapaxes(w, -1, -2)) + b[..., None, :]


def _logistic(z):
    out = np.empty_like(z)
    nonneg = z >= 0
    out[nonneg] = 1.0 / (1.0 + np.exp(-z[nonneg]))
    e = np.exp(z[~nonneg])
    out[~nonneg] = e / (1.0 + e)
    return out


def cell_forward(w, b, xe, de, trunk_layers=2, skip_layer=None):
    """mlp.py:238-266 on parameter dicts whose arrays share a leading stack."""
    h = np.maximum(_dense(w["trunk0"], b["trunk0"], xe), 0.0)
    for k in range(1, trunk_layers):
        inp = np.concatenate([xe, h], axis=-1) if k == skip_layer else h
        h = np.maximum(_dense(w[f"trunk{k}"], b[f"trunk{k}"], inp), 0.0)
    sigma = np.maximum(_dense(w["density"], b["density"], h)[..., 0], 0.0)
    feat = _dense(w["feature"], b["feature"], h)
    g = np.maximum(_dense(w["direction"], b["direction"], np.concatenate([feat, de], axis=-1)), 0.0)
    return _logistic(_dense(w["color"], b["color"], g)), sigma


# --------------------------------------------------------------------------
# grouping (batched.py:60-151)
# --------------------------------------------------------------------------


@dataclass
class Groups:
    order: np.ndarray
    inverse: np.ndarray
    offsets: np.ndarray


def group(keys, n_keys) -> Groups:
    """batched.py:60-85: stable counting sort by key."""
    keys = np.asarray(keys)
    if len(keys) and (keys.min() < 0 or keys.max() >= n_keys):
        raise ValueError(
            f"network index out of range [0, {n_keys}): min={keys.min()} max={keys.max()}"
        )
    order = np.argsort(keys, kind="stable")
    inverse = np.empty_like(order)
    inverse[order] = np.arange(len(order))
    offsets = np.concatenate([[0], np.cumsum(np.bincount(keys, minlength=n_keys))])
    return Groups(order, inverse, offsets)


def _stacks(offsets):
    """batched.py:88-117: segments grouped by power-of-two length class."""
    lengths = np.diff(offsets)
    used = np.flatnonzero(lengths)
    if not len(used):
        return
    cls = np.ceil(np.log2(np.maximum(lengths[used], 1))).astype(int)
    cls[lengths[used] == 1] = 0
    for c in np.unique(cls):
        cells = used[cls == c]
        ln = lengths[cells]
        width = int(ln.max())
        rows = offsets[cells][:, None] + np.arange(width)[None, :]
        if ln.min() == width:
            yield cells, rows, None
        else:
            valid = np.arange(width)[None, :] < ln[:, None]
            yield cells, np.where(valid, rows, 0), valid


def grouped_eval(lat: Lattice, pos_sorted, dir_sorted, groups: Groups):
    """batched.py:120-151: evaluate each segment with its own cell network and
    return results in the original query order."""
    n = len(groups.order)
    dtype = lat.weights["trunk0"].dtype
    rgb = np.zeros((n, 3), dtype=dtype)
    sig = np.zeros(n, dtype=dtype)
    for cells, rows, valid in _stacks(groups.offsets):
        p = pos_sorted[rows].astype(dtype)
        d = dir_sorted[rows].astype(dtype)
        if valid is not None:
            p[~valid] = 0.0
            d[~valid] = 0.0
        xe = encode(p, lat.pos_freqs, lat.include_raw)
        de = encode(d, lat.dir_freqs, lat.include_raw)
        w = {k: v[cells] for k, v in lat.weights.items()}
        b = {k: v[cells] for k, v in lat.biases.items()}
        c, s = cell_forward(w, b, xe, de, lat.trunk_layers, lat.skip_layer)
        if valid is None:
            rgb[rows.ravel()] = c.reshape(-1, 3)
            sig[rows.ravel()] = s.reshape(-1)
        else:
            rgb[rows[valid]] = c[valid]
            sig[rows[valid]] = s[valid]
    return rgb[groups.inverse], sig[groups.inverse]


def bulk_query_inputs(b_min, b_max, n, seed=0):
    """Reference bench.py:108-112 input recipe (BASELINE config 5): uniform
    float32 positions in the box, normalised float32 normal directions."""
    rng = np.random.default_rng(seed)
    b_min = np.asarray(b_min, np.float64)
    span = (np.asarray(b_max, np.float64) - b_min).astype(np.float32)
    pts = b_min.astype(np.float32) + rng.random((n, 3), dtype=np.float32) * span
    dirs = rng.normal(size=(n, 3)).astype(np.float32)
    dirs /= np.linalg.norm(dirs, axis=-1, keepdims=True)
    return pts, dirs


def query_points(lat: Lattice, positions, directions):
    """grid.py:50-56: bin at network resolution, group, evaluate."""
    keys = bin_cells(positions, lat.b_min, lat.b_max, lat.res)
    g = group(keys, lat.n_cells)
    return grouped_eval(lat, np.ascontiguousarray(positions[g.order]), np.ascontiguousarray(directions[g.order]), g)


# --------------------------------------------------------------------------
# occupancy (occupancy.py:65-79)
# --------------------------------------------------------------------------


@dataclass
class Occupancy:
    b_min: np.ndarray
    b_max: np.ndarray
    res: np.ndarray
    bits: np.ndarray  # packed little-endian uint8

    def lookup(self, x):
        f = bin_cells(x, self.b_min, self.b_max, self.res)
        return ((self.bits[f >> 3] >> (f & 7)) & 1).astype(bool)


def probe_points(b_min, b_max, res):
    """occupancy.py:112-123: every cell's 3x3x3 probe lattice in float64
    (lo = b_min + i*cell, then lo + offset*cell), cast to float32 and clipped
    into the box.  Returns (n_cells*27, 3) float32, cell-major, probes in
    meshgrid 'ij' order."""
    b_min = np.asarray(b_min, np.float64)
    b_max = np.asarray(b_max, np.float64)
    res = np.asarray(res, np.int64)
    n = int(np.prod(res))
    cell = (b_max - b_min) / res
    flat = np.arange(n)
    i3 = np.stack([flat % res[0], (flat // res[0]) % res[1], flat // (res[0] * res[1])], axis=-1)
    lo = b_min + i3 * cell
    offs = np.stack(np.meshgrid(*([np.array([0.0, 0.5, 1.0])] * 3), indexing="ij"), axis=-1).reshape(-1, 3)
    pts = (lo[:, None, :] + offs[None, :, :] * cell).astype(np.float32).reshape(-1, 3)
    return clamp_into_box(pts, b_min, b_max)


def extract_occupancy(density, b_min, b_max, res, tau, chunk_cells=16384):
    """occupancy.py:94-128: occupied iff any probe density > tau (numpy's
    comparison semantics: float32 densities against a Python scalar compare in
    float32).  Returns the packed little-endian bitmap."""
    res = np.asarray(res, np.int64)
    n = int(np.prod(res))
    pts = probe_points(b_min, b_max, res)
    occ = np.zeros(n, bool)
    for s in range(0, n, chunk_cells):
        e = min(n, s + chunk_cells)
        sigma = np.asarray(density(pts[27 * s : 27 * e]))
        occ[s:e] = (sigma.reshape(e - s, 27) > tau).any(axis=1)
    return np.packbits(occ, bitorder="little")


# --------------------------------------------------------------------------
# rays and marching (render.py:139-400)
# --------------------------------------------------------------------------


def pixel_rays(width, height, fx, fy, cx, cy, c2w):
    """render.py:139-148, restated per component: u,v in f64; world direction
    R.[u,v,1] in f64; normalise by the f64 Euclidean norm; cast to float32."""
    c2w = np.asarray(c2w, np.float64)
    u = (np.arange(width) + 0.5 - cx) / fx
    v = (np.arange(height) + 0.5 - cy) / fy
    uu, vv = np.meshgrid(u, v)
    uu, vv = uu.ravel(), vv.ravel()
    r = c2w[:3, :3]
    d = np.stack([uu * r[i, 0] + vv * r[i, 1] + r[i, 2] for i in range(3)], axis=-1)
    n = np.sqrt(d[:, 0] * d[:, 0] + d[:, 1] * d[:, 1] + d[:, 2] * d[:, 2])
    d = d / n[:, None]
    o = np.broadcast_to(c2w[:3, 3], d.shape)
    return o.astype(np.float32), d.astype(np.float32)


def slab(o, d, b_min, b_max):
    """render.py:151-171 slab test in f64; parallel components use the inside test."""
    o = np.asarray(o, np.float64)
    d = np.asarray(d, np.float64)
    with np.errstate(divide="ignore", invalid="ignore"):
        ta = (b_min - o) / d
        tb = (b_max - o) / d
    lo = np.minimum(ta, tb)
    hi = np.maximum(ta, tb)
    par = d == 0
    inside = (o >= b_min) & (o <= b_max)
    lo = np.where(par, np.where(inside, -np.inf, np.inf), lo)
    hi = np.where(par, np.where(inside, np.inf, -np.inf), hi)
    return np.maximum(lo.max(axis=-1), 0.0), hi.min(axis=-1)


@dataclass
class MarchConfig:
    k: int = 384
    epsilon: float = 0.01
    background: tuple = (1.0, 1.0, 1.0)
    ert_chunk: int = 32
    stratified: bool = True


@dataclass
class Counters:
    total_queries: int = 0
    ess_skipped: int = 0
    ert_terminated_rays: int = 0
    n_rays: int = 0
    rounds: list = field(default_factory=list)  # optional per-round trace

    def add(self, o: "Counters"):
        self.total_queries += o.total_queries
        self.ess_skipped += o.ess_skipped
        self.ert_terminated_rays += o.ert_terminated_rays
        self.n_rays += o.n_rays
        self.rounds.extend(o.rounds)


def march_block(query, b_min, b_max, occ, o64, d64, cfg: MarchConfig, gen, ray_base=0, trace=False):
    """render.py:287-348 for one ray block.  ``query(pos, dir) -> (rgb, sigma)``.

    Promotion rules reproduced: sample distance
    ``t = f64(t0_32) + (f64(j) + f64(jitter_32)) * f64(seg_32)``, position
    ``f32(f64(o32) + t * f64(d32))``; compositing entirely in float32; the ERT
    threshold compares float32 transmittance with the epsilon as numpy does
    for a Python float (NEP 50: the scalar adopts float32).
    """
    n = len(o64)
    ctr = Counters(n_rays=n)
    t0, t1 = slab(o64, d64, b_min, b_max)
    hit = t1 > t0
    seg = np.where(hit, (t1 - t0) / cfg.k, 0.0).astype(np.float32)
    if cfg.stratified:
        jit = gen.random((n, cfg.k), dtype=np.float32)
    else:
        jit = np.full((n, cfg.k), 0.5, dtype=np.float32)
    acc = np.zeros((n, 3), np.float32)
    trans = np.ones(n, np.float32)
    alive = hit.copy()
    dead_early = np.zeros(n, bool)
    o32, d32, t0_32 = o64.astype(np.float32), d64.astype(np.float32), t0.astype(np.float32)
    for s0 in range(0, cfg.k, cfg.ert_chunk):
        if not alive.any():
            break
        rays = np.flatnonzero(alive)
        slots = np.arange(s0, min(s0 + cfg.ert_chunk, cfg.k))
        m = len(slots)
        t = t0_32[rays, None] + (slots[None, :] + jit[rays][:, slots]) * seg[rays, None]
        p = (o32[rays, None, :] + t[..., None] * d32[rays, None, :]).astype(np.float32)
        p = clamp_into_box(p, b_min, b_max).reshape(-1, 3)
        keep = occ.lookup(p) if occ is not None else np.ones(len(p), bool)
        sig = np.zeros(len(p), np.float32)
        col = np.zeros((len(p), 3), np.float32)
        nq = int(keep.sum())
        ctr.ess_skipped += len(p) - nq
        if nq:
            c, s = query(p[keep], np.repeat(d32[rays], m, axis=0)[keep])
            col[keep] = c
            sig[keep] = s
            ctr.total_queries += nq
        if trace:
            kk = np.flatnonzero(keep)
            ctr.rounds.append((s0, ray_base + rays[kk // m], slots[kk % m], p[keep]))
        sig = sig.reshape(len(rays), m)
        col = col.reshape(len(rays), m, 3)
        a = alpha_of(sig, seg[rays, None])
        run = np.cumprod(1.0 - a, axis=1)
        before = np.concatenate([np.ones_like(run[:, :1]), run[:, :-1]], axis=1)
        acc[rays] += trans[rays, None] * (before[..., None] * a[..., None] * col).sum(axis=1)
        trans[rays] = trans[rays] * run[:, -1]
        if cfg.epsilon > 0.0:
            gone = rays[trans[rays] < cfg.epsilon]
            if s0 + m < cfg.k:
                dead_early[gone] = True
            alive[gone] = False
    ctr.ert_terminated_rays = int(dead_early.sum())
    out = acc + trans[:, None] * np.asarray(cfg.background, np.float32)[None, :]
    return np.clip(out, 0.0, 1.0), trans, ctr


def render_rays(query, b_min, b_max, occ, origins, directions, cfg: MarchConfig, seed=0, workers=1, trace=False):
    """render.py:351-384: fixed 4096-ray blocks, jitter stream per block from
    ``SeedSequence([seed, block_start])``, thread pool over blocks."""
    o = np.asarray(origins, np.float64).reshape(-1, 3)
    d = np.asarray(directions, np.float64).reshape(-1, 3)
    n = len(o)
    starts = list(range(0, n, RAY_BLOCK))

    def one(s):
        gen = np.random.default_rng(np.random.SeedSequence([seed, s]))
        e = min(s + RAY_BLOCK, n)
        return march_block(query, b_min, b_max, occ, o[s:e], d[s:e], cfg, gen, ray_base=s, trace=trace)

    if workers > 1 and len(starts) > 1:
        with ThreadPoolExecutor(max_workers=workers) as pool:
            res = list(pool.map(one, starts))
    else:
        res = [one(s) for s in starts]
    rgb = np.zeros((n, 3), np.float32)
    tot = Counters()
    for s, (c, _, ctr) in zip(starts, res):
        rgb[s : s + len(c)] = c
        tot.add(ctr)
    return rgb, tot


def render_image(lat: Lattice, occ: Occupancy | None, cam, cfg: MarchConfig, seed=0, workers=1, trace=False):
    """render.py:387-400 for a NetworkGrid field; ``cam`` has width, height,
    fx, fy, cx, cy, c2w."""
    o, d = pixel_rays(cam.width, cam.height, cam.fx, cam.fy, cam.cx, cam.cy, cam.c2w)
    q = lambda p, dd: query_points(lat, p, dd)
    rgb, ctr = render_rays(q, lat.b_min, lat.b_max, occ, o, d, cfg, seed, workers, trace)
    return rgb.reshape(cam.height, cam.width, 3), ctr


def composite(colors, alphas):
    """render.py:269-284 (front-to-back blending, batch dims allowed)."""
    colors = np.asarray(colors)
    alphas = np.asarray(alphas)
    if colors.shape[-2] == 0:
        return np.zeros((*alphas.shape[:-1], 3), colors.dtype), np.ones(alphas.shape[:-1], colors.dtype)
    run = np.cumprod(1.0 - alphas, axis=-1)
    before = np.concatenate([np.ones_like(run[..., :1]), run[..., :-1]], axis=-1)
    return (before[..., None] * alphas[..., None] * colors).sum(axis=-2), run[..., -1]
