"""Training-loop pieces of gridfield.train on the device (mirror of
/root/reference/pkg/src/gridfield/train.py).

What runs where:
* ``photometric_loss_and_grads`` (train.py:212-288): grouping, the fp32
  grouped forward, dense compositing + float64 loss + the rest-of-ray
  gradient recurrence (gf_photometric_loss), and the fused per-cell backward
  (gf_grouped_backward) all run on the device; the regularisation gradient is
  folded in on the device (gf_axpy) before one download of the gradients.
* ``distill_step`` (train.py:341-390): the teacher query, the student's
  grouped forward / backward, the loss terms (gf_distill_loss) and Adam run
  on the device.  The in-cell sample draws use the caller's numpy Generator,
  as in the reference, so the stream of random numbers is the same.
* ``adam_update`` (train.py:130-143) and ``regularization_term``
  (train.py:146-160): one kernel per parameter array (gf_adam_update,
  gf_sum_squares, gf_axpy).  Parameters stay numpy arrays in place, as the
  reference API requires; each step uploads them and writes them back.
* ``prepare_ray_samples`` (train.py:175-209): on the device; the caller's
  numpy Generator stream (PCG64) is reproduced there and the Generator is
  advanced exactly as rng.random((n, k), float32) would.
* ``density_probe`` (train.py:577-586): recognised by ``extract_occupancy``,
  which then runs the probe lattice on the device in one call.

``photometric_step``, ``train_photometric_loop``, ``run_distill_loop``,
``evaluate_psnr`` and ``mean_free_space_density`` are the reference's drivers
over these device steps (any dataset object with the reference dataset's
``indices`` / ``cameras`` / ``images`` / ``aabb`` works).  The device path
computes in float32, the reference's parameter dtype; float64 parameter stacks
are rejected.  Dataset generation, the pipeline driver (``run_pipeline``) and
CLI reporting are out of scope.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _device as D
from . import _native as N
from . import mlp
from .batched import GroupedLayout, QueryBatch, group_by_network, grouped_backward_device, grouped_forward_device
from .core import Aabb, clip_into

REGULARIZED_LAYERS = ("direction", "color")  # train.py:33


@dataclass
class TrainConfig:
    """train.py:36-110 (the fields the device steps read, same defaults)."""

    batch_size_pixels: int = 8192
    learning_rate: float = 5e-4
    lr_final_fraction: float = 0.1
    l2_reg_weight: float = 1e-6
    teacher_steps: int = 600_000
    distill_steps: int = 150_000
    finetune_steps: int = 1_000_000
    distill_points_per_cell: int = 32
    distill_alpha_weight: float = 1.0
    distill_delta: float | None = None
    k_train: int = 384
    density_noise_std: float = 0.0
    seed: int = 0
    adam_beta1: float = 0.9
    adam_beta2: float = 0.999
    adam_eps: float = 1e-8
    grid_max_dim: int = 16
    occupancy_factor: int = 16
    occupancy_tau: float = 10.0
    teacher_hidden_layers: int = 10
    teacher_hidden_width: int = 256
    teacher_direction_width: int = 128
    teacher_skip_layer: int | None = 5
    student_hidden_layers: int = 4
    student_hidden_width: int = 32
    background: tuple = (1.0, 1.0, 1.0)
    log_every: int = 100

    @classmethod
    def desk_preset(cls, seed: int = 0) -> "TrainConfig":
        """train.py:75-91: the scaled-down schedule (128x128 toy scenes); its
        6 x 96 skip-2 teacher runs on the generic device MLP."""
        return cls(batch_size_pixels=640, teacher_steps=3200, distill_steps=1200, finetune_steps=2600,
                   distill_points_per_cell=24, k_train=128, occupancy_factor=4, teacher_hidden_layers=6,
                   teacher_hidden_width=96, teacher_direction_width=64, teacher_skip_layer=2, seed=seed)

    def teacher_architecture(self, encoding) -> mlp.MlpArchitecture:
        return mlp.teacher_architecture(hidden_layers=self.teacher_hidden_layers,
                                        hidden_width=self.teacher_hidden_width,
                                        direction_layer_width=self.teacher_direction_width,
                                        skip_layer=self.teacher_skip_layer,
                                        position_input_dim=encoding.position_dim,
                                        direction_input_dim=encoding.direction_dim)

    def student_architecture(self, encoding) -> mlp.MlpArchitecture:
        return mlp.MlpArchitecture(hidden_layers=self.student_hidden_layers, hidden_width=self.student_hidden_width,
                                   position_input_dim=encoding.position_dim,
                                   direction_input_dim=encoding.direction_dim)


def lr_schedule(step: int, base_lr: float, horizon: int, final_fraction: float = 0.1) -> float:
    """train.py:112-116."""
    if horizon <= 0:
        return base_lr
    return float(base_lr * final_fraction ** (step / horizon))


class AdamState:
    """train.py:119-127.  The moments live on the device between steps
    (flat float32, MlpParams.arrays() order); ``m`` / ``v`` read them back
    into the host containers on access."""

    def __init__(self, m: mlp.MlpParams, v: mlp.MlpParams, step: int = 0):
        self._m, self._v = m, v
        self.step = step
        self._dev = None  # (m_flat, v_flat) on the device once adam_update ran

    @classmethod
    def for_params(cls, params: mlp.MlpParams) -> "AdamState":
        return cls(m=mlp.map_params(np.zeros_like, params), v=mlp.map_params(np.zeros_like, params))

    def _sync(self):
        if self._dev is not None:
            _scatter_flat(D.to_host(self._dev[0]), self._m)
            _scatter_flat(D.to_host(self._dev[1]), self._v)

    @property
    def m(self) -> mlp.MlpParams:
        self._sync()
        return self._m

    @property
    def v(self) -> mlp.MlpParams:
        self._sync()
        return self._v


def _flat_size(params: mlp.MlpParams) -> int:
    return sum(int(a.size) for _, a in params.arrays())


def _scatter_flat(flat: np.ndarray, params: mlp.MlpParams):
    off = 0
    for _, a in params.arrays():
        a[...] = flat[off : off + a.size].reshape(a.shape)
        off += a.size


class DeviceGrads(mlp.MlpParams):
    """Parameter gradients resident on the device (one flat buffer in
    MlpParams.arrays() order).  ``weights`` / ``biases`` are the reference's
    host arrays, downloaded on first access; ``adam_update`` consumes the
    device buffer directly, so a training step that never looks at the
    gradients on the host moves none of them over PCIe."""

    def __init__(self, arch, flat, shapes):
        self.arch = arch
        self._flat = flat
        self._shapes = shapes  # [(kind, name, shape)] in arrays() order
        self._w = self._b = None

    @property
    def materialized(self) -> bool:
        return self._w is not None

    def _materialize(self):
        if self._w is None:
            host = D.to_host(self._flat)  # the arrays view this pinned buffer
            w, b, off = {}, {}, 0
            for kind, name, shape in self._shapes:
                n = int(np.prod(shape))
                (w if kind == "w" else b)[name] = D.tracked(host[off : off + n].reshape(shape))
                off += n
            self._w, self._b = w, b
            self._dev_flat = (mlp.MlpParams.fingerprint(self), self._flat)

    @property
    def weights(self):
        self._materialize()
        return self._w

    @weights.setter
    def weights(self, v):
        self._w = v

    @property
    def biases(self):
        self._materialize()
        return self._b

    @biases.setter
    def biases(self, v):
        self._b = v


def device_flat(params: mlp.MlpParams):
    """Flat float32 device copy of ``params`` (arrays() order): the cached one
    when the host arrays are unchanged since it was made, else an upload."""
    if isinstance(params, DeviceGrads) and not params.materialized:
        return params._flat
    hit = getattr(params, "_dev_flat", None)
    if hit is not None and hit[0] == params.fingerprint():
        return hit[1]
    t = D.require_cuda()
    flat = D.empty((_flat_size(params),), t.float32)
    off = 0
    for _, a in params.arrays():
        flat[off : off + a.size].copy_(t.from_numpy(np.ascontiguousarray(a, dtype=np.float32).reshape(-1)))
        off += a.size
    return flat


def _f32(x) -> float:
    """A Python scalar as numpy's NEP 50 rule applies it to a float32 array."""
    return float(np.float32(x))


def _require_f32(params: mlp.MlpParams):
    if params.dtype != np.float32:
        raise N.NativeError(f"the device training path computes in float32, got {params.dtype} parameters")


def adam_update(params: mlp.MlpParams, grads: mlp.MlpParams, state: AdamState, lr: float, cfg: TrainConfig):
    """train.py:130-143: one Adam step, in place.  One gf_adam_update launch
    over the flat parameter vector (float32, numpy's operation order); the
    moments stay on the device, gradients from this package's device passes
    are used without re-upload, and the updated parameters are written back
    into the host arrays (the reference API) with their device copy kept for
    the next forward pass."""
    _require_f32(params)
    state.step += 1
    b1, b2, eps = cfg.adam_beta1, cfg.adam_beta2, cfg.adam_eps
    bc1 = 1.0 - b1**state.step
    bc2 = 1.0 - b2**state.step
    coef = (N.C.c_float * 8)(*[_f32(v) for v in (b1, 1.0 - b1, b2, 1.0 - b2, bc1, bc2, lr, eps)])
    if state._dev is None:
        state._dev = (device_flat(state._m).clone(), device_flat(state._v).clone())
    buf, views = _pinned_home(params)
    p = device_flat(params)
    g = device_flat(grads)
    N.check(N.lib().gf_adam_update(N.ptr(p), N.ptr(g), N.ptr(state._dev[0]), N.ptr(state._dev[1]), p.numel(), coef,
                                   D.stream_handle()), "adam_update")
    # one DMA of the updated parameters straight into their (page-locked) host arrays
    t = D.require_cuda()
    buf.copy_(p, non_blocking=True)
    t.cuda.current_stream().synchronize()
    for v in views:
        v._bump()  # written behind numpy's back: device caches must see a new version
    params._dev_flat = (params.fingerprint(), p)


def _pinned_home(params: mlp.MlpParams):
    """The parameter arrays, re-homed once into one page-locked flat buffer in
    arrays() order (values preserved), so the optimizer's result lands in them
    with a single DMA.  Re-homed again if the caller replaces an array."""
    home = getattr(params, "_pinned_home", None)
    if home is not None:
        buf, views = home
        cur = [a for _, a in params.arrays()]
        if len(cur) == len(views) and all(a is v for a, v in zip(cur, views)):
            return buf, views
    t = D.require_cuda()
    buf = t.empty((_flat_size(params),), dtype=t.float32, pin_memory=True)
    host = buf.numpy()
    views, off = [], 0
    for (kind, name), a in list(params.arrays()):
        v = D.TrackedArray(host[off : off + a.size].reshape(a.shape))
        v[...] = a
        (params.weights if kind == "w" else params.biases)[name] = v
        views.append(v)
        off += a.size
    params._pinned_home = (buf, views)
    return buf, views


def _sum_squares(x_dev) -> "object":
    t = D.require_cuda()
    out = D.empty((1,), t.float64)
    ws = D.workspace(N.lib().gf_sum_squares_workspace_bytes())
    N.check(N.lib().gf_sum_squares(N.ptr(x_dev), x_dev.numel(), N.ptr(out), N.ptr(ws), ws.numel(), D.stream_handle()),
            "sum_squares")
    return out


def _axpy(x_dev, y_dev, f: float, out_dev):
    N.check(N.lib().gf_axpy(N.ptr(x_dev), N.ptr(y_dev), x_dev.numel(), _f32(f), N.ptr(out_dev), D.stream_handle()),
            "axpy")


def _regularization_device(params: mlp.MlpParams, weight: float):
    """(value, {layer: (w_dev, b_dev)}) of the L2 term; device sums / scales."""
    t = D.require_cuda()
    value = 0.0
    dev = {}
    for name in REGULARIZED_LAYERS:
        w = D.to_device(params.weights[name], t.float32)
        b = D.to_device(params.biases[name], t.float32)
        value += float(_sum_squares(w).item() + _sum_squares(b).item())
        dev[name] = (w, b)
    return weight * value, dev


def regularization_term(params: mlp.MlpParams, weight: float):
    """train.py:146-160: L2 penalty on the view-dependent tail; gradient zero
    everywhere except those layers (2 * weight * x)."""
    _require_f32(params)
    t = D.require_cuda()
    value, dev = _regularization_device(params, weight)
    grads = mlp.map_params(np.zeros_like, params)
    for name, (w, b) in dev.items():
        gw, gb = D.empty(w.shape, t.float32), D.empty(b.shape, t.float32)
        _axpy(w, None, 2.0 * weight, gw)
        _axpy(b, None, 2.0 * weight, gb)
        grads.weights[name][...] = gw.cpu().numpy()
        grads.biases[name][...] = gb.cpu().numpy()
    return value, grads


@dataclass
class RaySamples:
    """train.py:163-172: retained quadrature points of a ray batch."""

    positions: np.ndarray
    directions: np.ndarray
    ray_index: np.ndarray
    slot: np.ndarray
    deltas: np.ndarray
    n_rays: int
    k: int


_M64 = (1 << 64) - 1


def _xsl_rr(state: int) -> int:
    """PCG64's output function (numpy pcg64.h pcg_output_xsl_rr_128_64)."""
    x = ((state >> 64) ^ state) & _M64
    rot = state >> 122
    return ((x >> rot) | (x << ((64 - rot) & 63))) & _M64


def _pcg_state(rng):
    bg = getattr(rng, "bit_generator", None)
    if bg is None or type(bg).__name__ != "PCG64":
        raise N.NativeError("prepare_ray_samples reproduces numpy's PCG64 Generator stream on the device; "
                            f"got {type(bg).__name__ if bg is not None else type(rng).__name__}")
    st = bg.state
    return bg, st


def _advance_float32_draws(bg, st, draws: int):
    """Leave the Generator exactly where rng.random((n, k), float32) would:
    each float32 takes one 32-bit half of a 64-bit output, low half first,
    after the buffered half if there is one (numpy pcg64_next32)."""
    if draws <= 0:
        return
    rem = draws - (1 if st["has_uint32"] else 0)
    words = (rem + 1) // 2
    if words:
        bg.advance(words)  # also clears the buffered half
    new = bg.state
    if rem % 2:
        new["has_uint32"], new["uinteger"] = 1, _xsl_rr(new["state"]["state"]) >> 32
    else:
        new["has_uint32"], new["uinteger"] = 0, 0
    bg.state = new


def prepare_ray_samples(origins, directions, aabb: Aabb, k: int, stratified: bool, rng, occ=None) -> RaySamples:
    """train.py:175-209 on the device (gf_prepare_samples_*): slab test,
    stratified jitter from the caller's Generator (its PCG64 stream is
    reproduced on the device and the Generator is advanced by the same n*k
    draws), float64 sample positions clamped into the box, the occupancy
    test, and np.nonzero's ordering.  Rays are float32 (generate_rays)."""
    t = D.require_cuda()
    o_h, d_h = np.asarray(origins), np.asarray(directions)
    if o_h.dtype != np.float32 or d_h.dtype != np.float32:
        raise N.NativeError("the device sample preparation takes float32 rays (as generate_rays returns)")
    n = len(o_h)
    o = D.to_device(o_h.reshape(-1, 3), t.float32)
    d = D.to_device(d_h.reshape(-1, 3), t.float32)
    box = (N.C.c_double * 6)(*[float(v) for v in aabb.b_min], *[float(v) for v in aabb.b_max])
    pcg = (N.C.c_uint64 * 4)()
    has, uint = 0, 0
    if stratified:
        bg, st = _pcg_state(rng)
        s, inc = st["state"]["state"], st["state"]["inc"]
        pcg[0], pcg[1], pcg[2], pcg[3] = s >> 64, s & _M64, inc >> 64, inc & _M64
        has, uint = int(st["has_uint32"]), int(st["uinteger"])
    geom, bits = None, None
    if occ is not None:
        if np.any(aabb.b_min < occ.aabb.b_min) or np.any(aabb.b_max > occ.aabb.b_max):
            raise N.NativeError("sample box must lie inside the occupancy grid's box")
        geom, bits = occ.native_geom(), occ.device_bits()
    offs = D.empty((n + 1,), t.int64)
    args = (N.ptr(o), N.ptr(d), n, int(k), int(bool(stratified)), box, pcg, has, uint, geom, N.ptr(bits))
    N.check(N.lib().gf_prepare_samples_count(*args, N.ptr(offs), D.stream_handle()), "prepare_ray_samples")
    q = int(offs[n].item()) if n else 0
    deltas = D.empty((n,), t.float32)
    pos = D.empty((q, 3), t.float64)
    dirs = D.empty((q, 3), t.float32)
    ri = D.empty((q,), t.int64)
    sl = D.empty((q,), t.int64)
    N.check(N.lib().gf_prepare_samples_write(*args, N.ptr(offs), N.ptr(deltas), N.ptr(pos), N.ptr(dirs), N.ptr(ri),
                                             N.ptr(sl), D.stream_handle()), "prepare_ray_samples")
    if stratified:
        _advance_float32_draws(bg, st, n * int(k))
    return RaySamples(positions=D.to_host(pos), directions=D.to_host(dirs), ray_index=D.to_host(ri),
                      slot=D.to_host(sl), deltas=D.to_host(deltas), n_rays=n, k=int(k))


def _grads_to_host(grid, gw, gb, flat) -> mlp.MlpParams:
    """The gradients as an MlpParams whose host arrays are downloaded only if
    the caller reads them (DeviceGrads)."""
    shapes = []
    for s, gwl, gbl in zip(grid.arch.layers(), gw, gb):
        shapes += [("w", s.name, tuple(gwl.shape)), ("b", s.name, tuple(gbl.shape))]
    return DeviceGrads(grid.arch, flat, shapes)


@dataclass
class _DeviceLayout:
    """GroupedLayout (batched.py:36-57) of a training batch, kept on the device."""

    n_queries: int
    order: object
    offsets: object
    pos: object   # (Q, 3) float32 rows in grouped order
    dirs: object  # (Q, 3) float32


def _device_layout(model, positions, directions) -> _DeviceLayout:
    """group_by_network(QueryBatch(x, d, model.cell_index(x)), n_cells)
    (batched.py:60-85, grid.py:44-45) without leaving the device: float64
    binning, stable grouping, rows gathered in grouped order."""
    from .core import raise_if_out_of_bounds

    t = D.require_cuda()
    x = np.asarray(positions)
    f64 = x.dtype != np.float32
    xd = D.to_device(x.reshape(-1, 3), t.float64 if f64 else t.float32)
    q = int(xd.shape[0])
    keys = D.empty((q,), t.int64)
    err = D.err_slot()
    N.check(N.lib().gf_bin_points(model.native_geom(), N.ptr(xd), int(f64), q, N.ptr(keys), N.ptr(err),
                                  D.stream_handle()), "cell_index")
    raise_if_out_of_bounds(err, x.reshape(-1, 3), model.aabb)
    order = D.empty((q,), t.int64)
    inverse = D.empty((q,), t.int64)
    offsets = D.empty((model.n_cells + 1,), t.int64)
    ws = D.workspace(N.lib().gf_group_workspace_bytes(q, model.n_cells))
    N.check(N.lib().gf_group_by_key(N.ptr(keys), q, model.n_cells, N.ptr(order), N.ptr(inverse), N.ptr(offsets),
                                    N.ptr(err), N.ptr(ws), ws.numel(), D.stream_handle()), "group_by_network")
    dd = D.to_device(np.asarray(directions, np.float32).reshape(-1, 3), t.float32)
    pos = D.empty((q, 3), t.float32)
    dirs = D.empty((q, 3), t.float32)
    N.check(N.lib().gf_gather_rows3(N.ptr(xd), int(f64), N.ptr(order), q, N.ptr(pos), D.stream_handle()), "gather")
    N.check(N.lib().gf_gather_rows3(N.ptr(dd), 0, N.ptr(order), q, N.ptr(dirs), D.stream_handle()), "gather")
    return _DeviceLayout(q, order, offsets, pos, dirs)


def photometric_loss_and_grads(model, samples: RaySamples, gt: np.ndarray, background, reg_weight: float = 0.0,
                               want_grads: bool = True, sigma_noise: np.ndarray | None = None):
    """train.py:212-288 on the device: mean squared pixel error of the
    composited batch (float64), plus parameter gradients (MlpParams)."""
    _require_f32(model.params)
    t = D.require_cuda()
    b, k = samples.n_rays, samples.k
    layout = _device_layout(model, samples.positions, samples.directions)
    cache = grouped_forward_device(model, layout, layout.pos, layout.dirs, keep_activations=True)
    q = layout.n_queries
    ri = D.to_device(np.asarray(samples.ray_index, np.int64), t.int64)
    sl = D.to_device(np.asarray(samples.slot, np.int64), t.int64)
    noise = None if sigma_noise is None else D.to_device(np.asarray(sigma_noise).astype(np.float32), t.float32)
    deltas = D.to_device(np.asarray(samples.deltas).astype(np.float32), t.float32)
    gtd = D.to_device(np.asarray(gt).astype(np.float32).reshape(-1, 3), t.float32)
    bg = (N.C.c_float * 3)(*[float(v) for v in np.asarray(background, dtype=np.float32).reshape(3)])
    dcq = D.empty((q, 3), t.float32) if want_grads else None
    dsq = D.empty((q,), t.float32) if want_grads else None
    loss_sum = D.empty((1,), t.float64)
    ws = D.workspace(N.lib().gf_photometric_workspace_bytes(b, k, q))
    N.check(N.lib().gf_photometric_loss(b, k, q, N.ptr(ri), N.ptr(sl), N.ptr(cache.rgb), N.ptr(cache.sigma),
                                        N.ptr(noise), N.ptr(deltas), N.ptr(gtd), bg, _f32(2.0 / b) if b else 0.0,
                                        N.ptr(dcq), N.ptr(dsq), N.ptr(loss_sum), N.ptr(ws), ws.numel(),
                                        D.stream_handle()), "photometric_loss")
    loss = float(loss_sum.item() / b) if b else float("nan")
    reg_dev = None
    if reg_weight > 0.0:
        reg_value, reg_dev = _regularization_device(model.params, reg_weight)
        loss += reg_value
    if not want_grads:
        return loss, None
    gw, gb, flat = grouped_backward_device(model, layout, cache, dcq, dsq)
    if reg_dev is not None:
        names = [s.name for s in model.arch.layers()]
        for name, (w, bias) in reg_dev.items():
            li = names.index(name)
            _axpy(w, gw[li], 2.0 * reg_weight, gw[li])  # g + (2 * weight) * w
            _axpy(bias, gb[li], 2.0 * reg_weight, gb[li])
    return loss, _grads_to_host(model, gw, gb, flat)


def _unit_sphere(rng, shape) -> np.ndarray:
    """train.py:335-338."""
    v = rng.normal(size=(*shape, 3)).astype(np.float32)
    v /= np.linalg.norm(v, axis=-1, keepdims=True)
    return v


def distill_step(student, teacher, cfg: TrainConfig, state: AdamState, rng, delta_ref: float) -> float:
    """train.py:341-390: regress every cell network onto the teacher at
    random in-cell points; loss terms, gradients and the update on the device."""
    _require_f32(student.params)
    t = D.require_cuda()
    n, p = student.n_cells, cfg.distill_points_per_cell
    res = student.resolution
    cell = student.aabb.cell_size(res).astype(np.float32)
    flat = np.arange(n)
    idx3 = np.stack([flat % res[0], (flat // res[0]) % res[1], flat // (res[0] * res[1])], axis=-1)
    lows = (student.aabb.b_min + idx3 * student.aabb.cell_size(res)).astype(np.float32)
    u = rng.random((n, p, 3), dtype=np.float32) * np.float32(1.0 - 2e-5) + np.float32(1e-5)
    positions = clip_into(lows[:, None, :] + u * cell[None, None, :], student.aabb).reshape(-1, 3)
    directions = _unit_sphere(rng, (n, p)).reshape(-1, 3)

    pos_d = D.to_device(positions, t.float32)
    dir_d = D.to_device(directions, t.float32)
    t_color, t_sigma = teacher.query_points(pos_d, dir_d)
    # the student lattice: cell c owns rows [c*p, (c+1)*p), identity order
    m = n * p
    layout = GroupedLayout(positions=positions, directions=directions, order=np.arange(m, dtype=np.int64),
                           inverse=np.arange(m, dtype=np.int64), offsets=np.arange(0, m + 1, p, dtype=np.int64),
                           n_networks=n)
    cache = grouped_forward_device(student, layout, pos_d, dir_d, keep_activations=True)
    w_a = cfg.distill_alpha_weight
    dc = D.empty((m, 3), t.float32)
    ds = D.empty((m,), t.float32)
    sums = D.empty((2,), t.float64)
    ws = D.workspace(N.lib().gf_distill_workspace_bytes(m))
    N.check(N.lib().gf_distill_loss(m, N.ptr(cache.rgb), N.ptr(cache.sigma), N.ptr(t_color), N.ptr(t_sigma),
                                    _f32(delta_ref), _f32(2.0 * w_a / m), _f32(2.0 / m), N.ptr(dc), N.ptr(ds),
                                    N.ptr(sums), N.ptr(ws), ws.numel(), D.stream_handle()), "distill_loss")
    s_a, s_c = sums.cpu().numpy()
    loss = float(w_a * s_a + s_c) / m
    gw, gb, flat = grouped_backward_device(student, layout, cache, dc, ds)
    grads = _grads_to_host(student, gw, gb, flat)
    lr = lr_schedule(state.step, cfg.learning_rate, cfg.distill_steps, cfg.lr_final_fraction)
    adam_update(student.params, grads, state, lr, cfg)
    return loss


def photometric_step(model, dataset, cfg: TrainConfig, state: AdamState, rng, occ=None, apply_reg: bool = False,
                     lr: float | None = None, train_indices: list | None = None, noise_std: float = 0.0) -> float:
    """train.py:291-332: one training image and pixel batch (the caller's
    Generator draws the view, the pixels, the jitter and the density noise in
    the reference's order), device rays / samples / loss / gradients / Adam.
    ``dataset`` is any object with the reference dataset's ``indices(split)``,
    ``cameras``, ``images`` and ``aabb``."""
    from .render import generate_rays

    idx = train_indices if train_indices is not None else dataset.indices("train")
    view = int(rng.choice(np.asarray(idx)))
    cam = dataset.cameras[view]
    n_px = cam.width * cam.height
    bsz = min(cfg.batch_size_pixels, n_px)
    pixels = rng.choice(n_px, size=bsz, replace=bsz > n_px)
    origins, dirs = generate_rays(cam)
    gt = dataset.images[view].reshape(-1, 3)[pixels]
    samples = prepare_ray_samples(origins[pixels], dirs[pixels], dataset.aabb, cfg.k_train, True, rng, occ=occ)
    noise = None
    if noise_std > 0.0:
        noise = rng.normal(0.0, noise_std, size=len(samples.positions)).astype(np.float32)
    loss, grads = photometric_loss_and_grads(model, samples, gt, cfg.background,
                                             reg_weight=cfg.l2_reg_weight if apply_reg else 0.0, sigma_noise=noise)
    adam_update(model.params, grads, state, cfg.learning_rate if lr is None else lr, cfg)
    return loss


def train_photometric_loop(model, dataset, cfg: TrainConfig, steps: int, rng, occ, apply_reg: bool, stage: str,
                           curve: list | None = None, noise_std: float = 0.0) -> None:
    """train.py:418-441: ``steps`` photometric updates with a fresh optimizer."""
    state = AdamState.for_params(model.params)
    for step in range(steps):
        lr = lr_schedule(step, cfg.learning_rate, steps, cfg.lr_final_fraction)
        loss = photometric_step(model, dataset, cfg, state, rng, occ=occ, apply_reg=apply_reg, lr=lr,
                                noise_std=noise_std)
        if curve is not None and (step % cfg.log_every == 0 or step == steps - 1):
            curve.append({"stage": stage, "step": step, "loss": loss})


def run_distill_loop(student, teacher, cfg: TrainConfig, delta_ref: float, rng, curve: list | None = None):
    """train.py:444-463: the distillation stage; returns (first, last) loss."""
    state = AdamState.for_params(student.params)
    first = last = float("nan")
    for step in range(cfg.distill_steps):
        last = distill_step(student, teacher, cfg, state, rng, delta_ref)
        if step == 0:
            first = last
        if curve is not None and (step % cfg.log_every == 0 or step == cfg.distill_steps - 1):
            curve.append({"stage": "distill", "step": step, "loss": last})
    return first, last


def evaluate_psnr(model, dataset, render_cfg, occ=None, split: str = "test", seed: int = 0, workers: int = 1) -> float:
    """train.py:393-407: mean PSNR over a split, rendered on the device."""
    from .render import compute_psnr, render_image

    psnrs = []
    for i in dataset.indices(split):
        img, _ = render_image(model, occ, dataset.cameras[i], render_cfg, seed=seed, workers=workers)
        psnrs.append(compute_psnr(img, dataset.images[i]))
    return float(np.mean(psnrs))


def mean_free_space_density(model, empty_cell_flat) -> float:
    """train.py:589-602: mean density over a fixed probe lattice of known-empty cells."""
    if len(empty_cell_flat) == 0:
        return 0.0
    res = model.resolution
    cell = model.aabb.cell_size(res)
    flat = np.asarray(empty_cell_flat)
    idx3 = np.stack([flat % res[0], (flat // res[0]) % res[1], flat // (res[0] * res[1])], axis=-1)
    lows = model.aabb.b_min + idx3 * cell
    offsets = np.stack(np.meshgrid(*([np.array([0.25, 0.5, 0.75])] * 3), indexing="ij"), axis=-1).reshape(-1, 3)
    pts = (lows[:, None, :] + offsets[None, :, :] * cell).reshape(-1, 3).astype(np.float32)
    return float(density_probe(model)(pts).mean())


class DensityProbe:
    """train.py:577-586: the model's density at a fixed canonical direction."""

    def __init__(self, model, direction=(0.0, 0.0, 1.0)):
        self.model = model
        self.direction = np.asarray(direction, dtype=np.float32)

    def __call__(self, points: np.ndarray) -> np.ndarray:
        dirs = np.broadcast_to(self.direction, (len(points), 3))
        _, sigma = self.model.query_points(np.asarray(points).astype(np.float32), dirs)
        return sigma


def density_probe(model, direction=(0.0, 0.0, 1.0)) -> DensityProbe:
    return DensityProbe(model, direction)
