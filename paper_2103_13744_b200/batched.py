"""Grouped execution of many per-cell networks (mirror of gridfield.batched,
/root/reference/pkg/src/gridfield/batched.py).

``group_by_network`` is a stable device counting sort; ``grouped_forward``
evaluates every segment with its own cell's MLP in one device pass and writes
results straight back to the original query order.
"""

from __future__ import annotations

from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass

import numpy as np

from . import _device as D
from . import _native as N


@dataclass
class QueryBatch:
    """batched.py:22-33."""

    positions: np.ndarray
    directions: np.ndarray
    network_index: np.ndarray

    def __post_init__(self):
        n = len(self.network_index)
        if len(self.positions) != n or len(self.directions) != n:
            raise ValueError("positions/directions/network_index lengths differ")


@dataclass
class GroupedLayout:
    """batched.py:36-57: ``order`` sorted slot -> original index, ``inverse``
    undoes it, ``offsets[i]:offsets[i+1]`` is network i's segment."""

    positions: np.ndarray
    directions: np.ndarray
    order: np.ndarray
    inverse: np.ndarray
    offsets: np.ndarray
    n_networks: int

    @property
    def n_queries(self) -> int:
        return len(self.order)

    def segment_lengths(self) -> np.ndarray:
        return np.diff(self.offsets)


def group_by_network(batch: QueryBatch, n_networks: int) -> GroupedLayout:
    """batched.py:60-85 on the device: stable counting sort by network index."""
    t = D.require_cuda()
    keys = np.asarray(batch.network_index).astype(np.int64, copy=False).reshape(-1)
    n = len(keys)
    kd = D.to_device(keys, t.int64)
    order = D.empty((n,), t.int64)
    inverse = D.empty((n,), t.int64)
    offsets = D.empty((n_networks + 1,), t.int64)
    err = D.err_slot()
    ws = D.workspace(N.lib().gf_group_workspace_bytes(n, n_networks))
    N.check(N.lib().gf_group_by_key(N.ptr(kd), n, n_networks, N.ptr(order), N.ptr(inverse), N.ptr(offsets),
                                    N.ptr(err), N.ptr(ws), ws.numel(), D.stream_handle()), "group_by_network")
    if int(err.item()) != N.INT64_MAX:
        raise ValueError(
            f"network index out of range [0, {n_networks}): "
            f"min={keys.min() if n else None} max={keys.max() if n else None}"
        )
    order_h = order.cpu().numpy()
    return GroupedLayout(
        positions=np.ascontiguousarray(np.asarray(batch.positions)[order_h]),
        directions=np.ascontiguousarray(np.asarray(batch.directions)[order_h]),
        order=order_h,
        inverse=inverse.cpu().numpy(),
        offsets=offsets.cpu().numpy(),
        n_networks=n_networks,
    )


ACT_FLOATS = 132  # gf_grouped_forward_act: [h0 | h1 | feature | g | sigma | 3 logits] per row (32-wide)


def grouped_forward_device(grid, layout: GroupedLayout, pos=None, dirs=None, precision="fp32",
                           keep_activations=False) -> "GroupedCache":
    """The fused grouped forward on device tensors (results in query order);
    ``pos``/``dirs`` may be given as device tensors already in grouped order.
    ``keep_activations`` (training, fp32): also keep the per-row activations
    the backward needs (batched.py:143-150's caches) when the kernel supports
    the manifest, so grouped_backward reads them instead of recomputing."""
    t = D.require_cuda()
    n = layout.n_queries
    packed = grid.device_params(precision)
    if pos is None:
        pos = D.to_device(np.asarray(layout.positions, np.float32).reshape(-1, 3), t.float32)
    if dirs is None:
        dirs = D.to_device(np.asarray(layout.directions, np.float32).reshape(-1, 3), t.float32)
    offs = D.to_device(layout.offsets if D.is_tensor(layout.offsets) else np.asarray(layout.offsets, np.int64),
                       t.int64)
    order = D.to_device(layout.order if D.is_tensor(layout.order) else np.asarray(layout.order, np.int64), t.int64)
    rgb = D.empty((n, 3), t.float32)
    sigma = D.empty((n,), t.float32)
    ws = D.workspace(N.lib().gf_grouped_workspace_bytes(grid.n_cells, n))
    arch = grid.native_arch()
    act = None
    if keep_activations and precision == "fp32" and grid.arch.hidden_width == 32:
        act = D.empty((max(n, 1) * ACT_FLOATS,), t.float32)
        rc = N.lib().gf_grouped_forward_act(arch, grid.n_cells, N.ptr(packed), N.ptr(pos), N.ptr(dirs), n,
                                            N.ptr(offs), N.ptr(order), N.ptr(rgb), N.ptr(sigma), N.ptr(act),
                                            N.ptr(ws), ws.numel(), D.stream_handle())
        if rc == N.GF_ERR_UNSUPPORTED:  # not the fused kernel's manifest: the backward recomputes
            act = None
        else:
            N.check(rc, "grouped_forward")
    if act is None:
        N.check(N.lib().gf_grouped_forward(arch, grid.n_cells, N.ptr(packed), N.PRECISION[precision],
                                           N.ptr(pos), N.ptr(dirs), n, N.ptr(offs), N.ptr(order), N.ptr(rgb),
                                           N.ptr(sigma), N.ptr(ws), ws.numel(), D.stream_handle()), "grouped_forward")
    return GroupedCache(packed, pos, dirs, offs, order, rgb, sigma, act)


def grouped_forward(grid, layout: GroupedLayout, caches: list | None = None, precision=None):
    """batched.py:120-151: evaluate each segment with its cell's network; the
    kernel writes row j's result to original index order[j], so the output is
    already in input order.

    With ``caches`` (training) the pass runs in fp32 and appends one
    ``GroupedCache`` holding the device-resident grouped rows and the packed
    parameters it used; ``grouped_backward`` recomputes the activations from
    them in its fused kernel instead of keeping (n, width) activation arrays."""
    p = "fp32" if caches is not None else grid.resolved_precision(precision)
    c = grouped_forward_device(grid, layout, precision=p, keep_activations=caches is not None)
    if caches is not None:
        caches.append(c)
    dtype = grid.params.dtype
    return c.rgb.cpu().numpy().astype(dtype, copy=False), c.sigma.cpu().numpy().astype(dtype, copy=False)


@dataclass
class GroupedCache:
    """What grouped_backward needs from its forward pass (the reference keeps
    per-bucket activations, batched.py:143-150): the fp32 parameter packing
    the forward used and the grouped rows, all on the device."""

    packed: object
    pos: object
    dirs: object
    offsets: object
    order: object
    rgb: object
    sigma: object
    act: object = None  # per-row activations (keep_activations), or None: the backward recomputes them


def grouped_backward_device(grid, layout: GroupedLayout, cache: GroupedCache, d_color, d_sigma):
    """gf_grouped_backward on device tensors -> per-layer (gw, gb) device lists
    in the reference layout (n_cells, out, in) / (n_cells, out)."""
    t = D.require_cuda()
    n = layout.n_queries
    dc = D.to_device(d_color, t.float32).reshape(-1, 3).contiguous()
    ds = D.to_device(d_sigma, t.float32).reshape(-1).contiguous()
    if dc.shape[0] != n or ds.shape[0] != n:
        raise ValueError("upstream gradients do not match the layout's query count")
    specs = grid.arch.layers()
    # one flat buffer in MlpParams.arrays() order (w, b per layer): the views
    # below are the per-layer outputs, the buffer feeds the optimizer directly
    nc = grid.n_cells
    flat = D.empty((nc * sum(s.out_dim * s.in_dim + s.out_dim for s in specs),), t.float32)
    gw, gb, off = [], [], 0
    for s in specs:
        gw.append(flat[off : off + nc * s.out_dim * s.in_dim].view(nc, s.out_dim, s.in_dim))
        off += nc * s.out_dim * s.in_dim
        gb.append(flat[off : off + nc * s.out_dim].view(nc, s.out_dim))
        off += nc * s.out_dim
    wp = (N.C.c_void_p * len(gw))(*[x.data_ptr() for x in gw])
    bp = (N.C.c_void_p * len(gb))(*[x.data_ptr() for x in gb])
    arch = grid.native_arch()
    ws_bytes = N.lib().gf_grouped_backward_workspace_bytes(arch, grid.n_cells, n)
    if ws_bytes == 0 and n > 0:
        _grouped_backward_dense(grid, cache, dc, ds, flat, gw, gb)
        return gw, gb, flat
    ws = D.workspace(ws_bytes)
    if cache.act is not None:
        N.check(N.lib().gf_grouped_backward_act(arch, grid.n_cells, N.ptr(cache.packed), N.ptr(cache.pos),
                                                N.ptr(cache.dirs), n, N.ptr(cache.offsets), N.ptr(cache.order),
                                                N.ptr(dc), N.ptr(ds), N.ptr(cache.act), wp, bp, N.ptr(ws), ws.numel(),
                                                D.stream_handle()), "grouped_backward")
        return gw, gb, flat
    N.check(N.lib().gf_grouped_backward(arch, grid.n_cells, N.ptr(cache.packed), N.ptr(cache.pos), N.ptr(cache.dirs),
                                        n, N.ptr(cache.offsets), N.ptr(cache.order), N.ptr(dc), N.ptr(ds), wp, bp,
                                        N.ptr(ws), ws.numel(), D.stream_handle()), "grouped_backward")
    return gw, gb, flat


def _grouped_backward_dense(grid, cache: GroupedCache, dc, ds, flat, gw, gb):
    """Manifests without a fused backward kernel (any depth / width / skip
    layer): each queried cell's rows go through the device encoding and
    mlp.backward's dense kernels (gf_mlp_forward / gf_mlp_backward)."""
    from . import mlp

    flat.zero_()
    offs = cache.offsets.cpu().numpy()
    order = cache.order.cpu().numpy()
    pos = cache.pos.cpu().numpy().reshape(-1, 3)
    dirs = cache.dirs.cpu().numpy().reshape(-1, 3)
    dc_h = dc.cpu().numpy()[order]
    ds_h = ds.cpu().numpy()[order]
    specs = grid.arch.layers()
    for c in np.nonzero(offs[1:] > offs[:-1])[0]:
        rows = slice(int(offs[c]), int(offs[c + 1]))
        x = grid.encoding.encode_position(pos[rows])
        d = grid.encoding.encode_direction(dirs[rows])
        g = mlp.backward(grid.params.at(int(c)).astype(np.float32), x, d, dc_h[rows], ds_h[rows])
        for s_, w_, b_ in zip(specs, gw, gb):
            w_[int(c)].copy_(D.to_device(g.weights[s_.name], w_.dtype))
            b_[int(c)].copy_(D.to_device(g.biases[s_.name], b_.dtype))


def grouped_backward(grid, layout: GroupedLayout, caches: list, d_color, d_sigma):
    """batched.py:154-187: parameter gradients of sum(d_color*color +
    d_sigma*sigma) stacked over all cells (zeros for unqueried networks), in
    one device pass (gf_grouped_backward: one CTA per cell, fused forward
    recompute + backward, fixed-order per-parameter sums).  Upstream
    gradients arrive in original query order (numpy or CUDA tensors)."""
    from . import mlp

    if not caches or not isinstance(caches[-1], GroupedCache):
        raise ValueError("grouped_backward needs the caches list filled by grouped_forward")
    gw, gb, _ = grouped_backward_device(grid, layout, caches[-1], d_color, d_sigma)
    specs = grid.arch.layers()
    dtype = grid.params.dtype
    return mlp.MlpParams(grid.arch, {s.name: w.cpu().numpy().astype(dtype, copy=False) for s, w in zip(specs, gw)},
                         {s.name: b.cpu().numpy().astype(dtype, copy=False) for s, b in zip(specs, gb)})


def parallel_map(fn, items, workers: int = 1) -> list:
    """batched.py:190-201: ordered results, identical for any worker count."""
    items = list(items)
    if workers <= 1 or len(items) <= 1:
        return [fn(item) for item in items]
    with ThreadPoolExecutor(max_workers=workers) as pool:
        return list(pool.map(fn, items))
