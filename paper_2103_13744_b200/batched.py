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


def grouped_forward(grid, layout: GroupedLayout, caches: list | None = None, precision=None):
    """batched.py:120-151: evaluate each segment with its cell's network; the
    kernel writes row j's result to original index order[j], so the output is
    already in input order.  ``caches`` (training backward) is out of scope."""
    if caches is not None:
        raise NotImplementedError("grouped_backward caches belong to training, which this build does not cover")
    t = D.require_cuda()
    n = layout.n_queries
    p = grid.resolved_precision(precision)
    packed = grid.device_params(p)
    pos = D.to_device(np.asarray(layout.positions, np.float32).reshape(-1, 3), t.float32)
    dirs = D.to_device(np.asarray(layout.directions, np.float32).reshape(-1, 3), t.float32)
    offs = D.to_device(np.asarray(layout.offsets, np.int64), t.int64)
    order = D.to_device(np.asarray(layout.order, np.int64), t.int64)
    rgb = D.empty((n, 3), t.float32)
    sigma = D.empty((n,), t.float32)
    ws = D.workspace(N.lib().gf_grouped_workspace_bytes(grid.n_cells, n))
    N.check(N.lib().gf_grouped_forward(grid.native_arch(), grid.n_cells, N.ptr(packed), N.PRECISION[p], N.ptr(pos),
                                       N.ptr(dirs), n, N.ptr(offs), N.ptr(order), N.ptr(rgb), N.ptr(sigma), N.ptr(ws),
                                       ws.numel(), D.stream_handle()), "grouped_forward")
    dtype = grid.params.dtype
    return rgb.cpu().numpy().astype(dtype, copy=False), sigma.cpu().numpy().astype(dtype, copy=False)


def parallel_map(fn, items, workers: int = 1) -> list:
    """batched.py:190-201: ordered results, identical for any worker count."""
    items = list(items)
    if workers <= 1 or len(items) <= 1:
        return [fn(item) for item in items]
    with ThreadPoolExecutor(max_workers=workers) as pool:
        return list(pool.map(fn, items))
