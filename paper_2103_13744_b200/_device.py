"""Device plumbing: CUDA device / stream selection, numpy<->device transfer,
versioned parameter arrays, and the per-object device caches (packed weights,
occupancy bits).  PyTorch is used only as the CUDA allocator and stream
provider; every computation runs in libgridfield_b200.so.
"""

from __future__ import annotations

import threading

import numpy as np

from . import _native as N

_torch = None


def torch():
    global _torch
    if _torch is None:
        import torch as t

        _torch = t
    return _torch


_cuda_ok = False


def require_cuda():
    # checked once per process (is_available() queries NVML: ~1 us per call,
    # and every render call passes through here several times)
    global _cuda_ok
    t = torch()
    if not _cuda_ok:
        if not t.cuda.is_available():
            raise N.NativeError("no CUDA device: the gridfield B200 hot path has no CPU fallback")
        N.lib()
        _cuda_ok = True
    return t


def device():
    t = require_cuda()
    return t.device("cuda", t.cuda.current_device())


def stream_handle() -> int:
    """The caller's current CUDA stream as a raw cudaStream_t."""
    t = torch()
    raw = getattr(t._C, "_cuda_getCurrentRawStream", None)
    if raw is not None:
        return int(raw(t.cuda.current_device()))
    return t.cuda.current_stream().cuda_stream


def is_tensor(a) -> bool:
    return isinstance(a, torch().Tensor)


def to_device(a, dtype) -> "object":
    """numpy array (or torch tensor) -> contiguous device tensor of ``dtype``."""
    t = require_cuda()
    if isinstance(a, t.Tensor):
        return a.to(device=device(), dtype=dtype).contiguous()
    arr = np.ascontiguousarray(a)
    return t.from_numpy(arr).to(device=device(), dtype=dtype, non_blocking=False).contiguous()


def to_host(x) -> np.ndarray:
    """Device tensor -> numpy array through page-locked memory (one DMA at
    full PCIe rate; torch's caching host allocator recycles the buffers).  The
    returned array views the pinned buffer and keeps it alive."""
    t = require_cuda()
    h = t.empty(tuple(x.shape), dtype=x.dtype, pin_memory=True)
    h.copy_(x, non_blocking=True)
    t.cuda.current_stream().synchronize()
    return h.numpy()


def empty(shape, dtype):
    t = require_cuda()
    return t.empty(shape, dtype=dtype, device=device())


def workspace(nbytes: int):
    t = require_cuda()
    return t.empty(max(int(nbytes), 1), dtype=t.uint8, device=device())


def err_slot():
    t = require_cuda()
    return t.full((1,), N.INT64_MAX, dtype=t.int64, device=device())


# ---------------------------------------------------------------------------
# versioned arrays: in-place writes bump a shared counter so device caches of
# parameters / occupancy bits never serve stale data (the reference's tests
# mutate grid.params.* in place and render again, test_grid.py:188-191).
# ---------------------------------------------------------------------------
class _Version:
    __slots__ = ("value",)

    def __init__(self):
        self.value = 0


_version_lock = threading.Lock()


class TrackedArray(np.ndarray):
    """ndarray whose in-place modifications (setitem, in-place ufuncs,
    np.copyto / np.put / fill) bump a version shared by all its views."""

    def __new__(cls, a):
        obj = np.asarray(a).view(cls)
        obj._gf_version = _Version()
        return obj

    def __array_finalize__(self, obj):
        v = getattr(obj, "_gf_version", None)
        self._gf_version = v if v is not None else _Version()

    def _bump(self):
        with _version_lock:
            self._gf_version.value += 1

    def __setitem__(self, key, value):
        super().__setitem__(key, value)
        self._bump()

    def __array_ufunc__(self, ufunc, method, *inputs, out=None, **kw):
        args = [x.view(np.ndarray) if isinstance(x, TrackedArray) else x for x in inputs]
        if out is not None:
            outs = tuple(x.view(np.ndarray) if isinstance(x, TrackedArray) else x for x in out)
            kw["out"] = outs
        res = getattr(ufunc, method)(*args, **kw)
        if out is not None:
            for x in out:
                if isinstance(x, TrackedArray):
                    x._bump()
            return out[0] if len(out) == 1 else out
        return res

    def __array_function__(self, func, types, args, kwargs):
        res = super().__array_function__(func, types, args, kwargs)
        if func in _MUTATING:
            target = args[0] if args else next(iter(kwargs.values()), None)
            if isinstance(target, TrackedArray):
                target._bump()
        return res

    def fill(self, value):
        super().fill(value)
        self._bump()

    @property
    def gf_version(self) -> int:
        return self._gf_version.value


_MUTATING = {np.copyto, np.put, np.place, np.putmask, np.fill_diagonal}


def tracked(a) -> TrackedArray:
    return a if isinstance(a, TrackedArray) else TrackedArray(a)


def fingerprint(arrays) -> tuple:
    """Identity + version of each array; changes whenever a cached device copy
    would go stale through the tracked paths.  Cheap on purpose (it runs on
    every render call): the dtype object, not its string (str(dtype) costs
    ~8 us per array), and no __array_interface__ dict."""
    return tuple((id(a), a.shape, a.dtype, a.strides, getattr(a, "gf_version", None)) for a in arrays)
