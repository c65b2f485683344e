"""ctypes binding of libgridfield_b200.so (include/gridfield_b200.h).

The library is built in-tree by ``__graft_entry__.build()`` (or ``make -C
paper_2103_13744_b200/csrc``).  There is no CPU fallback: if the library or a
CUDA device is missing, every device-backed function raises.
"""

from __future__ import annotations

import ctypes as C
import os
import threading
from pathlib import Path

import numpy as np

LIB_PATH = Path(os.environ.get("GF_LIB_PATH") or Path(__file__).resolve().parent / "_lib" / "libgridfield_b200.so")

GF_OK, GF_ERR_INVALID, GF_ERR_CUDA, GF_ERR_WORKSPACE, GF_ERR_UNSUPPORTED = range(5)
ABI_VERSION = 2  # include/gridfield_b200.h GF_ABI_VERSION
PRECISION = {"fp32": 0, "fp16": 1}
STAT_FIELDS = ("total_queries", "ess_skipped", "ert_terminated_rays", "n_rays")
INT64_MAX = np.iinfo(np.int64).max


class Arch(C.Structure):
    _fields_ = [
        ("hidden_layers", C.c_int32), ("width", C.c_int32), ("view_width", C.c_int32),
        ("pos_freqs", C.c_int32), ("dir_freqs", C.c_int32), ("include_raw", C.c_int32),
        ("skip_layer", C.c_int32),
    ]


# gf_field_fn: (user, srec, n, ray_dir, stride_shift, stride, res, stream) -> status
FIELD_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_int32, C.c_uint32, C.c_void_p,
                       C.c_void_p)


class Manifest(C.Structure):
    _fields_ = [
        ("hidden_layers", C.c_int32), ("width", C.c_int32), ("view_width", C.c_int32),
        ("pos_dim", C.c_int32), ("dir_dim", C.c_int32), ("skip_layer", C.c_int32),
    ]


def make_manifest(arch) -> Manifest:
    return Manifest(int(arch.hidden_layers), int(arch.hidden_width), int(arch.view_width),
                    int(arch.position_input_dim), int(arch.direction_input_dim), int(arch.skip_layer or 0))


class GridGeom(C.Structure):
    _fields_ = [("b_min", C.c_double * 3), ("b_max", C.c_double * 3), ("res", C.c_int32 * 3)]


class MarchCfg(C.Structure):
    _fields_ = [
        ("k", C.c_int32), ("ert_chunk", C.c_int32), ("stratified", C.c_int32), ("eps_compare_f64", C.c_int32),
        ("epsilon", C.c_double), ("background", C.c_float * 3), ("rays_f64", C.c_int32), ("seed", C.c_uint64),
    ]


class CameraT(C.Structure):
    _fields_ = [
        ("width", C.c_int32), ("height", C.c_int32), ("fx", C.c_double), ("fy", C.c_double),
        ("cx", C.c_double), ("cy", C.c_double), ("c2w", C.c_double * 12),
    ]


MAX_PRIMS = 16


class Prim(C.Structure):
    _fields_ = [("kind", C.c_int32), ("_pad", C.c_int32), ("a", C.c_double * 3), ("b", C.c_double * 3),
                ("color", C.c_double * 3), ("radius", C.c_double), ("density", C.c_double), ("feather", C.c_double)]


class Analytic(C.Structure):
    _fields_ = [("b_min", C.c_double * 3), ("b_max", C.c_double * 3), ("n_prims", C.c_int32), ("_pad", C.c_int32),
                ("prims", Prim * MAX_PRIMS), ("texture_freq", C.c_double), ("texture_amp", C.c_double),
                ("view_tint", C.c_double), ("tint_axis", C.c_double * 3)]


TRACE_DTYPE = np.dtype([("x", "<f4"), ("y", "<f4"), ("z", "<f4"), ("ray", "<u4"), ("slot", "<u4"), ("cell", "<u4")])

_P = C.c_void_p
_SIGS = {
    "gf_abi_version": (C.c_int, []),
    "gf_last_error": (C.c_char_p, []),
    "gf_param_count": (C.c_int64, [C.POINTER(Arch)]),
    "gf_packed_bytes": (C.c_size_t, [C.POINTER(Arch), C.c_int64, C.c_int]),
    "gf_pack_weights": (C.c_int, [C.POINTER(Arch), C.c_int64, C.POINTER(_P), C.POINTER(_P), _P, C.c_int, _P]),
    "gf_pack_weights_flat": (C.c_int, [C.POINTER(Arch), C.c_int64, _P, _P, C.c_int, _P]),
    "gf_query_workspace_bytes": (C.c_size_t, [C.POINTER(Arch), C.POINTER(GridGeom), C.c_int64]),
    "gf_query_points": (C.c_int, [C.POINTER(Arch), C.POINTER(GridGeom), _P, C.c_int, _P, _P, C.c_int64, _P, _P, _P,
                                  _P, C.c_size_t, _P]),
    "gf_grouped_workspace_bytes": (C.c_size_t, [C.c_int64, C.c_int64]),
    "gf_grouped_forward": (C.c_int, [C.POINTER(Arch), C.c_int64, _P, C.c_int, _P, _P, C.c_int64, _P, _P, _P, _P,
                                     _P, C.c_size_t, _P]),
    "gf_render_workspace_bytes": (C.c_size_t, [C.POINTER(Arch), C.POINTER(GridGeom), C.POINTER(MarchCfg), C.c_int64]),
    "gf_render_rays": (C.c_int, [C.POINTER(Arch), C.POINTER(GridGeom), _P, C.c_int, C.POINTER(GridGeom), _P,
                                 C.POINTER(MarchCfg), C.POINTER(CameraT), _P, _P, C.c_int64, C.c_int64, C.c_int64,
                                 _P, _P, _P,
                                 C.c_int64, _P, _P, C.c_size_t, _P]),
    "gf_group_workspace_bytes": (C.c_size_t, [C.c_int64, C.c_int64]),
    "gf_group_by_key": (C.c_int, [_P, C.c_int64, C.c_int64, _P, _P, _P, _P, _P, C.c_size_t, _P]),
    "gf_bin_points": (C.c_int, [C.POINTER(GridGeom), _P, C.c_int32, C.c_int64, _P, _P, _P]),
    "gf_occupied_at": (C.c_int, [C.POINTER(GridGeom), _P, _P, C.c_int32, C.c_int64, _P, _P, _P]),
    "gf_clip_into": (C.c_int, [C.POINTER(C.c_double), C.POINTER(C.c_double), _P, C.c_int64, _P, _P]),
    "gf_intersect_aabb": (C.c_int, [_P, _P, C.c_int64, C.POINTER(C.c_double), C.POINTER(C.c_double), _P, _P, _P]),
    "gf_ray_samples": (C.c_int, [C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_double, C.c_double, _P,
                                 C.c_int64, _P, _P]),
    "gf_positional_encode": (C.c_int, [_P, C.c_int32, C.c_int64, C.c_int32, C.c_int32, C.c_int32, _P, _P]),
    "gf_density_to_alpha": (C.c_int, [_P, _P, C.c_int32, C.c_int64, _P, _P]),
    "gf_composite": (C.c_int, [_P, _P, C.c_int64, C.c_int64, _P, _P, _P]),
    "gf_composite_f64": (C.c_int, [_P, _P, C.c_int64, C.c_int64, _P, _P, _P]),
    "gf_generate_rays": (C.c_int, [C.POINTER(CameraT), _P, _P, _P]),
    "gf_pcg64_block_state": (C.c_int, [C.c_uint64, C.c_uint64, C.POINTER(C.c_uint64)]),
    "gf_query_analytic": (C.c_int, [C.POINTER(Analytic), _P, _P, C.c_int64, _P, _P, _P]),
    "gf_render_analytic_workspace_bytes": (C.c_size_t, [C.POINTER(Analytic), C.POINTER(MarchCfg), C.c_int64]),
    "gf_render_rays_analytic": (C.c_int, [C.POINTER(Analytic), C.POINTER(GridGeom), _P, C.POINTER(MarchCfg),
                                          C.POINTER(CameraT), _P, _P, C.c_int64, C.c_int64, C.c_int64, _P, _P, _P,
                                          C.c_int64, _P, _P, C.c_size_t, _P]),
    "gf_extract_occupancy_analytic": (C.c_int, [C.POINTER(Analytic), C.POINTER(GridGeom), C.c_double, _P, _P]),
    "gf_extract_workspace_bytes": (C.c_size_t, [C.POINTER(Arch), C.POINTER(GridGeom), C.POINTER(GridGeom),
                                                C.c_int64]),
    "gf_extract_occupancy_network": (C.c_int, [C.POINTER(Arch), C.POINTER(GridGeom), _P, C.c_int,
                                               C.POINTER(C.c_float), C.POINTER(GridGeom), C.c_double, C.c_int64, _P,
                                               _P, _P, C.c_size_t, _P]),
    "gf_brute_force_workspace_bytes": (C.c_size_t, [C.c_int32, C.c_int64]),
    "gf_render_brute_force": (C.c_int, [C.POINTER(Analytic), C.POINTER(CameraT), C.c_int32, C.POINTER(C.c_float),
                                        C.c_int64, C.c_int64, _P, _P, C.c_size_t, _P]),
    "gf_analytic_empty_cells": (C.c_int, [C.POINTER(Analytic), C.POINTER(C.c_int32), _P, _P]),
    "gf_render_field_workspace_bytes": (C.c_size_t, [C.POINTER(GridGeom), C.POINTER(MarchCfg), C.c_int64]),
    "gf_render_rays_field": (C.c_int, [FIELD_FN, _P, C.POINTER(GridGeom), C.POINTER(GridGeom), _P,
                                       C.POINTER(MarchCfg), C.POINTER(CameraT), _P, _P, C.c_int64, C.c_int64,
                                       C.c_int64, _P, _P, _P, C.c_int64, _P, _P, C.c_size_t, _P]),
    "gf_field_gather": (C.c_int, [_P, C.c_int64, _P, C.c_int32, C.c_uint32, _P, _P, _P]),
    "gf_field_scatter": (C.c_int, [_P, C.c_int64, _P, _P, _P, _P]),
    "gf_mlp_forward": (C.c_int, [C.POINTER(Manifest), C.c_int32, C.c_int64, C.c_int64, C.POINTER(_P), C.POINTER(_P),
                                 _P, _P, _P, _P, C.POINTER(_P), _P, _P, _P]),
    "gf_mlp_backward_workspace_bytes": (C.c_size_t, [C.POINTER(Manifest), C.c_int32, C.c_int64, C.c_int64]),
    "gf_mlp_backward": (C.c_int, [C.POINTER(Manifest), C.c_int32, C.c_int64, C.c_int64, C.POINTER(_P), _P, _P,
                                  C.POINTER(_P), _P, _P, _P, _P, _P, _P, C.POINTER(_P), C.POINTER(_P), _P,
                                  C.c_size_t, _P]),
    "gf_grouped_backward_workspace_bytes": (C.c_size_t, [C.POINTER(Arch), C.c_int64, C.c_int64]),
    "gf_grouped_backward": (C.c_int, [C.POINTER(Arch), C.c_int64, _P, _P, _P, C.c_int64, _P, _P, _P, _P,
                                      C.POINTER(_P), C.POINTER(_P), _P, C.c_size_t, _P]),
    "gf_grouped_backward_act": (C.c_int, [C.POINTER(Arch), C.c_int64, _P, _P, _P, C.c_int64, _P, _P, _P, _P, _P,
                                          C.POINTER(_P), C.POINTER(_P), _P, C.c_size_t, _P]),
    "gf_grouped_forward_act": (C.c_int, [C.POINTER(Arch), C.c_int64, _P, _P, _P, C.c_int64, _P, _P, _P, _P, _P,
                                         _P, C.c_size_t, _P]),
    "gf_photometric_workspace_bytes": (C.c_size_t, [C.c_int64, C.c_int32, C.c_int64]),
    "gf_photometric_loss": (C.c_int, [C.c_int64, C.c_int32, C.c_int64, _P, _P, _P, _P, _P, _P, _P,
                                      C.POINTER(C.c_float), C.c_float, _P, _P, _P, _P, C.c_size_t, _P]),
    "gf_adam_update": (C.c_int, [_P, _P, _P, _P, C.c_int64, C.POINTER(C.c_float), _P]),
    "gf_sum_squares_workspace_bytes": (C.c_size_t, []),
    "gf_sum_squares": (C.c_int, [_P, C.c_int64, _P, _P, C.c_size_t, _P]),
    "gf_axpy": (C.c_int, [_P, _P, C.c_int64, C.c_float, _P, _P]),
    "gf_distill_workspace_bytes": (C.c_size_t, [C.c_int64]),
    "gf_distill_loss": (C.c_int, [C.c_int64, _P, _P, _P, _P, C.c_float, C.c_float, C.c_float, _P, _P, _P, _P,
                                  C.c_size_t, _P]),
    "gf_prepare_samples_count": (C.c_int, [_P, _P, C.c_int64, C.c_int32, C.c_int32, C.POINTER(C.c_double),
                                           C.POINTER(C.c_uint64), C.c_int32, C.c_uint32, C.POINTER(GridGeom), _P, _P,
                                           _P]),
    "gf_prepare_samples_write": (C.c_int, [_P, _P, C.c_int64, C.c_int32, C.c_int32, C.POINTER(C.c_double),
                                           C.POINTER(C.c_uint64), C.c_int32, C.c_uint32, C.POINTER(GridGeom), _P, _P,
                                           _P, _P, _P, _P, _P, _P]),
    "gf_gather_rows3": (C.c_int, [_P, C.c_int32, _P, C.c_int64, _P, _P]),
    "gf_stage_timing": (C.c_int, [C.c_int32]),
    "gf_stage_times": (C.c_int, [C.POINTER(C.c_double), C.POINTER(C.c_int64)]),
    "gf_launch_count": (C.c_int64, []),
    "gf_graph_counters": (C.c_int, [_P]),
}

STAGES = ("setup", "march", "scan", "scatter", "mlp")


def graph_counters() -> dict:
    """CUDA-graph activity of gf_render_rays since process start."""
    out = (C.c_int64 * 4)()
    check(lib().gf_graph_counters(C.addressof(out)), "gf_graph_counters")
    return dict(zip(("replays", "updates", "instantiations", "eager"), (int(v) for v in out)))


def stage_times() -> tuple[dict, dict]:
    """Accumulated (ms, launches) per stage since the last call (timing must
    have been enabled with lib().gf_stage_timing(1))."""
    ms = (C.c_double * len(STAGES))()
    n = (C.c_int64 * len(STAGES))()
    check(lib().gf_stage_times(ms, n), "gf_stage_times")
    return dict(zip(STAGES, list(ms))), dict(zip(STAGES, list(n)))

EXPORTED = tuple(_SIGS)

_lib = None
_lock = threading.Lock()


class NativeError(RuntimeError):
    pass


def lib():
    """Load the extension once; raise (never fall back) if it is missing."""
    global _lib
    if _lib is None:
        with _lock:
            if _lib is None:
                if not LIB_PATH.exists():
                    raise NativeError(
                        f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'`"
                    )
                h = C.CDLL(str(LIB_PATH))
                for name, (res, args) in _SIGS.items():
                    fn = getattr(h, name)
                    fn.restype = res
                    fn.argtypes = args
                if h.gf_abi_version() != ABI_VERSION:  # struct layouts below must match the library's
                    raise NativeError(f"{LIB_PATH} has ABI {h.gf_abi_version()}, this binding expects {ABI_VERSION}; "
                                      "rebuild it")
                _lib = h
    return _lib


def check(status: int, what: str):
    if status != GF_OK:
        msg = lib().gf_last_error().decode(errors="replace")
        raise NativeError(f"{what} failed (status {status}): {msg}")


def ptr(t) -> int:
    """Device pointer of a torch tensor (or None -> NULL)."""
    return None if t is None else t.data_ptr()


def make_arch(arch, encoding) -> Arch:
    return Arch(
        int(arch.hidden_layers), int(arch.hidden_width), int(arch.view_width),
        int(encoding.num_freqs_position), int(encoding.num_freqs_direction), int(bool(encoding.include_raw_input)),
        int(arch.skip_layer or 0),
    )


def make_geom(aabb, resolution) -> GridGeom:
    g = GridGeom()
    for a in range(3):
        g.b_min[a] = float(aabb.b_min[a])
        g.b_max[a] = float(aabb.b_max[a])
        g.res[a] = int(resolution[a])
    return g


def make_camera(cam) -> CameraT:
    c = CameraT()
    c.width, c.height = int(cam.width), int(cam.height)
    c.fx, c.fy, c.cx, c.cy = float(cam.fx), float(cam.fy), float(cam.cx), float(cam.cy)
    m = np.asarray(cam.c2w, np.float64)
    for r in range(3):
        for k in range(4):
            c.c2w[4 * r + k] = float(m[r, k])
    return c


def pcg64_block_state(seed: int, block_start: int) -> tuple[int, int]:
    out = (C.c_uint64 * 4)()
    check(lib().gf_pcg64_block_state(seed, block_start, out), "gf_pcg64_block_state")
    return (out[0] << 64) | out[1], (out[2] << 64) | out[3]


def library_path() -> str:
    return os.fspath(LIB_PATH)
