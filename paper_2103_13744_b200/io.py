"""Checkpoints (mirror of gridfield.io's checkpoint half,
/root/reference/pkg/src/gridfield/io.py:28-32, 142-224).

Same on-disk format, byte for byte: magic ``GFCKPT01``, little-endian u64
header length, a sorted-key JSON manifest, the float32 parameter payload in
layer-manifest order (each layer's weights (n_cells,out,in) then biases
(n_cells,out)) and an optional packed occupancy bitmap.

``load_checkpoint`` also keeps the payload so the first device use packs the
per-cell operand images straight from one copy of the file's parameter
block (``gf_pack_weights_flat``) instead of re-assembling them layer by
layer; any in-place edit of the parameters afterwards falls back to the
per-layer path.  Dataset directories and PNG IO stay out of scope.
"""

from __future__ import annotations

import dataclasses
import json
import struct
from pathlib import Path

import numpy as np

from . import _device as D
from .core import Aabb, PositionalEncoding
from .grid import NetworkGrid
from .mlp import MlpArchitecture, MlpParams
from .occupancy import OccupancyGrid

CHECKPOINT_MAGIC = b"GFCKPT01"


def save_checkpoint(path, grid: NetworkGrid, occ: OccupancyGrid | None = None) -> None:
    """io.py:150-175: serialize a lattice (and optional occupancy) to one file."""
    grid.params.validate()
    header = {
        "format_version": 1,
        "arch": dataclasses.asdict(grid.arch),
        "encoding": dataclasses.asdict(grid.encoding),
        "resolution": [int(v) for v in grid.resolution],
        "aabb": {"b_min": list(grid.aabb.b_min), "b_max": list(grid.aabb.b_max)},
        "param_dtype": "<f4",
        "param_count": int(grid.n_cells) * grid.arch.parameter_count(),
        "occupancy": None if occ is None else {"resolution": [int(v) for v in occ.resolution],
                                               "n_bytes": len(occ.bits)},
    }
    head = json.dumps(header, sort_keys=True, separators=(",", ":")).encode()
    payload = np.concatenate([np.asarray(a).astype("<f4", copy=False).ravel() for _, a in grid.params.arrays()])
    with open(path, "wb") as f:
        f.write(CHECKPOINT_MAGIC)
        f.write(struct.pack("<Q", len(head)))
        f.write(head)
        f.write(payload.tobytes())
        if occ is not None:
            f.write(np.asarray(occ.bits).tobytes())


def load_checkpoint(path) -> tuple[NetworkGrid, OccupancyGrid | None]:
    """io.py:178-224: validate magic, version and payload length, then build
    the lattice (parameters copied out of the file) and the occupancy grid."""
    blob = Path(path).read_bytes()
    if blob[:8] != CHECKPOINT_MAGIC:
        raise ValueError(f"{path}: not a checkpoint (bad magic)")
    (head_len,) = struct.unpack("<Q", blob[8:16])
    header = json.loads(blob[16 : 16 + head_len])
    if header.get("format_version") != 1:
        raise ValueError(f"{path}: unsupported format version {header.get('format_version')}")
    arch = MlpArchitecture(**header["arch"])
    enc = PositionalEncoding(**header["encoding"])
    resolution = np.array(header["resolution"], dtype=np.int64)
    aabb = Aabb(header["aabb"]["b_min"], header["aabb"]["b_max"])
    n_cells = int(np.prod(resolution))
    occ_info = header["occupancy"]
    occ_bytes = 0 if occ_info is None else occ_info["n_bytes"]
    param_bytes = header["param_count"] * 4
    expected = 16 + head_len + param_bytes + occ_bytes
    if len(blob) != expected:
        raise ValueError(f"{path}: payload length {len(blob)} != expected {expected}")
    flat = np.frombuffer(blob, dtype="<f4", count=header["param_count"], offset=16 + head_len).copy()
    weights, biases = {}, {}
    cursor = 0
    for spec in arch.layers():
        n = n_cells * spec.out_dim * spec.in_dim
        weights[spec.name] = D.tracked(flat[cursor : cursor + n].reshape(n_cells, spec.out_dim, spec.in_dim).copy())
        cursor += n
        n = n_cells * spec.out_dim
        biases[spec.name] = D.tracked(flat[cursor : cursor + n].reshape(n_cells, spec.out_dim).copy())
        cursor += n
    grid = NetworkGrid(aabb=aabb, resolution=resolution, arch=arch, encoding=enc,
                       params=MlpParams(arch, weights, biases))
    grid._payload = (grid.params.fingerprint(), flat)  # device packing straight from the file's block
    occ = None
    if occ_info is not None:
        bits = np.frombuffer(blob, dtype=np.uint8, offset=16 + head_len + param_bytes).copy()
        occ = OccupancyGrid(aabb, np.array(occ_info["resolution"], dtype=np.int64), bits)
    return grid, occ
