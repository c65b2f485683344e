"""The piece of gridfield.train the hot path needs (mirror of
/root/reference/pkg/src/gridfield/train.py:577-586).

``density_probe(model)`` is the density field occupancy extraction probes
(cli.py:155-160).  It is a plain callable, as in the reference; because it is
recognisable, ``extract_occupancy`` runs it on the device in one library call
(gf_extract_occupancy_network) instead of one host round trip per chunk.
Training itself (photometric fine-tuning, distillation) is out of scope.
"""

from __future__ import annotations

import numpy as np


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
