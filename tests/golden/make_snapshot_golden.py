"""Generate tests/golden/snapshot_ref.vpfv with the REAL reference writer
(/root/reference/pkg/src/vpfv/diagnostics.py:187-203); run in the build
container only:  python tests/golden/make_snapshot_golden.py

The field: 1D-2V grid (8, 8, 16) on [0, 2pi) x [-4, 4) x [-5, 5), interior
values 1 + 0.3 * default_rng(2024).random(N), species tag "e-", t = 1.25.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from vpfv.diagnostics import write_snapshot  # noqa: E402
from vpfv.grid import DistField, make_grid  # noqa: E402

N = (8, 8, 16)
g = make_grid(1, 2, N, (0.0, -4.0, -5.0), (2 * np.pi, 4.0, 5.0))
f = DistField(g, species="e-")
f.data[g.interior_slices()] = 1.0 + 0.3 * np.random.default_rng(2024).random(N)
write_snapshot(os.path.join(HERE, "snapshot_ref.vpfv"), f, 1.25)
