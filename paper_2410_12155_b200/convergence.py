"""Convergence ladders on the device.

The reference's ``vpfv convergence`` (/root/reference/pkg/src/vpfv/cli.py:144-181)
runs one problem at resolutions N, 2N, 4N, ... with a fixed dt shared by all
levels, compares consecutive levels with ``richardson_error``
(diagnostics.py:163-180: the fine field aggregated exactly onto the coarse
cells, L1 difference) and reports the observed orders log2(e_k / e_{k+1}).
Here every level steps on the GPU and the Richardson errors are computed from
the device states (``vpfv_richardson_partials``), so ladders reach
resolutions (e.g. 2D-2V 128^4 -> 256^4, 34 GB per state buffer) the CPU
reference cannot.
"""

from __future__ import annotations

import math

import numpy as np
import torch

from . import _lib
from .kernels import stream_handle
from .runner import Simulation


def richardson_error_device(coarse, fine, grid):
    """richardson_error of two padded device arrays (``grid`` = the coarse grid)."""
    nblocks = 592
    part = torch.empty(nblocks, dtype=torch.float64, device=coarse.device)
    _lib.call("vpfv_richardson_partials", coarse.data_ptr(), fine.data_ptr(), grid.ndim, _lib.int_array(grid.N),
              part.data_ptr(), nblocks, stream_handle(coarse.device))
    total = 0.0
    for x in part.cpu().numpy():  # in-order sum of the per-CTA partials
        total += float(x)
    return total / float(np.prod(grid.N))


def run_ladder(make_setup, levels, dt, t_end, device=None, csv_path=None):
    """Run ``make_setup(factor)`` for factor = 1, 2, 4, ... (``levels``
    levels) to ``t_end`` with the fixed ``dt``; returns (sizes, errors,
    orders) as cli.py:144-181 prints them, and writes its convergence.csv
    when ``csv_path`` is given.  Only two levels' states are alive at once."""
    if levels < 2:
        raise ValueError("a ladder needs at least two levels")
    sizes, errors = [], []
    prev = None
    for level in range(levels):
        sim = Simulation(make_setup(2 ** level), dt=dt, device=device)
        steps = int(round(t_end / dt))
        for _ in range(steps):
            sim.advance(dt)
        sizes.append(sim.grids[0].N[0])
        if prev is not None:
            errs = [richardson_error_device(a, b, g) for a, b, g in zip(prev.ctx.f0, sim.ctx.f0, prev.grids)]
            errors.append(sum(errs) / len(errs))
        prev = sim
    orders = [math.log2(errors[i] / errors[i + 1]) for i in range(len(errors) - 1)]
    if csv_path is not None:
        with open(csv_path, "w") as fh:
            fh.write("N,error,observed_order\n")
            for i, err in enumerate(errors):
                order = "" if i == 0 else "%.17g" % orders[i - 1]
                fh.write(f"{sizes[i]},{err:.17g},{order}\n")
    return sizes, errors, orders
