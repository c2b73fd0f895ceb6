"""Low-storage RK4 3/8ths stage protocol and the L1 CFL bound.

Mirrors /root/reference/pkg/src/vpfv/timestepping.py: ``StepContext``,
``rk4_38_low_storage_step``, ``rk4_butcher_step``, ``array_stage``,
``max_stable_dt``, ``DEFAULT_SIGMA``, ``RK_STAGE_TIMES``.  This is the
stage protocol the B200 drivers plug into:

    stage(dest, A, B, src, ca, cb, cd, cL, t):  dest = ca*A + cb*B + cd*dest + cL*L(src)

``RK4_STAGES`` is the same recurrence as data -- the drivers use it to
capture a whole step (four stages) in one CUDA graph with cL read on the
device as dt / cL_div.
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

DEFAULT_SIGMA = 1.73
RK_STAGE_TIMES = (0.0, 1.0 / 3.0, 2.0 / 3.0, 1.0)

# (dest, A, B, src, ca, cb, cd, cL_div): cL = dt / cL_div  (timestepping.py:80-83)
RK4_STAGES = (
    ("f1", "f0", "f0", "f0", 1.0, 0.0, 0.0, 3.0),
    ("fout", "f0", "f1", "f1", 2.0, -1.0, 0.0, 1.0),
    ("f1", "fout", "fout", "fout", -1.0, 0.0, 2.0, 1.0),
    ("fout", "f0", "f1", "f1", -0.125, 0.375, 0.75, 8.0),
)


@dataclass
class StepContext:
    """Three persistent buffers plus the clock (timestepping.py:39-52)."""

    f0: object
    f1: object
    fout: object
    t: float = 0.0
    step: int = 0

    def rotate(self):
        self.f0, self.fout = self.fout, self.f0
        self.step += 1


def rk4_butcher_step(u0, dt, L, t=0.0):
    """Classic tableau form, four stage derivatives (timestepping.py:55-66)."""
    u0 = np.asarray(u0)
    k1 = L(u0, t)
    k2 = L(u0 + (dt / 3.0) * k1, t + dt / 3.0)
    k3 = L(u0 + dt * (-k1 / 3.0 + k2), t + 2.0 * dt / 3.0)
    k4 = L(u0 + dt * (k1 - k2 + k3), t + dt)
    return u0 + (dt / 8.0) * (k1 + 3.0 * k2 + 3.0 * k3 + k4)


def rk4_38_low_storage_step(ctx: StepContext, dt, stage):
    """One step on the three buffers of ``ctx`` (timestepping.py:69-84)."""
    bufs = {"f0": ctx.f0, "f1": ctx.f1, "fout": ctx.fout}
    t = ctx.t
    times = (t, t + dt / 3.0, t + 2.0 * dt / 3.0, t + dt)
    for (dn, an, bn, sn, ca, cb, cd, div), ts in zip(RK4_STAGES, times):
        cL = dt / div if div != 1.0 else dt
        stage(bufs[dn], bufs[an], bufs[bn], bufs[sn], ca, cb, cd, cL, ts)
    ctx.t = t + dt


def array_stage(L):
    """Adapt a functional RHS to the stage protocol (timestepping.py:87-98)."""

    def stage(dest, A, B, src, ca, cb, cd, cL, t):
        rhs = L(src, t)
        dest[...] = ca * A + cb * B + cd * dest + cL * rhs

    return stage


def max_stable_dt(speeds, h, sigma=DEFAULT_SIGMA, safety=1.0):
    """sigma / sum_d(max|A_d|/h_d), min over species (timestepping.py:101-117)."""
    best = math.inf
    for per_dim in speeds:
        if len(per_dim) != len(h):
            raise ValueError("speed/width dimension mismatch")
        norm1 = sum(abs(a) / hd for a, hd in zip(per_dim, h))
        if norm1 > 0.0:
            best = min(best, sigma / norm1)
    return best * safety if best != math.inf else math.inf
