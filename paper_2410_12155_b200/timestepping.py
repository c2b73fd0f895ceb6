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


# Kutta's 3/8 rule as a tableau (the classic form of the recurrence above)
RK38_A = ((), (1.0 / 3.0,), (-1.0 / 3.0, 1.0), (1.0, -1.0, 1.0))
RK38_B = (0.125, 0.375, 0.375, 0.125)


def rk4_butcher_step(u0, dt, L, t=0.0):
    """Classic tableau form with four stored stage derivatives, for checks
    against the low-storage protocol (reference: timestepping.py:55-66).
    Driven by ``RK38_A`` / ``RK38_B`` / ``RK_STAGE_TIMES``, so its rounding
    is not the reference's expression grouping."""
    u0 = np.asarray(u0)
    ks = []
    for row, c in zip(RK38_A, RK_STAGE_TIMES):
        u = u0
        for a, k in zip(row, ks):
            u = u + (a * dt) * k
        ks.append(L(u, t + c * dt))
    incr = sum(b * k for b, k in zip(RK38_B, ks))
    return u0 + dt * incr


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
    """Wrap a functional RHS ``L(y, t)`` as a stage callable (reference:
    timestepping.py:87-98); materialises L(src), so host checks only."""

    def stage(dest, A, B, src, ca, cb, cd, cL, t):
        out = cL * L(src, t)
        for c, X in ((ca, A), (cb, B), (cd, dest)):
            if c != 0.0:
                out = out + c * X
        dest[...] = out

    return stage


def _l1_rate(per_dim, h):
    """sum_d max|A_d| / h_d for one species."""
    if len(per_dim) != len(h):
        raise ValueError("speed/width dimension mismatch")
    return sum(abs(a) / hd for a, hd in zip(per_dim, h))


def max_stable_dt(speeds, h, sigma=DEFAULT_SIGMA, safety=1.0):
    """L1 CFL bound sigma / rate, minimum over species, times ``safety``;
    ``math.inf`` when no species moves (reference: timestepping.py:101-117)."""
    rates = [_l1_rate(per_dim, h) for per_dim in speeds]
    fastest = max((r for r in rates if r > 0.0), default=0.0)
    return safety * (sigma / fastest) if fastest > 0.0 else math.inf
