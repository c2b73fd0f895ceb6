"""Species configuration and host-side speed helpers.

Mirrors ``SpeciesConfig``, ``advection_speeds``, ``max_speed_per_dim`` and
``correction_coeffs`` of /root/reference/pkg/src/vpfv/fvm.py.  These are the
host-side pieces around the hot path (the per-stage tables are computed on
the device by libvpfv in exactly this arithmetic; see kernels.StageTables).
The numerical operator itself lives only in the CUDA library.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class SpeciesConfig:
    """Charge, mass, normalisation constants and external fields (fvm.py:40-59).

    ``kappa2`` = (w_p0 t_0)^2, ``kappa_c`` = w_c0 t_0, ``G`` the external
    acceleration per velocity dim, ``Bz`` the static out-of-plane field.
    """

    name: str = "e"
    q: float = -1.0
    m: float = 1.0
    kappa2: float = 1.0
    kappa_c: float = 0.0
    Bz: float = 0.0
    G: tuple = (0.0,)

    @property
    def qm(self):
        return self.q / self.m


def _g(s):
    """External acceleration padded to two velocity components (fvm.py:72-74)."""
    return tuple(s.G) + (0.0,) * 2


def magnetic_factor(s):
    """cB = qm * kappa_c * Bz, the v x B rotation rate."""
    return s.qm * s.kappa_c * s.Bz


def advection_speeds(grid, species, E):
    """Per-dimension speeds broadcastable to the interior (fvm.py:77-122).

    Host numpy; used for the CFL bound and diagnostics, never per cell.
    """
    s = species
    gx, gy = _g(s)[:2]
    cB = magnetic_factor(s)
    E = {k: np.asarray(v) for k, v in E.items()}
    if (grid.d, grid.v) == (1, 1):
        return [grid.centers(1)[None, :], (s.qm * s.kappa2 * E["Ex"] + gx)[:, None]]
    if (grid.d, grid.v) == (1, 2):
        evx = s.qm * s.kappa2 * E["Ex"] + gx
        return [grid.centers(1)[None, :, None],
                evx[:, None, None] + cB * grid.centers(2)[None, None, :],
                (-cB * grid.centers(1) + gy)[None, :, None]]
    if (grid.d, grid.v) == (2, 2):
        evx = s.qm * s.kappa2 * E["Ex"] + gx
        evy = s.qm * s.kappa2 * E["Ey"] + gy
        return [grid.centers(2)[None, None, :, None],
                grid.centers(3)[None, None, None, :],
                evx[:, :, None, None] + cB * grid.centers(3)[None, None, None, :],
                evy[:, :, None, None] - cB * grid.centers(2)[None, None, :, None]]
    raise ValueError(f"unsupported dimensionality ({grid.d},{grid.v})")


def max_speed_per_dim(grid, species, E):
    """max |A^d| per dimension (fvm.py:125-127).

    Equal to the maximum over the broadcast speed arrays of
    ``advection_speeds`` without building them (at 128^4 those are 128^3-cell
    arrays, ~10 ms of host time per CFL step): a velocity-dim speed is
    fl(e(x) +- c(v)) with e the field part, and for fixed c that is monotone
    in e, so its largest magnitude sits at the smallest or largest e."""
    if grid.v == 1 or (grid.d, grid.v) not in ((1, 2), (2, 2)):
        return [float(np.max(np.abs(a))) for a in advection_speeds(grid, species, E)]
    s = species
    gx, gy = _g(s)[:2]
    cB = magnetic_factor(s)
    E = {k: np.asarray(v) for k, v in E.items()}

    def extreme(e, c, sign):  # max over (x, v) of |fl(e(x) + sign c(v))|
        lo, hi = np.min(e), np.max(e)
        return float(max(np.max(np.abs(lo + sign * c)), np.max(np.abs(hi + sign * c))))

    if (grid.d, grid.v) == (1, 2):
        evx = s.qm * s.kappa2 * E["Ex"] + gx
        return [float(np.max(np.abs(grid.centers(1)))), extreme(evx, cB * grid.centers(2), 1.0),
                float(np.max(np.abs(-cB * grid.centers(1) + gy)))]
    evx = s.qm * s.kappa2 * E["Ex"] + gx
    evy = s.qm * s.kappa2 * E["Ey"] + gy
    return [float(np.max(np.abs(grid.centers(2)))), float(np.max(np.abs(grid.centers(3)))),
            extreme(evx, cB * grid.centers(3), 1.0), extreme(evy, cB * grid.centers(2), -1.0)]


def correction_coeffs(grid, species, E):
    """Closed-form diagonal-correction coefficients (fvm.py:168-201), host numpy."""
    s = species
    h = grid.h
    qm = s.qm
    E = {k: np.asarray(v) for k, v in E.items()}
    if grid.d == 1:
        hx, hvx = h[0], h[1]
        dEx = np.roll(E["Ex"], -1) - np.roll(E["Ex"], 1)
        out = {"c1": hvx / (48.0 * hx) + qm * s.kappa2 * dEx / (96.0 * hvx)}
        if grid.v == 2:
            hvy = h[2]
            out["c2"] = qm * (s.kappa_c / 48.0) * s.Bz * (hvx / hvy - hvy / hvx)
        return out
    hx, hy, hvx, hvy = h
    Ex, Ey = E["Ex"], E["Ey"]
    d = lambda a, ax: np.roll(a, -1, axis=ax) - np.roll(a, 1, axis=ax)  # noqa: E731
    return {
        "c1": hvx / (48.0 * hx) + qm * s.kappa2 * d(Ex, 0) / (96.0 * hvx),
        "c2": qm * (s.kappa_c / 48.0) * s.Bz * (hvx / hvy - hvy / hvx),
        "c3": -qm * s.kappa2 * d(Ex, 1) / (96.0 * hvx),
        "c4": hvy / (48.0 * hy) + qm * s.kappa2 * d(Ey, 1) / (96.0 * hvy),
        "c5": -qm * s.kappa2 * d(Ey, 0) / (96.0 * hvy),
    }
