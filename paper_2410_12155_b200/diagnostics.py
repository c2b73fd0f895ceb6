"""Conserved-quantity rows, field amplitude, growth-rate fits (host side).

Mirrors /root/reference/pkg/src/vpfv/diagnostics.py: ``DiagnosticsRow``,
``DIAGNOSTICS_SCHEMA``, ``field_amplitude``, ``conserved_quantities``,
``rows_to_csv``, ``fit_growth_rate``, ``richardson_error`` with the
reference's signatures, return values and validation.  They run per output
cadence, not per stage; on device state the velocity sums run on the GPU
(``DeviceDiagnostics``).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

from .grid import NGHOST

DIAGNOSTICS_SCHEMA = "vpfv-diagnostics-1"


@dataclass(frozen=True)
class DiagnosticsRow:
    t: float
    dt: float
    mass: tuple
    momentum: float
    field_energy: float
    kinetic_energy: float
    total_energy: float
    field_amplitude: float

    @staticmethod
    def header(species_names):
        return (["t", "dt"] + [f"mass_{n}" for n in species_names]
                + ["momentum", "field_energy", "kinetic_energy", "total_energy", "field_amplitude"])

    def values(self):
        return ([self.t, self.dt] + [m for _, m in self.mass]
                + [self.momentum, self.field_energy, self.kinetic_energy, self.total_energy,
                   self.field_amplitude])


def _fold(x, axis):
    x = np.moveaxis(x, axis, -1)
    while x.shape[-1] > 1:
        n = x.shape[-1]
        m = n // 2
        s = x[..., 0:2 * m:2] + x[..., 1:2 * m:2]
        x = np.concatenate([s, x[..., 2 * m:]], axis=-1) if n % 2 else s
    return np.moveaxis(x, -1, axis)


def fold_tree_sum(x, axes):
    """Deterministic pairwise tree, fastest axis first (fields.py:42-47)."""
    out = np.array(x, dtype=np.float64, copy=True)
    for ax in sorted(axes, reverse=True):
        out = _fold(out, ax)
    return np.squeeze(out, axis=tuple(sorted(axes)))


def field_amplitude(E, grid):
    """sqrt(integral E.E dx) (diagnostics.py:74-82)."""
    vol = 1.0
    for k in range(grid.d):
        vol *= grid.h[k]
    total = 0.0
    for comp in E.values():
        total += float(np.sum(np.square(np.asarray(comp))))
    return math.sqrt(total * vol)


def higher_moments_arrays(data, grid):
    """Momentum and kinetic-energy densities with the midpoint-to-average lift
    (fields.py:131-161); ghosts of ``data`` must be synchronised."""
    g = grid
    inner = g.interior_slices()
    f = data[inner]
    vol = 1.0
    for k in g.velocity_dims:
        vol *= g.h[k]
    vaxes = tuple(g.velocity_dims)
    mom, kin = [], 0.0
    for d in g.velocity_dims:
        shape = [1] * g.ndim
        shape[d] = g.N[d]
        vc = g.centers(d).reshape(shape)
        h2 = g.h[d] ** 2
        lo = [0] * g.ndim
        hi = [0] * g.ndim
        lo[d], hi[d] = -1, 1
        sh = lambda off: data[tuple(slice(NGHOST + o, NGHOST + o + n) for o, n in zip(off, g.N))]  # noqa: E731
        dfd = (sh(hi) - sh(lo)) / (2.0 * g.h[d])
        mom.append((vc * f + (h2 / 12.0) * dfd).sum(axis=vaxes) * vol)
        kin = kin + ((vc ** 2 + h2 / 12.0) * f + (h2 / 6.0) * vc * dfd).sum(axis=vaxes) * vol
    return mom, 0.5 * kin


def _host_E(E):
    return {k: (v.cpu().numpy() if hasattr(v, "cpu") else np.asarray(v)) for k, v in E.items()}


def conserved_quantities(dists, species, state, t, dt):
    """One :class:`DiagnosticsRow` from synchronised fields
    (diagnostics.py:85-122, same signature and order of operations).

    ``dists`` are DistFields (host numpy data with current ghosts, or device
    tensors with stored velocity ghosts -- then the velocity sums run on the
    device through ``DeviceDiagnostics`` and only physical-grid arrays reach
    the host); ``state`` is the field solve of the same instant (``.E``)."""
    data0 = dists[0].data
    E = _host_E(state.E)
    if hasattr(data0, "is_cuda") and data0.is_cuda:
        from .kernels import stream_handle

        diag = DeviceDiagnostics([f.grid for f in dists], data0.device)
        return diag.row([f.data for f in dists], species, E, t, dt, stream_handle(data0.device))
    return conserved_quantities_arrays([np.asarray(f.data) for f in dists], [f.grid for f in dists], species,
                                       E, t, dt)


def conserved_quantities_arrays(datas, grids, species, E, t, dt):
    """``conserved_quantities`` on host padded arrays with synchronised ghosts
    (diagnostics.py:85-122)."""
    masses = []
    mom_tot = None
    kinetic = 0.0
    for data, g, sp in zip(datas, grids, species):
        cellvol = 1.0
        for w in g.h:
            cellvol *= w
        interior = data[g.interior_slices()]
        masses.append((sp.name, float(fold_tree_sum(interior, tuple(range(g.ndim)))) * cellvol))
        mom, kin = higher_moments_arrays(data, g)
        physvol = 1.0
        for k in range(g.d):
            physvol *= g.h[k]
        if mom_tot is None:
            mom_tot = [0.0] * len(mom)
        for k, mk in enumerate(mom):
            mom_tot[k] += sp.m * float(np.sum(mk)) * physvol
        kinetic += sp.m * float(np.sum(kin)) * physvol
    U = 0.5 * field_amplitude(E, grids[0]) ** 2
    return DiagnosticsRow(t=t, dt=dt, mass=tuple(masses), momentum=math.sqrt(sum(p * p for p in mom_tot)),
                          field_energy=U, kinetic_energy=kinetic, total_energy=U + kinetic,
                          field_amplitude=field_amplitude(E, grids[0]))


def rows_to_csv(rows, species_names):
    """Diagnostics rows as CSV text, 17 significant digits (diagnostics.py:125-130)."""
    lines = [",".join(DiagnosticsRow.header(species_names))]
    for row in rows:
        lines.append(",".join(f"{v:.17g}" for v in row.values()))
    return "\n".join(lines) + "\n"


def fit_growth_rate(t, amplitude, window):
    """Least-squares exponential rate of ``amplitude`` over ``window``
    (diagnostics.py:133-160): fits log(amplitude) = a + gamma t on the samples
    with window[0] <= t <= window[1] and returns ``(gamma, stderr)``; at least
    10 samples and positive amplitudes are required (ValueError otherwise)."""
    t = np.asarray(t, dtype=float)
    amplitude = np.asarray(amplitude, dtype=float)
    lo, hi = window
    keep = (t >= lo) & (t <= hi)
    count = int(np.count_nonzero(keep))
    if count < 10:
        raise ValueError(f"window [{lo}, {hi}] holds {count} samples; need >= 10")
    ts = t[keep]
    amps = amplitude[keep]
    if np.any(amps <= 0.0):
        raise ValueError("amplitude must be positive on the fit window")
    y = np.log(amps)
    n = ts.size
    tm = ts.mean()
    ym = y.mean()
    sxx = float(np.sum((ts - tm) ** 2))
    gamma = float(np.sum((ts - tm) * (y - ym)) / sxx)
    resid = y - (ym + gamma * (ts - tm))
    stderr = math.sqrt(float(np.sum(resid ** 2)) / max(n - 2, 1) / sxx)
    return gamma, stderr


def fit_peak_rate(t, amplitude, window):
    """Damping/growth rate fitted on the local maxima of ``amplitude`` inside
    ``window`` (the robust choice for oscillating, damped |E|):
    ``fit_growth_rate``'s least squares on the peaks only; returns
    ``(gamma, stderr)``.  Needs at least 3 peaks."""
    t = np.asarray(t, dtype=float)
    a = np.asarray(amplitude, dtype=float)
    lo, hi = window
    idx = [i for i in range(1, len(a) - 1) if a[i] >= a[i - 1] and a[i] > a[i + 1] and lo <= t[i] <= hi]
    if len(idx) < 3:
        raise ValueError(f"window [{lo}, {hi}] holds {len(idx)} amplitude peaks; need >= 3")
    ts, y = t[idx], np.log(a[idx])
    tm, ym = ts.mean(), y.mean()
    sxx = float(np.sum((ts - tm) ** 2))
    gamma = float(np.sum((ts - tm) * (y - ym)) / sxx)
    resid = y - (ym + gamma * (ts - tm))
    return gamma, math.sqrt(float(np.sum(resid ** 2)) / max(len(idx) - 2, 1) / sxx)


class DeviceDiagnostics:
    """``conserved_quantities`` from the device state without copying f to
    the host: per species the fold-tree velocity moment
    with unit volume (``vpfv_moment``, so the mass stays bitwise the
    reference's fold over all axes once the host folds the physical axes) and
    the momentum / kinetic-energy velocity sums (``vpfv_higher_moments``); only
    physical-grid arrays cross PCIe, and the host finishes in the reference's
    order of operations (diagnostics.py:85-122, fields.py:131-161)."""

    def __init__(self, grids, device):
        import torch

        from . import _lib

        self._lib = _lib
        self.grids = tuple(grids)
        self.device = device
        dev = lambda a: torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64), device=device)  # noqa: E731
        self.vc = [[dev(g.centers(k)) for k in g.velocity_dims] for g in self.grids]
        self.N = [_lib.int_array(g.N) for g in self.grids]
        self.n_raw = [torch.empty(tuple(g.N[:g.d]), dtype=torch.float64, device=device) for g in self.grids]
        self.hm = [torch.empty(tuple(g.N[:g.d]) + (2 * g.v,), dtype=torch.float64, device=device)
                   for g in self.grids]

    def row(self, arrays, species, E, t, dt, stream):
        """One DiagnosticsRow from the padded device arrays (velocity ghosts
        stored) and the host E dict of the same instant."""
        lib = self._lib
        for s, (g, f) in enumerate(zip(self.grids, arrays)):
            lib.call("vpfv_moment", f.data_ptr(), self.n_raw[s].data_ptr(), g.d, g.v, self.N[s], 1.0, stream)
            vcs = self.vc[s]
            hv = [g.h[k] for k in g.velocity_dims]
            lib.call("vpfv_higher_moments", f.data_ptr(), g.d, g.v, self.N[s], vcs[0].data_ptr(),
                     vcs[1].data_ptr() if len(vcs) > 1 else None, hv[0], hv[1] if len(hv) > 1 else 0.0,
                     self.hm[s].data_ptr(), stream)
        n_raw = [a.cpu().numpy() for a in self.n_raw]
        hm = [a.cpu().numpy() for a in self.hm]
        masses = []
        mom_tot = None
        kinetic = 0.0
        for g, sp, n0, h in zip(self.grids, species, n_raw, hm):
            cellvol = 1.0
            for w in g.h:
                cellvol *= w
            masses.append((sp.name, float(fold_tree_sum(n0, tuple(range(g.d)))) * cellvol))
            vol = 1.0
            for k in g.velocity_dims:
                vol *= g.h[k]
            mom = [h[..., 2 * k] * vol for k in range(g.v)]
            kin = 0.0
            for k in range(g.v):
                kin = kin + h[..., 2 * k + 1] * vol
            kin = 0.5 * kin
            physvol = 1.0
            for k in range(g.d):
                physvol *= g.h[k]
            if mom_tot is None:
                mom_tot = [0.0] * len(mom)
            for k, mk in enumerate(mom):
                mom_tot[k] += sp.m * float(np.sum(mk)) * physvol
            kinetic += sp.m * float(np.sum(kin)) * physvol
        U = 0.5 * field_amplitude(E, self.grids[0]) ** 2
        return DiagnosticsRow(t=t, dt=dt, mass=tuple(masses), momentum=math.sqrt(sum(p * p for p in mom_tot)),
                              field_energy=U, kinetic_energy=kinetic, total_energy=U + kinetic,
                              field_amplitude=field_amplitude(E, self.grids[0]))


def richardson_error(f_N, f_2N):
    """Volume-weighted L1 difference between a field and its refinement
    (diagnostics.py:163-180): the fine field aggregated exactly onto the
    coarse cells (mean of the 2^D children) before differencing."""
    a = np.asarray(f_N, dtype=float)
    b = np.asarray(f_2N, dtype=float)
    if a.ndim != b.ndim or any(2 * na != nb for na, nb in zip(a.shape, b.shape)):
        raise ValueError(f"refinement shape {b.shape} is not double of {a.shape} everywhere")
    shape = []
    for na in a.shape:
        shape += [na, 2]
    coarse = b.reshape(shape).mean(axis=tuple(range(1, 2 * a.ndim, 2)))
    return float(np.mean(np.abs(a - coarse)))
