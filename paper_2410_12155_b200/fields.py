"""Velocity moments, charge density and the spectral Poisson solve on the B200.

Mirrors /root/reference/pkg/src/vpfv/fields.py: ``zeroth_moment``,
``charge_density``, ``poisson_solve``, ``FieldState.solve``.  The device
``FieldSolver`` owns every table and scratch buffer the per-stage chain
needs (allocated once, so the chain can be captured in a CUDA graph):

    f (device, padded) --vpfv_moment--> n_s --vpfv_charge_density--> rho
      --vpfv_poisson_{1d,2d}--> E

The moment is bitwise the reference fold tree; the FFT is hand-written, so
E agrees with numpy's pocketfft to rounding (~1e-16 relative).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np
import torch

from . import _lib
from .kernels import stream_handle


def velocity_cell_volume(grid):
    vol = 1.0
    for k in grid.velocity_dims:
        vol *= grid.h[k]
    return vol


def _twiddles(n):
    m = np.arange(n)
    w = np.exp(-2j * np.pi * m / n)
    return np.ascontiguousarray(np.stack([w.real, w.imag], axis=-1).reshape(-1))


def _wavenumbers(n, h):
    """k = 2 pi fftfreq(n, h) and the derivative copy with the even-n Nyquist
    entry zeroed (fields.py:185-196)."""
    k = 2.0 * np.pi * np.fft.fftfreq(n, d=h)
    kd = k.copy()
    if n % 2 == 0:
        kd[n // 2] = 0.0
    return k, kd


class FieldSolver:
    """Device moment -> rho -> E chain for a set of species on one physical grid."""

    def __init__(self, grids, species, device, schedule="velocity-major"):
        if schedule not in ("velocity-major", "position-major", "free"):
            raise ValueError(f"unknown schedule {schedule!r}")
        self.schedule = schedule
        self._moment_fn = "vpfv_moment_seq" if schedule == "position-major" else "vpfv_moment"
        self.grids = list(grids)
        self.species = list(species)
        self.device = device
        g0 = self.grids[0]
        self.d = g0.d
        self.phys_shape = tuple(g0.N[:g0.d])
        self.nphys = int(np.prod(self.phys_shape))
        S = len(self.grids)
        f64 = dict(dtype=torch.float64, device=device)
        self.n = torch.empty((S,) + self.phys_shape, **f64)
        self.rho = torch.empty(self.phys_shape, **f64)
        self.E = {"Ex": torch.empty(self.phys_shape, **f64)}
        if self.d == 2:
            self.E["Ey"] = torch.empty(self.phys_shape, **f64)
        self.phi = torch.empty(self.phys_shape, **f64)
        self.q_host = _lib.dbl_array([s.q for s in self.species])
        self.vols = [velocity_cell_volume(g) for g in self.grids]
        self.N_arrays = [_lib.int_array(g.N) for g in self.grids]
        dev = lambda a: torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64), device=device)  # noqa: E731
        h = g0.h
        if self.d == 1:
            k, kd = _wavenumbers(g0.N[0], h[0])
            self.tw = dev(_twiddles(g0.N[0]))
            self.k2 = dev(k ** 2)
            self.kd = dev(kd)
            # the solve's Green's function K (E = K (*) rho), stored twice for vpfv_field_1d_conv
            ghat = np.zeros(g0.N[0], dtype=np.complex128)
            nz = k != 0.0
            ghat[nz] = -1j * kd[nz] / (k[nz] ** 2)
            green = np.fft.ifft(ghat).real
            self.green2 = dev(np.concatenate([green, green]))
        else:
            kx, kxd = _wavenumbers(g0.N[0], h[0])
            ky, kyd = _wavenumbers(g0.N[1], h[1])
            self.twx, self.twy = dev(_twiddles(g0.N[0])), dev(_twiddles(g0.N[1]))
            self.kx, self.ky, self.kxd, self.kyd = dev(kx), dev(ky), dev(kxd), dev(kyd)
            self.scratch = torch.empty(8 * self.nphys, **f64)

        self._field1d_args = {}

    # ------------------------------------------------------------------
    def field_1d_ok(self):
        """The fused 1D chain fits one CTA (poisson.cu vpfv_field_1d)."""
        return self.d == 1 and len(self.species) <= 8 and self.phys_shape[0] <= 2048

    def finish_in_field_1d(self, partial_shapes):
        """Fold the moment partials inside vpfv_field_1d too?  Only when they
        are small (one CTA reads them all): 1D-1V rows, or a few thousand
        doubles -- a 1D-2V 256^3 run's 8 MB of partials stay with the
        grid-wide vpfv_moment_partials."""
        if not partial_shapes:
            return False
        if all(sh[-2] == 1 for sh in partial_shapes):
            return True
        total = sum(int(np.prod(sh)) for sh in partial_shapes)
        return total <= 32768 and max(512 * sh[-2] for sh in partial_shapes) <= 200 * 1024

    def field_and_tables_1d(self, tables, packed, partials=None, stream=None, conv=False):
        """Moments-from-partials (when given) -> rho -> Ex -> every species'
        line tables in one launch.  ``conv=False``: one CTA with the FFT
        (vpfv_field_1d), bitwise the chain moments_from_partials / charge /
        poisson / StageTables.update; ``conv=True``: the Green's-function
        convolution over the whole GPU (vpfv_field_1d_conv; multi-row 1D-2V
        partials are finished by vpfv_moment_partials first).
        ``packed[s]``: species s gets the packed rows (1D-2V tiled kernel)."""
        stream = stream_handle(self.device) if stream is None else stream
        if conv:
            return self._field_conv_1d(tables, packed, partials, stream)
        key = (tuple(id(t) for t in tables), tuple(packed),
               None if partials is None else tuple(p.data_ptr() for p in partials))
        args = self._field1d_args.get(key)
        if args is None:
            S = len(tables)
            if partials is None:
                part = (None, None, None, None)
            else:
                part = (_lib.ptr_array([p.data_ptr() for p in partials]),
                        _lib.int_array([p.shape[-2] for p in partials]),
                        _lib.int_array([p.shape[-1] for p in partials]), _lib.dbl_array(self.vols))
            args = part + (
                self.n.data_ptr(), self.q_host, S, self.phys_shape[0], self.rho.data_ptr(),
                self.E["Ex"].data_ptr(), self.tw.data_ptr(), self.k2.data_ptr(), self.kd.data_ptr(),
                *self._table_args(tables, packed))
            self._field1d_args[key] = args
        _lib.call("vpfv_field_1d", *args, stream)
        return self.E

    @staticmethod
    def _table_args(tables, packed):
        """Per-species table outputs and constants of vpfv_field_1d[_conv]:
        packed rows for the tiled 1D-2V species, plain e/c1 otherwise."""
        pk = [bool(packed[s]) and t.grid.v == 2 for s, t in enumerate(tables)]
        return (_lib.ptr_array([0 if pk[s] else t.e.data_ptr() for s, t in enumerate(tables)]),
                _lib.ptr_array([0 if pk[s] else t.c1.data_ptr() for s, t in enumerate(tables)]),
                _lib.ptr_array([t.packed.data_ptr() if pk[s] else 0 for s, t in enumerate(tables)]),
                _lib.dbl_array([t.qmk2 for t in tables]), _lib.dbl_array([t.gx for t in tables]),
                _lib.dbl_array([t.t1 for t in tables]), _lib.dbl_array([t.den1 for t in tables]),
                _lib.int_array([1 if t.corrections else 0 for t in tables]))

    def _field_conv_1d(self, tables, packed, partials, stream):
        if partials is not None and any(p.shape[-2] != 1 for p in partials):
            self.moments_from_partials(partials, stream)
            partials = None
        key = ("conv", tuple(id(t) for t in tables), tuple(packed),
               None if partials is None else tuple(p.data_ptr() for p in partials))
        args = self._field1d_args.get(key)
        if args is None:
            S = len(tables)
            if partials is None:
                part = (None, None, None)
            else:
                part = (_lib.ptr_array([p.data_ptr() for p in partials]),
                        _lib.int_array([p.shape[-1] for p in partials]), _lib.dbl_array(self.vols))
            args = part + (
                self.n.data_ptr(), self.q_host, S, self.phys_shape[0], self.rho.data_ptr(),
                self.E["Ex"].data_ptr(), self.green2.data_ptr(), *self._table_args(tables, packed))
            self._field1d_args[key] = args
        _lib.call("vpfv_field_1d_conv", *args, stream)
        return self.E

    def moments(self, srcs, stream=None):
        stream = stream_handle(self.device) if stream is None else stream
        for s, (g, f) in enumerate(zip(self.grids, srcs)):
            _lib.call(self._moment_fn, f.data_ptr(), self.n[s].data_ptr(), g.d, g.v,
                      self.N_arrays[s], self.vols[s], stream)
        return self.n

    def moments_from_partials(self, partials, stream=None):
        """n_s from the fused-epilogue partials of each species' last stage."""
        stream = stream_handle(self.device) if stream is None else stream
        for s, (g, part) in enumerate(zip(self.grids, partials)):
            if part is None:
                raise ValueError("species without fused moment partials")
            _lib.call("vpfv_moment_partials", part.data_ptr(), self.n[s].data_ptr(), self.nphys,
                      part.shape[-2], part.shape[-1], self.vols[s], stream)  # partials [phys][rows][chunks]
        return self.n

    def solve_from_partials(self, partials, stream=None):
        self.moments_from_partials(partials, stream)
        self.charge(stream)
        return self.poisson(self.rho, False, stream)

    def poisson(self, rho, with_phi=False, stream=None):
        stream = stream_handle(self.device) if stream is None else stream
        phi = self.phi.data_ptr() if with_phi else None
        if self.d == 1:
            _lib.call("vpfv_poisson_1d", rho.data_ptr(), self.E["Ex"].data_ptr(), phi,
                      self.phys_shape[0], self.tw.data_ptr(), self.k2.data_ptr(),
                      self.kd.data_ptr(), stream)
        else:
            _lib.call("vpfv_poisson_2d", rho.data_ptr(), self.E["Ex"].data_ptr(),
                      self.E["Ey"].data_ptr(), phi, self.phys_shape[0], self.phys_shape[1],
                      self.twx.data_ptr(), self.twy.data_ptr(), self.kx.data_ptr(),
                      self.ky.data_ptr(), self.kxd.data_ptr(), self.kyd.data_ptr(),
                      self.scratch.data_ptr(), stream)
        return self.E

    def charge(self, stream=None):
        stream = stream_handle(self.device) if stream is None else stream
        _lib.call("vpfv_charge_density", self.n.data_ptr(), self.q_host, len(self.species),
                  self.nphys, self.rho.data_ptr(), stream)
        return self.rho

    def solve(self, srcs, with_phi=False, stream=None):
        """f -> n -> rho -> E on the device; returns the E dict (device)."""
        self.moments(srcs, stream)
        self.charge(stream)
        return self.poisson(self.rho, with_phi, stream)


# ---------------------------------------------------------------------------
# reference-shaped API functions (host or device inputs)


def _device_of(x):
    return x.device if isinstance(x, torch.Tensor) else torch.device("cuda", torch.cuda.current_device())


def _dev_array(a, device):
    if isinstance(a, torch.Tensor):
        return a.to(device=device, dtype=torch.float64).contiguous()
    return torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64), device=device)


def zeroth_moment(f, schedule="velocity-major"):
    """n(x) = sum_v f * prod(h_v) (fields.py:86-111).

    ``"velocity-major"``: the deterministic fold tree (``vpfv_moment``,
    bitwise the reference); ``"position-major"``: the per-cell sequential sum
    in C order (``vpfv_moment_seq``, bitwise the reference's compiled
    ``_seq_moment_*``); ``"free"``: the reference's library reduction with no
    fixed order ("performance experiments only") -- here the fold tree, one
    valid order of that sum.
    """
    if schedule not in ("velocity-major", "position-major", "free"):
        raise ValueError(f"unknown schedule {schedule!r}")
    g = f.grid
    device = _device_of(f.data)
    data = _dev_array(f.data, device)
    out = torch.empty(tuple(g.N[:g.d]), dtype=torch.float64, device=device)
    fn = "vpfv_moment_seq" if schedule == "position-major" else "vpfv_moment"
    _lib.call(fn, data.data_ptr(), out.data_ptr(), g.d, g.v, _lib.int_array(g.N),
              velocity_cell_volume(g), stream_handle(device))
    return out if isinstance(f.data, torch.Tensor) else out.cpu().numpy()


def higher_moments(f):
    """Momentum and kinetic-energy densities on the physical grid with the
    midpoint-to-average lift (fields.py:131-161): returns ``(momentum,
    kinetic)``, ``momentum`` one physical-grid array per velocity dim and
    ``kinetic`` = 1/2 sum_d <v_d^2 f>.  Ghosts must be synchronised.  Device
    data: the velocity sums run in ``vpfv_higher_moments``; host data: the
    reference's numpy arithmetic."""
    from .diagnostics import higher_moments_arrays

    g = f.grid
    if not isinstance(f.data, torch.Tensor):
        return higher_moments_arrays(np.asarray(f.data), g)
    device = f.data.device
    data = f.data.contiguous()
    vcs = [torch.as_tensor(g.centers(k), dtype=torch.float64, device=device) for k in g.velocity_dims]
    hv = [g.h[k] for k in g.velocity_dims]
    out = torch.empty(tuple(g.N[:g.d]) + (2 * g.v,), dtype=torch.float64, device=device)
    _lib.call("vpfv_higher_moments", data.data_ptr(), g.d, g.v, _lib.int_array(g.N), vcs[0].data_ptr(),
              vcs[1].data_ptr() if len(vcs) > 1 else None, hv[0], hv[1] if len(hv) > 1 else 0.0,
              out.data_ptr(), stream_handle(device))
    vol = velocity_cell_volume(g)
    mom = [out[..., 2 * k] * vol for k in range(g.v)]
    kin = 0.0
    for k in range(g.v):
        kin = kin + out[..., 2 * k + 1] * vol
    return mom, 0.5 * kin


def charge_density(densities, species):
    """rho = sum_s q_s n_s - mean (fields.py:164-169)."""
    as_np = not isinstance(densities[0], torch.Tensor)
    device = _device_of(densities[0])
    n = torch.stack([_dev_array(x, device) for x in densities])
    rho = torch.empty(n.shape[1:], dtype=torch.float64, device=device)
    _lib.call("vpfv_charge_density", n.data_ptr(), _lib.dbl_array([s.q for s in species]),
              len(species), int(rho.numel()), rho.data_ptr(), stream_handle(device))
    return rho.cpu().numpy() if as_np else rho


def poisson_solve(rho, grid):
    """Spectral periodic solve (fields.py:172-213); returns (phi, {"Ex"[, "Ey"]})."""
    as_np = not isinstance(rho, torch.Tensor)
    r = np.asarray(rho.detach().cpu().numpy() if not as_np else rho)
    if r.ndim != grid.d:
        raise ValueError("charge density must live on the physical grid")
    scale = np.max(np.abs(r)) if r.size else 0.0
    if abs(np.mean(r)) > 1e-10 * max(scale, 1.0):
        raise ValueError("poisson_solve requires zero-mean charge density")
    device = _device_of(rho)
    fs = _solver_for(grid, device)
    E = fs.poisson(_dev_array(r, device), with_phi=True)
    out_E = {k: (v.cpu().numpy() if as_np else v.clone()) for k, v in E.items()}
    phi = fs.phi.cpu().numpy() if as_np else fs.phi.clone()
    return phi, out_E


_SOLVERS = {}


def _solver_for(grid, device):
    from .fvm import SpeciesConfig

    key = (grid, str(device))
    if key not in _SOLVERS:
        _SOLVERS[key] = FieldSolver([grid], [SpeciesConfig()], device)
    return _SOLVERS[key]


@dataclass
class FieldState:
    """Densities and fields on the physical grid (fields.py:216-239)."""

    n: dict
    rho: object
    phi: object
    E: dict
    max_E: dict = field(default_factory=dict)

    @classmethod
    def solve(cls, dists, species, schedule="velocity-major"):
        dens = [zeroth_moment(f, schedule) for f in dists]
        rho = charge_density(dens, species)
        phi, E = poisson_solve(rho, dists[0].grid)
        max_E = {k: float(np.max(np.abs(np.asarray(v if not isinstance(v, torch.Tensor) else v.cpu()))))
                 for k, v in E.items()}
        return cls(n={sp.name: ns for sp, ns in zip(species, dens)}, rho=rho, phi=phi, E=E, max_E=max_E)
