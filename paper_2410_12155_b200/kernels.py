"""The fused stage operator on the B200: tables + launch + the drop-in API.

``fused_stage(dest, A, B, src, ca, cb, cd, cL, grid, species, E, check=True)``
is the drop-in replacement for the reference dispatcher
(/root/reference/pkg/src/vpfv/_kernels.py:320-373): same arguments, same
in-place semantics on the interior, same errors (``ValueError`` for
``dest is src`` or an unsupported dimensionality, ``FloatingPointError`` with
the interior multi-index of the first non-finite output).  Arrays may be
host numpy arrays (copied to/from the device around the call) or float64
CUDA tensors.  ``exact=True`` (the default here) evaluates in the reference
kernels' operation order and is bitwise equal to them; the drivers default to
the FMA fast path.

``StageTables`` holds one species' per-line tables on the device: static
ones (velocity centres, the magnetic factor, ...) built once on the host in
the reference's numpy arithmetic, and the E-dependent ones recomputed on the
device each stage by ``vpfv_tables_*``.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _lib
from .fvm import _g, magnetic_factor

SUPPORTED = ((1, 1), (1, 2), (2, 2))


def _ptr(t):
    return None if t is None else t.data_ptr()


def stream_handle(device=None):
    return torch.cuda.current_stream(device).cuda_stream


class StageTables:
    """Per-species device tables for the fused stage kernel."""

    def __init__(self, grid, species, device, corrections=True):
        if (grid.d, grid.v) not in SUPPORTED:
            raise ValueError(f"unsupported dimensionality ({grid.d},{grid.v})")
        self.grid, self.species, self.device = grid, species, device
        self.corrections = corrections
        s, g, h = species, grid, grid.h
        gx, gy = _g(s)[:2]
        cB = magnetic_factor(s)
        dev = lambda a: torch.as_tensor(np.ascontiguousarray(a, dtype=np.float64), device=device)  # noqa: E731
        self.gx, self.gy, self.cB = gx, gy, cB
        self.qmk2 = s.qm * s.kappa2            # (_kernels.py:337) qm*kappa2 first
        self.nqmk2 = -s.qm * s.kappa2          # (fvm.py:198) (-qm)*kappa2
        nphys = int(np.prod(g.N[:g.d]))
        phys_shape = tuple(g.N[:g.d])
        if (g.d, g.v) == (1, 1):
            self.ax = dev(g.centers(1))
            self.t1, self.den1 = h[1] / (48.0 * h[0]), 96.0 * h[1]
            self.e = torch.empty(phys_shape, dtype=torch.float64, device=device)   # avx
            self.c1 = torch.empty(phys_shape, dtype=torch.float64, device=device)
        elif (g.d, g.v) == (1, 2):
            self.vxc = dev(g.centers(1))
            vyc = np.empty(g.N[2] + 1)
            vyc[:-1] = g.centers(2)
            vyc[-1] = cB
            self.vyc = dev(vyc)
            self.avy = dev(-cB * g.centers(1) + gy)
            self.c2 = float(s.qm * (s.kappa_c / 48.0) * s.Bz * (h[1] / h[2] - h[2] / h[1]))
            self.t1, self.den1 = h[1] / (48.0 * h[0]), 96.0 * h[1]
            self.e = torch.empty(phys_shape, dtype=torch.float64, device=device)   # evx
            self.c1 = torch.empty(phys_shape, dtype=torch.float64, device=device)
            # packed (evx, c1) rows with periodic x ghost rows, for the tiled kernel
            self.packed = torch.zeros((g.N[0] + 2, 8), dtype=torch.float64, device=device)
        else:
            self.vxc = dev(g.centers(2))
            self.vyc = dev(g.centers(3))
            self.c2 = float(s.qm * (s.kappa_c / 48.0) * s.Bz * (h[2] / h[3] - h[3] / h[2]))
            self.t1, self.t4 = h[2] / (48.0 * h[0]), h[3] / (48.0 * h[1])
            self.denx, self.deny = 96.0 * h[2], 96.0 * h[3]
            mk = lambda: torch.empty(phys_shape, dtype=torch.float64, device=device)  # noqa: E731
            self.evx, self.evy, self.c1, self.c3, self.c4, self.c5 = (mk() for _ in range(6))
            # packed (evx, evy, c1, c3, c4, c5) rows with periodic x ghost rows, for the tiled kernel
            self.packed = torch.zeros((g.N[0] + 2, g.N[1], 8), dtype=torch.float64, device=device)
        if not corrections:
            self.c2 = 0.0
        self.nphys = nphys

    def fused_moment_ok(self, flags):
        """True when a TMA-tiled kernel (2D-2V or 1D-2V, with its fused
        moment epilogue) applies to this grid and these flags."""
        g = self.grid
        if flags & _lib.VPFV_EXACT:
            return False
        if (g.d, g.v) == (1, 1):
            return g.N[1] % 128 == 0
        if (g.d, g.v) == (2, 2):
            return bool(_lib.load().vpfv_stage_2d2v_tiled_ok(*g.N, flags))
        if (g.d, g.v) == (1, 2):
            return bool(_lib.load().vpfv_stage_1d2v_tiled_ok(*g.N, flags))
        return False

    def partials_shape(self):
        g = self.grid
        if (g.d, g.v) == (2, 2):
            return (g.N[0], g.N[1], g.N[2], g.N[3] // _lib.load().vpfv_stage_2d2v_partials_chunk())
        if (g.d, g.v) == (1, 1):
            return (g.N[0], 1, g.N[1] // 128)
        return (g.N[0], g.N[1], g.N[2] // _lib.load().vpfv_stage_1d2v_partials_chunk())

    # -- per-stage tables from E (device arrays on the physical grid) ---------
    def update(self, E, stream, packed=False):
        """Recompute the E-dependent tables; ``packed`` builds the layout the
        tiled 2D-2V kernel streams (instead of the separate arrays)."""
        g = self.grid
        if g.d == 1:
            Ex = E["Ex"]
            if packed and g.v == 2:  # the 1D-1V kernels read the plain tables
                _lib.call("vpfv_tables_1d_packed", Ex.data_ptr(), self.packed.data_ptr(), g.N[0],
                          self.qmk2, self.gx, self.t1, self.den1, stream)
                if not self.corrections:
                    self.packed[:, 1].zero_()
            else:
                _lib.call("vpfv_tables_1d", Ex.data_ptr(), self.e.data_ptr(), self.c1.data_ptr(),
                          g.N[0], self.qmk2, self.gx, self.t1, self.den1, stream)
                if not self.corrections:
                    self.c1.zero_()
        else:
            common = (g.N[0], g.N[1], self.qmk2, self.nqmk2, self.gx, self.gy, self.t1, self.t4,
                      self.denx, self.deny, stream)
            if packed:
                _lib.call("vpfv_tables_2d_packed", E["Ex"].data_ptr(), E["Ey"].data_ptr(),
                          self.packed.data_ptr(), *common)
                if not self.corrections:
                    self.packed[:, :, 2:6].zero_()
            else:
                _lib.call("vpfv_tables_2d", E["Ex"].data_ptr(), E["Ey"].data_ptr(),
                          self.evx.data_ptr(), self.evy.data_ptr(), self.c1.data_ptr(),
                          self.c3.data_ptr(), self.c4.data_ptr(), self.c5.data_ptr(), *common)
                if not self.corrections:
                    for c in (self.c1, self.c3, self.c4, self.c5):
                        c.zero_()

    # -- launch ---------------------------------------------------------------
    def launch(self, dest, A, B, src, ca, cb, cd, cL, flags, stream, dt_dev=None, cL_div=1.0,
               nonfinite=None, partials=None, packed=False, xsegments=0):
        g, h, N = self.grid, self.grid.h, self.grid.N
        common_tail = (flags, _ptr(dt_dev), float(cL_div), _ptr(nonfinite), stream)
        head = (dest.data_ptr(), A.data_ptr(), B.data_ptr(), src.data_ptr(),
                float(ca), float(cb), float(cd), float(cL))
        if (g.d, g.v) == (1, 1):
            if partials is not None:
                _lib.call("vpfv_stage_1d1v_fused", *head, self.ax.data_ptr(), self.e.data_ptr(),
                          self.c1.data_ptr(), h[0], h[1], N[0], N[1], flags, _ptr(dt_dev), float(cL_div),
                          _ptr(nonfinite), partials.data_ptr(), stream)
            else:
                _lib.call("vpfv_stage_1d1v", *head, self.ax.data_ptr(), self.e.data_ptr(),
                          self.c1.data_ptr(), h[0], h[1], N[0], N[1], *common_tail)
        elif (g.d, g.v) == (1, 2):
            args = (*head, self.vxc.data_ptr(), self.vyc.data_ptr(), self.e.data_ptr(),
                    self.avy.data_ptr(), self.c1.data_ptr(), self.c2, h[0], h[1], h[2], N[0], N[1], N[2])
            if packed or partials is not None:
                _lib.call("vpfv_stage_1d2v_fused", *args, flags, _ptr(dt_dev), float(cL_div),
                          _ptr(nonfinite), self.packed.data_ptr() if packed else None,
                          _ptr(partials), 0, stream)
            else:
                _lib.call("vpfv_stage_1d2v", *args, *common_tail)
        else:
            args = (*head, self.vxc.data_ptr(), self.vyc.data_ptr(), self.evx.data_ptr(),
                    self.evy.data_ptr(), self.cB, self.c1.data_ptr(), self.c2, self.c3.data_ptr(),
                    self.c4.data_ptr(), self.c5.data_ptr(), h[0], h[1], h[2], h[3], N[0], N[1], N[2], N[3])
            if packed or partials is not None:
                _lib.call("vpfv_stage_2d2v_fused", *args, flags, _ptr(dt_dev), float(cL_div),
                          _ptr(nonfinite), self.packed.data_ptr() if packed else None,
                          _ptr(partials), int(xsegments), stream)
            else:
                _lib.call("vpfv_stage_2d2v", *args, *common_tail)


def wrap_flags(grid, dims=None):
    """Stage flags reading the given (default: all periodic) dims by modular index."""
    f = 0
    for k in range(grid.ndim):
        if grid.periodic[k] and (dims is None or k in dims):
            f |= _lib.VPFV_WRAP(k)
    return f


def nonfinite_index(flag_value, grid):
    """Interior multi-index of a flat C-order interior offset."""
    return tuple(int(i) for i in np.unravel_index(int(flag_value), grid.N))


class _HostStager:
    """Host <-> device copies of padded fp64 arrays along axis 0 through two
    fixed pinned chunks (double-buffered; the numpy side of each chunk is
    copied by a small thread pool, overlapping the PCIe transfer of the other
    chunk).  Nothing field-sized is allocated per call: the drop-in keeps the
    reference's "no field-sized allocation while stepping" contract
    (/root/reference/pkg/tests/test_timestepping.py:234-254) on the host."""

    CHUNK_BYTES = 64 << 20
    THREADS = 8
    NBUF = 2

    def __init__(self, device, plane_shape):
        from concurrent.futures import ThreadPoolExecutor

        self.device = device
        self.plane_shape = tuple(plane_shape)
        self.plane = int(np.prod(plane_shape))
        self.nplanes = max(1, self.CHUNK_BYTES // (8 * self.plane))
        self.bufs = [torch.empty(self.nplanes * self.plane, dtype=torch.float64, pin_memory=True)
                     for _ in range(self.NBUF)]
        self.views = [b.numpy().reshape((self.nplanes,) + self.plane_shape) for b in self.bufs]
        self.events = [torch.cuda.Event() for _ in range(self.NBUF)]
        self.stream = torch.cuda.Stream(device)
        self.pool = ThreadPoolExecutor(self.THREADS)

    def _copy(self, dst, src):
        """np.copyto split over the pool along the largest leading axis."""
        ax = 0 if dst.shape[0] >= self.THREADS else 1
        n = dst.shape[ax]
        k = min(self.THREADS, n)
        cuts = [n * i // k for i in range(k + 1)]
        idx = lambda i: (slice(cuts[i], cuts[i + 1]),) if ax == 0 else (slice(None), slice(cuts[i], cuts[i + 1]))  # noqa: E731
        list(self.pool.map(lambda i: np.copyto(dst[idx(i)], src[idx(i)]), range(k)))

    def upload(self, host, dev, p0, p1, inner=None):
        """dev[p0:p1] <- host[p0:p1] (``inner``: only those trailing slices are
        read from the host; the rest of each staged plane is left as it was)."""
        main = torch.cuda.current_stream(self.device)
        self.stream.wait_stream(main)  # the device buffer is free once earlier work on it is done
        k = 0
        for a in range(p0, p1, self.nplanes):
            b = min(p1, a + self.nplanes)
            j = k % self.NBUF
            self.events[j].synchronize()  # the transfer that last used this chunk is done
            view = self.views[j][:b - a]
            if inner is None:
                self._copy(view, host[a:b])
            else:
                self._copy(view[(slice(None),) + inner], host[(slice(a, b),) + inner])
            with torch.cuda.stream(self.stream):
                dev[a:b].copy_(self.bufs[j][:(b - a) * self.plane].view((b - a,) + self.plane_shape),
                               non_blocking=True)
                self.events[j].record(self.stream)
            k += 1
        main.wait_stream(self.stream)

    def download(self, dev, host, p0, p1, inner):
        """host[p0:p1][inner] <- dev[p0:p1][inner] (the planes' other cells untouched)."""
        self.stream.wait_stream(torch.cuda.current_stream(self.device))
        chunks = [(a, min(p1, a + self.nplanes)) for a in range(p0, p1, self.nplanes)]

        def issue(k):
            a, b = chunks[k]
            j = k % self.NBUF
            with torch.cuda.stream(self.stream):
                self.bufs[j][:(b - a) * self.plane].view((b - a,) + self.plane_shape).copy_(dev[a:b], non_blocking=True)
                self.events[j].record(self.stream)

        nb = self.NBUF
        for k in range(min(nb, len(chunks))):
            issue(k)
        for k, (a, b) in enumerate(chunks):
            self.events[k % nb].synchronize()
            self._copy(host[(slice(a, b),) + inner], self.views[k % nb][:b - a][(slice(None),) + inner])
            if k + nb < len(chunks):  # chunk k's buffer is free again
                issue(k + nb)


class _DropIn:
    """Per-(grid, species, device, mode) state of the drop-in ``fused_stage``:
    four padded device buffers, the stage tables, E on the device, the
    non-finite word and the host stager -- allocated on the first call and
    reused by every later one."""

    def __init__(self, grid, species, device, exact):
        self.grid, self.device = grid, device
        # zeroed once: the chunked download moves whole planes (ghosts included)
        # and keeps only interiors; no copy then reads uninitialised memory
        self.bufs = [torch.zeros(grid.padded_shape, dtype=torch.float64, device=device) for _ in range(4)]
        self.tables = StageTables(grid, species, device)
        self.flags = _lib.VPFV_EXACT if exact else 0
        self.tiled = self.tables.fused_moment_ok(self.flags)
        self.E = {}
        self.flag = torch.full((1,), -1, dtype=torch.int64, device=device)
        self.stager = _HostStager(device, grid.padded_shape[1:])
        self.inner = tuple(slice(3, 3 + n) for n in grid.N)

    def e_dev(self, E):
        out = {}
        for k, v in E.items():
            if isinstance(v, torch.Tensor) and v.is_cuda:
                out[k] = v.to(torch.float64).contiguous()
                continue
            a = np.asarray(v, dtype=np.float64)
            t = self.E.get(k)
            if t is None or tuple(t.shape) != a.shape:
                t = self.E[k] = torch.empty(a.shape, dtype=torch.float64, device=self.device)
            t.copy_(torch.from_numpy(np.ascontiguousarray(a)))
            out[k] = t
        return out


_DROPIN = {}


def _dropin_for(grid, species, device, exact):
    key = (grid, repr(species), device.index, bool(exact))
    ctx = _DROPIN.get(key)
    if ctx is None:
        if len(_DROPIN) >= 2:  # bounded: at most two (grid, species) set-ups cached
            _DROPIN.pop(next(iter(_DROPIN)))
        ctx = _DROPIN[key] = _DropIn(grid, species, device, exact)
    return ctx


def _check_device_array(a):
    if not a.is_cuda or a.dtype != torch.float64 or not a.is_contiguous():
        raise ValueError("device arrays must be contiguous float64 CUDA tensors")
    return a


def fused_stage(dest, A, B, src, ca, cb, cd, cL, grid, species, E, check=True, exact=True):
    """Drop-in for the reference ``fused_stage`` (_kernels.py:320-373).

    Device (CUDA tensor) arguments are used in place.  Host (numpy) arguments
    go through a cached per-set-up context: src is uploaded whole (its ghost
    cells are read), the RK operands only over the interior x-planes (in fast
    mode only those with a nonzero coefficient), dest's interior is downloaded into the
    caller's array; aliasing between the host arrays is honoured (one device
    buffer per distinct array).  No field-sized host or device allocation
    happens after the first call for a set-up.
    """
    if dest is src:
        raise ValueError("dest must not alias src")
    if (grid.d, grid.v) not in SUPPORTED:
        raise ValueError(f"unsupported dimensionality ({grid.d},{grid.v})")
    arrays = (dest, A, B, src)
    on_device = [isinstance(x, torch.Tensor) for x in arrays]
    device = next((x.device for x, d in zip(arrays, on_device) if d), None)
    if device is None:
        device = torch.device("cuda", torch.cuda.current_device())
    _lib.check_device(device.index if device.index is not None else torch.cuda.current_device())
    for x in arrays:
        if tuple(x.shape) != grid.padded_shape:
            raise ValueError(f"array shape {tuple(x.shape)} != padded {grid.padded_shape}")
    ctx = _dropin_for(grid, species, device, exact)
    stream = stream_handle(device)
    # one device buffer per distinct host array (aliasing preserved)
    dev, slot = {}, 0
    for x, d in zip(arrays, on_device):
        if d:
            dev[id(x)] = _check_device_array(x)
        elif id(x) not in dev:
            if not isinstance(x, np.ndarray) or x.dtype != np.float64:
                raise ValueError("host arrays must be float64 numpy arrays")
            dev[id(x)] = ctx.bufs[slot]
            slot += 1
    d_dest, d_A, d_B, d_src = (dev[id(x)] for x in arrays)
    if d_dest.data_ptr() == d_src.data_ptr():
        raise ValueError("dest must not alias src")
    n0 = grid.padded_shape[0]
    rest = ctx.inner[1:]
    uploaded = set()
    if not on_device[3]:
        ctx.stager.upload(src, d_src, 0, n0)  # ghosts included: the stencil reads them
        uploaded.add(id(src))
    for x, c, d in ((A, ca, on_device[1]), (B, cb, on_device[2]), (dest, cd, on_device[0])):
        # read at the updated cell only; the exact kernels evaluate every term
        # in the reference's order (0 * inf is nan there too), the fast ones
        # skip zero coefficients
        if not d and (c != 0.0 or exact) and id(x) not in uploaded:
            ctx.stager.upload(x, dev[id(x)], 3, 3 + grid.N[0], inner=rest)
            uploaded.add(id(x))
    E_dev = ctx.e_dev(E)
    ctx.tables.update(E_dev, stream, packed=ctx.tiled)
    flag = None
    if check:
        flag = ctx.flag
        flag.fill_(-1)
    ctx.tables.launch(d_dest, d_A, d_B, d_src, ca, cb, cd, cL, ctx.flags, stream, nonfinite=flag,
                      packed=ctx.tiled)
    if not on_device[0]:
        ctx.stager.download(d_dest, dest, 3, 3 + grid.N[0], rest)
    if check:
        v = int(flag.item()) & 0xFFFFFFFFFFFFFFFF
        if v != _lib.VPFV_FINITE:
            mi = nonfinite_index(v, grid)
            raise FloatingPointError(f"non-finite stage output at interior index {mi}")
