"""Snapshot I/O: the reference's binary ``VPFV`` format, host and device.

Format (/root/reference/pkg/src/vpfv/diagnostics.py:184-234), all
little-endian: magic ``VPFV``, u32 version (1), u32 d, u32 v, u32 name length
+ utf-8 species tag, f64 time, per dimension u64 N, f64 lo, f64 hi, then the
interior cell averages row-major as f64.

* ``write_snapshot`` / ``read_snapshot`` mirror the reference on host
  ``DistField``s (byte-identical files, bitwise round trip);
* ``save_device`` / ``load_device`` stream one species of a device-resident
  state straight between the file and the device interior, a few x planes at
  a time through two pinned buffers (the copy of chunk k overlaps the file I/O
  of chunk k-1), so a 128^4 checkpoint never materialises the 2.6 GB padded
  array on the host.  ``Simulation.checkpoint`` and
  ``Simulation.restore`` (runner.py) use them.
"""

from __future__ import annotations

import struct

import numpy as np
import torch

from .grid import DistField, make_grid

SNAPSHOT_MAGIC = b"VPFV"
SNAPSHOT_VERSION = 1


def _header(grid, name, time):
    tag = name.encode("utf-8")
    parts = [SNAPSHOT_MAGIC, struct.pack("<III", SNAPSHOT_VERSION, grid.d, grid.v), struct.pack("<I", len(tag)),
             tag, struct.pack("<d", float(time))]
    for k in range(grid.ndim):
        parts.append(struct.pack("<Qdd", grid.N[k], grid.lo[k], grid.hi[k]))
    return b"".join(parts)


def _read_header(fh):
    magic = fh.read(4)
    if magic != SNAPSHOT_MAGIC:
        raise ValueError(f"not a snapshot file: magic {magic!r}")
    version, d, v = struct.unpack("<III", fh.read(12))
    if version != SNAPSHOT_VERSION:
        raise ValueError(f"unsupported snapshot version {version}")
    (nlen,) = struct.unpack("<I", fh.read(4))
    name = fh.read(nlen).decode("utf-8")
    (time,) = struct.unpack("<d", fh.read(8))
    N, lo, hi = [], [], []
    for _ in range(d + v):
        Nk, lok, hik = struct.unpack("<Qdd", fh.read(24))
        N.append(int(Nk))
        lo.append(lok)
        hi.append(hik)
    return name, time, make_grid(d, v, tuple(N), tuple(lo), tuple(hi))


def write_snapshot(path, dist: DistField, time, species=None):
    """One species' interior cell averages with grid metadata
    (diagnostics.py:187-203)."""
    g = dist.grid
    with open(path, "wb") as fh:
        fh.write(_header(g, species if species is not None else dist.species, time))
        fh.write(np.ascontiguousarray(dist.data[g.interior_slices()]).astype("<f8", copy=False).tobytes())


def read_snapshot(path):
    """(DistField, time) from a snapshot; bitwise round trip (diagnostics.py:206-234)."""
    with open(path, "rb") as fh:
        name, time, grid = _read_header(fh)
        count = int(np.prod(grid.N))
        raw = fh.read(count * 8)
        if len(raw) != count * 8:
            raise ValueError("snapshot truncated")
        interior = np.frombuffer(raw, dtype="<f8").reshape(tuple(grid.N))
    f = DistField(grid, species=name)
    f.data[grid.interior_slices()] = interior
    return f, time


def _chunks(grid, planes):
    n0 = grid.N[0]
    return [(i, min(i + planes, n0)) for i in range(0, n0, planes)]


def save_device(path, array, grid, name, time, planes=8):
    """Stream the interior of a padded device ``array`` (``grid``) into a
    snapshot file, ``planes`` x planes per chunk."""
    inner = grid.interior_slices()
    plane = tuple(grid.N[1:])
    bufs = [torch.empty((planes,) + plane, dtype=torch.float64).pin_memory() for _ in range(2)]
    copy = torch.cuda.Stream(array.device)
    done = [torch.cuda.Event(), torch.cuda.Event()]
    copy.wait_stream(torch.cuda.current_stream(array.device))  # the state is complete
    with open(path, "wb") as fh:
        fh.write(_header(grid, name, time))
        chunks = _chunks(grid, planes)
        pending = None
        for k, (a, b) in enumerate(chunks):
            buf = bufs[k & 1]
            with torch.cuda.stream(copy):
                buf[:b - a].copy_(array[(slice(inner[0].start + a, inner[0].start + b),) + inner[1:]],
                                  non_blocking=True)
                done[k & 1].record(copy)
            if pending is not None:  # write chunk k-1 while chunk k is copied
                pk, pn = pending
                done[pk & 1].synchronize()
                fh.write(bufs[pk & 1][:pn].numpy().tobytes())
            pending = (k, b - a)
        if pending is not None:
            pk, pn = pending
            done[pk & 1].synchronize()
            fh.write(bufs[pk & 1][:pn].numpy().tobytes())


def load_device(path, array, grid, planes=8, species=None):
    """Stream a snapshot's interior into the padded device ``array``
    (ghosts untouched); returns (species name, time).  The file's grid
    (extents, dimensionality, box bounds) must match ``grid`` and, when given,
    its species tag ``species``.  The copies are ordered after the work
    already queued on the caller's stream (e.g. a launched step still reading
    ``array``)."""
    inner = grid.interior_slices()
    plane = tuple(grid.N[1:])
    bufs = [torch.empty((planes,) + plane, dtype=torch.float64).pin_memory() for _ in range(2)]
    copy = torch.cuda.Stream(array.device)
    copy.wait_stream(torch.cuda.current_stream(array.device))
    done = [None, None]
    with open(path, "rb") as fh:
        name, time, g = _read_header(fh)
        if tuple(g.N) != tuple(grid.N) or (g.d, g.v) != (grid.d, grid.v):
            raise ValueError(f"snapshot grid {g.N} (d={g.d}, v={g.v}) does not match {grid.N}")
        if tuple(g.lo) != tuple(grid.lo) or tuple(g.hi) != tuple(grid.hi):
            raise ValueError(f"snapshot box {g.lo}..{g.hi} does not match {grid.lo}..{grid.hi}")
        if species is not None and name != species:
            raise ValueError(f"snapshot holds species {name!r}, expected {species!r}")
        per_plane = int(np.prod(plane)) * 8
        for k, (a, b) in enumerate(_chunks(grid, planes)):
            buf = bufs[k & 1]
            if done[k & 1] is not None:
                done[k & 1].synchronize()  # the copy out of this buffer (chunk k-2) finished
            view = buf[:b - a].numpy()  # read straight into the pinned buffer
            if fh.readinto(memoryview(view).cast("B")) != (b - a) * per_plane:
                raise ValueError("snapshot truncated")
            with torch.cuda.stream(copy):
                array[(slice(inner[0].start + a, inner[0].start + b),) + inner[1:]].copy_(buf[:b - a],
                                                                                          non_blocking=True)
                ev = torch.cuda.Event()
                ev.record(copy)
                done[k & 1] = ev
    copy.synchronize()
    torch.cuda.current_stream(array.device).wait_stream(copy)
    return name, time
