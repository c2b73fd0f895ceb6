"""Single-GPU driver: the reference ``Simulation`` with its state on the B200.

Mirrors /root/reference/pkg/src/vpfv/runner.py:126-256 (``Simulation``,
``RunDiverged``, ``stable_dt``): same constructor, ``advance``/``run``/
``current_dt``/``max_dt``/``interiors``/``state``/``diagnostics_row``/
``persistent_buffers`` and the three persistent buffers per species in a
``StepContext`` (here float64 CUDA tensors in the reference's padded layout).

Per stage (runner.py:183-191) the device runs
    moments (fold tree) -> rho -> Poisson/E -> line tables -> fused stage
and ``advance`` replays one CUDA graph holding all four stages of a step
(cL read on the device as dt / cL_div, so one graph serves every dt).
Ghosts: frozen velocity slabs are written into all three buffers once at
set-up (kernels write interiors only); periodic dims are read by modular
indexing inside the stage kernel, so no per-stage ghost fill exists.
The non-finite check of ``advance`` (runner.py:219-227) is the stage-4
epilogue flag, read back once per step, with the reference's rollback.
"""

from __future__ import annotations

import ctypes
import math
import os

import numpy as np
import torch

from . import _lib
from .diagnostics import conserved_quantities_arrays
from .fields import FieldSolver
from .fvm import max_speed_per_dim
from .grid import DistField, FrozenGhosts, fill_local_ghosts
from .kernels import StageTables, stream_handle, wrap_flags

_FINITE = np.uint64(_lib.VPFV_FINITE)
from .timestepping import DEFAULT_SIGMA, RK4_STAGES, StepContext, max_stable_dt


class RunDiverged(RuntimeError):
    """Non-finite state; f0 holds the last completed state (runner.py:64-66)."""


def stable_dt(grids, species, E, sigma=DEFAULT_SIGMA):
    """min over species of sigma / sum_d max|A_d|/h_d (runner.py:98-103)."""
    return min(max_stable_dt([max_speed_per_dim(g, sp, E)], g.h, sigma=sigma)
               for g, sp in zip(grids, species))


def _host_filled(f):
    """Padded float64 host copy of a set-up field with its ghosts filled the
    way the reference's first stage fills them, plus its frozen slabs."""
    data = f.data.detach().cpu().numpy() if isinstance(f.data, torch.Tensor) else f.data
    data = np.array(data, dtype=np.float64, copy=True)
    df = DistField(f.grid, f.species, data)
    frozen = FrozenGhosts.capture(df)
    fill_local_ghosts(df, frozen)
    return data, frozen


def _device_filled(f, device):
    """A device-resident set-up field with the ghosts _host_filled would
    give it: the velocity slabs are its own t=0 values (frozen), the periodic
    dims are wrapped whole-column in ascending order on the device
    (vpfv_wrap_fill, grid.py:263-277)."""
    g = f.grid
    data = f.data.to(device=device, dtype=torch.float64).contiguous().clone()
    mask = sum(1 << k for k in range(g.ndim) if g.periodic[k])
    if mask:
        _lib.call("vpfv_wrap_fill", data.data_ptr(), g.ndim, _lib.int_array(g.N), mask,
                  torch.cuda.current_stream(device).cuda_stream)
    return data


def require_cuda(device=None):
    if not torch.cuda.is_available():
        raise _lib.VpfvError("no CUDA device visible: the B200 path has no CPU fallback")
    dev = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
    if dev.index is None:
        dev = torch.device("cuda", torch.cuda.current_device())
    _lib.check_device(dev.index)
    return dev


class Simulation:
    """Whole-domain driver owning exactly three device buffers per species."""

    def __init__(self, setup, cfl_fraction=0.9, dt=None, corrections=True,
                 schedule="velocity-major", sigma=DEFAULT_SIGMA, *, device=None, exact=False,
                 use_graphs=True):
        if schedule not in ("velocity-major", "position-major", "free"):
            raise ValueError(f"unknown schedule {schedule!r}")
        self.device = require_cuda(device)
        self.species = tuple(setup.species)
        self.grids = tuple(f.grid for f in setup.dists)
        self.cfl_fraction = cfl_fraction
        self.fixed_dt = dt
        self.corrections = corrections
        self.schedule = schedule
        self.sigma = sigma
        self.exact = exact
        self.use_graphs = use_graphs
        self._names = [f.species for f in setup.dists]
        f0, self.frozen = [], []
        for f in setup.dists:
            if isinstance(f.data, torch.Tensor) and f.data.is_cuda:
                f0.append(_device_filled(f, self.device))  # built on the device (problems.separable_on_device)
                self.frozen.append(None)  # captured from the device buffer when a host view needs it
            else:
                data, frozen = _host_filled(f)
                f0.append(torch.from_numpy(data).to(self.device))
                self.frozen.append(frozen)
        # velocity ghosts are frozen: all three buffers start as the filled t=0 array
        self.ctx = StepContext(f0=f0, f1=[a.clone() for a in f0], fout=[a.clone() for a in f0])
        self.tables = [StageTables(g, sp, self.device, corrections) for g, sp in zip(self.grids, self.species)]
        self.fields = FieldSolver(self.grids, self.species, self.device, schedule)
        base = _lib.VPFV_EXACT if exact else 0
        self.flags = [base | wrap_flags(g) for g in self.grids]
        S = len(self.species)
        self.nonfinite = torch.full((4, S), -1, dtype=torch.int64, device=self.device)
        self._flags_host = torch.empty((4, S), dtype=torch.int64, pin_memory=True)
        self._flags_np = self._flags_host.numpy().view(np.uint64)  # the divergence check reads this view
        self._dt_set = None  # the dt value dt_dev holds (refilled only when it changes)
        self.dt_dev = torch.zeros(1, dtype=torch.float64, device=self.device)
        self._graphs = {}
        self._launches = {}
        # fused velocity moment: every stage emits the moment partials of its
        # dest, which is the next stage's src; stage 4's partials (of the new
        # f0) serve the next step's stage 1 unless f0 was modified in place
        # since (torch's version counter) -- then the standalone moment runs
        self.tiled = [t.fused_moment_ok(f) for t, f in zip(self.tables, self.flags)]
        # the fused epilogue partials are nodes of the fold tree: the
        # sequential "position-major" sum needs the standalone moment
        self.fuse_moment = all(self.tiled) and schedule != "position-major"
        mk = lambda: ([torch.empty(t.partials_shape(), dtype=torch.float64, device=self.device)  # noqa: E731
                       for t in self.tables] if self.fuse_moment else None)
        self.partials = mk()       # written by stages 1-3, read by stages 2-4
        self.partials_next = mk()  # written by stage 4 (moment of the new f0), read by the next stage 1
        self._moment_of = None  # (data_ptr, _version) of the f0 arrays the partials describe
        # d = 1: moments-from-partials, rho, Ex and every species' tables in
        # one single-CTA launch per stage instead of 2 + 2S small ones
        self.fuse_field = self.fields.field_1d_ok() and os.environ.get("VPFV_FIELD_SPLIT", "0") != "1"
        # ... over the whole GPU (Green's-function convolution) unless VPFV_FIELD_CONV=0
        self.field_conv = self.fuse_field and os.environ.get("VPFV_FIELD_CONV", "1") != "0"
        self._finish_in_field = self.fuse_moment and (
            all(t.partials_shape()[-2] == 1 for t in self.tables) if self.field_conv
            else self.fields.finish_in_field_1d([t.partials_shape() for t in self.tables]))
        self._side = [torch.cuda.Stream(self.device) for _ in self.species[1:]]  # concurrent species
        self._diag = None
        self._last_E = None
        self._timing = False
        self._events = None
        self._stage_ms = [0.0] * 4

    # -- state access --------------------------------------------------------
    @property
    def t(self):
        return self.ctx.t

    @property
    def step_count(self):
        return self.ctx.step

    def persistent_buffers(self):
        return (self.ctx.f0, self.ctx.f1, self.ctx.fout)

    # -- the stage protocol (timestepping.py:69-84 calls this) ---------------
    def _stage(self, dest, A, B, src, ca, cb, cd, cL, t, *, dt_dev=None, cL_div=1.0, slot=None, cached=False,
               emit_last=True):
        stream = stream_handle(self.device)
        use_partials = self.fuse_moment and slot is not None and (slot > 0 or cached)
        emit_partials = self.fuse_moment and slot is not None and (slot < 3 or emit_last)
        if self.fuse_field:
            if use_partials:
                part = self.partials if slot > 0 else self.partials_next
                if not self._finish_in_field:
                    self.fields.moments_from_partials(part, stream)
                    part = None
            else:
                part = None
                self.fields.moments(src, stream)
            E = self.fields.field_and_tables_1d(self.tables, self.tiled, part, stream=stream, conv=self.field_conv)
        elif use_partials:
            E = self.fields.solve_from_partials(self.partials if slot > 0 else self.partials_next, stream=stream)
        else:
            E = self.fields.solve(src, stream=stream)
        self._last_E = E
        main = torch.cuda.current_stream(self.device)
        forked = []
        for s, tab in enumerate(self.tables):
            # species > 0 run on side streams forked from this one, so their
            # stage kernels overlap (and fill each other's wave tails); the
            # fork/join is captured into the step graph as parallel branches
            side = self._side[s - 1] if (s > 0 and self._side) else None
            if side is not None:
                side.wait_stream(main)
                forked.append(side)
            with torch.cuda.stream(side if side is not None else main):
                st = stream_handle(self.device)
                if not self.fuse_field:
                    tab.update(E, st, packed=self.tiled[s])
                nf = None if slot is None else self.nonfinite[slot, s:s + 1]
                timed = self._timing and slot is not None
                if timed:
                    self._events[slot][s][0].record()
                tab.launch(dest[s], A[s], B[s], src[s], ca, cb, cd, cL, self.flags[s], st,
                           dt_dev=dt_dev, cL_div=cL_div, nonfinite=nf,
                           partials=(self.partials if slot < 3 else self.partials_next)[s] if emit_partials else None,
                           packed=self.tiled[s], xsegments=1 if len(self.tables) > 1 else 0)
                if timed:
                    self._events[slot][s][1].record()
        for side in forked:
            main.wait_stream(side)

    def _step_body(self, f0, f1, fout, cached=False, emit_last=True):
        bufs = {"f0": f0, "f1": f1, "fout": fout}
        start = _lib.launch_counter[0]
        self.nonfinite.fill_(-1)
        for slot, (dn, an, bn, sn, ca, cb, cd, div) in enumerate(RK4_STAGES):
            self._stage(bufs[dn], bufs[an], bufs[bn], bufs[sn], ca, cb, cd, 0.0, None,
                        dt_dev=self.dt_dev, cL_div=div, slot=slot, cached=cached, emit_last=emit_last)
        self._launches["step"] = _lib.launch_counter[0] - start
        # the divergence flags reach pinned host memory as part of the step (a
        # captured D2H node), so advance() needs only the stream sync
        self._flags_host.copy_(self.nonfinite, non_blocking=True)

    # -- in-step timing of the fused stage kernel (bench roofline) -----------
    def enable_stage_timing(self, on=True):
        """Record CUDA events around every stage-kernel launch of ``advance``
        (captured into the step graph as external event nodes)."""
        import torch as _t

        self._timing = bool(on)
        self._stage_ms = [0.0] * 4
        if on and self._events is None:
            S = len(self.species)
            self._events = [[(_t.cuda.Event(enable_timing=True, external=True),
                              _t.cuda.Event(enable_timing=True, external=True)) for _ in range(S)]
                            for _ in range(4)]

    def stage_kernel_ms(self):
        return list(self._stage_ms)

    def _accumulate_timing(self):
        if self._timing:
            for slot in range(4):
                for a, b in self._events[slot]:
                    self._stage_ms[slot] += a.elapsed_time(b)

    def launches_per_step(self):
        """libvpfv kernels launched per RK4 step (counted while capturing/running it)."""
        return self._launches.get("step", 0)

    def _graph_for(self, bufs, cached=False):
        key = (self._timing, cached) + tuple(tuple(a.data_ptr() for a in b) for b in bufs)
        g = self._graphs.get(key)
        if g is None:
            side = torch.cuda.Stream(self.device)
            side.wait_stream(torch.cuda.current_stream(self.device))
            with torch.cuda.stream(side):  # warm-up: first launches outside capture; it must
                self._step_body(*bufs, emit_last=False)  # leave the next-step partials untouched
            torch.cuda.current_stream(self.device).wait_stream(side)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g):
                self._step_body(*bufs, cached=cached)
            self._graphs[key] = g
        return g

    @staticmethod
    def _signature(arrays):
        return tuple((a.data_ptr(), a._version) for a in arrays)

    def launch_step(self, dt):
        """Enqueue one RK4 step (no host sync, no rotate)."""
        if dt != self._dt_set:
            self.dt_dev.fill_(float(dt))
            self._dt_set = dt
        bufs = (self.ctx.f0, self.ctx.f1, self.ctx.fout)
        # the partials left by the previous step's stage 4 describe f0 when f0
        # is that step's output and nothing wrote it since
        cached = self.fuse_moment and self._moment_of == self._signature(self.ctx.f0)
        if self.use_graphs:
            self._graph_for(bufs, cached).replay()
        else:
            self._step_body(*bufs, cached=cached)
        self._moment_of = self._signature(self.ctx.fout) if self.fuse_moment else None

    # -- timestep control -----------------------------------------------------
    def _E_host(self, arrays):
        if arrays is self.ctx.f0 and self.fuse_moment and self._moment_of == self._signature(self.ctx.f0):
            # stage 4 left the fused moment partials of this f0: the CFL mode's
            # extra field solve per step (runner.py:199-205) and the
            # diagnostics rows cost a moment finish, not a pass over f
            E = self.fields.solve_from_partials(self.partials_next)
        else:
            E = self.fields.solve(arrays)
        return {k: v.cpu().numpy() for k, v in E.items()}

    def max_dt(self):
        return stable_dt(self.grids, self.species, self._E_host(self.ctx.f0), self.sigma)

    def current_dt(self):
        if self.fixed_dt is not None:
            return self.fixed_dt
        bound = self.max_dt()
        if not math.isfinite(bound):
            raise RunDiverged("stability bound is not finite (empty flow?)")
        return bound * self.cfl_fraction

    # -- stepping ---------------------------------------------------------------
    def advance(self, dt):
        self.launch_step(dt)
        torch.cuda.current_stream(self.device).synchronize()
        self._accumulate_timing()
        self.ctx.t = self.ctx.t + dt
        self.ctx.rotate()
        bad = self._flags_np[3]
        if (bad != _FINITE).any():
            for s in range(len(self.species)):
                if bad[s] == _FINITE:
                    continue
                self.ctx.f0, self.ctx.fout = self.ctx.fout, self.ctx.f0
                self.ctx.t -= dt
                self.ctx.step -= 1
                raise RunDiverged(f"species {self._names[s]} non-finite")

    def interiors(self):
        return [a[g.interior_slices()].cpu().numpy().copy() for a, g in zip(self.ctx.f0, self.grids)]

    def _host_state(self):
        datas = []
        for s_, (a, g) in enumerate(zip(self.ctx.f0, self.grids)):
            if self.frozen[s_] is None:  # device-built set-up: the velocity slabs never change
                self.frozen[s_] = FrozenGhosts.capture(DistField(g, data=a.cpu().numpy()))
        for a, g, fr in zip(self.ctx.f0, self.grids, self.frozen):
            h = a.cpu().numpy().copy()
            fill_local_ghosts(DistField(g, data=h), fr)
            datas.append(h)
        return datas

    def state(self):
        from .fields import FieldState

        dists = [DistField(g, n, d) for g, n, d in zip(self.grids, self._names, self._host_state())]
        return FieldState.solve(dists, self.species, self.schedule)

    def diagnostics_row(self, dt):
        """conserved_quantities of the current state (diagnostics.py:85-122),
        computed on the device: only physical-grid arrays reach the host."""
        from .diagnostics import DeviceDiagnostics

        if self._diag is None:
            self._diag = DeviceDiagnostics(self.grids, self.device)
        E = self._E_host(self.ctx.f0)
        return self._diag.row(self.ctx.f0, self.species, E, self.ctx.t, dt, stream_handle(self.device))

    def checkpoint(self, directory, tag="ckpt"):
        """Write the current state as one VPFV snapshot per species
        (diagnostics.py:187-203 format; file name ``{tag}_{species}.vpfv``),
        streamed from the device a few x planes at a time."""
        import os

        from .snapshot import save_device

        os.makedirs(directory, exist_ok=True)
        paths = []
        for a, g, name in zip(self.ctx.f0, self.grids, self._names):
            path = os.path.join(directory, f"{tag}_{name}.vpfv")
            save_device(path, a, g, name, self.ctx.t)
            paths.append(path)
        return paths

    def restore(self, directory, tag="ckpt"):
        """Load the interiors written by ``checkpoint`` (the frozen velocity
        ghosts stay this set-up's t = 0 values, as in the reference) and the
        time; the next step recomputes the moment (tensor versions changed)."""
        import os

        from .snapshot import load_device

        t = None
        for a, g, name in zip(self.ctx.f0, self.grids, self._names):
            _, t = load_device(os.path.join(directory, f"{tag}_{name}.vpfv"), a, g, species=name)
        self.ctx.t = t
        return t

    def diagnostics_row_host(self, dt):
        """The same row from a host copy of the state (the reference path)."""
        E = self._E_host(self.ctx.f0)
        return conserved_quantities_arrays(self._host_state(), self.grids, self.species, E, self.ctx.t, dt)

    def field_amplitude(self):
        from .diagnostics import field_amplitude

        return field_amplitude(self._E_host(self.ctx.f0), self.grids[0])

    def run(self, t_end, cadence=10, max_steps=10 ** 7, on_row=None):
        rows = [self.diagnostics_row(0.0)]
        if on_row:
            on_row(rows[0])
        while self.ctx.t < t_end - 1e-12 and self.ctx.step < max_steps:
            dt = min(self.current_dt(), t_end - self.ctx.t)
            self.advance(dt)
            if self.ctx.step % cadence == 0 or self.ctx.t >= t_end - 1e-12:
                row = self.diagnostics_row(dt)
                rows.append(row)
                if on_row:
                    on_row(row)
        return rows


class HostPipeline:
    """Advance host-resident states through the device, one RK4 step each,
    with the copies overlapped: while state k steps on the compute stream,
    state k+1 is uploaded on one copy stream and the result of step k-1 is
    downloaded on another.

    This is the host-buffer entry of the library: the reference's stage and
    step functions take host (numpy) arrays, so every call moves the state
    both ways; a pipeline of such calls is bound by the two copy directions,
    not by the step.  Host states are interior arrays (``grid.N``): the ghost
    cells of the padded device buffers are frozen velocity slabs (written
    once, never by the kernels) or periodic images read by modular index, so
    only interiors cross PCIe.  There is no divergence rollback here -- the
    per-stage non-finite flags of the last step remain in ``sim.nonfinite``.

    The copy streams move contiguous device staging buffers only (pure DMA,
    double-buffered); the interior unpack into the padded input and the pack
    of the padded result are ``vpfv_box_copy`` launches on the compute stream
    around the step.  (Copying straight into / out of the strided interior
    views makes torch run a gather/scatter kernel on the copy stream, which
    waits for SMs behind the one-CTA-per-SM stage kernels and stalls the link
    (``staging=False`` keeps that path for comparison).)
    """

    def __init__(self, sim: Simulation, staging: bool = True):
        self.sim = sim
        self.staging = staging
        dev = sim.device
        nb = 1 if staging else 2
        self.din = [[a.clone() for a in sim.ctx.f0] for _ in range(nb)]   # ghosts included:
        self.dout = [[a.clone() for a in sim.ctx.f0] for _ in range(nb)]  # kernels write interiors only
        if staging:
            mk_st = lambda: [[torch.empty(tuple(g.N), dtype=torch.float64, device=dev)  # noqa: E731
                              for g in sim.grids] for _ in range(2)]
            self.sin, self.sout = mk_st(), mk_st()
        self.h2d = torch.cuda.Stream(dev)
        self.d2h = torch.cuda.Stream(dev)
        mk = lambda: [torch.cuda.Event() for _ in range(2)]  # noqa: E731
        self.in_ready, self.step_done, self.out_done = mk(), mk(), mk()

        self._inner = [g.interior_slices() for g in sim.grids]

    def bytes_per_step(self):
        return sum(math.prod(g.N) * 8 for g in self.sim.grids)

    def host_state(self):
        """Pinned host interiors of the simulation's current f0 (a valid input)."""
        return [a[sl].cpu().contiguous().pin_memory() for a, sl in zip(self.sim.ctx.f0, self._inner)]

    def run(self, host_in, host_out, dt, steps):
        """Step ``host_in(k)`` (a list of pinned per-species arrays) into
        ``host_out(k)`` for k < steps; returns after the last download."""
        sim, main = self.sim, torch.cuda.current_stream(self.sim.device)
        saved = (sim.ctx.f0, sim.ctx.fout)
        try:
            (self._run_staged if self.staging else self._run)(sim, main, host_in, host_out, dt, steps)
        finally:  # the simulation's own state buffers, not the pipeline's double buffers
            sim.ctx.f0, sim.ctx.fout = saved

    @staticmethod
    def _interior_copy(dst, src, g, pack, stream):
        """Interior of the padded ``src`` -> contiguous ``dst`` (pack) or the
        reverse (unpack), one ``vpfv_box_copy`` launch on ``stream``."""
        D = len(g.N)
        pad, flat = [sl.start for sl in g.interior_slices()], [0] * D
        so, do = (pad, flat) if pack else (flat, pad)
        _lib.call("vpfv_box_copy", dst.data_ptr(), _lib.ll_array(dst.stride()), _lib.int_array(do),
                  src.data_ptr(), _lib.ll_array(src.stride()), _lib.int_array(so), D,
                  _lib.int_array(g.N), ctypes.c_void_p(stream.cuda_stream))

    def _run_staged(self, sim, main, host_in, host_out, dt, steps):
        din, dout = self.din[0], self.dout[0]
        with torch.cuda.stream(self.h2d):
            for d, h in zip(self.sin[0], host_in(0)):
                d.copy_(h, non_blocking=True)
            self.in_ready[0].record()
        for k in range(steps):
            b = k & 1
            if k + 1 < steps:  # prefetch the next state once step k-1 has unpacked its staging buffer
                if k >= 1:
                    self.h2d.wait_event(self.step_done[1 - b])
                with torch.cuda.stream(self.h2d):
                    for d, h in zip(self.sin[1 - b], host_in(k + 1)):
                        d.copy_(h, non_blocking=True)
                    self.in_ready[1 - b].record()
            main.wait_event(self.in_ready[b])
            for d, s, g in zip(din, self.sin[b], sim.grids):
                self._interior_copy(d, s, g, False, main)
            sim.ctx.f0, sim.ctx.fout = din, dout
            sim.launch_step(dt)
            if k >= 2:
                main.wait_event(self.out_done[b])  # sout[b] drained by the download of step k-2
            for d, s, g in zip(self.sout[b], dout, sim.grids):
                self._interior_copy(d, s, g, True, main)
            self.step_done[b].record(main)
            self.d2h.wait_event(self.step_done[b])
            with torch.cuda.stream(self.d2h):
                for h, d in zip(host_out(k), self.sout[b]):
                    h.copy_(d, non_blocking=True)
                self.out_done[b].record()
        self.d2h.synchronize()
        self.h2d.synchronize()
        main.synchronize()

    def _run(self, sim, main, host_in, host_out, dt, steps):
        with torch.cuda.stream(self.h2d):
            for d, sl, h in zip(self.din[0], self._inner, host_in(0)):
                d[sl].copy_(h, non_blocking=True)
            self.in_ready[0].record()
        for k in range(steps):
            b = k & 1
            if k + 1 < steps:  # prefetch the next state once step k-1 no longer reads its buffer
                if k >= 1:
                    self.h2d.wait_event(self.step_done[1 - b])
                with torch.cuda.stream(self.h2d):
                    for d, sl, h in zip(self.din[1 - b], self._inner, host_in(k + 1)):
                        d[sl].copy_(h, non_blocking=True)
                    self.in_ready[1 - b].record()
            main.wait_event(self.in_ready[b])
            if k >= 2:
                main.wait_event(self.out_done[b])  # dout[b] drained by the download of step k-2
            sim.ctx.f0, sim.ctx.fout = self.din[b], self.dout[b]
            sim.launch_step(dt)
            self.step_done[b].record(main)
            self.d2h.wait_event(self.step_done[b])
            with torch.cuda.stream(self.d2h):
                for h, d, sl in zip(host_out(k), self.dout[b], self._inner):
                    h.copy_(d[sl], non_blocking=True)
                self.out_done[b].record()
        self.d2h.synchronize()
        self.h2d.synchronize()
        main.synchronize()
