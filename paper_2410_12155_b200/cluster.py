"""General phase-space box decompositions on the B200 (``SimulatedCluster``).

The reference's partitioned driver (/root/reference/pkg/src/vpfv/runner.py:
259-496) steps a ``PartitionPlan`` (partition.py) -- boxes split along any
of x, y, vx, vy, species co-located ``r`` per rank, ghost strategy
vp / fvm / all -- as isolated per-box states exchanged at stage barriers.
``ClusterSimulation`` runs the same plan on the device:

* every box is a padded device array stepped by the production stage
  kernels (the TMA-tiled ones where the box is eligible, else the generic
  ones) with its own table views: velocity tables sliced from the global
  grid's (the reference slices the global advection speeds, runner.py:
  418-431), physical tables copied from the global ones computed from the
  global E each stage;
* the ghost exchange moves exactly the plan's segments, one strided device
  box copy (``vpfv_box_copy``) per segment between local boxes, packed
  buffers over ``torch.distributed`` P2P between processes;
* the charge density is the reference's block-wise fold tree
  (runner.py:336-384): each box folds its trailing velocity axes, partials
  are combined across the boxes split along that axis in ascending index
  order (``combine_partials``), axis by axis -- bitwise the single-box fold
  when every span along a split velocity axis is a power of two;
* the TrafficLog records the rows the reference's simulated exchange
  writes (ghost per directed pair, reduce per combine message, field per
  box slab held off rank 0).

Without a process group (or with world size 1) every rank of the plan lives
in this process -- the reference's single-process "simulated cluster" with
device arrays.  Under ``torch.distributed`` with world size == plan.ranks
each process owns the boxes of its rank; densities are all-gathered after
the local folds and the combine is evaluated identically on every rank.
"""

from __future__ import annotations

import math

import numpy as np
import torch
import torch.distributed as dist

from . import _lib
from .fields import FieldSolver, velocity_cell_volume
from .grid import NGHOST
from .kernels import StageTables, stream_handle
from .partition import TrafficLog, combine_partials, padded_box_shape, plan_partitions
from .runner import RunDiverged, _host_filled, require_cuda, stable_dt
from .timestepping import DEFAULT_SIGMA, RK4_STAGES, StepContext

_FINITE = -1  # nonfinite word: VPFV_FINITE as int64


def fold_axis(x, axis):
    """The reference fold along one axis (fields.py:28-39): adjacent pairs
    level by level, an odd tail carried.  Elementwise torch adds, so the
    result is bitwise the numpy fold on any device."""
    n = x.shape[axis]
    while n > 1:
        m = n // 2
        even = x.narrow(axis, 0, 2 * m)
        pairs = even.unflatten(axis, (m, 2))
        s = pairs.select(axis + 1, 0) + pairs.select(axis + 1, 1)
        if n % 2:
            s = torch.cat([s, x.narrow(axis, 2 * m, 1)], dim=axis)
        x, n = s, s.shape[axis]
    return x


class BoxComm:
    """Ghost exchange and block-wise density fold of a plan for the boxes
    this process owns (all of them in-process).  Backend agnostic: device
    tensors move by ``vpfv_box_copy`` and NCCL, CPU tensors (the gloo tests)
    by torch slicing and gloo."""

    def __init__(self, plan, rank=0, world=1, group=None):
        self.plan, self.rank, self.world, self.group = plan, rank, world, group
        self.local = set(plan.rank_members[rank]) if world > 1 else {
            (s, b.lex) for s in range(plan.S) for b in plan.boxes[s]}
        self.pairs = plan.directed_pairs()

    # -- ghost exchange ------------------------------------------------------
    @staticmethod
    def _win(window):
        return tuple(slice(a, z) for a, z in window)

    @staticmethod
    def _copy(dst, dwin, src, swin):
        if dst.is_cuda:
            ext = [z - a for a, z in swin]
            _lib.call("vpfv_box_copy", dst.data_ptr(), _lib.ll_array(dst.stride()),
                      _lib.int_array([a for a, _ in dwin]), src.data_ptr(), _lib.ll_array(src.stride()),
                      _lib.int_array([a for a, _ in swin]), dst.ndim, _lib.int_array(ext),
                      stream_handle(dst.device))
        else:
            dst[BoxComm._win(dwin)].copy_(src[BoxComm._win(swin)])

    def exchange(self, fields, log=None, stage=0):
        """Fill every local box's exchanged ghost cells from their owners.
        ``fields`` maps (species, lex) -> padded local tensor (local boxes)."""
        sends, recvs = [], []
        for (src, dst), segs in self.pairs:
            s_loc, d_loc = src in self.local, dst in self.local
            if s_loc and d_loc:
                for seg in segs:  # owner-interior sources, ghost destinations: order is free
                    self._copy(fields[dst], seg.dst_window, fields[src], seg.src_window)
            elif s_loc:
                sends.append((segs, torch.cat([fields[src][self._win(x.src_window)].reshape(-1) for x in segs])))
            elif d_loc:
                n = sum(x.count for x in segs)
                recvs.append((dst, segs, torch.empty(n, dtype=torch.float64, device=fields[dst].device)))
            if log is not None:
                log.log(stage, "ghost", segs[0].src_rank, segs[0].dst_rank, sum(x.count for x in segs))
        if sends or recvs:
            self._p2p(sends, recvs)
            for dst, segs, buf in recvs:
                off = 0
                for seg in segs:
                    shape = tuple(z - a for a, z in seg.dst_window)
                    fields[dst][self._win(seg.dst_window)].copy_(buf[off:off + seg.count].view(shape))
                    off += seg.count

    def _p2p(self, sends, recvs):
        backend = dist.get_backend(self.group)
        stage_cpu = backend == "gloo"
        ops, back = [], []
        for segs, buf in sends:
            b = buf.cpu() if stage_cpu and buf.is_cuda else buf
            ops.append(dist.P2POp(dist.isend, b, self._grank(segs[0].dst_rank), self.group))
        for dst, segs, buf in recvs:
            b = torch.empty(buf.shape, dtype=buf.dtype) if stage_cpu and buf.is_cuda else buf
            back.append((buf, b))
            ops.append(dist.P2POp(dist.irecv, b, self._grank(segs[0].src_rank), self.group))
        for w in dist.batch_isend_irecv(ops):
            w.wait()
        for buf, b in back:
            if b is not buf:
                buf.copy_(b)

    def _grank(self, r):
        return dist.get_global_rank(self.group, r) if self.group is not None else r

    def log_field_distribution(self, log, stage, ncomp):
        """The rows of the E redistribution to every box held off rank 0
        (runner.py:429-432): ncomp components of the box's physical window."""
        if log is None:
            return
        for s in range(self.plan.S):
            d = self.plan.grids[s].d
            for b in self.plan.boxes[s]:
                if b.rank != 0:
                    log.log(stage, "field", 0, b.rank, ncomp * int(np.prod(b.shape[:d])))

    # -- block-wise density ----------------------------------------------------
    def _split_axes(self, s):
        g, n = self.plan.grids[s], self.plan.n[s]
        return [k for k in range(g.ndim - 1, g.d - 1, -1) if n[k] > 1]

    def local_partials(self, s, fields):
        """Per local box of species s: its interior folded along the velocity
        axes up to and including the first split one (innermost first), the
        part of the tree a box evaluates alone."""
        g = self.plan.grids[s]
        split = self._split_axes(s)
        stop = split[0] if split else g.d
        out = {}
        for b in self.plan.boxes[s]:
            if (s, b.lex) not in self.local:
                continue
            x = fields[(s, b.lex)][tuple(slice(NGHOST, NGHOST + w) for w in b.shape)]
            for ax in range(g.ndim - 1, stop - 1, -1):
                x = fold_axis(x, ax)
            out[b.lex] = x
        return out

    def _partial_shape(self, s, b):
        g = self.plan.grids[s]
        split = self._split_axes(s)
        stop = split[0] if split else g.d
        return tuple(w if k < stop else 1 for k, w in enumerate(b.shape))

    def gather_partials(self, s, mine):
        """Every box's local partial on every process (all-gather)."""
        boxes = self.plan.boxes[s]
        if self.world == 1:
            return {b.lex: mine[b.lex] for b in boxes}
        ref = next(iter(mine.values())) if mine else None
        device = ref.device if ref is not None else torch.device("cpu")
        sizes = [0] * self.world
        for b in boxes:
            sizes[b.rank] += int(np.prod(self._partial_shape(s, b)))
        cap = max(sizes)
        flat = torch.zeros(cap, dtype=torch.float64, device=device)
        off = 0
        for b in boxes:
            if b.rank == self.rank:
                v = mine[b.lex].reshape(-1)
                flat[off:off + v.numel()] = v
                off += v.numel()
        backend = dist.get_backend(self.group)
        src = flat.cpu() if backend == "gloo" and flat.is_cuda else flat
        parts = [torch.empty_like(src) for _ in range(self.world)]
        dist.all_gather(parts, src, group=self.group)
        offs = [0] * self.world
        out = {}
        for b in boxes:
            shp = self._partial_shape(s, b)
            n = int(np.prod(shp))
            out[b.lex] = parts[b.rank][offs[b.rank]:offs[b.rank] + n].view(shp).to(device)
            offs[b.rank] += n
        return out

    def density(self, s, fields, out, vol, log=None, stage=0):
        """Species s's charge-density input n (physical grid) into ``out``:
        the reference's block-wise fold tree (runner.py:336-384) and its
        reduce / field TrafficLog rows."""
        plan = self.plan
        g = plan.grids[s]
        d, D = g.d, g.ndim
        split = self._split_axes(s)
        first = split[0] if split else d
        parts = self.gather_partials(s, self.local_partials(s, fields))
        cur = {b.index: (parts[b.lex], b.rank) for b in plan.boxes[s]}
        for axis in range(D - 1, d - 1, -1):
            if axis < first:  # folds above the first split axis run on the gathered data
                cur = {i: (fold_axis(a, axis), r) for i, (a, r) in cur.items()}
            groups = {}
            for idx in sorted(cur):
                groups.setdefault(idx[:axis] + (0,) + idx[axis + 1:], []).append(idx)
            nxt = {}
            for key, members in groups.items():
                members.sort(key=lambda i: i[axis])
                arrs = [cur[m][0] for m in members]
                ranks = [cur[m][1] for m in members]
                nxt[key] = (arrs[0], ranks[0]) if len(arrs) == 1 else (
                    combine_partials(arrs, ranks=ranks, log=log, stage=stage), ranks[0])
            cur = nxt
        lex_of = {b.index: b.lex for b in plan.boxes[s]}
        for key, (arr, rank) in cur.items():
            b = plan.box(s, lex_of[key])
            win = tuple(slice(b.lo[k], b.hi[k]) for k in range(d))
            out[win] = arr.reshape([b.hi[k] - b.lo[k] for k in range(d)]) * vol
            if rank != 0 and log is not None:
                log.log(stage, "field", rank, 0, arr.numel())
        return out


class _BoxTables:
    """Stage tables of one box: a StageTables of the box grid whose velocity
    tables are replaced by slices of the global ones and whose physical
    tables are copied from the global tables every stage."""

    def __init__(self, gt: StageTables, box, lgrid, species, device, corrections):
        self.gt, self.box = gt, box
        self.t = StageTables(lgrid, species, device, corrections)
        g = gt.grid
        v0 = box.lo[g.d:]
        nv = box.shape[g.d:]
        t = self.t
        if (g.d, g.v) == (1, 1):
            t.ax = gt.ax[v0[0]:v0[0] + nv[0]].clone()
        elif (g.d, g.v) == (1, 2):
            t.vxc = gt.vxc[v0[0]:v0[0] + nv[0]].clone()
            t.avy = gt.avy[v0[0]:v0[0] + nv[0]].clone()
            t.vyc = torch.cat([gt.vyc[v0[1]:v0[1] + nv[1]], gt.vyc[-1:]])  # trailing slot: cB
        else:
            t.vxc = gt.vxc[v0[0]:v0[0] + nv[0]].clone()
            t.vyc = gt.vyc[v0[1]:v0[1] + nv[1]].clone()

    def refresh(self, packed):
        """Copy this box's rows of the global E-dependent tables."""
        g, b, t, gt = self.gt.grid, self.box, self.t, self.gt
        xs = slice(b.lo[0], b.hi[0])
        if g.d == 1:
            if packed and g.v == 2:
                t.packed.copy_(gt.packed[b.lo[0]:b.hi[0] + 2])  # rows x0-1 .. x1 (row = x + 1)
            else:
                t.e.copy_(gt.e[xs])
                t.c1.copy_(gt.c1[xs])
            return
        ys = slice(b.lo[1], b.hi[1])
        if packed:
            t.packed.copy_(gt.packed[b.lo[0]:b.hi[0] + 2, ys])
        else:
            for k in ("evx", "evy", "c1", "c3", "c4", "c5"):
                getattr(t, k).copy_(getattr(gt, k)[xs, ys])


class ClusterSimulation:
    """Step a PartitionPlan's boxes on the device (reference SimulatedCluster
    signature, runner.py:268-279, plus device / exact / group)."""

    def __init__(self, setup, n, ranks=None, species_per_rank=1, strategy="vp", cfl_fraction=0.9, dt=None,
                 corrections=True, sigma=DEFAULT_SIGMA, *, device=None, exact=False, group=None):
        self.device = require_cuda(device)
        self.species = tuple(setup.species)
        self.globals = tuple(f.grid for f in setup.dists)
        self.plan = plan_partitions(self.globals, n, ranks=ranks, r=species_per_rank, strategy=strategy)
        self.cfl_fraction, self.fixed_dt, self.corrections, self.sigma = cfl_fraction, dt, corrections, sigma
        self.exact = exact
        self.log = TrafficLog()
        self._names = [f.species for f in setup.dists]
        self._stage_no = 0
        distributed = dist.is_initialized() and dist.get_world_size(group) > 1
        self.rank = dist.get_rank(group) if distributed else 0
        self.world = dist.get_world_size(group) if distributed else 1
        if distributed and self.world != self.plan.ranks:
            raise ValueError(f"the plan has {self.plan.ranks} ranks but the process group {self.world}")
        self.comm = BoxComm(self.plan, self.rank, self.world, group)
        self.keys = sorted(self.comm.local)
        f0 = {}
        for s, f in enumerate(setup.dists):
            data, _ = _host_filled(f)  # global ghosts current (scatter_field semantics)
            for b in self.plan.boxes[s]:
                if (s, b.lex) in self.comm.local:
                    win = tuple(slice(a, z + 2 * NGHOST) for a, z in zip(b.lo, b.hi))
                    f0[(s, b.lex)] = torch.from_numpy(np.ascontiguousarray(data[win])).to(self.device)
        self.ctx = StepContext(f0=f0, f1={k: v.clone() for k, v in f0.items()},
                               fout={k: v.clone() for k, v in f0.items()})
        self.lgrids = {k: self.plan.box_grid(*k) for k in self.keys}
        self.gtables = [StageTables(g, sp, self.device, corrections) for g, sp in zip(self.globals, self.species)]
        base = _lib.VPFV_EXACT if exact else 0
        self.flags = {k: base | sum(_lib.VPFV_WRAP(j) for j in range(lg.ndim) if lg.periodic[j])
                      for k, lg in self.lgrids.items()}
        self.btables = {k: _BoxTables(self.gtables[k[0]], self.plan.box(*k), self.lgrids[k], self.species[k[0]],
                                      self.device, corrections) for k in self.keys}
        self.tiled = {k: self.btables[k].t.fused_moment_ok(self.flags[k]) for k in self.keys}
        self.fields = FieldSolver(self.globals, self.species, self.device)
        self.vols = [velocity_cell_volume(g) for g in self.globals]
        self.nonfinite = {k: torch.full((1,), _FINITE, dtype=torch.int64, device=self.device) for k in self.keys}
        self.dt_dev = torch.zeros(1, dtype=torch.float64, device=self.device)

    # ------------------------------------------------------------------
    @property
    def t(self):
        return self.ctx.t

    @property
    def step_count(self):
        return self.ctx.step

    def local_cells(self):
        return sum(int(np.prod(self.plan.box(*k).shape)) for k in self.keys)

    def _field_solve(self, bufs, log=None):
        stage = self._stage_no
        for s in range(len(self.species)):
            self.comm.density(s, bufs, self.fields.n[s], self.vols[s], log=log, stage=stage)
        stream = stream_handle(self.device)
        self.fields.charge(stream)
        return self.fields.poisson(self.fields.rho, False, stream)

    def _stage(self, dest, A, B, src, ca, cb, cd, cL, t):
        """One stage on every local box (reference stage protocol,
        runner.py:394-437): exchange, global field solve, tables, kernels."""
        self.comm.exchange(src, log=self.log, stage=self._stage_no)
        E = self._field_solve(src, log=self.log)
        stream = stream_handle(self.device)
        for s, gt in enumerate(self.gtables):
            gt.update(E, stream, packed=False)
            if any(self.tiled[k] for k in self.keys if k[0] == s):
                gt.update(E, stream, packed=True)
        self.comm.log_field_distribution(self.log, self._stage_no, len(E))
        for k in self.keys:
            bt = self.btables[k]
            bt.refresh(self.tiled[k])
            bt.t.launch(dest[k], A[k], B[k], src[k], ca, cb, cd, cL, self.flags[k], stream,
                        nonfinite=self.nonfinite[k], packed=self.tiled[k])
        self._stage_no += 1

    # ------------------------------------------------------------------
    def max_dt(self):
        E = self._field_solve(self.ctx.f0, log=self.log)  # logged like the reference's (runner.py:440-442)
        return stable_dt(self.globals, self.species, {k: v.cpu().numpy() for k, v in E.items()}, self.sigma)

    def current_dt(self):
        if self.fixed_dt is not None:
            return self.fixed_dt
        bound = self.max_dt()
        if not math.isfinite(bound):
            raise RunDiverged("stability bound is not finite (empty flow?)")
        return bound * self.cfl_fraction

    def advance(self, dt):
        for v in self.nonfinite.values():
            v.fill_(_FINITE)
        bufs = {"f0": self.ctx.f0, "f1": self.ctx.f1, "fout": self.ctx.fout}
        for dn, an, bn, sn, ca, cb, cd, div in RK4_STAGES:
            self._stage(bufs[dn], bufs[an], bufs[bn], bufs[sn], ca, cb, cd, dt / div, self.ctx.t)
        self.ctx.t = self.ctx.t + dt
        self.ctx.rotate()
        bad = [k for k in self.keys if int(self.nonfinite[k].item()) != _FINITE]
        if self.world > 1:
            flag = torch.tensor([1 if bad else 0], dtype=torch.int64)
            dist.all_reduce(flag, op=dist.ReduceOp.MAX, group=self.comm.group)
            any_bad = bool(flag.item())
        else:
            any_bad = bool(bad)
        if any_bad:
            self.ctx.f0, self.ctx.fout = self.ctx.fout, self.ctx.f0
            self.ctx.t -= dt
            self.ctx.step -= 1
            if bad:
                s, lex = bad[0]
                raise RunDiverged(f"species {self._names[s]} non-finite on box {lex}")
            raise RunDiverged("non-finite state on another rank")

    def gather(self, s):
        """Global interior array of species s (every process gets it)."""
        g = self.globals[s]
        out = torch.empty(tuple(g.N), dtype=torch.float64, device=self.device)
        for b in self.plan.boxes[s]:
            if (s, b.lex) in self.comm.local:
                inner = tuple(slice(NGHOST, NGHOST + w) for w in b.shape)
                out[tuple(slice(a, z) for a, z in zip(b.lo, b.hi))] = self.ctx.f0[(s, b.lex)][inner]
        if self.world > 1:
            backend = dist.get_backend(self.comm.group)
            for b in self.plan.boxes[s]:
                win = tuple(slice(a, z) for a, z in zip(b.lo, b.hi))
                buf = out[win].contiguous()
                if backend == "gloo":
                    h = buf.cpu()
                    dist.broadcast(h, self.comm._grank(b.rank), group=self.comm.group)
                    buf = h.to(self.device)
                else:
                    dist.broadcast(buf, self.comm._grank(b.rank), group=self.comm.group)
                out[win] = buf
        return out.cpu().numpy()

    def run(self, t_end, max_steps=10 ** 7):
        steps = 0
        while self.t < t_end - 1e-12 and steps < max_steps:
            self.advance(min(self.current_dt(), t_end - self.t))
            steps += 1
        return steps


# the reference's name for the partitioned driver
SimulatedCluster = ClusterSimulation
