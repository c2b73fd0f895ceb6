"""Multi-rank (world size 2, gloo, CPU) coverage of the x-slab layer.

The communication logic of paper_2410_12155_b200.parallel (SlabExchange,
slab_bounds, local_grid, global-table slicing) drives the oracle's stage on
each rank; the gathered state must equal the single-rank oracle run bitwise
-- the reference's SimulatedCluster == Simulation property
(/root/reference/pkg/tests/test_runner.py:107-155).
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import golden_io as G
from oracle import vpfv_oracle as O
from paper_2410_12155_b200 import parallel as PL
from paper_2410_12155_b200.grid import NGHOST


def _collect(q, procs, timeout):
    """The rank-0 result, failing fast when any worker dies."""
    import queue
    import time

    t0 = time.time()
    while time.time() - t0 < timeout:
        try:
            return q.get(timeout=2)
        except queue.Empty:
            dead = [p.exitcode for p in procs if p.exitcode not in (None, 0)]
            if dead:
                for p in procs:
                    if p.is_alive():
                        p.kill()
                raise AssertionError(f"a worker failed (exit codes {dead})")
    raise AssertionError("workers timed out")


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _cases():
    """(name, grids, species, init padded arrays, dt) with Nx divisible into
    two slabs of >= 8 cells."""
    out = []
    for name in ("twostream", "landau1d"):
        c = G.step_case(name)
        out.append((name, c["grids"], c["species"], c["init"], c["dt"]))
    # 2D-2V two-species (different velocity boxes), built from oracle pieces
    sp = [O.Species("i", 1.0, 1.0, 1.0, 0.1, 1.0, (0.0, 0.01)), O.Species("e", -1.0, 0.04, 1.0, 0.1, 1.0, (0.0, 0.01))]
    grids, init = [], []
    rng = np.random.default_rng(11)
    for vmax in (3.0, 6.0):
        g = O.Grid(2, 2, (16, 8, 8, 8), (0.0, 0.0, -vmax, -vmax), (4 * np.pi, 4 * np.pi, vmax, vmax))
        a = 1.0 + 0.2 * rng.random(g.padded_shape)
        grids.append(g)
        init.append(O.fill_ghosts(a, g, O.capture_frozen(a, g)))
    out.append(("2d2v-2sp", grids, sp, init, 0.01))
    return out


def _run_slabs(rank, world, grids, species, init, dt, steps):
    comm = PL.SlabExchange(rank, world)
    x0, nloc = PL.slab_bounds(grids[0].N[0], world, rank)
    lgrids = [O.grid_from(PL.local_grid(g, x0, nloc)) for g in grids]
    filled = [O.fill_ghosts(np.array(d), g, O.capture_frozen(d, g)) for d, g in zip(init, grids)]
    f0 = [torch.from_numpy(np.ascontiguousarray(a[x0:x0 + nloc + 2 * NGHOST])) for a in filled]
    local_frozen = [O.capture_frozen(f.numpy(), lg) for f, lg in zip(f0, lgrids)]
    ctx = O.StepContext(f0=f0, f1=[t.clone() for t in f0], fout=[t.clone() for t in f0])
    S = len(species)

    def stage(dest, A, B, src, ca, cb, cd, cL, t):
        for s in range(S):  # local fill (frozen velocity slabs, unsplit periodic dims)
            O.fill_ghosts(src[s].numpy(), lgrids[s], local_frozen[s])
        comm.exchange_x(src)
        n_loc = torch.from_numpy(np.stack([O.zeroth_moment(src[s].numpy(), lgrids[s]) for s in range(S)]))
        gathered = torch.empty((world,) + tuple(n_loc.shape), dtype=torch.float64)
        comm.gather_x(n_loc.unsqueeze(0), gathered)
        dens = list(gathered.transpose(0, 1).reshape((S, grids[0].N[0]) + tuple(n_loc.shape[2:])).numpy())
        _, E = O.poisson_solve(O.charge_density(dens, species), grids[0])
        for s in range(S):
            T = O.slice_tables(O.stage_tables(grids[s], species[s], E), x0, nloc)
            O.fused_stage(dest[s].numpy(), A[s].numpy(), B[s].numpy(), src[s].numpy(), ca, cb, cd, cL,
                          lgrids[s], species[s], E, check=False, tables=T)

    for _ in range(steps):
        O.rk4_38_low_storage_step(ctx, dt, stage)
        ctx.rotate()
    out = []
    for s in range(S):
        local = torch.from_numpy(np.ascontiguousarray(ctx.f0[s].numpy()[lgrids[s].inner()]))
        full = torch.empty(tuple(grids[s].N), dtype=torch.float64)
        comm.gather_x(local, full)
        out.append(full.numpy())
    return out


def _worker(rank, world, port, steps, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        res = {}
        for name, grids, species, init, dt in _cases():
            res[name] = _run_slabs(rank, world, grids, species, init, dt, steps)
        if rank == 0:
            q.put(res)
    finally:
        dist.destroy_process_group()


def test_two_rank_slabs_equal_single_rank_bitwise():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, 2, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = _collect(q, procs, 300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for name, grids, species, init, dt in _cases():
        ref = O.OracleSimulation(grids, species, init, dt=dt, rhs="fused")
        for _ in range(2):
            ref.advance(dt)
        for a, b in zip(got[name], ref.interiors()):
            assert np.array_equal(a, b), name


def test_slab_bounds_rules():
    assert PL.slab_bounds(128, 8, 3) == (48, 16)
    with pytest.raises(ValueError):
        PL.slab_bounds(128, 3, 0)
    with pytest.raises(ValueError):
        PL.slab_bounds(16, 4, 0)


def test_local_grid_keeps_global_widths():
    from paper_2410_12155_b200.grid import make_grid

    g = make_grid(2, 2, (16, 8, 8, 8), (0, 0, -1, -1), (1.3, 1, 1, 1))
    lg = PL.local_grid(g, 8, 8)
    assert lg.h == g.h and lg.periodic == (False, True, False, False)
    assert lg.centers(2).tolist() == g.centers(2).tolist()


# ---------------------------------------------------------------------------
# x-slabs x velocity partitions (the north star's "allreduce of the charge
# density across velocity partitions", here a deterministic gather + fold)


def _box_cases():
    """Cases whose first velocity dim splits into two spans of >= 8 (and x
    into two when four ranks are used)."""
    out = []
    for name in ("twostream", "landau1d"):  # 1D-1V 16 x 16
        c = G.step_case(name)
        out.append((name, c["grids"], c["species"], c["init"], c["dt"]))
    sp = [O.Species("i", 1.0, 1.0, 1.0, 0.1, 1.0, (0.0, 0.01)), O.Species("e", -1.0, 0.04, 1.0, 0.1, 1.0, (0.0, 0.01))]
    rng = np.random.default_rng(12)
    grids, init = [], []
    for vmax in (3.0, 6.0):  # 2D-2V, two species, Nvx = 16
        g = O.Grid(2, 2, (16, 8, 16, 8), (0.0, 0.0, -vmax, -vmax), (4 * np.pi, 4 * np.pi, vmax, vmax))
        a = 1.0 + 0.2 * rng.random(g.padded_shape)
        grids.append(g)
        init.append(O.fill_ghosts(a, g, O.capture_frozen(a, g)))
    out.append(("2d2v-2sp-v16", grids, sp, init, 0.01))
    sp12 = [O.Species("e", -1.0, 1.0, 1.2, 0.4, 1.0, (0.0, 0.0))]  # 1D-2V with a magnetic field (cB != 0)
    g = O.Grid(1, 2, (16, 16, 12), (0.0, -4.0, -5.0), (2 * np.pi, 4.0, 5.0))
    a = 1.0 + 0.2 * np.random.default_rng(13).random(g.padded_shape)
    out.append(("1d2v-B", [g], sp12, [O.fill_ghosts(a, g, O.capture_frozen(a, g))], 0.01))
    return out


def _slice_v(T, g, v0, nv):
    """Velocity-centre tables sliced to the box's range of the first velocity dim."""
    out = dict(T)
    keys = {(1, 1): ("ax",), (1, 2): ("vxc", "avy"), (2, 2): ("vxc",)}[(g.d, g.v)]
    for k in keys:
        out[k] = np.asarray(out[k])[v0:v0 + nv]
    return out


def _run_boxes(rank, world, vparts, grids, species, init, dt, steps):
    comm = PL.SlabExchange(rank, world, vparts=vparts)
    g0 = grids[0]
    vd = g0.d
    x0, nloc = PL.slab_bounds(g0.N[0], comm.px, comm.ix)
    lgrids, f0, boxes = [], [], []
    for g, d in zip(grids, init):
        v0, nv = PL.slab_bounds(g.N[vd], comm.pv, comm.iv)
        boxes.append((v0, nv))
        lgrids.append(O.grid_from(PL.local_grid(g, x0, nloc, v0, nv)))
        filled = O.fill_ghosts(np.array(d), g, O.capture_frozen(d, g))
        idx = [slice(None)] * g.ndim
        idx[0] = slice(x0, x0 + nloc + 2 * NGHOST)
        idx[vd] = slice(v0, v0 + nv + 2 * NGHOST)
        f0.append(torch.from_numpy(np.ascontiguousarray(filled[tuple(idx)])))
    local_frozen = [O.capture_frozen(f.numpy(), lg) for f, lg in zip(f0, lgrids)]
    ctx = O.StepContext(f0=f0, f1=[t.clone() for t in f0], fout=[t.clone() for t in f0])
    S = len(species)

    def stage(dest, A, B, src, ca, cb, cd, cL, t):
        for s in range(S):
            O.fill_ghosts(src[s].numpy(), lgrids[s], local_frozen[s])
        comm.exchange_v(src, vd)
        comm.exchange_x(src)
        sub = torch.from_numpy(np.stack([O.fold_tree_sum(src[s].numpy()[lgrids[s].inner()], lgrids[s].velocity_dims)
                                         for s in range(S)]))
        full = torch.empty((S, g0.N[0]) + tuple(sub.shape[2:]), dtype=torch.float64)
        comm.gather_density(sub, full)
        dens = [full[s].numpy() * O.velocity_volume(grids[s]) for s in range(S)]
        _, E = O.poisson_solve(O.charge_density(dens, species), g0)
        for s in range(S):
            T = _slice_v(O.slice_tables(O.stage_tables(grids[s], species[s], E), x0, nloc), grids[s], *boxes[s])
            O.fused_stage(dest[s].numpy(), A[s].numpy(), B[s].numpy(), src[s].numpy(), ca, cb, cd, cL,
                          lgrids[s], species[s], E, check=False, tables=T)

    for _ in range(steps):
        O.rk4_38_low_storage_step(ctx, dt, stage)
        ctx.rotate()
    out = []
    for s in range(S):
        local = torch.from_numpy(np.ascontiguousarray(ctx.f0[s].numpy()[lgrids[s].inner()]))
        full = torch.empty(tuple(grids[s].N), dtype=torch.float64)
        comm.gather_state(local, full, vd)
        out.append(full.numpy())
    return out


def _box_worker(rank, world, vparts, port, steps, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        res = {}
        for name, grids, species, init, dt in _box_cases():
            res[name] = _run_boxes(rank, world, vparts, grids, species, init, dt, steps)
        if rank == 0:
            q.put(res)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,vparts", [(2, 2), (4, 2)])
def test_velocity_partitions_equal_single_rank_bitwise(world, vparts):
    """x-slabs x partitions of the first velocity dim: faces exchanged along
    velocity, subtree sums of the fold tree combined across the velocity
    partitions -- bitwise the single-rank run (power-of-two spans,
    /root/reference/pkg/tests/test_partition.py:736-767)."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_box_worker, args=(r, world, vparts, port, 2, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = _collect(q, procs, 600)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for name, grids, species, init, dt in _box_cases():
        ref = O.OracleSimulation(grids, species, init, dt=dt, rhs="fused")
        for _ in range(2):
            ref.advance(dt)
        for a, b in zip(got[name], ref.interiors()):
            assert np.array_equal(a, b), name


def test_fold_pairs_is_the_fold_tree():
    x = np.random.default_rng(3).random(12)
    for n in (1, 2, 3, 4, 5, 8):
        assert PL.fold_pairs(list(x[:n])) == O.fold_tree_sum(x[:n], (0,))


def test_traffic_report_counts_halo_bytes():
    """The per-stage byte accounting of a (2 x-slabs, 2 velocity partitions)
    box layout, from shapes alone (no communication)."""

    class _Comm:
        px, pv, vlo, vhi = 2, 2, None, 3

    class _Sim:
        pass

    from paper_2410_12155_b200.grid import make_grid

    g = make_grid(2, 2, (8, 8, 16, 8), (0, 0, -1, -1), (1, 1, 1, 1))
    sim = _Sim()
    sim.lgrids = [PL.local_grid(g, 0, 8, 0, 8)]
    sim.comm, sim.nloc, sim.vdim, sim.world = _Comm(), 8, 2, 4
    sim.n_local = torch.empty((1, 8, 8), dtype=torch.float64)
    t = PL.DistributedSimulation.traffic_report(sim)
    plane = 14 * 14 * 14
    assert t["x_halo_bytes"] == 2 * 3 * plane * 8
    assert t["v_face_bytes"] == 1 * 8 * 3 * 14 * 14 * 8
    assert t["density_bytes"] == 3 * 64 * 8


def test_peer_halo_linked_pointer_tables():
    """PeerHalo.linked: each slab's buffers map to the same-role buffers of its
    periodic x neighbours, and it bumps the low neighbour's "from high" word
    (offset 8) and the high neighbour's "from low" word (offset 0)."""
    from paper_2410_12155_b200.parallel import PeerHalo

    R = 3
    states = [[torch.zeros(4, dtype=torch.float64) for _ in range(3)] for _ in range(R)]
    sigs = [torch.zeros(2, dtype=torch.int64) for _ in range(R)]
    peers = PeerHalo.linked(states, sigs, 2, "cpu")
    for r, p in enumerate(peers):
        lo, hi = (r - 1) % R, (r + 1) % R
        for k in range(3):
            assert p.peer_of[states[r][k].data_ptr()] == (states[lo][k].data_ptr(), states[hi][k].data_ptr())
        assert p.sig_lo_ptr == sigs[lo].data_ptr() + 8 and p.sig_hi_ptr == sigs[hi].data_ptr()
        assert p.push_args(states[r][1], 1)[:4] == (states[lo][1].data_ptr(), states[hi][1].data_ptr(),
                                                    sigs[lo].data_ptr() + 8, sigs[hi].data_ptr())
        assert p.done.numel() == 2


def test_peer_halo_mode_validation():
    """halo='peer' is refused where the fused push does not apply."""
    from paper_2410_12155_b200 import problems as P
    from paper_2410_12155_b200.parallel import DistributedSimulation

    with pytest.raises(ValueError):
        DistributedSimulation(P.make_problem(P.landau_spec(), 8, 8), halo="bogus", device="cpu")
