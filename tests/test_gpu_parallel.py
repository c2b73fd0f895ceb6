"""GPU coverage of DistributedSimulation on the one GPU a test box has.

* world size 1: the slab driver (x from halo storage, tables by pointer
  offset, eager launches) equals the single-GPU Simulation;
* world size 2 on the same device with the gloo transport (device tensors
  staged through the host): both slabs step on the GPU, the gathered state
  equals the single-GPU Simulation -- the bitwise SimulatedCluster property
  (/root/reference/pkg/tests/test_runner.py:107-155).
"""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _setup(name):
    from paper_2410_12155_b200 import problems as P

    if name == "landau2d":
        return P.make_problem(P.landau_spec(), 32, 32)
    if name == "twostream":
        return P.make_problem(P.ProblemSpec("two-stream"), 64, 64)
    if name == "lhdi":
        return P.make_problem(P.ProblemSpec("lhdi"), 16, 32)
    if name == "lhdi64":  # velocity boxes of 32 after a 2-way velocity split: tiled 1D-2V kernel on both sides
        return P.make_problem(P.ProblemSpec("lhdi"), 16, 64)
    return P.make_electron_proton_2d2v(16, 32)


def _reference(name, steps):
    from paper_2410_12155_b200 import runner as R

    sim = R.Simulation(_setup(name))
    dt = 0.9 * sim.max_dt()
    sim.fixed_dt = dt
    for _ in range(steps):
        sim.advance(dt)
    return dt, sim.interiors()


def _collect(q, procs, timeout):
    """The rank-0 result, failing fast when any worker dies (instead of
    waiting out the queue timeout while the survivors block in a collective)."""
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


def _worker(rank, world, port, names, dts, steps, q, vparts=1, halo="nccl"):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2410_12155_b200 import parallel as PL

        torch.cuda.set_device(0)
        out = {}
        for name, dt in zip(names, dts):
            sim = PL.DistributedSimulation(_setup(name), dt=dt, device="cuda:0", velocity_parts=vparts, halo=halo)
            for _ in range(steps):
                sim.advance(dt)
            out[name] = [sim.gather(s) for s in range(len(sim.species))]
            out[name + ":graphs"] = len(getattr(sim, "_graphs", {}))
        if rank == 0:
            q.put(out)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name", ["landau2d", "twostream", "lhdi", "ep"])
def test_world1_slab_driver_equals_simulation(name):
    from paper_2410_12155_b200 import parallel as PL

    dt, want = _reference(name, 3)
    sim = PL.DistributedSimulation(_setup(name), dt=dt)
    for _ in range(3):
        sim.advance(dt)
    for a, b in zip(sim.interiors(), want):
        assert np.array_equal(a, b)


def test_two_ranks_same_gpu_equal_simulation():
    names = ["landau2d", "lhdi", "ep"]
    refs = {n: _reference(n, 2) for n in names}
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, names, [refs[n][0] for n in names], 2, q))
             for r in range(2)]
    for p in procs:
        p.start()
    got = _collect(q, procs, 600)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for n in names:
        for a, b in zip(got[n], refs[n][1]):
            assert np.array_equal(a, b), n


@pytest.mark.parametrize("world,vparts", [(2, 2), (4, 2)])
def test_velocity_partitions_same_gpu_equal_simulation(world, vparts):
    """x-slabs x velocity partitions on the GPU kernels (velocity faces
    exchanged, fold-tree subtree sums combined across the partitions, the
    overlapped x exchange when there are two slabs): bitwise the single-GPU
    run."""
    names = ["landau2d", "twostream", "lhdi64", "ep"]
    refs = {n: _reference(n, 2) for n in names}
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, names, [refs[n][0] for n in names], 2, q, vparts))
             for r in range(world)]
    for p in procs:
        p.start()
    got = _collect(q, procs, 900)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    for n in names:
        for a, b in zip(got[n], refs[n][1]):
            assert np.array_equal(a, b), n


# ---------------------------------------------------------------------------
# fused x-halo push over peer memory (csrc/peer.cu, vpfv_stage_2d2v_fused_peer)


@pytest.mark.parametrize("nslabs", [2, 4])
def test_peer_halo_push_linked_slabs_equal_simulation(nslabs):
    """nslabs x-slabs of a 2D-2V Landau run on one GPU, each on its own
    stream: every slab's stage kernel stores its 3 boundary planes into its
    neighbours' ghost planes and signals them; each slab waits on its own
    signal words before its next stage.  The slabs step bitwise like the
    single-GPU Simulation, and every wait consumed exactly its signals."""
    from paper_2410_12155_b200 import _lib, parallel as PL, runner as R
    from paper_2410_12155_b200.fields import FieldSolver
    from paper_2410_12155_b200.grid import NGHOST
    from paper_2410_12155_b200.kernels import StageTables, stream_handle
    from paper_2410_12155_b200.timestepping import RK4_STAGES

    steps = 3
    dt, want = _reference("landau2d", steps)
    setup = _setup("landau2d")
    dev = torch.device("cuda:0")
    g, sp = setup.dists[0].grid, setup.species[0]
    data, _ = R._host_filled(setup.dists[0])
    nloc = g.N[0] // nslabs
    lgrid = PL.local_grid(g, 0, nloc)
    states, sigs, views = [], [], []
    gt = StageTables(g, sp, dev)
    for r in range(nslabs):
        x0 = r * nloc
        f0 = torch.from_numpy(np.ascontiguousarray(data[x0:x0 + nloc + 2 * NGHOST])).to(dev)
        states.append([f0, f0.clone(), f0.clone()])  # (f0, f1, fout)
        sigs.append(torch.zeros(2, dtype=torch.int64, device=dev))
        views.append(PL._LocalTables(gt, lgrid, x0))
    peers = PL.PeerHalo.linked(states, sigs, 1, dev)
    fields = FieldSolver([g], [sp], dev)
    flags = sum(_lib.VPFV_WRAP(k) for k in range(1, 4) if lgrid.periodic[k])
    assert _lib.load().vpfv_stage_2d2v_tiled_ok(nloc, g.N[1], g.N[2], g.N[3], flags)
    nloc_arr = _lib.int_array(lgrid.N)
    dt_dev = torch.full((1,), dt, dtype=torch.float64, device=dev)
    streams = [torch.cuda.Stream(dev) for _ in range(nslabs)]
    main = torch.cuda.current_stream(dev)
    torch.cuda.synchronize()
    for r in range(nslabs):
        peers[r].signal(stream_handle(dev))  # the t = 0 ghosts came with the global array
    Ny = g.N[1]
    for _ in range(steps):
        for (dn, an, bn, sn, ca, cb, cd, div) in RK4_STAGES:
            names = {"f0": 0, "f1": 1, "fout": 2}
            for st in streams:
                main.wait_stream(st)
            for r in range(nslabs):  # this slab's rows of the global density
                _lib.call("vpfv_moment", states[r][names[sn]].data_ptr(),
                          fields.n.data_ptr() + r * nloc * Ny * 8, 2, 2, nloc_arr, fields.vols[0], stream_handle(dev))
            fields.charge()
            E = fields.poisson(fields.rho)
            gt.update(E, stream_handle(dev), packed=True)
            for r in range(nslabs):
                streams[r].wait_stream(main)
                with torch.cuda.stream(streams[r]):
                    h = stream_handle(dev)
                    st_ = states[r]
                    dest = st_[names[dn]]
                    peers[r].wait(h)
                    PL.launch_stage_peer(views[r], dest, st_[names[an]], st_[names[bn]], st_[names[sn]], ca, cb, cd,
                                         0.0, flags, h, peers[r].push_args(dest, 0), dt_dev=dt_dev, cL_div=div)
        for r in range(nslabs):  # rotate f0 <-> fout
            states[r][0], states[r][2] = states[r][2], states[r][0]
    torch.cuda.synchronize()
    for r in range(nslabs):
        peers[r].check()
        assert peers[r].consumed.tolist() == [4 * steps] * 2
        assert sigs[r].tolist() == [4 * steps + 1] * 2  # the last stage's signal awaits the next stage
    got = np.concatenate([s[0][lgrid.interior_slices()].cpu().numpy() for s in states], axis=0)
    assert np.array_equal(got, want[0])


def test_peer_halo_two_processes_same_gpu():
    """DistributedSimulation(halo="peer") with two processes sharing the GPU:
    each maps the other's state buffers and signal words by CUDA IPC, the
    stage kernels push the x halo across the processes, and the gathered
    state is bitwise the single-GPU Simulation (2D-2V and 1D-2V, one and
    two species: the waits count one signal per species and neighbour)."""
    names = ["landau2d", "ep", "lhdi64"]  # 2D-2V one and two species, 1D-2V two species
    refs = {n: _reference(n, 5) for n in names}  # step 1 eager, then graphs for both rotations, replayed
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, names, [refs[n][0] for n in names], 5, q, 1, "peer"))
             for r in range(2)]
    for p in procs:
        p.start()
    out = _collect(q, procs, 300)
    for p in procs:
        p.join(60)
    for n in names:
        for a, b in zip(out[n], refs[n][1]):
            assert np.array_equal(a.cpu().numpy() if hasattr(a, "cpu") else a, b)
        assert out[n + ":graphs"] == 2  # steady-state steps ran as graphs (both buffer rotations)


def _diverge_worker(rank, world, port, name, dt, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2410_12155_b200 import parallel as PL
        from paper_2410_12155_b200.runner import RunDiverged

        torch.cuda.set_device(0)
        sim = PL.DistributedSimulation(_setup(name), dt=dt, device="cuda:0", halo="peer")
        for _ in range(3):  # the steady state runs as graphs with the verdict exchanged inside
            sim.advance(dt)
        t_ok, f_ok = sim.t, [a.clone() for a in sim.ctx.f0]
        if rank == 1:  # poison one interior cell on rank 1 only
            sim.ctx.f0[0][5, 5, 5, 5] = float("nan")
        msg = None
        try:
            sim.advance(dt)
        except RunDiverged as e:
            msg = str(e)
        rolled = sim.t == t_ok and (rank == 1 or all(torch.equal(a, b) for a, b in zip(sim.ctx.f0, f_ok)))
        q.put((rank, msg, rolled, len(sim._graphs)))
        dist.barrier()
    finally:
        dist.destroy_process_group()


def test_peer_divergence_verdict_reaches_every_rank():
    """A non-finite cell on one rank makes every rank raise RunDiverged for
    the same step and roll back (runner.py:453-464) -- the verdict travels
    through vpfv_flag_exchange inside the step, no host collective."""
    dt = _reference("landau2d", 1)[0]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_diverge_worker, args=(r, 2, port, "landau2d", dt, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = sorted([_collect(q, procs, 300), _collect(q, procs, 300)])
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    (r0, m0, ok0, g0), (r1, m1, ok1, g1) = got
    assert m1 is not None and "non-finite" in m1 and "rank 1" in m1
    # rank 0 raises too: through the verdict, or its own cells when the nan
    # already reached them through the shared density within the step
    assert m0 is not None and "non-finite" in m0
    assert ok0 and ok1 and g0 >= 1


def test_nccl_c_abi_single_rank_ring():
    """The NCCL-mode C ABI (csrc/comm.cu) on a one-rank communicator: the x
    halo exchange with itself is the periodic wrap of the x ghost planes,
    the density all-gather a copy, the flag all-reduce the identity.  (A
    communicator needs one GPU per rank: the multi-rank exchange is the
    same calls with lo != hi.)"""
    import ctypes

    from paper_2410_12155_b200 import _lib
    from paper_2410_12155_b200.kernels import stream_handle

    L = _lib.load()
    n = L.vpfv_comm_id_size()
    uid = (ctypes.c_ubyte * n)()
    _lib.call("vpfv_comm_unique_id", uid)
    comm = ctypes.c_void_p()
    _lib.call("vpfv_comm_init", ctypes.byref(comm), 1, 0, uid, 0)
    try:
        dev = torch.device("cuda", 0)
        N = (8, 10, 12)
        f = torch.rand(tuple(x + 6 for x in N), dtype=torch.float64, device=dev)
        want = f.clone()
        want[:3] = f[N[0]:N[0] + 3]
        want[N[0] + 3:] = f[3:6]
        s = stream_handle(dev)
        _lib.call("vpfv_halo_exchange_x", comm, f.data_ptr(), 3, _lib.int_array(N), s)
        nl = torch.rand(37, dtype=torch.float64, device=dev)
        ng = torch.zeros(37, dtype=torch.float64, device=dev)
        _lib.call("vpfv_density_allgather", comm, nl.data_ptr(), ng.data_ptr(), 37, s)
        flag = torch.tensor([5], dtype=torch.int64, device=dev)
        _lib.call("vpfv_flag_allreduce", comm, flag.data_ptr(), s)
        torch.cuda.synchronize()
        assert torch.equal(f, want)
        assert torch.equal(nl, ng)
        assert int(flag.item()) == 5
    finally:
        _lib.call("vpfv_comm_destroy", comm)
