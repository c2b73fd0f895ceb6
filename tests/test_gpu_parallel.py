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


def _worker(rank, world, port, names, dts, steps, q, vparts=1):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2410_12155_b200 import parallel as PL

        torch.cuda.set_device(0)
        out = {}
        for name, dt in zip(names, dts):
            sim = PL.DistributedSimulation(_setup(name), dt=dt, device="cuda:0", velocity_parts=vparts)
            for _ in range(steps):
                sim.advance(dt)
            out[name] = [sim.gather(s) for s in range(len(sim.species))]
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
