"""General box decompositions (partition plans split along x, y, vx, vy, species
co-located per rank) -- cluster.BoxComm / ClusterSimulation.

CPU (gloo, one process per plan rank): the exchange and the block-wise
density of cluster.BoxComm drive the oracle's fused stage on every box; the
gathered state must equal the single-rank oracle run bitwise -- the
reference's SimulatedCluster == Simulation property
(/root/reference/pkg/tests/test_runner.py:107-155) -- and the TrafficLog
totals must equal those the reference's SimulatedCluster recorded
(tests/golden/cluster_*.npz, make_partition_golden.py).

GPU: ClusterSimulation with every rank in one process (the reference's
simulated cluster on device arrays) against the reference SimulatedCluster
fixtures (<= 1e-12 rel L2 after two steps, TrafficLog totals exact) and
against this package's single-box Simulation (bitwise).
"""

import json
import os

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import golden_io as G  # noqa: F401  (sys.path set-up for oracle imports)
from oracle import vpfv_oracle as O
from paper_2410_12155_b200 import cluster as CL
from paper_2410_12155_b200 import partition as P
from paper_2410_12155_b200 import problems
from paper_2410_12155_b200.grid import NGHOST
from test_parallel import _collect, _free_port

HERE = os.path.dirname(os.path.abspath(__file__))

CASES = {  # name: (set-up builder, plan counts, species per rank, dt)
    "landau2d_xy": (lambda: problems.make_problem(problems.landau_spec(), 16, 16), (2, 2, 1, 1), 1, 0.05),
    "landau2d_vv": (lambda: problems.make_problem(problems.landau_spec(), 16, 16), (1, 1, 2, 2), 1, 0.05),
    "landau2d_xv": (lambda: problems.make_problem(problems.landau_spec(), 16, 16), (2, 1, 1, 2), 1, 0.05),
    "lhdi_x_r2": (lambda: problems.make_problem(problems.ProblemSpec("lhdi"), 16, 16), (2, 1, 1), 2, 0.002),
    "lhdi_vv": (lambda: problems.make_problem(problems.ProblemSpec("lhdi"), 16, 16), (1, 2, 2), 1, 0.002),
}


def _fixture(name):
    d = np.load(os.path.join(HERE, "golden", f"cluster_{name}.npz"))
    meta = json.loads(str(d["meta"]))
    return meta, [d[f"f{s}"] for s in range(len([k for k in d.files if k.startswith("f")]))]


def _box_tables(T, b, d, v):
    """Global oracle tables sliced to box b (physical rows, velocity centres)."""
    out = dict(T)
    phys = tuple(slice(b.lo[k], b.hi[k]) for k in range(d))
    vs = [slice(b.lo[d + k], b.hi[d + k]) for k in range(v)]
    for k in ("avx", "evx", "evy", "c1", "c3", "c4", "c5"):
        if k in out and isinstance(out[k], np.ndarray):
            out[k] = out[k][phys]
    if (d, v) == (1, 1):
        out["ax"] = T["ax"][vs[0]]
    elif (d, v) == (1, 2):
        out["vxc"] = T["vxc"][vs[0]]
        out["avy"] = T["avy"][vs[0]]
        out["vyc"] = np.concatenate([T["vyc"][:-1][vs[1]], T["vyc"][-1:]])
    else:
        out["vxc"] = T["vxc"][vs[0]]
        out["vyc"] = T["vyc"][vs[1]]
    return out


def _run_boxes(rank, world, name, steps):
    mk, n, r, dt = CASES[name]
    setup = mk()
    grids = [f.grid for f in setup.dists]
    species = [O.species_from(s) for s in setup.species]
    plan = P.plan_partitions(grids, n, r=r)
    assert plan.ranks == world
    comm = CL.BoxComm(plan, rank, world)
    keys = sorted(comm.local)
    fields, ogrids, frozen = {}, {}, {}
    for s, f in enumerate(setup.dists):
        og = O.grid_from(grids[s])
        glob = O.fill_ghosts(np.array(f.data, dtype=np.float64), og, O.capture_frozen(np.asarray(f.data), og))
        for (ks, lex), arr in P.scatter_field(plan, s, glob).items():
            if (ks, lex) in comm.local:
                fields[(ks, lex)] = torch.from_numpy(arr)
    for k in keys:
        ogrids[k] = O.grid_from(plan.box_grid(*k))
        frozen[k] = O.capture_frozen(fields[k].numpy(), ogrids[k])
    ctx = O.StepContext(f0=fields, f1={k: v.clone() for k, v in fields.items()},
                        fout={k: v.clone() for k, v in fields.items()})
    log = P.TrafficLog()
    gglob = [O.grid_from(g) for g in grids]
    stage_no = [0]

    def stage(dest, A, B, src, ca, cb, cd, cL, t):
        for k in keys:  # local fill: frozen velocity slabs, wraps of unsplit periodic dims
            O.fill_ghosts(src[k].numpy(), ogrids[k], frozen[k])
        comm.exchange(src, log=log, stage=stage_no[0])
        dens = []
        for s in range(len(species)):
            out = torch.zeros(tuple(grids[s].N[:grids[s].d]), dtype=torch.float64)
            comm.density(s, src, out, O.velocity_volume(gglob[s]), log=log, stage=stage_no[0])
            dens.append(out.numpy())
        _, E = O.poisson_solve(O.charge_density(dens, species), gglob[0])
        comm.log_field_distribution(log, stage_no[0], len(E))
        T = [O.stage_tables(gglob[s], species[s], E) for s in range(len(species))]
        for k in keys:
            s = k[0]
            b = plan.box(*k)
            Tb = _box_tables(T[s], b, grids[s].d, grids[s].v)
            O.fused_stage(dest[k].numpy(), A[k].numpy(), B[k].numpy(), src[k].numpy(), ca, cb, cd, cL,
                          ogrids[k], species[s], E, check=False, tables=Tb)
        stage_no[0] += 1

    for _ in range(steps):
        O.rk4_38_low_storage_step(ctx, dt, stage)
        ctx.rotate()
    # gather the global interiors (broadcast each box from its owner)
    out = []
    for s in range(len(species)):
        full = np.empty(grids[s].N)
        for b in plan.boxes[s]:
            buf = torch.empty(b.shape, dtype=torch.float64)
            if (s, b.lex) in comm.local:
                buf.copy_(ctx.f0[(s, b.lex)][tuple(slice(NGHOST, NGHOST + w) for w in b.shape)])
            dist.broadcast(buf, b.rank)
            full[tuple(slice(a, z) for a, z in zip(b.lo, b.hi))] = buf.numpy()
        out.append(full)
    return out, {k: log.total(k) for k in ("ghost", "reduce", "field")}


def _worker(rank, world, port, name, steps, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.set_num_threads(1)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        res = _run_boxes(rank, world, name, steps)
        if rank == 0:
            q.put(res)
    finally:
        dist.destroy_process_group()


def _single(name, steps):
    mk, _, _, dt = CASES[name]
    setup = mk()
    sim = O.OracleSimulation([f.grid for f in setup.dists], setup.species,
                             [np.array(f.data) for f in setup.dists], dt=dt, rhs="fused")
    for _ in range(steps):
        sim.advance(dt)
    return sim.interiors()


@pytest.mark.parametrize("name", list(CASES))
def test_multirank_boxes_equal_single_rank_bitwise(name):
    mk, n, r, _ = CASES[name]
    plan = P.plan_partitions([f.grid for f in mk().dists], n, r=r)
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(k, plan.ranks, port, name, 2, q)) for k in range(plan.ranks)]
    for p in procs:
        p.start()
    got, totals = _collect(q, procs, 600)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = _single(name, 2)
    meta, ref = _fixture(name)
    for a, b, c in zip(got, want, ref):
        assert np.array_equal(a, b)  # bitwise the single-rank fused-operator run
        assert np.linalg.norm(a - c) / np.linalg.norm(c) <= 1e-12  # the reference SimulatedCluster
    assert totals == meta["totals"]  # the reference's TrafficLog


def test_fold_axis_is_the_reference_fold():
    rng = np.random.default_rng(5)
    for shape, axis in (((5, 7, 12), 2), ((3, 16, 9), 1), ((11,), 0)):
        x = rng.standard_normal(shape)
        assert np.array_equal(CL.fold_axis(torch.from_numpy(x), axis).numpy(), O.fold_axis(x, axis))


# ---------------------------------------------------------------------------
# device


@pytest.mark.gpu
@pytest.mark.parametrize("name", list(CASES))
def test_device_simulated_cluster_vs_reference(name):
    from paper_2410_12155_b200 import runner as R

    mk, n, r, dt = CASES[name]
    meta, ref = _fixture(name)
    cl = CL.SimulatedCluster(mk(), n, species_per_rank=r, dt=dt)
    sim = R.Simulation(mk(), dt=dt)
    for _ in range(2):
        cl.advance(dt)
        sim.advance(dt)
    single = sim.interiors()
    # same kernel family on both sides (every box and the full grid TMA-tiled)
    # -> the same per-cell operation order -> bitwise; boxes too narrow for the
    # tiled kernels take the generic fast kernel (FMA order differs: ~1e-16)
    same = all(cl.tiled.values()) and all(sim.tiled)
    for s, want in enumerate(ref):
        got = cl.gather(s)
        assert np.linalg.norm(got - want) / np.linalg.norm(want) <= 1e-12
        if same:
            assert np.array_equal(got, single[s]), "boxes must reproduce the single-box run bitwise"
        else:
            assert np.linalg.norm(got - single[s]) / np.linalg.norm(single[s]) <= 1e-14
    assert {k: cl.log.total(k) for k in ("ghost", "reduce", "field")} == meta["totals"]


@pytest.mark.gpu
def test_device_cluster_exact_mode_and_strategies():
    """Exact-mode kernels on a 4-way box split, every ghost strategy: the
    result does not depend on the strategy (the extra segments only refresh
    cells no stencil reads) and matches the fused single-rank oracle."""
    mk, n, r, dt = CASES["landau2d_vv"]
    outs = []
    for strat in ("vp", "fvm", "all"):
        cl = CL.ClusterSimulation(mk(), (2, 1, 2, 1), strategy=strat, dt=dt, exact=True)
        cl.advance(dt)
        outs.append(cl.gather(0))
    assert np.array_equal(outs[0], outs[1]) and np.array_equal(outs[0], outs[2])
    want = _single("landau2d_vv", 1)[0]
    assert np.linalg.norm(outs[0] - want) / np.linalg.norm(want) <= 1e-13


def _device_worker(rank, world, port, name, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        mk, n, r, dt = CASES[name]
        cl = CL.ClusterSimulation(mk(), n, species_per_rank=r, dt=dt)
        for _ in range(2):
            cl.advance(dt)
        out = [cl.gather(s) for s in range(len(cl.species))]
        if rank == 0:
            q.put((out, {k: cl.log.total(k) for k in ("ghost", "reduce", "field")}))
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
@pytest.mark.parametrize("name", ["landau2d_xv", "lhdi_x_r2"])
def test_device_cluster_one_process_per_rank_equals_in_process(name):
    """Every plan rank in its own process (all on GPU 0, gloo transport with
    host staging -- the NCCL path needs one GPU per rank): P2P ghost segments
    and the all-gathered density fold give bitwise the in-process cluster."""
    mk, n, r, dt = CASES[name]
    ref = CL.ClusterSimulation(mk(), n, species_per_rank=r, dt=dt)
    for _ in range(2):
        ref.advance(dt)
    want = [ref.gather(s) for s in range(len(ref.species))]
    totals = {k: ref.log.total(k) for k in ("ghost", "reduce", "field")}
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_device_worker, args=(k, ref.plan.ranks, port, name, q))
             for k in range(ref.plan.ranks)]
    for p in procs:
        p.start()
    got, got_totals = _collect(q, procs, 600)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for a, b in zip(got, want):
        assert np.array_equal(a, b)
    assert got_totals == totals
