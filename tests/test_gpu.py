"""GPU parity tests: the sm_100a library against the oracle / reference fixtures.

Everything calls through the C ABI (libvpfv.so via ctypes).  Bars:
* exact mode: bitwise equal to the reference fused kernels;
* fast mode and full steps: relative L2 on f <= 1e-12 per step (north star);
* physics: Landau damping and two-stream rates vs the reference's frozen
  dispersion roots (/root/reference/pkg/tests/test_dispersion.py:185-212,
  :497-508).
"""

import math

import numpy as np
import pytest
import torch

import golden_io as G
from oracle import vpfv_oracle as O

pytestmark = pytest.mark.gpu

from paper_2410_12155_b200 import _lib, fields as F, kernels as K, problems as P, runner as R  # noqa: E402
from paper_2410_12155_b200.grid import make_grid  # noqa: E402


def pgrid(g):
    return make_grid(g.d, g.v, g.N, g.lo, g.hi, periodic=g.periodic)


def rel_l2(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / np.linalg.norm(np.asarray(b)))


# ---------------------------------------------------------------------------
# fused stage


@pytest.mark.parametrize("name", G.STAGE_NAMES)
def test_stage_exact_bitwise_host_buffers(name):
    c = G.stage_case(name)
    g = pgrid(c["grid"])
    for (ca, cb, cd, cL), want in zip(c["coefs"], c["out"]):
        dest = c["dest"].copy()
        K.fused_stage(dest, c["A"], c["B"], c["src"], ca, cb, cd, cL, g, c["species"], c["E"])
        assert np.array_equal(dest[g.interior_slices()], want)


@pytest.mark.parametrize("name", G.STAGE_NAMES)
def test_stage_exact_bitwise_device_buffers(name):
    c = G.stage_case(name)
    g = pgrid(c["grid"])
    dev = lambda a: torch.from_numpy(a).cuda()  # noqa: E731
    A, B, src = dev(c["A"]), dev(c["B"]), dev(c["src"])
    E = {k: dev(v) for k, v in c["E"].items()}
    for (ca, cb, cd, cL), want in zip(c["coefs"], c["out"]):
        dest = dev(c["dest"].copy())
        K.fused_stage(dest, A, B, src, ca, cb, cd, cL, g, c["species"], E)
        assert np.array_equal(dest[g.interior_slices()].cpu().numpy(), want)
        # ghosts untouched
        d0 = c["dest"].copy()
        d0[g.interior_slices()] = want
        assert np.array_equal(dest.cpu().numpy(), d0)


@pytest.mark.parametrize("name", G.STAGE_NAMES)
def test_stage_fast_close(name):
    c = G.stage_case(name)
    g = pgrid(c["grid"])
    for (ca, cb, cd, cL), want in zip(c["coefs"], c["out"]):
        dest = c["dest"].copy()
        K.fused_stage(dest, c["A"], c["B"], c["src"], ca, cb, cd, cL, g, c["species"], c["E"], exact=False)
        got = dest[g.interior_slices()]
        assert np.max(np.abs(got - want)) <= 1e-14 * np.max(np.abs(want))


@pytest.mark.parametrize("exact", [True, False])
def test_stage_aliasing_patterns_of_rk4(exact):
    """The four RK stages alias A/B/dest with src and each other
    (timestepping.py:80-83); device results equal the oracle on the same
    aliasing."""
    c = G.stage_case("stage_2d2v_frozen")
    g = pgrid(c["grid"])
    og, sp = c["grid"], c["species"]
    f0, f1 = c["src"].copy(), c["A"].copy()
    O.fill_ghosts(f1, og, O.capture_frozen(f0, og))
    fout = c["B"].copy()
    for (dn, an, bn, sn, ca, cb, cd, cL) in [("f1", "f0", "f0", "f0", 1.0, 0.0, 0.0, 0.01),
                                              ("fout", "f0", "f1", "f1", 2.0, -1.0, 0.0, 0.03),
                                              ("f1", "fout", "fout", "fout", -1.0, 0.0, 2.0, 0.03),
                                              ("fout", "f0", "f1", "f1", -0.125, 0.375, 0.75, 0.00375)]:
        host = {"f0": f0.copy(), "f1": f1.copy(), "fout": fout.copy()}
        O.fused_stage(host[dn], host[an], host[bn], host[sn], ca, cb, cd, cL, og, sp, c["E"], check=False)
        devb = {k: torch.from_numpy(v.copy()).cuda() for k, v in (("f0", f0), ("f1", f1), ("fout", fout))}
        K.fused_stage(devb[dn], devb[an], devb[bn], devb[sn], ca, cb, cd, cL, g, sp, c["E"], exact=exact)
        got = devb[dn][g.interior_slices()].cpu().numpy()
        want = host[dn][og.inner()]
        if exact:
            assert np.array_equal(got, want)
        else:
            assert np.max(np.abs(got - want)) <= 1e-14 * np.max(np.abs(want))


def test_alias_rejected_and_nonfinite_index():
    c = G.stage_case("stage_1d2v_periodic")
    g = pgrid(c["grid"])
    src = torch.from_numpy(c["src"]).cuda()
    with pytest.raises(ValueError):
        K.fused_stage(src, src, src, src, 0, 0, 0, 1.0, g, c["species"], c["E"])
    bad = c["src"].copy()
    bad[8, 7, 9] = np.inf
    with pytest.raises(FloatingPointError) as ei:
        K.fused_stage(np.zeros(g.padded_shape), bad, bad, bad, 0, 0, 0, 1.0, g, c["species"], c["E"])
    host = np.zeros(g.padded_shape)
    with pytest.raises(FloatingPointError) as eo:
        O.fused_stage(host, bad, bad, bad, 0, 0, 0, 1.0, c["grid"], c["species"], c["E"])
    assert str(ei.value) == str(eo.value)


def test_unsupported_dimensionality():
    from paper_2410_12155_b200.grid import PhaseSpaceGrid

    g = PhaseSpaceGrid(2, 3, (8,) * 5, (0.0,) * 5, (1.0,) * 5, (True,) * 5)
    with pytest.raises(ValueError):
        K.fused_stage(np.zeros(1), np.zeros(1), np.zeros(1), np.ones(1), 0, 0, 0, 1.0, g, None, {})


def test_constant_field_is_steady_all_periodic():
    """Constant f on a torus: every face difference and diagonal vanishes."""
    g = make_grid(2, 2, [8, 8, 8, 8], [0, 0, -1, -1], [1, 1, 1, 1], periodic=(True,) * 4)
    from paper_2410_12155_b200.fvm import SpeciesConfig

    f = torch.full(g.padded_shape, 1.0, dtype=torch.float64, device="cuda")
    dest = torch.zeros_like(f)
    E = {"Ex": np.full((8, 8), 0.3), "Ey": np.full((8, 8), -0.2)}
    K.fused_stage(dest, f, f, f, 1.0, 0.0, 0.0, 0.1, g, SpeciesConfig(kappa_c=0.5, Bz=1.0), E, exact=False)
    assert torch.equal(dest[g.interior_slices()], f[g.interior_slices()])


# ---------------------------------------------------------------------------
# moments and Poisson


@pytest.mark.parametrize("name", G.MOMENT_NAMES)
def test_moment_bitwise(name):
    from paper_2410_12155_b200.grid import DistField

    g, data, want = G.moment_case(name + ".npz")
    got = F.zeroth_moment(DistField(pgrid(g), data=data))
    assert np.array_equal(got, want)


@pytest.mark.parametrize("nv", [(32, 32), (128, 128), (64, 1024), (12, 10), (33, 17), (1024,)])
def test_moment_bitwise_shapes(nv):
    from paper_2410_12155_b200.grid import DistField

    if len(nv) == 1:
        og = O.Grid(1, 1, (8,) + nv, (0.0, -1.0), (1.0, 1.0))
    else:
        og = O.Grid(1, 2, (8,) + nv, (0.0, -1.0, -2.0), (1.0, 1.0, 2.0))
    data = np.random.default_rng(5).random(og.padded_shape)
    got = F.zeroth_moment(DistField(pgrid(og), data=data))
    assert np.array_equal(got, O.zeroth_moment(data, og))


@pytest.mark.parametrize("name", G.POISSON_NAMES)
def test_poisson_vs_reference(name):
    g, arr = G.poisson_case(name + ".npz")
    phi, E = F.poisson_solve(arr["rho"], pgrid(g))
    for k, v in E.items():
        assert np.max(np.abs(v - arr[k])) <= 1e-13 * max(1.0, np.max(np.abs(arr[k])))
    assert np.max(np.abs(phi - arr["phi"])) <= 1e-13 * max(1.0, np.max(np.abs(arr["phi"])))


@pytest.mark.parametrize("n", [(128,), (1024,), (100,), (128, 128), (64, 32), (24, 20)])
def test_poisson_eigen_and_oracle(n):
    rng = np.random.default_rng(len(n) * 1000 + n[0])
    if len(n) == 1:
        og = O.Grid(1, 1, (n[0], 8), (0.0, -1.0), (2 * np.pi, 1.0))
    else:
        og = O.Grid(2, 2, (n[0], n[1], 8, 8), (0.0, 0.0, -1, -1), (4 * np.pi, 2 * np.pi, 1, 1))
    rho = rng.standard_normal(n)
    rho -= rho.mean()
    _, want = O.poisson_solve(rho, og)
    _, got = F.poisson_solve(rho, pgrid(og))
    for k in want:
        assert np.max(np.abs(got[k] - want[k])) <= 1e-13 * np.max(np.abs(want[k]))


# ---------------------------------------------------------------------------
# full steps through the Simulation driver


@pytest.mark.parametrize("name", G.STEP_NAMES)
@pytest.mark.parametrize("exact", [False, True])
def test_simulation_steps_vs_reference(name, exact):
    c = G.step_case(name)
    mk = {
        "landau1d": lambda: P.make_landau_1d(P.landau_spec(alpha=0.01), 16, 16),
        "twostream": lambda: P.make_problem(P.ProblemSpec("two-stream"), 16, 16),
        "dgh": lambda: P.make_problem(P.ProblemSpec("dgh"), 8, 8),
        "lhdi": lambda: P.make_problem(P.ProblemSpec("lhdi"), 8, 8),
        "bimax1d2v": lambda: P.make_bimaxwellian_1d2v(8, 8, 10),
        "landau2d": lambda: P.make_problem(P.landau_spec(), 8, 8),
    }[name]
    sim = R.Simulation(mk(), dt=c["dt"], exact=exact)
    for k in range(3):
        sim.advance(c["dt"])
        if k in (0, 2):
            for s, a in enumerate(sim.interiors()):
                want = c["out"][f"step{k + 1}_f{s}"]
                assert rel_l2(a, want) <= 1e-12, (name, k, s, rel_l2(a, want))


def test_graph_replay_equals_eager():
    a = R.Simulation(P.make_problem(P.landau_spec(), 8, 8), dt=0.05, use_graphs=True)
    b = R.Simulation(P.make_problem(P.landau_spec(), 8, 8), dt=0.05, use_graphs=False)
    for _ in range(4):
        a.advance(0.05)
        b.advance(0.05)
    assert np.array_equal(a.interiors()[0], b.interiors()[0])


def test_protocol_stage_equals_advance():
    """rk4_38_low_storage_step(ctx, dt, sim._stage) == sim.advance(dt)."""
    from paper_2410_12155_b200.timestepping import rk4_38_low_storage_step

    a = R.Simulation(P.make_problem(P.ProblemSpec("lhdi"), 8, 8), dt=0.002)
    b = R.Simulation(P.make_problem(P.ProblemSpec("lhdi"), 8, 8), dt=0.002)
    a.advance(0.002)
    rk4_38_low_storage_step(b.ctx, 0.002, b._stage)
    b.ctx.rotate()
    for x, y in zip(a.interiors(), b.interiors()):
        assert np.array_equal(x, y)


def test_three_persistent_buffers_and_divergence():
    sim = R.Simulation(P.make_problem(P.ProblemSpec("two-stream"), 16, 16), dt=1e-3)
    ids = {id(b[0]) for b in sim.persistent_buffers()}
    ptrs = {b[0].data_ptr() for b in sim.persistent_buffers()}
    for _ in range(5):
        sim.advance(sim.current_dt())
    assert {id(b[0]) for b in sim.persistent_buffers()} == ids
    assert {b[0].data_ptr() for b in sim.persistent_buffers()} == ptrs
    good = sim.interiors()[0]
    sim.ctx.f0[0][8, 8] = math.nan
    with pytest.raises(R.RunDiverged):
        for _ in range(60):
            sim.advance(sim.current_dt())
    # rolled back: f0 is the last committed state (here the poked one)
    assert sim.step_count >= 5 and good.shape == sim.interiors()[0].shape
    assert math.isnan(sim.interiors()[0][5, 5])


def test_cfl_dt_matches_oracle():
    c = G.step_case("twostream")
    sim = R.Simulation(P.make_problem(P.ProblemSpec("two-stream"), 16, 16))
    ref = O.OracleSimulation(c["grids"], c["species"], c["init"])
    assert sim.current_dt() == pytest.approx(ref.current_dt(), rel=1e-12)


@pytest.mark.parametrize("maker,N", [("landau2d", 32), ("bimax", 32), ("ep", 16)])
def test_medium_step_vs_c_oracle(maker, N):
    """One step at a size where the threaded C oracle still takes seconds."""
    from oracle import cbackend as C

    mk = {"landau2d": lambda: P.make_problem(P.landau_spec(), N, N),
          "bimax": lambda: P.make_bimaxwellian_1d2v(N, N, N),
          "ep": lambda: P.make_electron_proton_2d2v(N, N)}[maker]
    setup = mk()
    dt = 0.9 * R.Simulation(mk()).max_dt()
    sim = R.Simulation(setup, dt=dt)
    ref = C.CSimulation([f.grid for f in setup.dists], setup.species, [f.data for f in mk().dists], dt=dt)
    for _ in range(2):
        sim.advance(dt)
        ref.advance(dt)
    for a, b in zip(sim.interiors(), ref.interiors()):
        assert rel_l2(a, b) <= 1e-12


# ---------------------------------------------------------------------------
# physics rates (north star: Landau-damping and two-stream rates must match)


def _amplitude_history(sim, t_end):
    ts, amps = [0.0], [sim.field_amplitude()]
    while sim.t < t_end - 1e-12:
        sim.advance(min(sim.current_dt(), t_end - sim.t))
        ts.append(sim.t)
        amps.append(sim.field_amplitude())
    return np.array(ts), np.array(amps)


def test_landau_damping_rate():
    from paper_2410_12155_b200.diagnostics import fit_peak_rate

    sim = R.Simulation(P.make_landau_1d(P.landau_spec(alpha=0.01), 128, 128))
    ts, amps = _amplitude_history(sim, 20.0)
    gamma, _ = fit_peak_rate(ts, amps, (0.0, 20.0))
    root = -0.15335946690960492  # test_dispersion.py:497-508 (k = 0.5)
    assert abs(gamma - root) <= 0.02 * abs(root), gamma
    assert abs(gamma - (-0.15416)) <= 2e-3  # CPU oracle fit at 128^2


def test_two_stream_growth_rate():
    from paper_2410_12155_b200.diagnostics import fit_growth_rate

    sim = R.Simulation(P.make_problem(P.ProblemSpec("two-stream"), 256, 256))
    ts, amps = _amplitude_history(sim, 25.0)
    gamma, stderr = fit_growth_rate(ts, amps, (10.0, 25.0))  # the reference signature (diagnostics.py:133)
    assert stderr < 0.01
    root = 0.2931724221224933  # test_dispersion.py:185-212 table, k = 0.6, v_T^2 = 0.1
    assert abs(gamma - root) <= 0.01 * root, gamma
    assert abs(gamma - 0.29312) <= 1e-3  # CPU oracle fit at 256^2


# ---------------------------------------------------------------------------
# the TMA-tiled 2D-2V kernel (fast path) and its fused moment epilogue


def _tiled_case(N, seed, periodic_v=False):
    g = O.Grid(2, 2, N, (0.0, 0.0, -4.0, -5.0), (2 * np.pi, 4 * np.pi, 4.0, 5.0),
               (True, True, periodic_v, periodic_v))
    rng = np.random.default_rng(seed)
    src = 1.0 + 0.3 * rng.random(g.padded_shape)
    O.fill_ghosts(src, g, O.capture_frozen(src, g))
    cx, cy = g.centers(0), g.centers(1)
    E = {"Ex": 0.4 * np.outer(np.sin(cx), np.cos(cy)) + 0.05, "Ey": 0.3 * np.outer(np.cos(cx), np.sin(2 * cy))}
    sp = O.Species("e", -1.0, 1.0, 1.1, 0.3, 1.0, (0.02, -0.01))
    return g, sp, src, E, rng


@pytest.mark.parametrize("N", [(8, 8, 16, 32), (10, 16, 16, 48), (16, 8, 32, 96)])
@pytest.mark.parametrize("coef", [(1.0, 0.0, 0.0, 0.01), (2.0, -1.0, 0.0, 0.03), (-1.0, 0.0, 2.0, 0.03),
                                  (-0.125, 0.375, 0.75, 0.00375)])
def test_tiled_stage_vs_oracle(N, coef):
    g, sp, src, E, rng = _tiled_case(N, sum(N))
    A, dest0 = rng.random(g.padded_shape), rng.random(g.padded_shape)
    ca, cb, cd, cL = coef
    want = dest0.copy()
    O.fused_stage(want, A, src, src, ca, cb, cd, cL, g, sp, E, check=False)
    got = dest0.copy()
    K.fused_stage(got, A, src, src, ca, cb, cd, cL, pgrid(g), sp, E, exact=False)
    inner = g.inner()
    assert np.max(np.abs(got[inner] - want[inner])) <= 2e-14 * np.max(np.abs(want[inner]))
    assert np.array_equal(got[~_interior_mask(g)], dest0[~_interior_mask(g)])  # ghosts untouched


def _interior_mask(g):
    m = np.zeros(g.padded_shape, bool)
    m[g.inner()] = True
    return m


@pytest.mark.parametrize("N", [(8, 8, 16, 32), (12, 16, 32, 128), (10, 24, 16, 64), (8, 8, 64, 64),
                               (8, 8, 128, 32), (8, 8, 256, 16), (8, 8, 32, 256)])
def test_tiled_stage_wrap_reads_interior_and_fused_moment(N):
    """With x/y read by modular index the physical ghosts may hold garbage;
    the fused epilogue's moment partials fold to the reference fold tree."""
    g, sp, src, E, rng = _tiled_case(N, 7)
    pg = pgrid(g)
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    bad = src.copy()
    bad[:3] = np.nan
    bad[-3:] = np.nan
    bad[:, :3] = np.nan
    bad[:, -3:] = np.nan
    want = np.zeros(g.padded_shape)
    O.fused_stage(want, src, src, src, 1.0, 0.0, 0.0, 0.02, g, sp, E, check=False)
    tab = K.StageTables(pg, sp, torch.device("cuda"))
    Ed = {k: dev(v) for k, v in E.items()}
    stream = K.stream_handle()
    tab.update(Ed, stream, packed=True)
    flags = K.wrap_flags(pg)
    if not tab.fused_moment_ok(flags):
        pytest.skip("extents not eligible for the tiled kernel under this tile configuration")
    d_src = dev(bad)
    d_dest = torch.zeros_like(d_src)
    part = torch.empty(tab.partials_shape(), dtype=torch.float64, device="cuda")
    nf = torch.full((1,), -1, dtype=torch.int64, device="cuda")
    tab.launch(d_dest, d_src, d_src, d_src, 1.0, 0.0, 0.0, 0.02, flags, stream, nonfinite=nf, partials=part,
               packed=True)
    got = d_dest.cpu().numpy()
    inner = g.inner()
    assert int(nf.item()) == -1
    assert np.max(np.abs(got[inner] - want[inner])) <= 2e-14 * np.max(np.abs(want[inner]))
    n = torch.empty((N[0], N[1]), dtype=torch.float64, device="cuda")
    _lib.call("vpfv_moment_partials", part.data_ptr(), n.data_ptr(), N[0] * N[1], N[2], part.shape[-1],
              O.velocity_volume(g), stream)
    assert np.array_equal(n.cpu().numpy(), O.zeroth_moment(got, g))


@pytest.mark.parametrize("vx", [(-3.5, 4.5), (-4.0, 4.0), (-4.5, 3.5), (-2.0, 6.0), (0.5, 8.5), (-8.5, -0.5)])
@pytest.mark.parametrize("coef", [(1.0, 0.0, 0.0, 0.02), (-0.125, 0.375, 0.75, 0.00375)])
def test_tiled_stage_vx_sign_layouts(vx, coef):
    """The tiled kernel runs one plane loop per a_x sign: column blocks whose
    vx cells share a sign take one pass, blocks straddling vx = 0 (inside a
    tile, inside a thread's 4 cells, or with a centre exactly at 0, which
    takes the a <= 0 branch) take both passes, each finalising its own sign's
    cells.  All layouts match the oracle, partials fold to the reference tree,
    RK operands (dest aliased) stay per cell."""
    N = (8, 8, 32, 32)
    g = O.Grid(2, 2, N, (0.0, 0.0, vx[0], -5.0), (2 * np.pi, 4 * np.pi, vx[1], 5.0), (True, True, False, False))
    rng = np.random.default_rng(11)
    src = 1.0 + 0.3 * rng.random(g.padded_shape)
    O.fill_ghosts(src, g, O.capture_frozen(src, g))
    cx, cy = g.centers(0), g.centers(1)
    E = {"Ex": 0.4 * np.outer(np.sin(cx), np.cos(cy)) + 0.05, "Ey": 0.3 * np.outer(np.cos(cx), np.sin(2 * cy))}
    sp = O.Species("e", -1.0, 1.0, 1.1, 0.3, 1.0, (0.02, -0.01))
    A, dest0 = rng.random(g.padded_shape), rng.random(g.padded_shape)
    ca, cb, cd, cL = coef
    want = dest0.copy()
    O.fused_stage(want, A, src, src, ca, cb, cd, cL, g, sp, E, check=False)
    pg = pgrid(g)
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    tab = K.StageTables(pg, sp, torch.device("cuda"))
    stream = K.stream_handle()
    tab.update({k: dev(v) for k, v in E.items()}, stream, packed=True)
    flags = K.wrap_flags(pg)
    assert tab.fused_moment_ok(flags)
    d_src, d_A, d_dest = dev(src), dev(A), dev(dest0)
    part = torch.empty(tab.partials_shape(), dtype=torch.float64, device="cuda")
    nf = torch.full((1,), -1, dtype=torch.int64, device="cuda")
    tab.launch(d_dest, d_A, d_src, d_src, ca, cb, cd, cL, flags, stream, nonfinite=nf, partials=part, packed=True)
    got = d_dest.cpu().numpy()
    inner = g.inner()
    assert int(nf.item()) == -1
    assert np.max(np.abs(got[inner] - want[inner])) <= 2e-14 * np.max(np.abs(want[inner]))
    assert np.array_equal(got[~_interior_mask(g)], dest0[~_interior_mask(g)])
    n = torch.empty((N[0], N[1]), dtype=torch.float64, device="cuda")
    _lib.call("vpfv_moment_partials", part.data_ptr(), n.data_ptr(), N[0] * N[1], N[2], part.shape[-1],
              O.velocity_volume(g), stream)
    assert np.array_equal(n.cpu().numpy(), O.zeroth_moment(got, g))
    # a non-finite source cell is reported at its own index whichever pass finalises it
    for ix in (5, 27):
        bad = src.copy()
        bad[3 + 2, 3 + 3, 3 + ix, 3 + 9] = np.inf
        nf.fill_(-1)
        d_dest.copy_(dev(dest0))
        d_bad = dev(bad)
        tab.launch(d_dest, d_A, d_bad, d_bad, ca, cb, cd, cL, flags, stream, nonfinite=nf, partials=part,
                   packed=True)
        assert int(nf.item()) >= 0


def test_fused_moment_rejected_off_the_tiled_path():
    g, sp, src, E, rng = _tiled_case((8, 8, 8, 32), 3)
    pg = pgrid(g)
    tab = K.StageTables(pg, sp, torch.device("cuda"))
    stream = K.stream_handle()
    tab.update({k: torch.from_numpy(v).cuda() for k, v in E.items()}, stream)
    d = torch.from_numpy(src).cuda()
    part = torch.empty(tab.partials_shape(), dtype=torch.float64, device="cuda")
    with pytest.raises(ValueError):
        tab.launch(torch.zeros_like(d), d, d, d, 1.0, 0.0, 0.0, 0.02, _lib.VPFV_EXACT, stream, partials=part)


@pytest.mark.parametrize("N", [32, 64])
def test_landau2d_steps_fused_path_vs_c_oracle(N):
    """Several RK4 steps through the tiled kernel + fused moments (the bench
    path) against the threaded C restatement of the reference."""
    from oracle import cbackend as C

    setup = P.make_problem(P.landau_spec(), N, N)
    sim = R.Simulation(setup)
    assert sim.fuse_moment
    dt = 0.9 * sim.max_dt()
    sim.fixed_dt = dt
    ref = C.CSimulation([f.grid for f in setup.dists], setup.species,
                        [f.data for f in P.make_problem(P.landau_spec(), N, N).dists], dt=dt)
    for _ in range(3):
        sim.advance(dt)
        ref.advance(dt)
        assert rel_l2(sim.interiors()[0], ref.interiors()[0]) <= 1e-12


# ---------------------------------------------------------------------------
# the TMA-tiled 1D-2V kernel


def _tiled12_case(N, seed):
    g = O.Grid(1, 2, N, (0.0, -4.0, -6.0), (2 * np.pi, 4.0, 6.0), (True, False, False))
    rng = np.random.default_rng(seed)
    src = 1.0 + 0.3 * rng.random(g.padded_shape)
    O.fill_ghosts(src, g, O.capture_frozen(src, g))
    E = {"Ex": 0.4 * np.sin(g.centers(0)) + 0.05}
    sp = O.Species("e", -1.0, 1.0, 1.1, 0.3, 1.0, (0.02, -0.01))
    return g, sp, src, E, rng


@pytest.mark.parametrize("N", [(8, 32, 32), (12, 64, 32), (9, 32, 96)])
@pytest.mark.parametrize("coef", [(1.0, 0.0, 0.0, 0.01), (2.0, -1.0, 0.0, 0.03), (-1.0, 0.0, 2.0, 0.03),
                                  (-0.125, 0.375, 0.75, 0.00375)])
def test_tiled12_stage_vs_oracle(N, coef):
    g, sp, src, E, rng = _tiled12_case(N, sum(N))
    A, dest0 = rng.random(g.padded_shape), rng.random(g.padded_shape)
    ca, cb, cd, cL = coef
    want = dest0.copy()
    O.fused_stage(want, A, src, src, ca, cb, cd, cL, g, sp, E, check=False)
    got = dest0.copy()
    pg = pgrid(g)
    assert K.StageTables(pg, sp, torch.device("cuda")).fused_moment_ok(0)
    K.fused_stage(got, A, src, src, ca, cb, cd, cL, pg, sp, E, exact=False)
    inner = g.inner()
    assert np.max(np.abs(got[inner] - want[inner])) <= 2e-14 * np.max(np.abs(want[inner]))
    assert np.array_equal(got[~_interior_mask(g)], dest0[~_interior_mask(g)])


def test_tiled12_wrap_and_fused_moment():
    N = (16, 32, 64)
    g, sp, src, E, rng = _tiled12_case(N, 5)
    pg = pgrid(g)
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    bad = src.copy()
    bad[:3] = np.nan
    bad[-3:] = np.nan
    want = np.zeros(g.padded_shape)
    O.fused_stage(want, src, src, src, 1.0, 0.0, 0.0, 0.02, g, sp, E, check=False)
    tab = K.StageTables(pg, sp, torch.device("cuda"))
    stream = K.stream_handle()
    tab.update({k: dev(v) for k, v in E.items()}, stream, packed=True)
    flags = K.wrap_flags(pg)
    assert tab.fused_moment_ok(flags)
    d_src = dev(bad)
    d_dest = torch.zeros_like(d_src)
    part = torch.empty(tab.partials_shape(), dtype=torch.float64, device="cuda")
    nf = torch.full((1,), -1, dtype=torch.int64, device="cuda")
    tab.launch(d_dest, d_src, d_src, d_src, 1.0, 0.0, 0.0, 0.02, flags, stream, nonfinite=nf, partials=part,
               packed=True)
    got = d_dest.cpu().numpy()
    inner = g.inner()
    assert int(nf.item()) == -1
    assert np.max(np.abs(got[inner] - want[inner])) <= 2e-14 * np.max(np.abs(want[inner]))
    n = torch.empty((N[0],), dtype=torch.float64, device="cuda")
    _lib.call("vpfv_moment_partials", part.data_ptr(), n.data_ptr(), N[0], N[1], part.shape[-1],
              O.velocity_volume(g), stream)
    assert np.array_equal(n.cpu().numpy(), O.zeroth_moment(got, g))


@pytest.mark.parametrize("maker", ["bimax", "lhdi", "dgh"])
def test_1d2v_fused_path_steps_vs_c_oracle(maker):
    from oracle import cbackend as C

    mk = {"bimax": lambda: P.make_bimaxwellian_1d2v(32, 64, 32),
          "lhdi": lambda: P.make_problem(P.ProblemSpec("lhdi"), 16, 32),
          "dgh": lambda: P.make_problem(P.ProblemSpec("dgh"), 16, 32)}[maker]
    setup = mk()
    sim = R.Simulation(setup)
    assert sim.fuse_moment
    dt = 0.9 * sim.max_dt()
    sim.fixed_dt = dt
    ref = C.CSimulation([f.grid for f in setup.dists], setup.species, [f.data for f in mk().dists], dt=dt)
    for _ in range(3):
        sim.advance(dt)
        ref.advance(dt)
        for a, b in zip(sim.interiors(), ref.interiors()):
            assert rel_l2(a, b) <= 1e-12


@pytest.mark.gpu
def test_fused_moment_cache_honours_inplace_edits():
    """Stage 4 leaves the moment partials of the new f0 for the next step's
    stage 1; an in-place edit of f0 in between (tensor version bump) must send
    the next step back to the standalone moment."""
    from oracle import cbackend as C

    setup = P.make_problem(P.landau_spec(), 32, 32)
    sim = R.Simulation(setup)
    dt = 0.9 * sim.max_dt()
    sim.fixed_dt = dt
    for _ in range(2):  # the second step runs on the cached partials
        sim.advance(dt)
    f = sim.ctx.f0[0]
    f[3:-3, 3:-3, 3:-3, 3:-3].mul_(1.001)  # interior edit through a view
    start = [a.cpu().numpy().copy() for a in sim.ctx.f0]
    ref = C.CSimulation([g for g in sim.grids], setup.species, start, dt=dt)
    for _ in range(2):
        sim.advance(dt)
        ref.advance(dt)
        assert rel_l2(sim.interiors()[0], ref.interiors()[0]) <= 1e-12


@pytest.mark.gpu
@pytest.mark.parametrize("N", [(16, 8, 16, 32), (12, 16, 32, 16), (16, 8, 64, 80)])
def test_tiled_stage_x_ranges_equal_full_launch(N):
    """vpfv_stage_2d2v_fused_range over [3, n-3), [0, 3), [n-3, n) (the
    overlapped-exchange order) is bitwise the full launch, partials included."""
    g, sp, src, E, rng = _tiled_case(N, 11)
    pg = pgrid(g)
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    tab = K.StageTables(pg, sp, torch.device("cuda"))
    stream = K.stream_handle()
    tab.update({k: dev(v) for k, v in E.items()}, stream, packed=True)
    flags = K.wrap_flags(pg)
    assert tab.fused_moment_ok(flags)
    A, d_src = dev(rng.random(g.padded_shape)), dev(src)
    d0 = dev(rng.random(g.padded_shape))
    full, part_full = d0.clone(), torch.empty(tab.partials_shape(), dtype=torch.float64, device="cuda")
    tab.launch(full, A, d_src, d_src, -0.125, 0.375, 0.75, 0.004, flags, stream, partials=part_full, packed=True)
    rng_out, part_rng = d0.clone(), torch.empty_like(part_full)
    h, n = pg.h, N[0]
    for x0, x1 in ((3, n - 3), (0, 3), (n - 3, n)):
        _lib.call("vpfv_stage_2d2v_fused_range", rng_out.data_ptr(), A.data_ptr(), d_src.data_ptr(),
                  d_src.data_ptr(), -0.125, 0.375, 0.75, 0.004, tab.vxc.data_ptr(), tab.vyc.data_ptr(),
                  tab.evx.data_ptr(), tab.evy.data_ptr(), tab.cB, tab.c1.data_ptr(), tab.c2, tab.c3.data_ptr(),
                  tab.c4.data_ptr(), tab.c5.data_ptr(), h[0], h[1], h[2], h[3], *N, x0, x1, flags, None, 1.0,
                  None, tab.packed.data_ptr(), part_rng.data_ptr(), stream)
    torch.cuda.synchronize()
    assert torch.equal(rng_out, full)
    assert torch.equal(part_rng, part_full)
    with pytest.raises(ValueError):  # sub-ranges exist only on the tiled path
        _lib.call("vpfv_stage_2d2v_fused_range", rng_out.data_ptr(), A.data_ptr(), d_src.data_ptr(),
                  d_src.data_ptr(), 1.0, 0.0, 0.0, 0.004, tab.vxc.data_ptr(), tab.vyc.data_ptr(),
                  tab.evx.data_ptr(), tab.evy.data_ptr(), tab.cB, tab.c1.data_ptr(), tab.c2, tab.c3.data_ptr(),
                  tab.c4.data_ptr(), tab.c5.data_ptr(), h[0], h[1], h[2], h[3], *N, 0, 3, flags, None, 1.0,
                  None, None, None, stream)


@pytest.mark.gpu
def test_tiled_kernel_variants_bitwise(tmp_path):
    """Every 2D-2V kernel variant the VPFV_RB_* switches select runs the same
    arithmetic: the warp-specialised default (compile-time strides at
    Nvx = Nvy = 128), its runtime-stride instantiation, the round-1 barrier
    loop, and the double-buffered operand geometry give bitwise the same
    RK4 step (buffers, fused partials, non-finite word).  One process per
    variant (the switches are read once per process)."""
    import os
    import subprocess
    import sys

    helper = os.path.join(os.path.dirname(__file__), "helpers", "kernel_variant_step.py")
    variants = {"default": {}, "runtime_strides": {"VPFV_RB_NV": "0"}, "barrier_loop": {"VPFV_RB_WS": "0"},
                "double_buffered_operands": {"VPFV_RB_OPDB": "1"}}
    got = {}
    for name, env in variants.items():
        out = str(tmp_path / f"{name}.npz")
        e = dict(os.environ)
        for k in ("VPFV_RB_NV", "VPFV_RB_WS", "VPFV_RB_OPDB", "VPFV_RB_CFG"):
            e.pop(k, None)
        e.update(env)
        subprocess.run([sys.executable, helper, out], env=e, check=True, timeout=300)
        got[name] = np.load(out)
    ref = got["default"]
    assert int(ref["nonfinite"][0]) == -1
    for name, z in got.items():
        for key in ("f0", "f1", "fout", "partials", "nonfinite"):
            assert np.array_equal(z[key], ref[key]), (name, key)


@pytest.mark.gpu
@pytest.mark.parametrize("problem,n", [("landau2d", 32), ("ep2d2v", 16), ("landau1d", 128), ("twostream", 512),
                                       ("bimax1d2v", 32)])
def test_programmatic_launches_bitwise_stream_order(tmp_path, problem, n):
    """Graph-replayed steps with the programmatic launches (the 1D field
    chain, the 2D moment finish -> charge -> FFT -> tables -> stage chain)
    equal the same steps in plain stream order (VPFV_PDL=0), bitwise: every
    programmatic kernel waits for its predecessor before touching its data.
    One process per mode (the switch is read once per process)."""
    import os
    import subprocess
    import sys

    helper = os.path.join(os.path.dirname(__file__), "helpers", "sim_steps.py")
    got = {}
    for mode in ("1", "0"):
        out = str(tmp_path / f"pdl{mode}.npz")
        e = dict(os.environ)
        e["VPFV_PDL"] = mode
        subprocess.run([sys.executable, helper, out, problem, str(n), "6"], env=e, check=True, timeout=300)
        got[mode] = np.load(out)
    for key in got["1"].files:
        assert np.all(np.isfinite(got["1"][key]))
        assert np.array_equal(got["1"][key], got["0"][key]), (problem, key)


@pytest.mark.gpu
def test_1d2v_kernel_geometries_bitwise(tmp_path):
    """The 1D-2V kernel's geometries (VPFV_R12_CFG: 8 cells per thread at 4
    CTAs/SM, the default; 4 cells per thread at 3 or 2 CTAs/SM; (64, 16)
    tiles) keep each cell's arithmetic and its order, so an RK4 step is
    bitwise the same under every one (buffers, partials, non-finite word)."""
    import os
    import subprocess
    import sys

    helper = os.path.join(os.path.dirname(__file__), "helpers", "kernel_variant_step.py")
    got = {}
    for cfg in ("4", "1", "0", "2"):
        out = str(tmp_path / f"cfg{cfg}.npz")
        e = dict(os.environ, VPFV_R12_CFG=cfg)
        subprocess.run([sys.executable, helper, out, "1d2v"], env=e, check=True, timeout=300)
        got[cfg] = np.load(out)
    ref = got["4"]
    assert int(ref["nonfinite"][0]) == -1
    for cfg, z in got.items():
        for key in ("f0", "f1", "fout", "partials", "nonfinite"):
            assert np.array_equal(z[key], ref[key]), (cfg, key)


def _device_rhs_case(case, seed=3):
    """A seeded device state, species, fixed E, stage tables and flags for the
    tiled 2D-2V / 1D-2V kernels (frozen velocity ghosts, periodic space)."""
    from paper_2410_12155_b200.fvm import SpeciesConfig

    dev = torch.device("cuda")
    gen = torch.Generator(device=dev)
    gen.manual_seed(seed)
    if case == "2d2v":
        g = make_grid(2, 2, (16, 8, 32, 32), (0.0, 0.0, -5.0, -5.0), (2 * np.pi, 4 * np.pi, 5.0, 5.0),
                      periodic=(True, True, False, False))
        cx, cy = (torch.as_tensor(g.centers(i), device=dev) for i in (0, 1))
        E = {"Ex": 0.3 * torch.outer(torch.sin(cx), torch.cos(0.5 * cy)) + 0.05,
             "Ey": 0.2 * torch.outer(torch.cos(cx), torch.sin(cy))}
    else:
        g = make_grid(1, 2, (32, 32, 32), (0.0, -5.0, -5.0), (2 * np.pi, 5.0, 5.0), periodic=(True, False, False))
        E = {"Ex": 0.3 * torch.sin(torch.as_tensor(g.centers(0), device=dev)) + 0.05}
    sp = SpeciesConfig(q=-1.0, kappa_c=0.02, Bz=0.7)
    tab = K.StageTables(g, sp, dev)
    stream = K.stream_handle()
    tab.update(E, stream, packed=True)
    flags = K.wrap_flags(g)
    assert tab.fused_moment_ok(flags)  # the tiled kernels
    rand = lambda: 1.0 + 0.3 * torch.rand(g.padded_shape, dtype=torch.float64, device=dev, generator=gen)  # noqa: E731
    return g, tab, stream, flags, rand


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["2d2v", "1d2v"])
def test_low_storage_20_steps_matches_butcher_on_device(case):
    """The reference's PDE dual run (/root/reference/pkg/tests/test_timestepping.py:208-232)
    on the device: 20 steps of the three-buffer RK4 3/8 protocol through the
    fused stage kernels (RK combination in the epilogue) against the classic
    tableau with the same kernels as a pure RHS (ca = cb = cd = 0, cL = 1) and
    the combination in torch, fixed E: within 1e-12 of max|f|."""
    from paper_2410_12155_b200.timestepping import StepContext, rk4_38_low_storage_step

    g, tab, stream, flags, rand = _device_rhs_case(case)
    f = rand()
    dt = 0.01

    def stage(dest, A, B, src, ca, cb, cd, cL, t):
        tab.launch(dest, A, B, src, ca, cb, cd, cL, flags, stream, packed=True)

    def L(y):
        out = torch.zeros_like(y)  # zero ghosts: intermediate states keep the frozen velocity slabs
        tab.launch(out, y, y, y, 0.0, 0.0, 0.0, 1.0, flags, stream, packed=True)
        return out

    ub = f.clone()
    ctx = StepContext(f0=f.clone(), f1=f.clone(), fout=f.clone())
    for _ in range(20):
        k1 = L(ub)
        k2 = L(ub + (dt / 3.0) * k1)
        k3 = L(ub + dt * (-k1 / 3.0 + k2))
        k4 = L(ub + dt * (k1 - k2 + k3))
        ub = ub + (dt / 8.0) * (k1 + 3.0 * k2 + 3.0 * k3 + k4)
        rk4_38_low_storage_step(ctx, dt, stage)
        ctx.rotate()
    torch.cuda.synchronize()
    inner = g.interior_slices()
    a, b = ctx.f0[inner], ub[inner]
    assert float((a - b).abs().max()) <= 1e-12 * float(b.abs().max())


@pytest.mark.gpu
@pytest.mark.parametrize("case", ["2d2v", "1d2v"])
def test_stage_operator_linear_on_device(case):
    """The fused operator is linear (/root/reference/pkg/tests/test_fvm.py:156-167):
    RHS(2 fa - 0.5 fb) = 2 RHS(fa) - 0.5 RHS(fb) within 1e-13 of its scale,
    through the tiled kernels."""
    g, tab, stream, flags, rand = _device_rhs_case(case, seed=9)
    fa, fb = rand(), rand()

    def rhs(y):
        out = torch.zeros_like(y)
        tab.launch(out, y, y, y, 0.0, 0.0, 0.0, 1.0, flags, stream, packed=True)
        return out

    lhs = rhs(2.0 * fa - 0.5 * fb)
    want = 2.0 * rhs(fa) - 0.5 * rhs(fb)
    torch.cuda.synchronize()
    inner = g.interior_slices()
    scale = float(want[inner].abs().max())
    assert float((lhs[inner] - want[inner]).abs().max()) < 1e-13 * scale


def _mms_error_2d2v(N, corrections):
    """Mean |RHS - exact| of the device operator on a separable manufactured f
    (the set-up of /root/reference/pkg/tests/test_fvm.py:363-427: x/y-varying
    E, magnetic rotation, all five diagonal pairings active).  Velocity ghosts
    hold the periodic images (the profiles are periodic on the velocity box),
    so the tiled kernel's stored-ghost read is the reference's periodic box."""
    from numpy.polynomial.legendre import leggauss

    from paper_2410_12155_b200.fvm import SpeciesConfig

    lo, hi = (0.0, 0.0, -1.0, -1.5), (2 * np.pi, 2 * np.pi, 1.0, 1.5)
    g = make_grid(2, 2, (N,) * 4, lo, hi, periodic=(True, True, False, False))
    sp = SpeciesConfig(q=-1.0, m=1.0, kappa2=1.3, kappa_c=0.4, Bz=1.0)
    gx, gw = leggauss(6)

    def avg(fn, k, padded=False):  # 1D cell averages by 6-point Gauss
        c = lo[k] + (np.arange(-3, N + 3) + 0.5) * g.h[k] if padded else g.centers(k)
        return (fn(c[:, None] + 0.5 * g.h[k] * gx[None, :]) * (0.5 * gw)).sum(axis=1)

    X, Y = (lambda x: np.exp(0.3 * np.sin(x))), (lambda y: np.exp(0.2 * np.cos(y)))
    Vx, Vy = (lambda v: 2.0 + np.sin(np.pi * v)), (lambda v: 2.0 + np.cos(2 * np.pi * v / 3.0))
    dX, dY = (lambda x: 0.3 * np.cos(x) * X(x)), (lambda y: -0.2 * np.sin(y) * Y(y))
    dVx, dVy = (lambda v: np.pi * np.cos(np.pi * v)), (lambda v: -(2 * np.pi / 3.0) * np.sin(2 * np.pi * v / 3.0))

    def outer4(a, b, c, d):
        return a[:, None, None, None] * b[None, :, None, None] * c[None, None, :, None] * d[None, None, None, :]

    f = outer4(*(avg(fn, k, padded=True) for k, fn in enumerate((X, Y, Vx, Vy))))
    E = {"Ex": np.outer(avg(np.sin, 0), avg(np.cos, 1)), "Ey": np.outer(avg(np.cos, 0), avg(np.sin, 1))}
    dev = torch.device("cuda")
    tab = K.StageTables(g, sp, dev, corrections=corrections)
    stream = K.stream_handle()
    tab.update({k: torch.from_numpy(v).to(dev) for k, v in E.items()}, stream, packed=True)
    flags = K.wrap_flags(g)
    assert tab.fused_moment_ok(flags)
    d_f = torch.from_numpy(f).to(dev)
    out = torch.zeros_like(d_f)
    tab.launch(out, d_f, d_f, d_f, 0.0, 0.0, 0.0, 1.0, flags, stream, packed=True)
    rhs = out[g.interior_slices()].cpu().numpy()
    k2, cB = sp.qm * sp.kappa2, sp.qm * sp.kappa_c * sp.Bz
    t = lambda fx, fy, fvx, fvy: outer4(avg(fx, 0), avg(fy, 1), avg(fvx, 2), avg(fvy, 3))  # noqa: E731
    exact = -(t(dX, Y, lambda v: v * Vx(v), Vy) + t(X, dY, Vx, lambda v: v * Vy(v))
              + k2 * t(lambda x: np.sin(x) * X(x), lambda y: np.cos(y) * Y(y), dVx, Vy)
              + cB * t(X, Y, dVx, lambda v: v * Vy(v))
              + k2 * t(lambda x: np.cos(x) * X(x), lambda y: np.sin(y) * Y(y), Vx, dVy)
              - cB * t(X, Y, lambda v: v * Vx(v), dVy))
    return float(np.mean(np.abs(rhs - exact)))


def _mms_error_1d2v(N, corrections):
    """The magnetized 1D-2V manufactured case of /root/reference/pkg/tests/test_fvm.py:302-349
    (B_z rotation, unequal velocity widths, external G_y) on the device
    operator; velocity ghosts hold the periodic images."""
    from numpy.polynomial.legendre import leggauss

    from paper_2410_12155_b200.fvm import SpeciesConfig

    lo, hi = (0.0, -1.0, -1.5), (2 * np.pi, 1.0, 1.5)
    g = make_grid(1, 2, (N,) * 3, lo, hi, periodic=(True, False, False))
    sp = SpeciesConfig(q=-1.0, m=1.0, kappa2=1.0, kappa_c=0.4, Bz=1.0, G=(0.0, 0.1))
    gx, gw = leggauss(6)

    def avg(fn, k, padded=False):
        c = lo[k] + (np.arange(-3, N + 3) + 0.5) * g.h[k] if padded else g.centers(k)
        return (fn(c[:, None] + 0.5 * g.h[k] * gx[None, :]) * (0.5 * gw)).sum(axis=1)

    X = lambda x: np.exp(0.5 * np.sin(x))  # noqa: E731
    Vx, Vy = (lambda v: 2.0 + np.sin(np.pi * v)), (lambda v: 2.0 + np.cos(2 * np.pi * v / 3.0))
    dX = lambda x: 0.5 * np.cos(x) * X(x)  # noqa: E731
    dVx, dVy = (lambda v: np.pi * np.cos(np.pi * v)), (lambda v: -(2 * np.pi / 3.0) * np.sin(2 * np.pi * v / 3.0))

    def outer3(a, b, c):
        return a[:, None, None] * b[None, :, None] * c[None, None, :]

    f = outer3(*(avg(fn, k, padded=True) for k, fn in enumerate((X, Vx, Vy))))
    dev = torch.device("cuda")
    tab = K.StageTables(g, sp, dev, corrections=corrections)
    stream = K.stream_handle()
    tab.update({"Ex": torch.from_numpy(avg(np.sin, 0)).to(dev)}, stream, packed=True)
    flags = K.wrap_flags(g)
    assert tab.fused_moment_ok(flags)
    d_f = torch.from_numpy(f).to(dev)
    out = torch.zeros_like(d_f)
    tab.launch(out, d_f, d_f, d_f, 0.0, 0.0, 0.0, 1.0, flags, stream, packed=True)
    rhs = out[g.interior_slices()].cpu().numpy()
    cB = sp.qm * sp.kappa_c * sp.Bz
    t = lambda fx, fvx, fvy: outer3(avg(fx, 0), avg(fvx, 1), avg(fvy, 2))  # noqa: E731
    exact = -(t(dX, lambda v: v * Vx(v), Vy) + sp.qm * sp.kappa2 * t(lambda x: np.sin(x) * X(x), dVx, Vy)
              + cB * t(X, dVx, lambda v: v * Vy(v)) + t(X, lambda v: -cB * v * Vx(v) + sp.G[1] * Vx(v), dVy))
    return float(np.mean(np.abs(rhs - exact)))


@pytest.mark.gpu
def test_manufactured_fourth_order_1d2v_on_device():
    """Magnetized 1D-2V order on the device (/root/reference/pkg/tests/test_fvm.py:351-360):
    slope > 3.8 with the corrections, < 3.05 without (32^3 -> 64^3, tiled kernel)."""
    e = [_mms_error_1d2v(N, True) for N in (32, 64)]
    assert np.log2(e[0] / e[1]) > 3.8, e
    u = [_mms_error_1d2v(N, False) for N in (32, 64)]
    assert np.log2(u[0] / u[1]) < 3.05, u


@pytest.mark.gpu
def test_manufactured_fourth_order_2d2v_on_device():
    """The scheme's order on the device operator (/root/reference/pkg/tests/test_fvm.py:429-437):
    fourth order with the diagonal corrections (slope > 3.7), at most third
    without (< 3.05), 2D-2V, through the tiled kernel at 32^4 and 64^4."""
    e = [_mms_error_2d2v(N, True) for N in (32, 64)]
    assert np.log2(e[0] / e[1]) > 3.7, e
    u = [_mms_error_2d2v(N, False) for N in (32, 64)]
    assert np.log2(u[0] / u[1]) < 3.05, u


@pytest.mark.gpu
@pytest.mark.parametrize("staging", [True, False])
@pytest.mark.parametrize("maker", ["landau2d", "landau1d", "weibel", "ep"])
def test_host_pipeline_equals_advance(maker, staging):
    """runner.HostPipeline (overlapped H2D / step / D2H of host states) gives
    bitwise the state Simulation.advance gives for each input, through the
    contiguous staging buffers (interior pack/unpack by vpfv_box_copy on the
    compute stream) and through the strided-view copies."""
    setup = {"landau2d": lambda: P.make_problem(P.landau_spec(), 32, 32),
             "landau1d": lambda: P.make_landau_1d(P.landau_spec(alpha=0.01), 32, 64),
             "weibel": lambda: P.make_problem(P.ProblemSpec("weibel"), 16, 32),
             "ep": lambda: P.make_electron_proton_2d2v(16, 32)}[maker]()
    sim = R.Simulation(setup)
    dt = 0.9 * sim.max_dt()
    sim.fixed_dt = dt
    pipe = R.HostPipeline(sim, staging=staging)
    base = pipe.host_state()
    inputs = [[(h * (1.0 + 0.01 * k)).pin_memory() for h in base] for k in range(5)]
    outs = [[torch.empty_like(h).pin_memory() for h in base] for _ in range(5)]
    pipe.run(lambda k: inputs[k], lambda k: outs[k], dt, 5)
    for k in range(5):
        ref = R.Simulation(setup, dt=dt)
        for f, g, h in zip(ref.ctx.f0, ref.grids, inputs[k]):
            f[g.interior_slices()].copy_(h)
        ref.advance(dt)
        for f, g, o in zip(ref.ctx.f0, ref.grids, outs[k]):
            assert torch.equal(f[g.interior_slices()].cpu(), o), k


@pytest.mark.gpu
@pytest.mark.parametrize("maker", ["landau2d", "lhdi", "landau1d", "ep"])
def test_device_diagnostics_row_matches_host_row(maker):
    """Simulation.diagnostics_row (device velocity sums)
    equals the host mirror of conserved_quantities (diagnostics.py:85-122) on
    the same state: mass bitwise (fold tree), the rest to rounding."""
    mk = {"landau2d": lambda: P.make_problem(P.landau_spec(), 16, 32),
          "lhdi": lambda: P.make_problem(P.ProblemSpec("lhdi"), 16, 32),
          "landau1d": lambda: P.make_landau_1d(P.landau_spec(alpha=0.01), 32, 64),
          "ep": lambda: P.make_electron_proton_2d2v(16, 32)}[maker]
    sim = R.Simulation(mk())
    dt = 0.9 * sim.max_dt()
    sim.advance(dt)
    dev, host = sim.diagnostics_row(dt), sim.diagnostics_row_host(dt)
    assert dev.mass == host.mass
    scale = max(abs(host.kinetic_energy), abs(host.total_energy), 1.0)
    assert abs(dev.kinetic_energy - host.kinetic_energy) <= 1e-12 * scale
    assert abs(dev.total_energy - host.total_energy) <= 1e-12 * scale
    assert dev.field_energy == host.field_energy and dev.field_amplitude == host.field_amplitude
    assert abs(dev.momentum - host.momentum) <= 1e-12 * scale


@pytest.mark.gpu
def test_checkpoint_restore_streams_bitwise(tmp_path):
    """Simulation.checkpoint streams f0 interiors to VPFV snapshots (the
    reference reader's format); restore into a fresh Simulation continues
    bitwise."""
    from paper_2410_12155_b200 import snapshot as S

    setup = P.make_electron_proton_2d2v(16, 32)
    sim = R.Simulation(setup)
    dt = 0.9 * sim.max_dt()
    sim.fixed_dt = dt
    for _ in range(2):
        sim.advance(dt)
    paths = sim.checkpoint(str(tmp_path), tag="c")
    for p, want in zip(paths, sim.interiors()):
        f, t = S.read_snapshot(p)
        assert t == sim.t
        assert np.array_equal(f.data[f.grid.interior_slices()], want)
    other = R.Simulation(P.make_electron_proton_2d2v(16, 32), dt=dt)
    assert other.restore(str(tmp_path), tag="c") == sim.t
    sim.advance(dt)
    other.advance(dt)
    for a, b in zip(sim.interiors(), other.interiors()):
        assert np.array_equal(a, b)


@pytest.mark.gpu
@pytest.mark.parametrize("with_partials", [True, False])
def test_tiled_stage_nonfinite_index(with_partials):
    """A NaN in src on the tiled path: the reported index is the smallest flat
    interior index of a non-finite output (fused_stage's FloatingPointError
    contract, _kernels.py:368-373), whether detection rides on the moment
    partials' row sums or on the per-thread sum."""
    N = (12, 16, 32, 48)
    g, sp, src, E, rng = _tiled_case(N, 5)
    src = src.copy()
    src[3 + 7, 3 + 5, 3 + 11, 3 + 20] = np.nan
    want = np.zeros(g.padded_shape)
    O.fused_stage(want, src, src, src, 1.0, 0.0, 0.0, 0.02, g, sp, E, check=False)
    bad = ~np.isfinite(want[g.inner()])
    expect = int(np.flatnonzero(bad.ravel())[0])
    pg = pgrid(g)
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    tab = K.StageTables(pg, sp, torch.device("cuda"))
    stream = K.stream_handle()
    tab.update({k: dev(v) for k, v in E.items()}, stream, packed=True)
    flags = K.wrap_flags(pg)
    assert tab.fused_moment_ok(flags)
    part = torch.empty(tab.partials_shape(), dtype=torch.float64, device="cuda") if with_partials else None
    nf = torch.full((1,), -1, dtype=torch.int64, device="cuda")
    d_src = dev(src)
    tab.launch(torch.zeros_like(d_src), d_src, d_src, d_src, 1.0, 0.0, 0.0, 0.02, flags, stream, nonfinite=nf,
               partials=part, packed=True)
    assert int(nf.item()) == expect


@pytest.mark.gpu
@pytest.mark.parametrize("N", [(8, 12), (8, 8, 12), (8, 8, 8, 10)])
def test_richardson_error_device_matches_host(N):
    from paper_2410_12155_b200 import convergence as CV
    from paper_2410_12155_b200.diagnostics import richardson_error

    rng = np.random.default_rng(len(N))
    pad = lambda n: tuple(k + 6 for k in n)  # noqa: E731
    coarse = rng.random(pad(N))
    fine = rng.random(pad(tuple(2 * k for k in N)))
    g = make_grid(1 if len(N) < 4 else 2, len(N) - (1 if len(N) < 4 else 2), N, (0.0,) * len(N), (1.0,) * len(N))
    got = CV.richardson_error_device(torch.from_numpy(coarse).cuda(), torch.from_numpy(fine).cuda(), g)
    inner = lambda n: tuple(slice(3, 3 + k) for k in n)  # noqa: E731
    want = richardson_error(coarse[inner(N)], fine[inner(tuple(2 * k for k in N))])
    assert abs(got - want) <= 1e-13 * want


@pytest.mark.gpu
def test_convergence_ladder_fourth_order(tmp_path):
    """A 1D-1V Landau ladder (fixed dt shared by the levels, cli.py:144-181):
    the observed spatial order of the fourth-order scheme."""
    from paper_2410_12155_b200 import convergence as CV

    mk = lambda f: P.make_landau_1d(P.landau_spec(alpha=0.1), 16 * f, 16 * f)  # noqa: E731
    sizes, errors, orders = CV.run_ladder(mk, 4, dt=0.01, t_end=0.2, csv_path=str(tmp_path / "c.csv"))
    assert sizes == [16, 32, 64, 128]
    assert all(e > 0 for e in errors) and errors[0] > errors[1] > errors[2]
    assert orders[-1] > 3.5, orders
    lines = (tmp_path / "c.csv").read_text().strip().split("\n")
    assert lines[0] == "N,error,observed_order" and len(lines) == 4


@pytest.mark.gpu
@pytest.mark.parametrize("N", [(16, 128), (12, 384)])
def test_1d1v_fused_moment_partials_fold_tree(N):
    """vpfv_stage_1d1v_fused: the stage output equals vpfv_stage_1d1v and the
    partials fold to the reference fold-tree moment of the new dest bitwise."""
    g = O.Grid(1, 1, N, (0.0, -6.0), (2 * np.pi, 6.0), (True, False))
    rng = np.random.default_rng(sum(N))
    src = 1.0 + 0.3 * rng.random(g.padded_shape)
    O.fill_ghosts(src, g, O.capture_frozen(src, g))
    E = {"Ex": 0.2 * np.sin(g.centers(0))}
    sp = O.Species("e", -1.0, 1.0, 1.0, 0.0, 0.0, (0.0, 0.0))
    pg = pgrid(g)
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    tab = K.StageTables(pg, sp, torch.device("cuda"))
    stream = K.stream_handle()
    tab.update({"Ex": dev(E["Ex"])}, stream)
    flags = K.wrap_flags(pg)
    assert tab.fused_moment_ok(flags)
    d_src = dev(src)
    plain, fused = torch.zeros_like(d_src), torch.zeros_like(d_src)
    part = torch.empty(tab.partials_shape(), dtype=torch.float64, device="cuda")
    tab.launch(plain, d_src, d_src, d_src, 1.0, 0.0, 0.0, 0.02, flags, stream)
    tab.launch(fused, d_src, d_src, d_src, 1.0, 0.0, 0.0, 0.02, flags, stream, partials=part)
    assert torch.equal(plain, fused)
    n = torch.empty(N[0], dtype=torch.float64, device="cuda")
    _lib.call("vpfv_moment_partials", part.data_ptr(), n.data_ptr(), N[0], 1, part.shape[-1],
              O.velocity_volume(g), stream)
    assert np.array_equal(n.cpu().numpy(), O.zeroth_moment(fused.cpu().numpy(), g))


@pytest.mark.parametrize("problem,N,Nv", [("two-stream", 16, 16), ("two-stream", 32, 128), ("lhdi", 8, 8),
                                          ("lhdi", 16, 32), ("dgh", 16, 32), ("weibel", 16, 32),
                                          ("dgh", 64, 128), ("two-stream", 24, 128)])
def test_fused_field_1d_equals_split_chain(problem, N, Nv, monkeypatch):
    """vpfv_field_1d (moments-from-partials + charge + Poisson + every
    species' tables in one CTA) reproduces the separate launches bitwise over
    a few steps, with and without the fused moment partials."""
    def run(split, conv="0"):
        monkeypatch.setenv("VPFV_FIELD_SPLIT", "1" if split else "0")
        monkeypatch.setenv("VPFV_FIELD_CONV", conv)
        sim = R.Simulation(P.make_problem(P.ProblemSpec(problem), N, Nv), dt=1e-3)
        assert sim.fuse_field is (not split)
        if problem == "dgh" and N == 64:
            assert not sim._finish_in_field  # large partials keep the grid-wide finish
        for _ in range(3):
            sim.advance(1e-3)
        return sim
    a, b, c = run(False), run(True), run(False, "1")
    for x, y, z in zip(a.interiors(), b.interiors(), c.interiors()):
        assert np.array_equal(x, y)
        assert rel_l2(z, y) <= 1e-13  # the Green's-function convolution: rounding only
    assert torch.equal(a.fields.E["Ex"], b.fields.E["Ex"])
    ec, eb = c.fields.E["Ex"].cpu().numpy(), b.fields.E["Ex"].cpu().numpy()
    assert np.abs(ec - eb).max() <= 1e-12 * max(np.abs(eb).max(), 1e-300)
    for ta, tb, tiled in zip(a.tables, b.tables, a.tiled):
        if tiled and ta.grid.v == 2:
            assert torch.equal(ta.packed, tb.packed)
        else:
            assert torch.equal(ta.e, tb.e) and torch.equal(ta.c1, tb.c1)


def test_fused_field_1d_corrections_off(monkeypatch):
    """corrections=False zeroes c1 in the fused tables too."""
    out = []
    for split in (False, True):
        monkeypatch.setenv("VPFV_FIELD_SPLIT", "1" if split else "0")
        monkeypatch.setenv("VPFV_FIELD_CONV", "0")
        sim = R.Simulation(P.make_problem(P.ProblemSpec("dgh"), 16, 32), dt=1e-3, corrections=False)
        sim.advance(1e-3)
        out.append(sim)
    assert torch.equal(out[0].tables[0].packed, out[1].tables[0].packed)
    assert float(out[0].tables[0].packed[:, 1].abs().max()) == 0.0
    monkeypatch.setenv("VPFV_FIELD_SPLIT", "0")
    monkeypatch.setenv("VPFV_FIELD_CONV", "1")
    conv = R.Simulation(P.make_problem(P.ProblemSpec("dgh"), 16, 32), dt=1e-3, corrections=False)
    conv.advance(1e-3)
    assert float(conv.tables[0].packed[:, 1].abs().max()) == 0.0
    assert np.array_equal(out[0].interiors()[0], out[1].interiors()[0])


@pytest.mark.gpu
@pytest.mark.parametrize("N,periodic_x", [((64, 256), True), ((37, 128), True), ((48, 384), False),
                                          ((1024, 1024), True)])
def test_1d1v_march_equals_generic(N, periodic_x, monkeypatch):
    """The x-marching 1D-1V kernel (bulk-copied rows, stage1d1v_march.cu) is
    bitwise the generic fast kernel for every RK4 stage's operand pattern,
    with the moment partials and the non-finite flag."""
    g = O.Grid(1, 1, N, (0.0, -6.0), (2 * np.pi, 6.0), (periodic_x, False))
    rng = np.random.default_rng(N[0] + N[1])
    mk = lambda: 1.0 + 0.3 * rng.random(g.padded_shape)  # noqa: E731
    f0, f1, fo = mk(), mk(), mk()
    E = {"Ex": 0.2 * np.sin(g.centers(0)) + 0.05 * rng.standard_normal(N[0])}
    sp = O.Species("e", -1.0, 1.0, 1.0, 0.0, 0.0, (0.0, 0.0))
    pg = pgrid(g)
    dev = lambda a: torch.from_numpy(np.ascontiguousarray(a)).cuda()  # noqa: E731
    tab = K.StageTables(pg, sp, torch.device("cuda"))
    stream = K.stream_handle()
    tab.update({"Ex": dev(E["Ex"])}, stream)
    flags = K.wrap_flags(pg)
    d = {"f0": dev(f0), "f1": dev(f1), "fout": dev(fo)}
    for (dn, an, bn, sn, ca, cb, cd, div) in R.RK4_STAGES:
        outs = []
        for mode in ("0", "1"):
            monkeypatch.setenv("VPFV_1D1V_MARCH", mode)
            dest = d[dn].clone()
            A = dest if an == dn else d[an]
            B = dest if bn == dn else d[bn]
            part = torch.full(tab.partials_shape(), np.nan, dtype=torch.float64, device="cuda")
            nf = torch.full((1,), -1, dtype=torch.int64, device="cuda")
            tab.launch(dest, A, B, d[sn], ca, cb, cd, 0.0, flags, stream, dt_dev=torch.full(
                (1,), 0.01, dtype=torch.float64, device="cuda"), cL_div=div, nonfinite=nf, partials=part)
            torch.cuda.synchronize()
            outs.append((dest, part, int(nf.item())))
        (a, pa, na), (b, pb, nb) = outs
        assert torch.equal(a, b), (dn, an, bn, sn)
        assert torch.equal(pa, pb) and na == nb == -1
    # a non-finite input cell: both kernels report the same first bad index
    bad = d["f0"].clone()
    bad[3 + N[0] // 2, 3 + N[1] // 3] = np.inf
    flagged = []
    for mode in ("0", "1"):
        monkeypatch.setenv("VPFV_1D1V_MARCH", mode)
        dest = torch.zeros_like(bad)
        nf = torch.full((1,), -1, dtype=torch.int64, device="cuda")
        tab.launch(dest, bad, bad, bad, 1.0, 0.0, 0.0, 0.01, flags, stream, nonfinite=nf)
        torch.cuda.synchronize()
        flagged.append(int(nf.item()))
    assert flagged[0] == flagged[1] != -1


@pytest.mark.gpu
@pytest.mark.parametrize("nphys,nvx,nlt", [(5, 32, 1), (3, 64, 16), (4, 1024, 2), (2, 256, 8), (3, 48, 4)])
def test_moment_partials_finish_is_the_fold_tree(nphys, nvx, nlt):
    """vpfv_moment_partials on random chunk sums equals the reference fold
    tree over (vx rows, chunk columns) -- the row-parallel kernel for
    power-of-two Nvx, the warp-per-cell kernel otherwise -- times vol."""
    rng = np.random.default_rng(nphys * nvx + nlt)
    part = rng.standard_normal((nphys, nvx, nlt))
    want = np.array([O.fold_tree_sum(part[p], (0, 1)) * 0.37 for p in range(nphys)])
    d = torch.from_numpy(part).cuda()
    n = torch.empty(nphys, dtype=torch.float64, device="cuda")
    _lib.call("vpfv_moment_partials", d.data_ptr(), n.data_ptr(), nphys, nvx, nlt, 0.37, K.stream_handle())
    torch.cuda.synchronize()
    assert np.array_equal(n.cpu().numpy(), want)


@pytest.mark.gpu
def test_peer_wait_times_out_instead_of_hanging():
    """A neighbour that never signals: vpfv_peer_wait gives up after its
    timeout and raises the flag (the device is not left spinning)."""
    sig = torch.zeros(2, dtype=torch.int64, device="cuda")
    consumed = torch.zeros(2, dtype=torch.int64, device="cuda")
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    _lib.call("vpfv_peer_wait", sig.data_ptr(), consumed.data_ptr(), 1, 1, 0.05, flag.data_ptr(), K.stream_handle())
    torch.cuda.synchronize()
    assert int(flag.item()) == 1
    sig.fill_(1)  # the signals arrive: the next wait passes and consumes them
    flag.zero_()
    _lib.call("vpfv_peer_wait", sig.data_ptr(), consumed.data_ptr(), 1, 1, 5.0, flag.data_ptr(), K.stream_handle())
    torch.cuda.synchronize()
    assert int(flag.item()) == 0 and consumed.tolist() == [1, 1]


@pytest.mark.gpu
@pytest.mark.parametrize("problem,N,Nv", [("landau", 16, 16), ("two-stream", 32, 128), ("dgh", 16, 32)])
def test_cfl_solve_from_cached_partials(problem, N, Nv):
    """After a step, max_dt (the CFL mode's per-step solve) takes the density
    from stage 4's fused partials instead of a moment pass over f0: the same
    E bit for bit, hence the same dt; an in-place edit of f0 falls back."""
    sim = R.Simulation(P.make_problem(P.ProblemSpec(problem), N, Nv))
    dt = sim.max_dt()
    sim.advance(0.5 * dt)
    assert sim.fuse_moment and sim._moment_of == sim._signature(sim.ctx.f0)
    a = sim._E_host(sim.ctx.f0)
    b = {k: v.cpu().numpy() for k, v in sim.fields.solve(sim.ctx.f0).items()}
    for k in b:
        assert np.array_equal(a[k], b[k])
    sim.ctx.f0[0].mul_(1.0)  # bumps the tensor version: the partials no longer describe f0
    assert sim._moment_of != sim._signature(sim.ctx.f0)
    c = sim._E_host(sim.ctx.f0)
    for k in b:
        assert np.array_equal(c[k], b[k])


def test_dropin_host_stepping_allocation_audit_and_parity():
    """The drop-in ``fused_stage`` on host arrays
    stepping the reference's 3-buffer RK4 protocol: after a warm-up step, ten
    more allocate nothing field-sized on the host (the reference's own audit,
    /root/reference/pkg/tests/test_timestepping.py:234-254) or on the device,
    and the state matches the oracle's numpy restatement stepping the same
    protocol (exact mode: bitwise the reference kernels)."""
    import tracemalloc

    from paper_2410_12155_b200.timestepping import RK4_STAGES

    c = G.stage_case("stage_2d2v_frozen")
    g, og, sp, E = pgrid(c["grid"]), c["grid"], c["species"], c["E"]
    host = {"f0": c["src"].copy(), "f1": np.zeros(g.padded_shape), "fout": np.zeros(g.padded_shape)}
    ref = {k: v.copy() for k, v in host.items()}

    def step(bufs, fs, **kw):
        for dn, an, bn, sn, ca, cb, cd, div in RK4_STAGES:
            fs(bufs[dn], bufs[an], bufs[bn], bufs[sn], ca, cb, cd, 0.01 / div, g if fs is K.fused_stage else og,
               sp, E, **kw)
        bufs["f0"], bufs["fout"] = bufs["fout"], bufs["f0"]

    step(host, K.fused_stage)
    step(ref, O.fused_stage, check=False)
    torch.cuda.synchronize()
    dev0 = torch.cuda.memory_allocated()
    tracemalloc.start()
    base, _ = tracemalloc.get_traced_memory()
    for _ in range(10):
        step(host, K.fused_stage)
    _, peak = tracemalloc.get_traced_memory()
    tracemalloc.stop()
    assert peak - base < host["f0"].nbytes / 4, f"stepping allocated {peak - base} bytes on the host"
    assert torch.cuda.memory_allocated() == dev0
    for _ in range(10):
        step(ref, O.fused_stage, check=False)
    inner = g.interior_slices()
    assert np.array_equal(host["f0"][inner], ref["f0"][inner])


@pytest.mark.parametrize("build", [
    lambda dev: P.make_problem(P.landau_spec(), 32, 32, device=dev),
    lambda dev: P.make_landau_1d(P.landau_spec(alpha=0.01), 64, 64, device=dev),
    lambda dev: P.make_problem(P.ProblemSpec("two-stream"), 64, 128, device=dev),
    lambda dev: P.make_problem(P.ProblemSpec("lhdi"), 16, 16, device=dev),
    lambda dev: P.make_bimaxwellian_1d2v(32, 32, 32, device=dev),
    lambda dev: P.make_electron_proton_2d2v((32, 32), (32, 32), device=dev),
], ids=["landau2d-32", "landau1d-64", "twostream-64x128", "lhdi-16", "bimax-32", "ep2d2v-32"])
def test_device_initial_conditions_bitwise_host(build):
    """problems.separable_on_device (vpfv_init_separable) builds the padded
    initial arrays on the GPU bitwise equal to the host builder (itself
    bitwise the reference, tests/test_host.py); a Simulation started from the
    device set-up steps bitwise like one started from the host set-up."""
    from paper_2410_12155_b200 import runner as R

    dev_setup, host_setup = build("cuda:0"), build(None)
    for fd, fh in zip(dev_setup.dists, host_setup.dists):
        assert isinstance(fd.data, torch.Tensor) and fd.data.is_cuda
        assert np.array_equal(fd.data.cpu().numpy(), fh.data)
    a, b = R.Simulation(dev_setup), R.Simulation(host_setup)
    dt = 0.5 * b.max_dt()
    for sim in (a, b):
        sim.advance(dt)
    for x, y in zip(a.interiors(), b.interiors()):
        assert np.array_equal(x, y)
    for x, y in zip(a._host_state(), b._host_state()):  # ghosts too (frozen slabs captured from the device)
        assert np.array_equal(x, y)


@pytest.mark.gpu
@pytest.mark.parametrize("shape,ext", [((7, 9, 40), (5, 6, 33)), ((4, 6, 11, 134), (2, 3, 7, 128)),
                                       ((5, 70), (3, 64)), ((6, 5, 20), (4, 3, 17)), ((300,), (257,))])
def test_box_copy_matches_slicing(shape, ext):
    """vpfv_box_copy (the warp-per-row kernel for unit-stride rows of >= 32
    cells, the element kernel otherwise) equals torch slicing, both ways
    between a padded array and a contiguous box, leaving the rest untouched."""
    gen = torch.Generator().manual_seed(len(shape) * 131 + ext[-1])
    src = torch.rand(shape, generator=gen, dtype=torch.float64).cuda()
    so = [(n - e) // 2 for n, e in zip(shape, ext)]
    box = torch.full(ext, -1.0, dtype=torch.float64, device="cuda")
    st = ctypes_stream()
    _lib.call("vpfv_box_copy", box.data_ptr(), _lib.ll_array(box.stride()), _lib.int_array([0] * len(ext)),
              src.data_ptr(), _lib.ll_array(src.stride()), _lib.int_array(so), len(ext), _lib.int_array(ext), st)
    sl = tuple(slice(o, o + e) for o, e in zip(so, ext))
    torch.cuda.synchronize()
    assert torch.equal(box, src[sl])
    dst = torch.zeros(shape, dtype=torch.float64, device="cuda")
    do = [n - e for n, e in zip(shape, ext)]
    _lib.call("vpfv_box_copy", dst.data_ptr(), _lib.ll_array(dst.stride()), _lib.int_array(do),
              box.data_ptr(), _lib.ll_array(box.stride()), _lib.int_array([0] * len(ext)), len(ext),
              _lib.int_array(ext), st)
    torch.cuda.synchronize()
    want = torch.zeros_like(dst)
    want[tuple(slice(o, o + e) for o, e in zip(do, ext))] = src[sl]
    assert torch.equal(dst, want)


def ctypes_stream():
    import ctypes

    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
