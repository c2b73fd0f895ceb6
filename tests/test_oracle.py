"""Pin the CPU oracle against fixtures produced by the real reference.

CPU only.  Bitwise wherever the reference itself is bitwise reproducible.
"""

import numpy as np
import pytest

import golden_io as G
from oracle import vpfv_oracle as O


@pytest.mark.parametrize("name", G.STAGE_NAMES)
def test_fused_stage_bitwise_vs_reference(name):
    c = G.stage_case(name)
    for (ca, cb, cd, cL), want in zip(c["coefs"], c["out"]):
        dest = c["dest"].copy()
        O.fused_stage(dest, c["A"], c["B"], c["src"], ca, cb, cd, cL, c["grid"], c["species"], c["E"])
        assert np.array_equal(dest[c["grid"].inner()], want)


@pytest.mark.parametrize("name", G.STAGE_NAMES)
def test_numpy_rhs_bitwise_vs_reference(name):
    c = G.stage_case(name)
    got = O.vlasov_rhs(c["src"], c["grid"], c["species"], c["E"])
    assert np.array_equal(got, c["rhs"])


@pytest.mark.parametrize("name", G.STAGE_NAMES)
def test_correction_coeffs_bitwise(name):
    c = G.stage_case(name)
    cc = O.correction_coeffs(c["grid"], c["species"], c["E"])
    for k, v in cc.items():
        assert np.array_equal(np.asarray(v), c["arrays"]["coef_" + k])


@pytest.mark.parametrize("name", G.MOMENT_NAMES)
def test_fold_tree_moment_bitwise(name):
    g, data, want = G.moment_case(name + ".npz")
    assert np.array_equal(O.zeroth_moment(data, g), want)


@pytest.mark.parametrize("name", G.POISSON_NAMES)
def test_poisson_bitwise(name):
    g, arr = G.poisson_case(name + ".npz")
    phi, E = O.poisson_solve(arr["rho"], g)
    assert np.array_equal(phi, arr["phi"])
    for k, v in E.items():
        assert np.array_equal(v, arr[k])


@pytest.mark.parametrize("name", G.STEP_NAMES)
def test_simulation_steps_bitwise(name):
    c = G.step_case(name)
    sim = O.OracleSimulation(c["grids"], c["species"], c["init"], dt=c["dt"])
    for k in range(3):
        sim.advance(c["dt"])
        if k in (0, 2):
            for s, a in enumerate(sim.interiors()):
                assert np.array_equal(a, c["out"][f"step{k + 1}_f{s}"]), (name, k, s)


def test_fused_driver_close_to_production():
    """The fused-kernel arithmetic drives the same trajectory to ~1e-16."""
    c = G.step_case("landau2d")
    sim = O.OracleSimulation(c["grids"], c["species"], c["init"], dt=c["dt"], rhs="fused")
    for _ in range(3):
        sim.advance(c["dt"])
    got = sim.interiors()[0]
    want = c["out"]["step3_f0"]
    assert np.linalg.norm(got - want) <= 1e-14 * np.linalg.norm(want)


def test_alias_and_nonfinite():
    c = G.stage_case("stage_1d1v_periodic")
    g, sp = c["grid"], c["species"]
    with pytest.raises(ValueError):
        O.fused_stage(c["src"], c["src"], c["src"], c["src"], 0, 0, 0, 1.0, g, sp, c["E"])
    src = c["src"].copy()
    src[8, 8] = np.inf
    with pytest.raises(FloatingPointError):
        O.fused_stage(np.zeros(g.padded_shape), src, src, src, 0, 0, 0, 1.0, g, sp, c["E"])


def test_combine_partials_pow2_bitwise():
    rng = np.random.default_rng(7)
    x = rng.random((5, 16))
    want = O.fold_tree_sum(x, (1,))
    for nb in (2, 4, 8, 16):
        span = 16 // nb
        parts = [O.fold_axis(x[:, i * span:(i + 1) * span], 1)[:, 0] for i in range(nb)]
        assert np.array_equal(O.combine_partials(parts), want)


# --- the threaded C restatement (CPU baseline) is bitwise the same oracle ---

@pytest.mark.parametrize("name", G.STAGE_NAMES)
def test_c_stage_bitwise_vs_reference(name):
    from oracle import cbackend as C
    c = G.stage_case(name)
    for (ca, cb, cd, cL), want in zip(c["coefs"], c["out"]):
        dest = c["dest"].copy()
        C.fused_stage(dest, c["A"], c["B"], c["src"], ca, cb, cd, cL, c["grid"], c["species"], c["E"])
        assert np.array_equal(dest[c["grid"].inner()], want)


@pytest.mark.parametrize("name", G.MOMENT_NAMES)
def test_c_moment_bitwise_vs_reference(name):
    from oracle import cbackend as C
    g, data, want = G.moment_case(name + ".npz")
    assert np.array_equal(C.zeroth_moment(data, g), want)
