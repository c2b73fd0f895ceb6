"""Parity at the benchmarked sizes: every BASELINE workload, at the size
``bench.py`` times it, stepped on the GPU and by the threaded C restatement
of the reference (oracle/stage_ref.c, bitwise = the reference numba kernels,
/root/reference/pkg/src/vpfv/_kernels.py:92-317) from the same initial
state with the same fixed dt.

Bar (north star): relative L2 on f <= 1e-12 after every step, per species.
These are the code paths the small parity cases never reach: the multi-wave
CTA order and super-tile walk of the 2D-2V kernel at 128^4 (1024 column
blocks on 148 SMs), the 1D-2V Geo<32,3> tiles at Nvx = 256, the 1D-1V x-march
with the GPU-wide field chain at 1024^2, and the m_r = 1836 velocity boxes of
the two-species 2D-2V run.  The reference's own pin of the kernels against
the numpy operator is /root/reference/pkg/tests/test_timestepping.py:123-184.

The C oracle steps 128^4 in ~2 s on 16 host cores; the whole file runs in a
few minutes on the GPU box.
"""

import gc

import numpy as np
import pytest

import bench

pytestmark = pytest.mark.gpu

STEPS = {"landau1d-128": 5, "twostream-1024": 3, "weibel-256": 2, "landau2d-128": 2, "ep2d2v-64": 2}


def _rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.mark.parametrize("workload", ["landau1d-128", "twostream-1024", "weibel-256", "ep2d2v-64",
                                      "landau2d-128"])
def test_bench_workload_steps_vs_c_oracle(workload):
    import torch

    from oracle import cbackend as C
    from paper_2410_12155_b200 import runner as R

    setup = bench.make_setup(workload)
    sim = R.Simulation(setup)
    assert all(sim.tiled), "the bench path (tiled / fused kernels) must be the one under test"
    dt = 0.9 * sim.max_dt()
    sim.fixed_dt = dt
    ref = C.CSimulation([f.grid for f in setup.dists], setup.species,
                        [np.array(f.data) for f in bench.make_setup(workload).dists], dt=dt)
    for step in range(STEPS[workload]):
        sim.advance(dt)
        ref.advance(dt)
        got = sim.interiors()
        for s, (a, b) in enumerate(zip(got, ref.interiors())):
            r = _rel(a, b)
            assert r <= 1e-12, f"{workload}: step {step + 1}, species {s}: rel L2 {r:.3e}"
        del got
    del sim, ref
    gc.collect()
    torch.cuda.empty_cache()
