"""Child process for the launch-mode tests: a few graph-replayed RK4 steps
of a problem through runner.Simulation under whatever VPFV_* switches the
parent set (read once per process), interiors written to an .npz.  Test
infrastructure only.

    python tests/helpers/sim_steps.py OUT.npz PROBLEM N STEPS
"""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2410_12155_b200 import problems as P  # noqa: E402
from paper_2410_12155_b200.runner import Simulation  # noqa: E402


def main(out, problem, n, steps):
    dev = torch.device("cuda", 0)
    setup = {
        "landau2d": lambda: P.make_problem(P.landau_spec(), n, n),
        "landau1d": lambda: P.make_landau_1d(P.landau_spec(alpha=0.01), n, n),
        "twostream": lambda: P.make_problem(P.ProblemSpec("two-stream"), n, n),
        "bimax1d2v": lambda: P.make_bimaxwellian_1d2v(n, n, n),
        "ep2d2v": lambda: P.make_electron_proton_2d2v(n, n),
    }[problem]()
    sim = Simulation(setup, device=dev)
    dt = 0.5 * sim.max_dt()
    for _ in range(steps):
        sim.advance(dt)
    torch.cuda.synchronize()
    np.savez(out, *sim.interiors())


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2], int(sys.argv[3]), int(sys.argv[4]))
