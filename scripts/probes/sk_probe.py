"""Stream-K probe: one RK4 step of a single-species 2D-2V Landau set-up at
N^4 (default 64), device-timed over 20 graph replays, under whatever
VPFV_RB_SK / VPFV_XSEG the environment sets; and, for two species, whether
the side-stream stage launches overlap (sum of per-species stage times vs the
step).  python scripts/probes/sk_probe.py [N]"""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
import torch  # noqa: E402

from paper_2410_12155_b200 import problems as PB  # noqa: E402
from paper_2410_12155_b200.runner import Simulation  # noqa: E402


def timed(sim, dt, steps=20):
    sim.advance(dt)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(steps):
        sim.advance(dt)
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / steps


N = int(sys.argv[1]) if len(sys.argv) > 1 else 64
dev = torch.device("cuda", 0)
setup = PB.make_problem(PB.landau_spec(), N, N, device=dev)
sim = Simulation(setup, device=dev)
dt = 0.5 * sim.max_dt()
print(f"landau2d {N}^4 single species: {timed(sim, dt):.4f} ms/step  "
      f"(VPFV_RB_SK={os.environ.get('VPFV_RB_SK', '1')}, VPFV_XSEG={os.environ.get('VPFV_XSEG', 'auto')})")
