"""Where the non-stage time of a 2D-2V 128^4 RK4 step goes: device time of
the per-stage field chain (moment finish -> charge -> FFT Poisson -> packed
tables) alone, captured four times into one CUDA graph, against the full
step graph.  python scripts/probes/chain_probe.py [N]"""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
import torch  # noqa: E402

from paper_2410_12155_b200 import problems as PB  # noqa: E402
from paper_2410_12155_b200.kernels import stream_handle  # noqa: E402
from paper_2410_12155_b200.runner import Simulation  # noqa: E402


def graph_time(fn, reps=20):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn()
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        fn()
    g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps


N = int(sys.argv[1]) if len(sys.argv) > 1 else 128
dev = torch.device("cuda", 0)
sim = Simulation(PB.make_problem(PB.landau_spec(), N, N, device=dev), device=dev)
dt = 0.5 * sim.max_dt()
for _ in range(3):
    sim.advance(dt)
torch.cuda.synchronize()
a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(10):
    sim.advance(dt)
b.record()
torch.cuda.synchronize()
step = a.elapsed_time(b) / 10


def chain():
    st = stream_handle(dev)
    for _ in range(4):
        E = sim.fields.solve_from_partials(sim.partials, stream=st)
        for s, tab in enumerate(sim.tables):
            tab.update(E, st, packed=sim.tiled[s])


print(f"{N}^4: step {step:.4f} ms; field chain x4 {graph_time(chain):.4f} ms")
