"""Where a small step's time goes: advance() (host sync per step) vs graph
replays back to back vs the Python cost of advance's host side.

    python scripts/probes/step_overhead.py WORKLOAD [steps]
"""
import sys
import time

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2410_12155_b200 import runner as R  # noqa: E402

wl = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 200
for timing in (False, True):
    sim = R.Simulation(bench.make_setup(wl))
    dt = sim.max_dt()
    sim.enable_stage_timing(timing)
    for _ in range(5):
        sim.advance(dt)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    s.record()
    for _ in range(n):
        sim.advance(dt)
    e.record()
    torch.cuda.synchronize()
    wall = (time.perf_counter() - t0) / n * 1e6
    dev = s.elapsed_time(e) / n * 1e3
    # back-to-back graph replays (no per-step host sync)
    bufs = (sim.ctx.f0, sim.ctx.f1, sim.ctx.fout)
    g = sim._graph_for(bufs, sim.fuse_moment)
    g.replay()
    torch.cuda.synchronize()
    s.record()
    for _ in range(n):
        g.replay()
    e.record()
    torch.cuda.synchronize()
    rep = s.elapsed_time(e) / n * 1e3
    t0 = time.perf_counter()
    for _ in range(n):
        sim.dt_dev.fill_(float(dt))
    torch.cuda.synchronize()
    fill = (time.perf_counter() - t0) / n * 1e6
    t0 = time.perf_counter()
    for _ in range(n):
        g.replay()
    cpu_replay = (time.perf_counter() - t0) / n * 1e6
    torch.cuda.synchronize()
    print(f"{wl} timing={timing}: advance wall {wall:.1f} us, device {dev:.1f} us/step; "
          f"replay-only {rep:.1f} us/step; host: fill {fill:.1f} us, replay call {cpu_replay:.1f} us")
