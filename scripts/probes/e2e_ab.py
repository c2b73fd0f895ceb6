"""A/B of runner.HostPipeline's copy paths at one workload (interleaved):
contiguous staging + compute-stream pack/unpack (staging=True, default) vs
copies straight into / out of the strided interior views (staging=False).
python scripts/probes/e2e_ab.py [workload] [steps] [reps]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2410_12155_b200 import runner as R  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "landau2d-128"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 32
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
dev = torch.device("cuda:0")
setup = bench.make_setup(wl, device=dev)
sim = R.Simulation(setup, device=dev)
dt = 0.9 * sim.max_dt()
sim.fixed_dt = dt
cells = sum(int(torch.tensor(g.N).prod()) for g in sim.grids)
pipes = {s: R.HostPipeline(sim, staging=s) for s in (True, False)}
host_in = pipes[True].host_state()
host_out = [[torch.empty_like(h).pin_memory() for h in host_in] for _ in range(2)]
res = {True: [], False: []}
for p in pipes.values():
    p.run(lambda k: host_in, lambda k: host_out[k & 1], dt, 3)
for r in range(reps):
    for s, p in pipes.items():
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        p.run(lambda k: host_in, lambda k: host_out[k & 1], dt, steps)
        el = time.perf_counter() - t0
        res[s].append(cells * steps / el)
print(json.dumps({"workload": wl, "steps": steps, "staging": res[True], "strided": res[False],
                  "ms_per_step_staging": [cells / v * 1e3 for v in res[True]],
                  "ms_per_step_strided": [cells / v * 1e3 for v in res[False]]}))
