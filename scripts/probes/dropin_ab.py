"""Drop-in fused_stage host staging sweep (kernels._HostStager THREADS /
NBUF / CHUNK_BYTES) at one workload: RK4 steps of four host-array
fused_stage calls, interleaved settings, wall clock.
python scripts/probes/dropin_ab.py [workload] [reps]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2410_12155_b200 import kernels as K  # noqa: E402
from paper_2410_12155_b200 import runner as R  # noqa: E402

wl = sys.argv[1] if len(sys.argv) > 1 else "landau2d-128"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
dev = torch.device("cuda:0")
setup = bench.make_setup(wl, device=dev)
sim = R.Simulation(setup, device=dev)
dt = 0.9 * sim.max_dt()
cells = sum(int(torch.tensor(g.N).prod()) for g in sim.grids)
E_host = sim._E_host(sim.ctx.f0)
h0 = sim._host_state()[0]
del sim
torch.cuda.empty_cache()
settings = [(8, 2, 64), (16, 2, 64), (16, 3, 64), (16, 4, 32), (16, 2, 128), (12, 3, 128)]
res = {str(s): [] for s in settings}
for r in range(reps):
    for th, nb, mb in settings:
        K._HostStager.THREADS, K._HostStager.NBUF, K._HostStager.CHUNK_BYTES = th, nb, mb << 20
        K._DROPIN.clear()
        out = bench.e2e_dropin_measure(setup, h0.copy(), E_host, dt, dev, cells, steps=1)
        res[str((th, nb, mb))].append(round(out["seconds"], 4))
        print(th, nb, mb, out["seconds"], file=sys.stderr, flush=True)
print(json.dumps({"workload": wl, "seconds_per_step": res, "cores": os.cpu_count()}))
