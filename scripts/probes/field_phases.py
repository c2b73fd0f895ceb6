"""Per-phase globaltimer stamps of vpfv_field_1d (library built with
-DVPFV_FIELD_PROBE: scripts/build_variant.sh probe -DVPFV_FIELD_PROBE, run with
VPFV_LIB=exp/libvpfv_probe.so).   python scripts/probes/field_phases.py WORKLOAD"""
import ctypes
import sys

import torch

sys.path.insert(0, ".")
import bench  # noqa: E402
from paper_2410_12155_b200 import _lib, runner as R  # noqa: E402

sim = R.Simulation(bench.make_setup(sys.argv[1]), use_graphs=False)
dt = sim.max_dt()
names = ["finish+rho", "tree", "put", "fwd fft", "ph/put", "inv fft", "Ex out", "tables"]
acc = [0.0] * 8
n = 0
for it in range(30):
    sim.advance(dt)
    torch.cuda.synchronize()
    buf = (ctypes.c_ulonglong * 16)()
    _lib.load().vpfv_field_probe(buf)
    if it >= 5:
        st = list(buf)[:9]
        for k in range(8):
            acc[k] += (st[k + 1] - st[k]) / 1e3
        n += 1
print(sys.argv[1], " ".join(f"{nm}={a / n:.2f}us" for nm, a in zip(names, acc)), f"total={sum(acc) / n:.2f}us")
