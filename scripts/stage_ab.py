"""Time the four RK4 stage launches of the tiled 2D-2V kernel on a synthetic
128^4 state, for one or more library builds (A/B of kernel variants).

    python scripts/stage_ab.py [--N 128] [--reps 10] LIB [LIB ...]

LIB is a path to a libvpfv.so build ("main" = the in-tree one).  Every LIB
runs in its own process (the library is bound at import); each prints one
line: per-stage milliseconds (mean over reps, CUDA events on the launch
stream) and their sum, plus a checksum of the stage-4 output so variants can
be compared for equality.  Uses random f (1 + 0.3 U[0,1)) and smooth E; not
on any product path.
"""

import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def child(N, reps, lib, nopart=False, nonf=False):
    sys.path.insert(0, ROOT)
    import numpy as np
    import torch

    from paper_2410_12155_b200 import _lib
    from paper_2410_12155_b200.fvm import SpeciesConfig
    from paper_2410_12155_b200.grid import make_grid
    from paper_2410_12155_b200.kernels import StageTables, stream_handle, wrap_flags
    from paper_2410_12155_b200.timestepping import RK4_STAGES

    dev = torch.device("cuda", 0)
    g = make_grid(2, 2, (N, N, N, N), (0.0, 0.0, -8.0, -8.0), (4 * np.pi, 4 * np.pi, 8.0, 8.0),
                  periodic=(True, True, False, False))
    sp = SpeciesConfig(q=-1.0, kappa_c=0.02, Bz=1.0)
    gen = torch.Generator(device=dev)
    gen.manual_seed(1)
    bufs = {k: 1.0 + 0.3 * torch.rand(g.padded_shape, dtype=torch.float64, device=dev, generator=gen)
            for k in ("f0", "f1", "fout")}
    cx = torch.as_tensor(g.centers(0), device=dev)
    cy = torch.as_tensor(g.centers(1), device=dev)
    E = {"Ex": 0.4 * torch.outer(torch.sin(0.5 * cx), torch.cos(0.5 * cy)) + 0.05,
         "Ey": 0.3 * torch.outer(torch.cos(0.5 * cx), torch.sin(cy))}
    tab = StageTables(g, sp, dev)
    stream = stream_handle(dev)
    tab.update(E, stream, packed=True)
    flags = wrap_flags(g)
    part = torch.empty(tab.partials_shape(), dtype=torch.float64, device=dev)
    nf = torch.full((1,), -1, dtype=torch.int64, device=dev)
    dt = 0.01
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(2)] for _ in range(4)]
    times = [0.0] * 4

    def step(record):
        for s, (dn, an, bn, sn, ca, cb, cd, div) in enumerate(RK4_STAGES):
            if record:
                ev[s][0].record()
            tab.launch(bufs[dn], bufs[an], bufs[bn], bufs[sn], ca, cb, cd, dt / div, flags, stream,
                       nonfinite=None if nonf else nf, partials=None if nopart else part, packed=True)
            if record:
                ev[s][1].record()
        bufs["f0"], bufs["fout"] = bufs["fout"], bufs["f0"]

    for _ in range(3):
        step(False)
    torch.cuda.synchronize()
    for _ in range(reps):
        step(True)
        torch.cuda.synchronize()
        for s in range(4):
            times[s] += ev[s][0].elapsed_time(ev[s][1]) / reps
    cs = float(bufs["f0"][3:-3, 3:-3, 3:-3, 3:-3].double().sum().item())
    print(json.dumps({"lib": lib + (" nopart" if nopart else "") + (" nonf" if nonf else ""), "stage_ms": [round(t, 4) for t in times], "sum_ms": round(sum(times), 4),
                      "checksum": cs, "nonfinite": int(nf.item())}), flush=True)


def main():
    args = sys.argv[1:]
    N, reps = 128, 10
    if "--N" in args:
        i = args.index("--N")
        N = int(args[i + 1])
        del args[i:i + 2]
    if "--reps" in args:
        i = args.index("--reps")
        reps = int(args[i + 1])
        del args[i:i + 2]
    flags = [a for a in args if a in ("--nopart", "--nonf")]
    args = [a for a in args if a not in flags]
    if args and args[0] == "--child":
        child(N, reps, args[1], "--nopart" in flags, "--nonf" in flags)
        return
    for lib in args:
        env = dict(os.environ)
        if lib != "main":
            env["VPFV_LIB"] = os.path.abspath(lib)
        subprocess.run([sys.executable, __file__, "--N", str(N), "--reps", str(reps), *flags, "--child", lib],
                       env=env, check=False)


if __name__ == "__main__":
    main()
