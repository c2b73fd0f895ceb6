"""Child process for the kernel-variant tests: one RK4 step's four fused stage
launches (the RK4 3/8 aliasing, fused partials, non-finite word) on a seeded
state -- 2D-2V 8 x 8 x 128 x 128 or, with MODE 1d2v, 1D-2V 24 x 64 x 64 --
with whatever VPFV_RB_* / VPFV_R12_* switches the parent set in the
environment; writes the three buffers and the last partials to an .npz.
The switches are read once per process, so every variant runs in its own
process.  Test infrastructure only.

    python tests/helpers/kernel_variant_step.py OUT.npz [2d2v|1d2v]
"""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2410_12155_b200.fvm import SpeciesConfig  # noqa: E402
from paper_2410_12155_b200.grid import make_grid  # noqa: E402
from paper_2410_12155_b200.kernels import StageTables, stream_handle, wrap_flags  # noqa: E402
from paper_2410_12155_b200.timestepping import RK4_STAGES  # noqa: E402


def main(out, mode="2d2v"):
    dev = torch.device("cuda", 0)
    sp = SpeciesConfig(q=-1.0, kappa_c=0.02, Bz=0.5)
    gen = torch.Generator(device=dev)
    gen.manual_seed(5)
    if mode == "1d2v":
        g = make_grid(1, 2, (24, 64, 64), (0.0, -6.0, -6.0), (2 * np.pi, 6.0, 6.0), periodic=(True, False, False))
        cx = torch.as_tensor(g.centers(0), device=dev)
        E = {"Ex": 0.4 * torch.sin(cx) + 0.05}
    else:
        g = make_grid(2, 2, (8, 8, 128, 128), (0.0, 0.0, -6.0, -6.0), (2 * np.pi, 4 * np.pi, 6.0, 6.0),
                      periodic=(True, True, False, False))
        cx = torch.as_tensor(g.centers(0), device=dev)
        cy = torch.as_tensor(g.centers(1), device=dev)
        E = {"Ex": 0.4 * torch.outer(torch.sin(cx), torch.cos(0.5 * cy)) + 0.05,
             "Ey": 0.3 * torch.outer(torch.cos(cx), torch.sin(cy))}
    bufs = {k: 1.0 + 0.3 * torch.rand(g.padded_shape, dtype=torch.float64, device=dev, generator=gen)
            for k in ("f0", "f1", "fout")}
    tab = StageTables(g, sp, dev)
    stream = stream_handle(dev)
    tab.update(E, stream, packed=True)
    flags = wrap_flags(g)
    part = torch.empty(tab.partials_shape(), dtype=torch.float64, device=dev)
    nf = torch.full((1,), -1, dtype=torch.int64, device=dev)
    for dn, an, bn, sn, ca, cb, cd, div in RK4_STAGES:
        tab.launch(bufs[dn], bufs[an], bufs[bn], bufs[sn], ca, cb, cd, 0.01 / div, flags, stream, nonfinite=nf,
                   partials=part, packed=True)
    torch.cuda.synchronize()
    np.savez(out, nonfinite=nf.cpu().numpy(), partials=part.cpu().numpy(),
             **{k: v.cpu().numpy() for k, v in bufs.items()})


if __name__ == "__main__":
    main(sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else "2d2v")
