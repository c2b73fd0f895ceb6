import sys, os, numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from oracle import vpfv_oracle as O
from paper_2410_12155_b200 import kernels as K, _lib
from paper_2410_12155_b200.grid import make_grid
N = (8, 8, 8, 32)
g = O.Grid(2, 2, N, (0.0, 0.0, -4.0, -5.0), (2 * np.pi, 4 * np.pi, 4.0, 5.0), (True, True, False, False))
rng = np.random.default_rng(1)
src = 1.0 + 0.3 * rng.random(g.padded_shape)
O.fill_ghosts(src, g, O.capture_frozen(src, g))
E = {"Ex": np.zeros((8, 8)) + 0.1, "Ey": np.zeros((8, 8)) - 0.1}
sp = O.Species("e", -1.0, 1.0, 1.1, 0.3, 1.0, (0.02, -0.01))
pg = make_grid(2, 2, N, g.lo, g.hi, periodic=g.periodic)
want = np.zeros(g.padded_shape)
O.fused_stage(want, src, src, src, 1.0, 0.0, 0.0, 0.02, g, sp, E, check=False)
got = np.zeros(g.padded_shape)
K.fused_stage(got, src, src, src, 1.0, 0.0, 0.0, 0.02, pg, sp, E, exact=False)
torch.cuda.synchronize()
print("maxdiff", np.max(np.abs(got[g.inner()] - want[g.inner()])))
