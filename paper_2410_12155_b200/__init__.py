"""B200-native VP-FV (arXiv 2410.12155) stage hot path behind the reference `vpfv` API.

Host-side Python mirrors the reference package's public surface for the hot
path (grid, species, problems, stage protocol, Simulation, fused_stage,
fields); every per-stage operation runs in libvpfv.so, hand-written CUDA for
sm_100a loaded through ctypes (include/vpfv.h is the C ABI).  There is no CPU
fallback: without the library or an sm_100 device the compute calls raise.
"""

from .grid import NGHOST, DistField, FrozenGhosts, PhaseSpaceGrid, fill_local_ghosts, make_grid
from .fvm import SpeciesConfig

__all__ = ["NGHOST", "DistField", "FrozenGhosts", "PhaseSpaceGrid", "fill_local_ghosts",
           "make_grid", "SpeciesConfig"]
