"""ctypes binding of the compiled C restatement (oracle/stage_ref.c).

TEST / CPU-BASELINE INFRASTRUCTURE ONLY.  Built by ``oracle/Makefile`` (called
from ``__graft_entry__.build()``) into ``oracle/_build/libvpfv_oracle.so``.
"""

from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

from . import vpfv_oracle as O

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_build", "libvpfv_oracle.so")

_dp = ctypes.POINTER(ctypes.c_double)
_lib = None


def build():
    subprocess.check_call(["make", "-s", "-C", HERE])


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = ctypes.CDLL(LIB_PATH)
        d, i = ctypes.c_double, ctypes.c_int
        L.oracle_stage_1d1v.argtypes = [_dp] * 4 + [d] * 4 + [_dp] * 3 + [d, d, i, i]
        L.oracle_stage_1d2v.argtypes = [_dp] * 4 + [d] * 4 + [_dp] * 5 + [d] * 4 + [i] * 3
        L.oracle_stage_2d2v.argtypes = ([_dp] * 4 + [d] * 4 + [_dp] * 4 + [d, _dp, d]
                                        + [_dp] * 3 + [d] * 4 + [i] * 4)
        L.oracle_moment.argtypes = [_dp, _dp, i, ctypes.POINTER(ctypes.c_int),
                                    ctypes.POINTER(ctypes.c_int), i, d]
        L.oracle_num_threads.restype = i
        _lib = L
    return _lib


def _p(a):
    assert a.dtype == np.float64 and a.flags.c_contiguous
    return a.ctypes.data_as(_dp)


def num_threads():
    return lib().oracle_num_threads()


def fused_stage(dest, A, B, src, ca, cb, cd, cL, g, s, E):
    """C twin of ``vpfv_oracle.fused_stage`` (no check, no alias test)."""
    L = lib()
    T = {k: (np.ascontiguousarray(v, dtype=np.float64) if isinstance(v, np.ndarray) else v)
         for k, v in O.stage_tables(g, s, E).items()}
    h = g.h
    if (g.d, g.v) == (1, 1):
        L.oracle_stage_1d1v(_p(dest), _p(A), _p(B), _p(src), ca, cb, cd, cL,
                            _p(T["ax"]), _p(T["avx"]), _p(T["c1"]), h[0], h[1], *g.N)
    elif (g.d, g.v) == (1, 2):
        L.oracle_stage_1d2v(_p(dest), _p(A), _p(B), _p(src), ca, cb, cd, cL,
                            _p(T["vxc"]), _p(T["vyc"]), _p(T["evx"]), _p(T["avy"]), _p(T["c1"]),
                            T["c2"], h[0], h[1], h[2], *g.N)
    else:
        L.oracle_stage_2d2v(_p(dest), _p(A), _p(B), _p(src), ca, cb, cd, cL,
                            _p(T["vxc"]), _p(T["vyc"]), _p(T["evx"]), _p(T["evy"]), T["cB"],
                            _p(T["c1"]), T["c2"], _p(T["c3"]), _p(T["c4"]), _p(T["c5"]),
                            *h, *g.N)


def zeroth_moment(data, g):
    out = np.empty(g.N[:g.d])
    Npad = (ctypes.c_int * 4)(*g.padded_shape)
    N = (ctypes.c_int * 4)(*g.N)
    lib().oracle_moment(_p(data), _p(out), g.d, Npad, N, g.v, O.velocity_volume(g))
    return out


class CSimulation(O.OracleSimulation):
    """OracleSimulation whose stages and moments run in the threaded C
    restatement -- the multi-core CPU baseline (bitwise = ``rhs='fused'``)."""

    def _solve(self, arrays):
        for a, g, fr in zip(arrays, self.grids, self.frozen):
            O.fill_ghosts(a, g, fr)
        dens = [zeroth_moment(a, g) for a, g in zip(arrays, self.grids)]
        rho = O.charge_density(dens, self.species)
        _, E = O.poisson_solve(rho, self.grids[0])
        return dens, rho, E

    def _stage(self, dest, A, B, src, ca, cb, cd, cL, t):
        _, _, E = self._solve(src)
        self.last_E = E
        for s, (g, sp) in enumerate(zip(self.grids, self.species)):
            fused_stage(dest[s], A[s], B[s], src[s], ca, cb, cd, cL, g, sp, E)
