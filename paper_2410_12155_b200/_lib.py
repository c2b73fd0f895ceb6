"""ctypes binding of libvpfv.so (the sm_100a CUDA library behind include/vpfv.h).

There is no fallback: if the library is missing, or the device is not an
sm_100 part, every compute entry point raises.  The library is built
in-tree by ``__graft_entry__.build()`` (or ``python -m
paper_2410_12155_b200.build``) so it travels with the repository snapshot.
"""

from __future__ import annotations

import ctypes
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("VPFV_LIB") or os.path.join(HERE, "lib", "libvpfv.so")

VPFV_OK = 0
VPFV_EALIAS = 1
VPFV_EDIM = 2
VPFV_ENONFINITE = 3
VPFV_ECUDA = 4
VPFV_EARG = 5
VPFV_ENCCL = 6

VPFV_EXACT = 0x1
VPFV_FINITE = 0xFFFFFFFFFFFFFFFF


def VPFV_WRAP(k):
    return 1 << (1 + k)


_d = ctypes.c_double
_i = ctypes.c_int
_u = ctypes.c_uint
_p = ctypes.c_void_p

# (name, restype, argtypes) -- must match include/vpfv.h
SIGNATURES = {
    "vpfv_stage_1d1v": (_i, [_p] * 4 + [_d] * 4 + [_p] * 3 + [_d, _d, _i, _i, _u, _p, _d, _p, _p]),
    "vpfv_stage_1d1v_fused": (_i, [_p] * 4 + [_d] * 4 + [_p] * 3 + [_d, _d, _i, _i, _u, _p, _d, _p, _p, _p]),
    "vpfv_stage_1d2v": (_i, [_p] * 4 + [_d] * 4 + [_p] * 5 + [_d] * 4 + [_i] * 3 + [_u, _p, _d, _p, _p]),
    "vpfv_stage_2d2v": (_i, [_p] * 4 + [_d] * 4 + [_p] * 4 + [_d, _p, _d] + [_p] * 3 + [_d] * 4
                        + [_i] * 4 + [_u, _p, _d, _p, _p]),
    "vpfv_stage_2d2v_fused": (_i, [_p] * 4 + [_d] * 4 + [_p] * 4 + [_d, _p, _d] + [_p] * 3
                              + [_d] * 4 + [_i] * 4 + [_u, _p, _d, _p, _p, _p, _i, _p]),
    "vpfv_stage_2d2v_fused_range": (_i, [_p] * 4 + [_d] * 4 + [_p] * 4 + [_d, _p, _d] + [_p] * 3
                                    + [_d] * 4 + [_i] * 6 + [_u, _p, _d, _p, _p, _p, _p]),
    "vpfv_stage_2d2v_fused_peer": (_i, [_p] * 4 + [_d] * 4 + [_p] * 4 + [_d] + [_p] + [_d] + [_p] * 3 + [_d] * 4
                                   + [_i] * 4 + [_u, _p, _d, _p, _p, _p, _p, _p, _p, _p, _p, _p]),
    "vpfv_peer_signal": (_i, [_p, _p, _p]),
    "vpfv_flag_exchange": (_i, [_p, _i, _p, _i, _p, _p, _p, _d, _p, _p]),
    "vpfv_moment_partials_push": (_i, [_p, _i, _i, _i, _d, _p, _i, _p, _i, _p, _p]),
    "vpfv_peer_wait": (_i, [_p, _p, _i, _i, _d, _p, _p]),
    "vpfv_ipc_handle_size": (_i, []),
    "vpfv_ipc_export": (_i, [_p, _p, _p]),
    "vpfv_ipc_open": (_i, [_p, ctypes.c_longlong, _p]),
    "vpfv_stage_2d2v_generic": (_i, [_p] * 4 + [_d] * 4 + [_p] * 4 + [_d, _p, _d] + [_p] * 3
                                + [_d] * 4 + [_i] * 4 + [_u, _p, _d, _p, _p]),
    "vpfv_moment_partials": (_i, [_p, _p, _i, _i, _i, _d, _p]),
    "vpfv_stage_2d2v_tiled_ok": (_i, [_i, _i, _i, _i, _u]),
    "vpfv_stage_1d2v_fused": (_i, [_p] * 4 + [_d] * 4 + [_p] * 5 + [_d] * 4 + [_i] * 3
                              + [_u, _p, _d, _p, _p, _p, _i, _p]),
    "vpfv_stage_1d2v_fused_peer": (_i, [_p] * 4 + [_d] * 4 + [_p] * 5 + [_d] * 4 + [_i] * 3
                                   + [_u, _p, _d, _p, _p, _p, _p, _p, _p, _p, _p, _p]),
    "vpfv_stage_1d2v_tiled_ok": (_i, [_i, _i, _i, _u]),
    "vpfv_tables_1d_packed": (_i, [_p, _p, _i, _d, _d, _d, _d, _p]),
    "vpfv_stage_2d2v_partials_chunk": (_i, []),
    "vpfv_stage_1d2v_partials_chunk": (_i, []),
    "vpfv_moment": (_i, [_p, _p, _i, _i, _p, _d, _p]),
    "vpfv_moment_seq": (_i, [_p, _p, _i, _i, _p, _d, _p]),
    "vpfv_higher_moments": (_i, [_p, _i, _i, _p, _p, _p, _d, _d, _p, _p]),
    "vpfv_richardson_partials": (_i, [_p, _p, _i, _p, _p, _i, _p]),
    "vpfv_scale": (_i, [_p, _d, ctypes.c_longlong, _p]),
    "vpfv_field_1d_max_cells": (_i, []),
    "vpfv_field_1d_conv": (_i, [_p, _p, _p, _p, _p, _i, _i, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p]),
    "vpfv_field_1d": (_i, [_p, _p, _p, _p, _p, _p, _i, _i, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p, _p]),
    "vpfv_charge_density": (_i, [_p, _p, _i, _i, _p, _p]),
    "vpfv_poisson_1d": (_i, [_p, _p, _p, _i, _p, _p, _p, _p]),
    "vpfv_poisson_2d": (_i, [_p] * 4 + [_i, _i] + [_p] * 7 + [_p]),
    "vpfv_tables_1d": (_i, [_p, _p, _p, _i, _d, _d, _d, _d, _p]),
    "vpfv_tables_2d": (_i, [_p] * 8 + [_i, _i] + [_d] * 8 + [_p]),
    "vpfv_tables_2d_packed": (_i, [_p] * 3 + [_i, _i] + [_d] * 8 + [_p]),
    "vpfv_wrap_fill": (_i, [_p, _i, _p, _u, _p]),
    "vpfv_box_copy": (_i, [_p, _p, _p, _p, _p, _p, _i, _p, _p]),
    "vpfv_version": (_i, []),
    "vpfv_moment_chunk_partials": (_i, [_p, _p, _i, _p, _p]),
    "vpfv_comm_id_size": (_i, []),
    "vpfv_comm_unique_id": (_i, [_p]),
    "vpfv_comm_init": (_i, [_p, _i, _i, _p, _i]),
    "vpfv_comm_destroy": (_i, [_p]),
    "vpfv_halo_exchange_x": (_i, [_p, _p, _i, _p, _p]),
    "vpfv_density_allgather": (_i, [_p, _p, _p, ctypes.c_longlong, _p]),
    "vpfv_flag_allreduce": (_i, [_p, _p, _p]),
    "vpfv_init_separable": (_i, [_p, ctypes.c_longlong, _i, _i] + [_p] * 6 + [_i, _p]),
    "vpfv_check_device": (_i, [_i]),
    "vpfv_last_error": (ctypes.c_char_p, []),
}

_lib = None
_checked_devices = set()


class VpfvError(RuntimeError):
    pass


def load():
    """Load libvpfv.so (no device needed) and declare every entry point."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise VpfvError(
                f"{LIB_PATH} is not built; run `python -c 'import __graft_entry__ as g; g.build()'` "
                "(the B200 path has no CPU fallback)"
            )
        lib = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
    return _lib


def check_device(dev: int):
    if dev in _checked_devices:
        return
    rc = load().vpfv_check_device(dev)
    if rc != VPFV_OK:
        raise VpfvError(f"libvpfv: {load().vpfv_last_error().decode()}")
    _checked_devices.add(dev)


# kernels launched per entry-point call (for launch accounting); default 1
KERNELS_PER_CALL = {"vpfv_poisson_2d": 3, "vpfv_version": 0, "vpfv_check_device": 0,
                    "vpfv_last_error": 0, "vpfv_stage_2d2v_tiled_ok": 0,
                    "vpfv_stage_2d2v_partials_chunk": 0, "vpfv_stage_1d2v_tiled_ok": 0}
launch_counter = [0]


def call(name, *args):
    """Invoke an entry point and map its status to the reference exceptions."""
    launch_counter[0] += KERNELS_PER_CALL.get(name, 1)
    rc = getattr(load(), name)(*args)
    if rc == VPFV_OK:
        return
    msg = load().vpfv_last_error().decode()
    if rc in (VPFV_EALIAS, VPFV_EDIM, VPFV_EARG):
        raise ValueError(msg)
    if rc == VPFV_ENONFINITE:
        raise FloatingPointError(msg)
    raise VpfvError(f"{name}: {msg} (status {rc})")


def int_array(vals):
    return (ctypes.c_int * len(vals))(*[int(v) for v in vals])


def ll_array(vals):
    return (ctypes.c_longlong * len(vals))(*[int(v) for v in vals])


def ptr_array(vals):
    return (ctypes.c_void_p * len(vals))(*[int(v) if v else None for v in vals])


def dbl_array(vals):
    return (ctypes.c_double * len(vals))(*[float(v) for v in vals])
