"""ctypes binding of the sm_100a C-ABI library ``libzt.so`` (include/zt.h).

There is no CPU fallback: if the library is missing this module raises at
import time, and every public op needs a CUDA device.
"""

from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("ZT_LIB_PATH") or os.path.join(_HERE, "libzt.so")

ZT_OK, ZT_EINVAL, ZT_ESTRUCTURE, ZT_ENOCONV, ZT_ELINALG, ZT_ECUDA, ZT_ENCCL, ZT_ENOMEM = range(8)

# (name, restype, argtypes) for every symbol include/zt.h declares
_c_int, _c_i64, _c_sz, _c_dbl, _vp = ctypes.c_int, ctypes.c_int64, ctypes.c_size_t, ctypes.c_double, ctypes.c_void_p
_PI, _PD = ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_double)
SIGNATURES = {
    "zt_version": (_c_int, []),
    "zt_strerror": (ctypes.c_char_p, [_c_int]),
    "zt_last_error": (ctypes.c_char_p, []),
    "zt_op_create": (_c_int, [_c_int, _c_int, ctypes.POINTER(_vp)]),
    "zt_op_destroy": (_c_int, [_vp]),
    "zt_op_n": (_c_int, [_vp]),
    "zt_op_factors": (_c_int, [_vp, _vp, _vp]),
    "zt_stream_solve": (_c_int, [_vp, _vp, _c_i64, _c_i64, _vp, _c_i64, _c_i64, _c_int, _vp]),
    "zt_solve_workspace_bytes": (_c_sz, [_c_int, _c_int]),
    "zt_stream_solve_ws": (_c_int, [_vp, _vp, _c_i64, _c_i64, _vp, _c_i64, _c_i64, _c_int, _vp, _c_sz, _vp]),
    "zt_apply_laplacian": (_c_int, [_vp, _vp, _c_i64, _c_i64, _vp, _c_i64, _c_i64, _c_int, _c_int, _vp]),
    "zt_residuals": (_c_int, [_c_int, _vp, _c_i64, _vp, _vp]),
    "zt_resid_workspace_bytes": (_c_sz, [_c_int]),
    "zt_residuals_ws": (_c_int, [_c_int, _vp, _c_i64, _vp, _vp, _vp]),
    "zt_zgemm": (_c_int, [_c_int, _vp, _c_i64, _vp, _c_i64, _vp, _c_i64, _c_int, _vp]),
    "zt_step_workspace_bytes": (_c_sz, [_c_int]),
    "zt_zgemm_rect": (_c_int, [_c_int, _c_int, _c_int, _vp, _c_i64, _vp, _c_i64, _vp, _c_i64, _c_int, _vp]),
    "zt_zgemm_update_rows": (
        _c_int,
        [_c_int, _c_int, _vp, _vp, _vp, _vp, _vp, _vp, _c_i64, _c_dbl, _c_dbl, _vp, _vp],
    ),
    "zt_fixed_point": (_c_int, [_vp, _vp, _vp, _c_dbl, _c_dbl, _c_int, _vp, _c_sz, _PI, _PD, _vp]),
    "zt_oz_modgemm": (_c_int, [_c_int, _c_int, _c_int, _c_int, _vp, _vp, _vp, _c_int, _vp]),
    "zt_oz_moduli": (_c_int, [_vp, _c_int]),
    "zt_oz_iotas": (_c_int, [_vp, _c_int]),
    "zt_oz_bits": (_c_int, [_c_int]),
    "zt_oz_plane_bytes": (_c_sz, [_c_int, _c_int]),
    "zt_oz_convert_rows": (_c_int, [_c_int, _c_int, _vp, _c_i64, _c_int, _c_int, _c_int, _vp, _vp, _vp, _vp]),
    "zt_oz_convert_cols": (_c_int, [_c_int, _c_int, _vp, _c_i64, _c_int, _vp, _vp, _vp, _vp]),
    "zt_oz_reconstruct": (_c_int, [_c_int, _c_int, _vp, _vp, _vp, _vp, _c_i64, _vp, _c_int, _c_int, _vp, _c_i64,
                                   _c_int, _vp]),
    "zt_oz_workspace_bytes": (_c_sz, [_c_int]),
    "zt_oz_profile_read": (_c_int, [_vp, _vp, _c_int]),
    "zt_oz_zgemm": (_c_int, [_c_int, _vp, _c_i64, _vp, _c_i64, _c_int, _vp, _c_i64, _c_int, _vp, _c_sz, _vp]),
    "zt_midpoint_step_host": (
        _c_int,
        [_vp, _vp, _vp, _vp, _c_dbl, _c_dbl, _c_int, _vp, _c_sz, _PI, _PD, _vp],
    ),
    "zt_midpoint_step": (
        _c_int,
        [_vp, _vp, _vp, _c_dbl, _c_dbl, _c_int, _vp, _c_sz, _PI, _PD, _PD, _vp],
    ),
    "zt_commutator": (_c_int, [_c_int, _vp, _vp, _vp, _vp, _vp]),
    "zt_sandwich": (_c_int, [_c_int, _vp, _vp, _c_dbl, _vp, _vp, _vp]),
    "zt_basis_vectors": (_c_int, [_c_int, _c_int, _c_int, _vp, _vp, _vp]),
    "zt_basis_extract": (_c_int, [_c_int, _c_int, _c_int, _vp, _vp, _vp, _vp, _c_i64, _vp, _vp, _vp]),
    "zt_basis_project": (_c_int, [_c_int, _c_int, _c_int, _vp, _vp, _vp, _vp, _vp, _vp, _c_i64, _vp]),
    "zt_grid_eval": (_c_int, [_c_int, _c_int, _c_int, _c_int, _vp, _vp, _vp, _vp, _vp]),
    "zt_zgemm_rect_scatter": (
        _c_int, [_c_int, _c_int, _c_int, _vp, _c_i64, _vp, _c_i64, _vp, _c_i64, _vp, _c_int, _c_int, _c_int, _vp]),
    "zt_zgemm_update_rows_peer": (
        _c_int,
        [_c_int, _c_int, _vp, _vp, _vp, _c_int, _vp, _vp, _vp, _c_i64, _c_dbl, _c_dbl, _vp, _vp, _c_int, _c_int, _vp],
    ),
    "zt_rows_broadcast": (_c_int, [_c_int, _c_int, _vp, _c_i64, _vp, _c_int, _c_int, _vp]),
    "zt_zgemm_rect_mirror": (_c_int, [_c_int, _c_int, _c_int, _vp, _c_i64, _vp, _c_i64, _vp, _c_i64, _vp, _c_i64, _vp]),
    "zt_update_rows_ew": (
        _c_int,
        [_c_int, _c_int, _vp, _vp, _c_int, _vp, _vp, _vp, _vp, _c_i64, _c_dbl, _c_dbl, _vp, _vp, _c_int, _c_int, _vp],
    ),
    "zt_launch_count": (_c_i64, []),
    "zt_set_graph": (_c_int, [_c_int]),
    "zt_loop_graph_begin": (_c_int, [_vp, ctypes.POINTER(_vp)]),
    "zt_loop_graph_gate": (_c_int, [_vp, _vp, _vp]),
    "zt_loop_graph_body_begin": (_c_int, [_vp, _vp, _vp]),
    "zt_loop_graph_decide": (_c_int, [_vp, _vp, _c_int, _vp, _c_dbl, _c_int, _vp]),
    "zt_loop_graph_body_end": (_c_int, [_vp, _vp]),
    "zt_loop_graph_end": (_c_int, [_vp, _vp]),
    "zt_loop_graph_launch": (_c_int, [_vp, _vp]),
    "zt_loop_graph_destroy": (_c_int, [_vp]),
    "zt_peer_put_u64": (_c_int, [_vp, _vp, _c_int, _c_int, _vp]),
    "zt_step_algo": (_c_int, []),
    "zt_profile_enable": (_c_int, [_c_int]),
    "zt_profile_read": (_c_int, [_vp, _vp, _c_int]),
}


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"{LIB_PATH} is missing: build the sm_100a library first "
            "(python -c 'import __graft_entry__ as g; g.build()'); there is no CPU fallback"
        )
    lib = ctypes.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


lib = _load()


class ZTError(RuntimeError):
    pass


def last_error() -> str:
    msg = lib.zt_last_error()
    return msg.decode() if msg else ""


def check(rc: int, structure_error=None):
    """Map a zt_status to the reference's exception types."""
    if rc == ZT_OK:
        return
    msg = last_error() or lib.zt_strerror(rc).decode()
    if rc == ZT_EINVAL:
        raise ValueError(msg)
    if rc == ZT_ESTRUCTURE and structure_error is not None:
        raise structure_error(msg)
    if rc == ZT_ELINALG:
        raise np.linalg.LinAlgError(msg)
    raise ZTError(f"[{lib.zt_strerror(rc).decode()}] {msg}")


def launch_count() -> int:
    return int(lib.zt_launch_count())
