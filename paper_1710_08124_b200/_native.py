"""ctypes binding of ``libfepll_b200.so`` (the C ABI in include/fepll_b200.h).

The library is built in-tree (``python -m paper_1710_08124_b200.build``).
There is no fallback: if it is missing or fails to load, every entry point
raises :class:`DeviceError`.
"""

from __future__ import annotations

import ctypes as C
from pathlib import Path

from .errors import DataError, DeviceError, NumericalError

LIB_PATH = Path(__file__).resolve().parent / "libfepll_b200.so"

i32, i64, f64, vp = C.c_int32, C.c_int64, C.c_double, C.c_void_p
P_i32, P_i64, P_f64, P_f32 = (C.POINTER(C.c_int32), C.POINTER(C.c_int64),
                              C.POINTER(C.c_double), C.POINTER(C.c_float))


class PlanDesc(C.Structure):
    _fields_ = [
        ("patch_dim", i32), ("n_nodes", i32), ("n_components", i32), ("iterations", i32),
        ("child_start", P_i32), ("child_count", P_i32), ("child_list", P_i32),
        ("leaf_index", P_i32), ("depth", P_i32), ("node_rank", P_i32),
        ("grp_width", P_i32), ("grp_col_off", P_i32), ("child_col_off", P_i32),
        ("grp_off64", P_i64), ("grp_basis", P_f64), ("grp_basis_len", i64),
        ("grp_cols_total", i32),
        ("node_const", P_f64), ("node_nu_tail", P_f64), ("grp_sqw", P_f64),
        ("model_rank", P_i32), ("model_col_off", P_i32), ("model_off64", P_i64),
        ("model_basis", P_f64), ("model_basis_len", i64), ("model_cols_total", i32),
        ("model_shrink", P_f64), ("model_gamma_tail", P_f64),
        ("grp_tc_hi", P_f32), ("grp_tc_lo", P_f32), ("grp_tc_len", i64),
        ("grp_tc_off", P_i64), ("grp_tc_npad", P_i32),
        ("grp_tc_child_col", P_i32), ("grp_tc_w", P_f32), ("grp_tc_w_off", P_i32),
        ("grp_tc_w_cols", i32),
        ("grp_tc_x", P_f32),
    ]


# name -> (restype, argtypes)
_SIGS = {
    "fepll_abi_version": (i32, []),
    "fepll_launch_count": (i64, []),
    "fepll_last_error": (C.c_char_p, []),
    "fepll_plan_create": (i32, [C.POINTER(PlanDesc), C.POINTER(vp)]),
    "fepll_plan_reserve": (i32, [vp, i64]),
    "fepll_plan_destroy": (i32, [vp]),
    "fepll_plan_set_option": (i32, [vp, C.c_char_p, i64]),
    "fepll_plan_get_option": (i32, [vp, C.c_char_p, C.POINTER(i64)]),
    "fepll_plan_profile": (i32, [vp, i32]),
    "fepll_plan_profile_read": (i32, [vp, C.POINTER(f64), C.POINTER(i32)]),
    "fepll_grid_scratch_ints": (i32, []),
    "fepll_sample_grid": (i32, [C.c_uint64, C.c_uint64, i32, i32, i32, i32, i32, C.c_uint32, vp, vp, vp, vp]),
    "fepll_extract": (i32, [vp, i32, i32, i32, i32, vp, i32, i32, vp, vp, i32, vp, vp, vp]),
    "fepll_select": (i32, [vp, i32, vp, i32, i32, vp, i32, vp, vp, vp, vp, i64, i32, f64, vp, vp, vp]),
    "fepll_wiener_reads_image": (i32, [vp]),
    "fepll_wiener": (i32, [vp, i32, vp, i32, i32, vp, i32, vp, vp, i64, vp, i32, vp]),
    "fepll_select_rescored": (i32, [vp, vp, vp]),
    "fepll_wiener_f32": (i32, [vp, i32, vp, i32, i32, vp, i32, vp, vp, i32, i64, vp, i32, vp]),
    "fepll_aggregate_strip_f32": (i32, [vp, vp, vp, i32, i32, i32, i32, i32, i32, i32, i32,
                                        i32, i32, i32, i32, i32, i32, vp, vp, f64, i32, vp, vp, vp, vp]),
    "fepll_aggregate_cover_ex": (i32, [vp, vp, vp, vp, vp, i32, i32, i32, i32, i32, i32, i32, i32, vp, vp,
                                       f64, i32, vp, vp, vp, i32, vp]),
    "fepll_aggregate_cover_f32": (i32, [vp, vp, vp, vp, i32, i32, i32, i32, i32, i32, i32, i32, vp, vp,
                                        f64, i32, vp, vp, vp, vp]),
    "fepll_aggregate": (i32, [vp, vp, vp, i32, i32, i32, i32, i32, i32, i32, i32, vp, vp, f64,
                              i32, vp, vp, vp, vp]),
    "fepll_aggregate_strip": (i32, [vp, vp, vp, i32, i32, i32, i32, i32, i32, i32, i32,
                                    i32, i32, i32, i32, i32, i32, vp, vp, f64, i32, vp, vp, vp, vp]),
    "fepll_cover_scratch_ints": (i64, [i64]),
    "fepll_cover_build": (i32, [vp, i32, i32, i32, i32, i32, i32, i32, i32, i32, i32, i32, i32,
                                vp, vp, i64, vp, vp]),
    "fepll_tiles_seg_cap": (i32, [i32, i32, i32]),
    "fepll_tiles_width": (i32, []),
    "fepll_debug_level_spans": (i32, [vp]),
    "fepll_stamp": (i32, [vp, vp]),
    "fepll_tiles_smem_bytes": (i64, [i32, i32, i32, i32, i32]),
    "fepll_tiles_build": (i32, [vp, vp, i32, i32, i32, i32, i32, vp, vp, vp, vp, vp, vp]),
    "fepll_aggregate_tiles": (i32, [vp, vp, vp, i32, vp, vp, vp, vp, i32, i32, i32, i32, i32, i32, i32, i32, i32,
                                    vp, vp, f64, i32, vp, vp, vp, vp]),
    "fepll_aggregate_cover": (i32, [vp, vp, vp, vp, i32, i32, i32, i32, i32, i32, i32, i32, vp, vp, f64,
                                    i32, vp, vp, vp, vp]),
    "fepll_op_create": (i32, [i32, i32, i32, i32, vp, i32, i32, vp, C.POINTER(vp)]),
    "fepll_op_destroy": (i32, [vp]),
    "fepll_op_adjoint": (i32, [vp, vp, vp, vp]),
    "fepll_op_lambda": (i32, [vp, vp, f64, f64, C.POINTER(f64), C.POINTER(f64)]),
    "fepll_op_init": (i32, [vp, vp, vp, f64, f64, f64, i32, vp, vp, vp]),
    "fepll_op_solve": (i32, [vp, vp, vp, f64, f64, i32, vp, vp, vp, vp]),
    "fepll_op_normal": (i32, [vp, vp, f64, vp, vp]),
    "fepll_tree_kl": (i32, [vp, vp, i32, i32, vp, vp, vp]),
    "fepll_cluster_swap": (i32, [vp, i32, i32, vp, vp, i32, vp, vp]),
}

_lib = None


def lib():
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise DeviceError(f"{LIB_PATH.name} is not built; run python -m paper_1710_08124_b200.build")
        try:
            h = C.CDLL(str(LIB_PATH))
        except OSError as e:
            raise DeviceError(f"cannot load {LIB_PATH}: {e}") from e
        for name, (res, args) in _SIGS.items():
            fn = getattr(h, name)
            fn.restype = res
            fn.argtypes = args
        _lib = h
    return _lib


def exported_symbols() -> list:
    return list(_SIGS)


def check(rc: int, what: str) -> None:
    if rc == 0:
        return
    msg = lib().fepll_last_error().decode(errors="replace")
    text = f"{what}: {msg}"
    if rc == 3:
        raise DataError(text)
    if rc == 4:
        raise NumericalError(text)
    raise DeviceError(text)


def call(name: str, *args) -> None:
    check(getattr(lib(), name)(*args), name)


def ptr(t) -> int | None:
    """Device pointer of a torch tensor (None passes NULL)."""
    return None if t is None else t.data_ptr()
