"""ctypes binding of libdaspmm.so (include/daspmm.h). Loads the in-tree library and
fails loudly when it is missing — there is no CPU fallback."""
from __future__ import annotations

import ctypes as C
import os

PKG = os.path.dirname(os.path.abspath(__file__))
# DASPMM_LIB overrides the library path (tuning aid: compare builds of the same sources)
LIB_PATH = os.environ.get("DASPMM_LIB") or os.path.join(PKG, "libdaspmm.so")

OK = 0
ERR_INVALID_CONFIG = 1
ERR_DIMS = 2
ERR_LAYOUT = 3
ERR_INVALID_ARG = 4
ERR_OUT_OF_RANGE = 5
ERR_MODEL_FORMAT = 6
ERR_CUDA = 7
ERR_NCCL = 8
ERR_UNSUPPORTED = 9

F32, F64 = 0, 1
ROW_MAJOR, COL_MAJOR = 0, 1
EXACT = 1
RESELECT = 2
CONVERT_LAYOUT = 4
SPLIT_AUTO, SPLIT_ROWS, SPLIT_COLS = -1, 0, 1

_vp = C.c_void_p
_i64 = C.c_int64
_i64p = C.POINTER(C.c_int64)
_ip = C.POINTER(C.c_int)

# name -> (restype, argtypes); every symbol here is declared in include/daspmm.h.
SIGNATURES = {
    "daspmm_last_error": (C.c_char_p, []),
    "daspmm_version": (C.c_int, []),
    "daspmm_device_count": (C.c_int, []),
    "daspmm_csr_create_host": (C.c_int, [_i64, _i64, _i64, _vp, _vp, _vp, C.c_int, C.POINTER(_vp)]),
    "daspmm_csr_create_device": (C.c_int, [_i64, _i64, _i64, _vp, _vp, _vp, C.c_int, C.c_int, _vp,
                                           C.POINTER(_vp)]),
    "daspmm_csr_create_coo_device": (C.c_int, [_i64, _i64, _i64, _vp, _vp, _vp, C.c_int, _vp,
                                               C.POINTER(_vp)]),
    "daspmm_csr_create_panel": (C.c_int, [_vp, _i64, _i64, _vp, C.POINTER(_vp)]),
    "daspmm_csr_destroy": (C.c_int, [_vp]),
    "daspmm_csr_values_updated": (C.c_int, [_vp]),
    "daspmm_debug_std_chain": (C.c_int, [_vp, C.POINTER(C.c_double)]),
    "daspmm_csr_info": (C.c_int, [_vp, _i64p, _i64p, _i64p, _ip, _i64p, _i64p]),
    "daspmm_csr_device_arrays": (C.c_int, [_vp, C.POINTER(_vp), C.POINTER(_vp), C.POINTER(_vp)]),
    "daspmm_spmm": (C.c_int, [_vp, C.c_int, _i64, _i64, _i64, _vp, C.c_int, _i64, _i64, _vp, _i64,
                              C.c_uint, _vp]),
    "daspmm_spmm_host": (C.c_int, [_vp, C.c_int, _i64, _i64, _i64, _vp, C.c_int, _i64, _vp,
                                   C.c_uint]),
    "daspmm_spmm_auto_layout": (C.c_int, [_vp, C.c_int, _i64, _i64, _i64, _vp, C.c_int, _i64, _i64,
                                          _vp, _i64, C.c_uint, _vp]),
    "daspmm_extract_features": (C.c_int, [_vp, _i64, _i64p, _i64p, C.POINTER(C.c_double)]),
    "daspmm_partition": (C.c_int, [_vp, _i64, _vp, _vp, _vp]),
    "daspmm_model_parse": (C.c_int, [C.c_char_p, C.c_size_t, C.POINTER(_vp)]),
    "daspmm_model_destroy": (C.c_int, [_vp]),
    "daspmm_model_info": (C.c_int, [_vp, _ip, _ip, _ip, _ip]),
    "daspmm_model_predict_host": (C.c_int, [_vp, _i64, _i64, C.c_double, _i64, _i64, _ip]),
    "daspmm_select": (C.c_int, [_vp, _vp, _i64, _i64, _vp, _vp]),
    "daspmm_spmm_selected": (C.c_int, [_vp, _vp, _i64, _vp, C.c_int, _i64, _i64, _vp, _i64, _i64,
                                       C.c_uint, _vp, _vp]),
    "daspmm_debug_tree_reduce_f64": (C.c_int, [_vp, _i64, _vp]),
    "daspmm_spmm_rows_to": (C.c_int, [_vp, _vp, _i64, _i64, _vp, C.c_int, _i64, _vp]),
    "daspmm_reload_env": (C.c_int, []),
    "daspmm_plan_info": (C.c_int, [_vp, C.c_int, _i64, _vp, _i64, _vp, _i64, C.c_uint, _vp, _vp]),
    "daspmm_debug_conditional_scan_f64": (C.c_int, [_vp, _vp, _i64, _vp]),
    "daspmm_selected_cache_info": (C.c_int, [_vp, _i64p, _i64p, _i64p]),
    "daspmm_comm_unique_id": (C.c_int, [_vp]),
    "daspmm_comm_create": (C.c_int, [C.c_int, C.c_int, _vp, C.POINTER(_vp)]),
    "daspmm_comm_destroy": (C.c_int, [_vp]),
    "daspmm_multi_plan": (C.c_int, [_vp, C.c_int, _i64, C.c_int, _ip, _vp]),
    "daspmm_multi_spmm": (C.c_int, [_vp, _vp, _vp, _i64, _vp, _i64, _i64, _vp, _i64, C.c_int,
                                    C.c_int, _vp, _vp]),
}

_lib = None


class DaspmmError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(msg)
        self.code = code


class ModelFormatError(DaspmmError):
    """spmmkit::ModelFormatError (gbdt.hpp:301-303)."""


class InvalidArgument(DaspmmError, ValueError):
    """std::invalid_argument."""


class OutOfRange(DaspmmError, IndexError):
    """std::out_of_range."""


def lib():
    """The loaded library. Raises if the in-tree build is missing."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} not built — run `python -m paper_2202_08556_b200.build` "
                "(daspmm has no CPU fallback)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in SIGNATURES.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def check(rc: int) -> None:
    if rc == OK:
        return
    msg = lib().daspmm_last_error().decode(errors="replace")
    if rc in (ERR_INVALID_CONFIG, ERR_DIMS, ERR_LAYOUT, ERR_INVALID_ARG):
        raise InvalidArgument(rc, msg)
    if rc == ERR_OUT_OF_RANGE:
        raise OutOfRange(rc, msg)
    if rc == ERR_MODEL_FORMAT:
        raise ModelFormatError(rc, msg)
    raise DaspmmError(rc, msg)
