"""TEST INFRASTRUCTURE ONLY — ctypes front-end for the CPU oracle.

Loads ``oracle/libdaspmm_oracle.so`` (plain-C restatement of the reference's hot
path, oracle/daspmm_oracle.c) and, when present, ``oracle/_ref/libspmmkit_ref.so``
(the unmodified reference headers behind a C-ABI shim, oracle/ref_driver.cpp).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline legs may
import this module. The product package (``paper_2202_08556_b200``) never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "libdaspmm_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libspmmkit_ref.so")

_i64p = np.ctypeslib.ndpointer(np.int64, flags="C_CONTIGUOUS")
_i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")
_f64p = np.ctypeslib.ndpointer(np.float64, flags="C_CONTIGUOUS")
_f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")


def build(ref: bool = True) -> None:
    """Compile the oracle (and the reference shim when /root/reference exists)."""
    targets = ["oracle"] + (["ref"] if ref else [])
    subprocess.run(["make", "-s", "-C", HERE] + targets, check=True)


_lib = None
_ref = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(ORACLE_SO):
            build(ref=False)
        L = C.CDLL(ORACLE_SO)
        for sfx, fp in (("f64", _f64p), ("f32", _f32p)):
            f = getattr(L, f"oracle_spmm_reference_{sfx}")
            f.argtypes = [C.c_int64, C.c_int64, C.c_int64, _i64p, _i64p, fp, fp, C.c_int, fp]
            f.restype = None
            f = getattr(L, f"oracle_spmm_{sfx}")
            f.argtypes = [C.c_int, C.c_int64, C.c_int64, C.c_int64, C.c_int64, C.c_int64,
                          C.c_int64, _i64p, _i64p, fp, fp, fp]
            f.restype = C.c_int
            f = getattr(L, f"oracle_tree_reduce_lanes_{sfx}")
            f.argtypes = [fp, C.c_int64, C.c_int64]
            f.restype = None
            f = getattr(L, f"oracle_conditional_scan_lanes_{sfx}")
            f.argtypes = [fp, _i64p, C.c_int64, C.c_int64]
            f.restype = None
        L.oracle_row_of_element.argtypes = [C.c_int64, _i64p, C.c_int64]
        L.oracle_row_of_element.restype = C.c_int64
        L.oracle_partition_elements.argtypes = [C.c_int64, _i64p, C.c_int64, _i64p, _i64p, _i64p]
        L.oracle_partition_elements.restype = C.c_int
        L.oracle_extract_features.argtypes = [C.c_int64, _i64p, C.POINTER(C.c_double)]
        L.oracle_extract_features.restype = C.c_int
        L.oracle_encode_features.argtypes = [C.c_int64, C.c_int64, C.c_double, C.c_int64,
                                             C.c_int, C.c_int64, _f64p]
        L.oracle_encode_features.restype = C.c_int
        L.oracle_predict_class.argtypes = [C.c_int, C.c_int, _i64p, _i32p, _f64p, _i32p, _i32p,
                                           _f64p, _f64p, _f64p]
        L.oracle_predict_class.restype = C.c_int
        _lib = L
    return _lib


def have_ref() -> bool:
    return os.path.exists(REF_SO)


def ref():
    """The reference shim, or None when oracle/_ref was not built (e.g. GPU box
    without a prebuilt copy)."""
    global _ref
    if _ref is None and have_ref():
        R = C.CDLL(REF_SO)
        R.ref_last_error.restype = C.c_char_p
        R.ref_rmat.argtypes = [C.c_int, C.c_int64] + [C.c_double] * 4 + [C.c_uint64]
        R.ref_rmat.restype = C.c_void_p
        R.ref_csr_from_coo.argtypes = [C.c_int64, C.c_int64, C.c_int64, _i64p, _i64p, _f64p]
        R.ref_csr_from_coo.restype = C.c_void_p
        R.ref_csr_from_csr.argtypes = [C.c_int64, C.c_int64, _i64p, _i64p, _f64p]
        R.ref_csr_from_csr.restype = C.c_void_p
        R.ref_read_matrix_market.argtypes = [C.c_char_p]
        R.ref_read_matrix_market.restype = C.c_void_p
        R.ref_csr_info.argtypes = [C.c_void_p] + [C.POINTER(C.c_int64)] * 3
        R.ref_csr_copy.argtypes = [C.c_void_p, _i64p, _i64p, _f64p]
        R.ref_csr_free.argtypes = [C.c_void_p]
        R.ref_dense_random_f64.argtypes = [C.c_int64, C.c_int64, C.c_int, C.c_uint64, _f64p]
        R.ref_dense_random_f32.argtypes = [C.c_int64, C.c_int64, C.c_int, C.c_uint64, _f32p]
        for sfx, fp in (("f64", _f64p), ("f32", _f32p)):
            f = getattr(R, f"ref_spmm_reference_{sfx}")
            f.argtypes = [C.c_void_p, fp, C.c_int64, C.c_int, fp]
            f.restype = C.c_int
            f = getattr(R, f"ref_spmm_{sfx}")
            f.argtypes = [C.c_void_p, C.c_int, C.c_int64, C.c_int64, C.c_int64, fp, C.c_int64,
                          C.c_int, fp]
            f.restype = C.c_int
        R.ref_time_spmm_f32.argtypes = [C.c_void_p, C.c_int, C.c_int64, C.c_int64, C.c_int64,
                                        _f32p, C.c_int64, C.c_int, C.c_int] + \
            [C.POINTER(C.c_double)] * 3
        R.ref_time_spmm_f32.restype = C.c_int
        R.ref_dense_f32.argtypes = [_f32p, C.c_int64, C.c_int64, C.c_int]
        R.ref_dense_f32.restype = C.c_void_p
        R.ref_dense_free.argtypes = [C.c_void_p]
        R.ref_time_spmm_once_f32.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int64,
                                             C.c_int64, C.c_int64, C.POINTER(C.c_double)]
        R.ref_time_spmm_once_f32.restype = C.c_int
        R.ref_time_spmm_dense_reference_f32.argtypes = [C.c_void_p, C.c_void_p,
                                                        C.POINTER(C.c_double)]
        R.ref_time_spmm_dense_reference_f32.restype = C.c_int
        R.ref_partition.argtypes = [C.c_void_p, C.c_int, _i64p, _i64p, _i64p]
        R.ref_partition.restype = C.c_int
        R.ref_row_index_of.argtypes = [C.c_void_p, C.c_int64, C.POINTER(C.c_int64)]
        R.ref_row_index_of.restype = C.c_int
        R.ref_tree_reduce_f64.argtypes = [_f64p, C.c_int64, C.POINTER(C.c_double)]
        R.ref_tree_reduce_f64.restype = C.c_int
        R.ref_conditional_reduce_f64.argtypes = [_f64p, _i64p, C.c_int64, _i64p, _f64p,
                                                 C.POINTER(C.c_int64)]
        R.ref_conditional_reduce_f64.restype = C.c_int
        R.ref_extract_features.argtypes = [C.c_void_p, C.c_int64, C.POINTER(C.c_int64),
                                           C.POINTER(C.c_int64), C.POINTER(C.c_double)]
        R.ref_extract_features.restype = C.c_int
        R.ref_selector_load.argtypes = [C.c_char_p]
        R.ref_selector_load.restype = C.c_void_p
        R.ref_selector_free.argtypes = [C.c_void_p]
        R.ref_selector_predict.argtypes = [C.c_void_p, C.c_int64, C.c_int64, C.c_double,
                                           C.c_int64, C.c_int64, C.POINTER(C.c_int)]
        R.ref_selector_predict.restype = C.c_int
        R.ref_selector_train.argtypes = [C.c_int64, C.c_int64, _f64p, C.c_void_p, _f64p,
                                         C.c_int, C.c_int, C.c_int]
        R.ref_selector_train.restype = C.c_void_p
        R.ref_free.argtypes = [C.c_void_p]
        _ref = R
    return _ref


# ---------------------------------------------------------------- numpy helpers
class Csr:
    """Host CSR with int64 indices, as the reference's CsrMatrix (types.hpp:28-35)."""

    def __init__(self, rows, cols, rp, ci, vals):
        self.num_rows = int(rows)
        self.num_cols = int(cols)
        self.row_offsets = np.ascontiguousarray(rp, dtype=np.int64)
        self.col_indices = np.ascontiguousarray(ci, dtype=np.int64)
        self.values = np.ascontiguousarray(vals, dtype=np.float64)

    @property
    def nnz(self) -> int:
        return int(self.row_offsets[-1])


def spmm_reference(a: Csr, x: np.ndarray, x_colmajor: bool = False, dtype=np.float64):
    """spmm_reference (spmm.hpp:16-32). ``x`` is given in its memory order
    (shape K x N RowMajor, or the flat ColMajor buffer when x_colmajor)."""
    L = lib()
    sfx = "f64" if dtype == np.float64 else "f32"
    n = x.shape[1] if not x_colmajor else x.size // max(a.num_cols, 1)
    if x_colmajor and a.num_cols == 0:
        n = 0
    y = np.zeros((a.num_rows, n), dtype=dtype)
    xv = np.ascontiguousarray(x, dtype=dtype).reshape(-1)
    getattr(L, f"oracle_spmm_reference_{sfx}")(a.num_rows, a.num_cols, n, a.row_offsets,
                                               a.col_indices, a.values.astype(dtype), xv,
                                               int(x_colmajor), y.reshape(-1))
    return y


def spmm_kernel(kernel: int, a: Csr, x_logical: np.ndarray, P=1, W=8, Cb=4,
                dtype=np.float64):
    """One of the 8 design-space kernels (spmm.hpp:194-271), run serially with
    workers in index order. ``x_logical`` is K x N (logical); it is laid out as the
    kernel's N-loop choice requires (CM kernels read ColMajor)."""
    L = lib()
    sfx = "f64" if dtype == np.float64 else "f32"
    K, n = x_logical.shape
    cm = (kernel >> 1) & 1
    xmem = np.ascontiguousarray(x_logical.T if cm else x_logical, dtype=dtype).reshape(-1)
    y = np.zeros((a.num_rows, n), dtype=dtype)
    rc = getattr(L, f"oracle_spmm_{sfx}")(kernel, P, W, Cb, a.num_rows, a.num_cols, n,
                                          a.row_offsets, a.col_indices,
                                          a.values.astype(dtype), xmem, y.reshape(-1))
    if rc:
        raise ValueError(f"oracle_spmm rc={rc}")
    return y


def partition_elements(a: Csr, p: int):
    L = lib()
    b = np.zeros(p, np.int64)
    e = np.zeros(p, np.int64)
    r = np.zeros(p, np.int64)
    if L.oracle_partition_elements(a.num_rows, a.row_offsets, p, b, e, r):
        raise ValueError("partition_elements: need p >= 1")
    return b, e, r


def extract_features(a: Csr):
    L = lib()
    s = C.c_double()
    if L.oracle_extract_features(a.num_rows, a.row_offsets, C.byref(s)):
        raise ValueError("extract_features: matrix has no rows to summarize")
    return a.nnz, a.num_rows, s.value


def tree_reduce_lanes(v: np.ndarray, w: int, lanes: int) -> np.ndarray:
    out = np.ascontiguousarray(v, dtype=np.float64).copy()
    lib().oracle_tree_reduce_lanes_f64(out, w, lanes)
    return out


def conditional_scan_lanes(v: np.ndarray, ids: np.ndarray, w: int, lanes: int) -> np.ndarray:
    out = np.ascontiguousarray(v, dtype=np.float64).copy()
    lib().oracle_conditional_scan_lanes_f64(out, np.ascontiguousarray(ids, np.int64), w, lanes)
    return out


def encode_features(nnz, mat_size, std_row, n_cols, uses_hw=False, hw=-1):
    out = np.zeros(5, np.float64)
    k = lib().oracle_encode_features(nnz, mat_size, std_row, n_cols, int(uses_hw), hw, out)
    if k < 0:
        raise ValueError("encode_features: model expects a hardware_id but the sample has none")
    return out[:k]


def predict_class(flat, f: np.ndarray) -> int:
    """flat: dict from parse_model_text (tests/helpers)."""
    scores = np.zeros(flat["num_classes"], np.float64)
    return lib().oracle_predict_class(flat["num_classes"], flat["num_rounds"], flat["tree_off"],
                                      flat["feat"], flat["thr"], flat["left"], flat["right"],
                                      flat["value"], np.ascontiguousarray(f, np.float64), scores)


def parse_selector_text(text: str) -> dict:
    """Minimal parser for the reference's selector text v1 (selector.hpp:113-132,
    gbdt.hpp:336-453) into flat arrays for oracle_predict_class."""
    tok = text.split()
    i = 0

    def nxt():
        nonlocal i
        i += 1
        return tok[i - 1]

    assert nxt() == "spmmkit-selector" and nxt() == "v1"
    assert nxt() == "uses_hardware"
    uses_hw = int(nxt()) != 0
    assert nxt() == "spmmkit-gbdt" and nxt() == "v1"
    assert nxt() == "classes"
    ncls = int(nxt())
    assert nxt() == "features"
    nfeat = int(nxt())
    assert nxt() == "best_round"
    nxt()
    assert nxt() == "config"
    for _ in range(7):
        nxt()
        nxt()
    assert nxt() == "feature_names"
    for _ in range(int(nxt())):
        nxt()
    assert nxt() == "rounds"
    nrounds = int(nxt())
    feat, thr, left, right, value, off = [], [], [], [], [], [0]
    for r in range(nrounds):
        for c in range(ncls):
            assert nxt() == "tree"
            assert int(nxt()) == r and int(nxt()) == c
            nn = int(nxt())
            for _ in range(nn):
                assert nxt() == "node"
                kind = nxt()
                if kind == "split":
                    feat.append(int(nxt()))
                    thr.append(float(nxt()))
                    left.append(int(nxt()))
                    right.append(int(nxt()))
                    nxt()  # gain
                    value.append(0.0)
                else:
                    feat.append(-1)
                    thr.append(0.0)
                    left.append(-1)
                    right.append(-1)
                    value.append(float(nxt()))
            off.append(off[-1] + nn)
    assert nxt() == "end"
    return dict(uses_hardware=uses_hw, num_classes=ncls, num_features=nfeat,
                num_rounds=nrounds, tree_off=np.array(off, np.int64),
                feat=np.array(feat, np.int32), thr=np.array(thr, np.float64),
                left=np.array(left, np.int32), right=np.array(right, np.int32),
                value=np.array(value, np.float64))
