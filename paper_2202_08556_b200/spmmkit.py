"""spmmkit's hot-path API (proj/include/spmmkit) over the B200 library.

Same names, argument meaning and error behaviour as the reference's C++ API, so the
parity tests read like the reference's own tests:

  reference (C++)                                   here
  ------------------------------------------------  -------------------------------------
  CsrMatrix<T> (types.hpp:28-91)                    CsrMatrix  (host, int64 indices)
  DenseMatrix<T>, Layout (types.hpp:16, 158-206)    DenseMatrix, Layout
  KernelId, all_kernels (kernel_id.hpp:12-76)       KernelId, all_kernels
  WorkerConfig, make_config (worker.hpp:18-55)      WorkerConfig, make_config, ...
  spmm / spmm_auto_layout (spmm.hpp:194-281)        spmm / spmm_auto_layout  (run on the GPU)
  extract_features (features.hpp:21-41)             extract_features           (GPU)
  partition_elements (partition.hpp:45-64)          partition_elements         (GPU kernel)
  load_selector / predict_kernel (selector.hpp)     load_selector / predict_kernel
  —                                                 DeviceCsr: device-resident handle,
                                                    spmm_device / select_device /
                                                    spmm_selected (torch tensors)

std::invalid_argument -> ValueError (InvalidArgument), std::out_of_range ->
IndexError (OutOfRange), ModelFormatError -> ModelFormatError.
"""
from __future__ import annotations

import ctypes as C
import enum
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

from . import _lib
from ._lib import InvalidArgument, ModelFormatError, OutOfRange, check, lib

__all__ = [
    "Layout", "KernelId", "all_kernels", "kNumKernels", "WorkerConfig", "validate_config",
    "is_valid", "recommended_col_block", "make_config", "CsrMatrix", "DenseMatrix",
    "convert_layout", "DeviceCsr", "spmm", "spmm_auto_layout", "spmm_device",
    "extract_features", "FeatureVector", "partition_elements", "SelectorModel", "load_selector",
    "predict_kernel", "Tolerance", "tolerance_equal", "InvalidArgument", "OutOfRange",
    "ModelFormatError", "spmm_selected", "SpmmBatch", "selected_cache_info",
]


class Layout(enum.IntEnum):
    RowMajor = _lib.ROW_MAJOR
    ColMajor = _lib.COL_MAJOR


# ------------------------------------------------------------------ kernel_id.hpp
_M = ("RB", "EB")
_N = ("RM", "CM")
_K = ("SR", "PR")
kNumKernels = 8


@dataclass(frozen=True)
class KernelId:
    """One point of the 2x2x2 design space; index = 4m + 2n + k (kernel_id.hpp:25-27)."""
    m: int = 0
    n: int = 0
    k: int = 0

    def index(self) -> int:
        return self.m * 4 + self.n * 2 + self.k

    @staticmethod
    def from_index(idx: int) -> "KernelId":
        if idx < 0 or idx > 7:
            raise OutOfRange(_lib.ERR_OUT_OF_RANGE, "KernelId index must be 0..7")
        return KernelId(idx // 4, (idx // 2) % 2, idx % 2)

    def name(self) -> str:
        return f"{_M[self.m]}+{_N[self.n]}+{_K[self.k]}"

    @staticmethod
    def parse(s: str) -> Optional["KernelId"]:
        if len(s) != 8 or s[2] != "+" or s[5] != "+":
            return None
        try:
            return KernelId(_M.index(s[0:2]), _N.index(s[3:5]), _K.index(s[6:8]))
        except ValueError:
            return None

    def __int__(self):
        return self.index()

    def __repr__(self):
        return f"KernelId({self.name()})"


def all_kernels():
    return [KernelId.from_index(i) for i in range(kNumKernels)]


# ------------------------------------------------------------------ worker.hpp
@dataclass
class WorkerConfig:
    num_workers: int = 1  # P
    group_width: int = 8  # W
    col_block: int = 4    # C


def validate_config(cfg: WorkerConfig):
    """worker.hpp:29-40 — list of issues, empty when valid."""
    issues = []
    if cfg.num_workers < 1:
        issues.append(f"num_workers must be >= 1, got {cfg.num_workers}")
    w = cfg.group_width
    if w < 2 or (w & (w - 1)) != 0:
        issues.append(f"group_width must be a power of two >= 2, got {w}")
    if cfg.col_block < 1:
        issues.append(f"col_block must be >= 1, got {cfg.col_block}")
    return issues


def is_valid(cfg: WorkerConfig) -> bool:
    return not validate_config(cfg)


def recommended_col_block(kernel: KernelId, n_cols: int) -> int:
    """worker.hpp:47-50."""
    cap = 4 if kernel.k == 1 else 8
    return max(1, min(n_cols, cap))


def make_config(kernel: KernelId, n_cols: int, num_workers: int = 1, group_width: int = 8):
    return WorkerConfig(num_workers, group_width, recommended_col_block(kernel, n_cols))


# ------------------------------------------------------------------ types.hpp
class CsrMatrix:
    """Host CSR with int64 offsets/indices (types.hpp:28-35)."""

    def __init__(self, num_rows=0, num_cols=0, row_offsets=None, col_indices=None, values=None,
                 dtype=np.float64):
        self.num_rows = int(num_rows)
        self.num_cols = int(num_cols)
        self.row_offsets = np.zeros(1, np.int64) if row_offsets is None else \
            np.ascontiguousarray(row_offsets, np.int64)
        self.col_indices = np.zeros(0, np.int64) if col_indices is None else \
            np.ascontiguousarray(col_indices, np.int64)
        self.values = np.zeros(0, dtype) if values is None else np.ascontiguousarray(values, dtype)

    def nnz(self) -> int:
        return int(self.col_indices.size)

    def row_nnz(self, m: int) -> int:
        return int(self.row_offsets[m + 1] - self.row_offsets[m])

    @staticmethod
    def identity(n: int, dtype=np.float64) -> "CsrMatrix":
        return CsrMatrix(n, n, np.arange(n + 1), np.arange(n), np.ones(n, dtype), dtype)

    @staticmethod
    def from_coo(num_rows, num_cols, triplets, dtype=np.float64) -> "CsrMatrix":
        """types.hpp:56-90: sort by (row, col), sum duplicates."""
        if len(triplets) == 0:
            return CsrMatrix(num_rows, num_cols, np.zeros(num_rows + 1, np.int64), None, None, dtype)
        r = np.array([t[0] for t in triplets], np.int64)
        c = np.array([t[1] for t in triplets], np.int64)
        v = np.array([t[2] for t in triplets], dtype)
        if (r < 0).any() or (r >= num_rows).any() or (c < 0).any() or (c >= num_cols).any():
            raise InvalidArgument(_lib.ERR_INVALID_ARG, "from_coo: coordinate out of bounds")
        order = np.lexsort((c, r))
        r, c, v = r[order], c[order], v[order]
        keep = np.ones(r.size, bool)
        keep[1:] = (r[1:] != r[:-1]) | (c[1:] != c[:-1])
        grp = np.cumsum(keep) - 1
        vs = np.zeros(int(keep.sum()), dtype)
        # duplicates summed in sorted order, left to right (types.hpp:67-80)
        for i in range(v.size):
            vs[grp[i]] = vs[grp[i]] + v[i] if not keep[i] else v[i]
        r, c = r[keep], c[keep]
        rp = np.zeros(num_rows + 1, np.int64)
        np.add.at(rp, r + 1, 1)
        return CsrMatrix(num_rows, num_cols, np.cumsum(rp), c, vs, dtype)

    def astype(self, dtype) -> "CsrMatrix":
        return CsrMatrix(self.num_rows, self.num_cols, self.row_offsets, self.col_indices,
                         self.values.astype(dtype), dtype)


class DenseMatrix:
    """Dense operand with explicit layout (types.hpp:158-194). ``data`` is the flat
    buffer in memory order, as the reference's std::vector."""

    def __init__(self, rows, cols, layout=Layout.RowMajor, data=None, dtype=np.float64):
        self.num_rows = int(rows)
        self.num_cols = int(cols)
        self.layout = Layout(layout)
        self.data = np.zeros(self.num_rows * self.num_cols, dtype) if data is None else \
            np.ascontiguousarray(data, dtype).reshape(-1)

    @property
    def dtype(self):
        return self.data.dtype

    def index_of(self, r, c):
        return r * self.num_cols + c if self.layout == Layout.RowMajor else c * self.num_rows + r

    def at(self, r, c):
        return self.data[self.index_of(r, c)]

    def logical(self) -> np.ndarray:
        """rows x cols array in logical order."""
        if self.layout == Layout.RowMajor:
            return self.data.reshape(self.num_rows, self.num_cols)
        return self.data.reshape(self.num_cols, self.num_rows).T

    @staticmethod
    def from_logical(a: np.ndarray, layout=Layout.RowMajor) -> "DenseMatrix":
        a = np.asarray(a)
        buf = a if layout == Layout.RowMajor else a.T
        return DenseMatrix(a.shape[0], a.shape[1], layout, np.ascontiguousarray(buf).reshape(-1),
                           a.dtype)

    @staticmethod
    def zeros(rows, cols, layout=Layout.RowMajor, dtype=np.float64):
        return DenseMatrix(rows, cols, layout, None, dtype)


def convert_layout(m: DenseMatrix, target: Layout) -> DenseMatrix:
    """types.hpp:198-206."""
    if m.layout == target:
        return DenseMatrix(m.num_rows, m.num_cols, m.layout, m.data.copy(), m.dtype)
    return DenseMatrix.from_logical(m.logical(), target)


# ------------------------------------------------------------------ device handle
def _dtype_code(dtype) -> int:
    dt = np.dtype(dtype)
    if dt == np.float32:
        return _lib.F32
    if dt == np.float64:
        return _lib.F64
    raise InvalidArgument(_lib.ERR_INVALID_ARG, f"unsupported value type {dt}")


class DeviceCsr:
    """Device-resident CSR handle (int32 offsets/cols on the GPU)."""

    def __init__(self, handle: int, dtype, keepalive=None, device: Optional[int] = None):
        self._h = C.c_void_p(handle)
        self.dtype = np.dtype(dtype)
        self._keep = keepalive
        self.device = _current_device() if device is None else int(device)
        M, K, nnz, dt, ne, ct = (C.c_int64(), C.c_int64(), C.c_int64(), C.c_int(), C.c_int64(),
                                 C.c_int64())
        check(lib().daspmm_csr_info(self._h, C.byref(M), C.byref(K), C.byref(nnz), C.byref(dt),
                                    C.byref(ne), C.byref(ct)))
        self.num_rows, self.num_cols, self._nnz = M.value, K.value, nnz.value
        self.empty_rows, self.cols_touched = ne.value, ct.value

    @staticmethod
    def from_host(a: CsrMatrix, dtype=None) -> "DeviceCsr":
        dtype = np.dtype(dtype or a.values.dtype)
        vals = np.ascontiguousarray(a.values, dtype)
        rp = np.ascontiguousarray(a.row_offsets, np.int64)
        ci = np.ascontiguousarray(a.col_indices, np.int64)
        out = C.c_void_p()
        check(lib().daspmm_csr_create_host(a.num_rows, a.num_cols, a.nnz(), rp.ctypes.data,
                                           ci.ctypes.data, vals.ctypes.data, _dtype_code(dtype),
                                           C.byref(out)))
        return DeviceCsr(out.value, dtype)

    @staticmethod
    def from_device(num_rows, num_cols, row_offsets, col_indices, values, copy=False,
                    stream=None) -> "DeviceCsr":
        """torch int32 offsets/cols and float32/float64 values on the GPU."""
        import torch

        assert row_offsets.dtype == torch.int32 and col_indices.dtype == torch.int32
        dtype = np.float32 if values.dtype == torch.float32 else np.float64
        out = C.c_void_p()
        check(lib().daspmm_csr_create_device(num_rows, num_cols, col_indices.numel(),
                                             row_offsets.data_ptr(), col_indices.data_ptr(),
                                             values.data_ptr(), _dtype_code(dtype), int(copy),
                                             _stream_ptr(stream), C.byref(out)))
        keep = None if copy else (row_offsets, col_indices, values)
        return DeviceCsr(out.value, dtype, keep, row_offsets.device.index)

    @staticmethod
    def from_coo_device(num_rows, num_cols, rows, cols, values, stream=None) -> "DeviceCsr":
        """CsrMatrix::from_coo (types.hpp:54-90) on the device: torch int64 row / column
        tensors and float32/float64 values on the GPU, any order; duplicates summed in
        input order; out-of-bounds coordinates raise InvalidArgument with the reference's
        message (daspmm_csr_create_coo_device)."""
        import torch

        assert rows.dtype == torch.int64 and cols.dtype == torch.int64
        assert rows.numel() == cols.numel() == values.numel()
        dtype = np.float32 if values.dtype == torch.float32 else np.float64
        rows, cols, values = rows.contiguous(), cols.contiguous(), values.contiguous()
        out = C.c_void_p()
        check(lib().daspmm_csr_create_coo_device(num_rows, num_cols, rows.numel(),
                                                 rows.data_ptr(), cols.data_ptr(),
                                                 values.data_ptr(), _dtype_code(dtype),
                                                 _stream_ptr(stream), C.byref(out)))
        return DeviceCsr(out.value, dtype, None, rows.device.index)

    def values_updated(self):
        """The borrowed values tensor was changed in place (same structure): drop the
        handle's derived copies of the values (daspmm_csr_values_updated)."""
        check(lib().daspmm_csr_values_updated(self._h))

    def panel(self, r0: int, r1: int, stream=None) -> "DeviceCsr":
        out = C.c_void_p()
        check(lib().daspmm_csr_create_panel(self._h, r0, r1, _stream_ptr(stream), C.byref(out)))
        return DeviceCsr(out.value, self.dtype, device=self.device)

    def nnz(self) -> int:
        return self._nnz

    def device_arrays(self):
        rp, ci, va = C.c_void_p(), C.c_void_p(), C.c_void_p()
        check(lib().daspmm_csr_device_arrays(self._h, C.byref(rp), C.byref(ci), C.byref(va)))
        return rp.value, ci.value, va.value

    def close(self):
        if self._h:
            lib().daspmm_csr_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _current_device() -> int:
    try:
        import torch

        if torch.cuda.is_available():
            return torch.cuda.current_device()
    except Exception:
        pass
    return 0


_TORCH_DT = {np.dtype(np.float32): "torch.float32", np.dtype(np.float64): "torch.float64"}


def _check_operands(a: DeviceCsr, B, C_out, b_layout, what: str = "spmm"):
    """The checks the C ABI cannot make on raw pointers (spmm.hpp:197-209 for the
    dimensions): 2-D CUDA tensors on the handle's device, the handle's value type,
    unit column stride, B with K rows (K x N row-major, or the N x K buffer of a
    column-major B) and C of M x N."""
    for name, t in (("B", B), ("C", C_out)):
        if getattr(t, "dim", lambda: -1)() != 2:
            raise InvalidArgument(_lib.ERR_INVALID_ARG, f"{what}: {name} must be a 2-D tensor")
        if not t.is_cuda or t.device.index != a.device:
            raise InvalidArgument(_lib.ERR_INVALID_ARG,
                                  f"{what}: {name} must be a CUDA tensor on cuda:{a.device}, "
                                  f"got {t.device}")
        if str(t.dtype) != _TORCH_DT.get(a.dtype):
            raise InvalidArgument(_lib.ERR_INVALID_ARG,
                                  f"{what}: {name} is {t.dtype} but A holds {a.dtype}")
        if t.shape[1] > 1 and t.stride(1) != 1:
            raise InvalidArgument(_lib.ERR_INVALID_ARG,
                                  f"{what}: {name} needs unit column stride, got {t.stride(1)}")
    k_rows = B.shape[0] if b_layout == Layout.RowMajor else B.shape[1]
    n = B.shape[1] if b_layout == Layout.RowMajor else B.shape[0]
    if k_rows != a.num_cols:
        raise InvalidArgument(_lib.ERR_DIMS, f"{what}: A is {a.num_rows}x{a.num_cols} but X has "
                                             f"{k_rows} rows")
    if tuple(C_out.shape) != (a.num_rows, n):
        raise InvalidArgument(_lib.ERR_DIMS, f"{what}: C is {C_out.shape[0]}x{C_out.shape[1]}, "
                                             f"expected {a.num_rows}x{n}")
    return n


def _stream_ptr(stream):
    if stream is None:
        try:
            import torch

            if torch.cuda.is_available():
                return torch.cuda.current_stream().cuda_stream
        except Exception:
            pass
        return None
    return getattr(stream, "cuda_stream", stream)


def _ld(t) -> int:
    """Leading dimension of a row-major 2-D tensor (torch ignores the stride of a
    size-1 dimension when deciding contiguity, so do not trust it there)."""
    return int(t.stride(0)) if t.shape[0] > 1 else int(max(t.shape[1], 1))


def _as_device(a) -> DeviceCsr:
    return a if isinstance(a, DeviceCsr) else DeviceCsr.from_host(a)


# ------------------------------------------------------------------ spmm.hpp
def spmm(kernel: KernelId, a, x: DenseMatrix, cfg: WorkerConfig, exact: bool = False) -> DenseMatrix:
    """spmm() — spmm.hpp:194-271, computed on the GPU. Same checks and messages:
    config, then dimensions, then layout. Returns a RowMajor DenseMatrix.

    ``exact`` selects the reference evaluation order (bit-identical results; EB
    honours cfg.num_workers as the chunk count). Otherwise the library fuses
    multiply-adds and picks the EB chunking itself (tolerance parity)."""
    issues = validate_config(cfg)
    if issues:
        raise InvalidArgument(_lib.ERR_INVALID_CONFIG, "spmm: invalid config; " + "; ".join(issues))
    if a.num_cols != x.num_rows:
        raise InvalidArgument(_lib.ERR_DIMS, f"spmm: A is {a.num_rows}x{a.num_cols} but X has "
                                              f"{x.num_rows} rows")
    want = Layout.ColMajor if kernel.n == 1 else Layout.RowMajor
    if x.layout != want:
        raise InvalidArgument(_lib.ERR_LAYOUT, f"spmm: kernel {kernel.name()} needs {want.name} X, "
                                                f"got {x.layout.name}")
    d = _as_device(a)
    if d.dtype != x.dtype:
        raise InvalidArgument(_lib.ERR_INVALID_ARG, "spmm: A and X value types differ")
    n = x.num_cols
    y = np.zeros(a.num_rows * n, x.dtype)
    P = cfg.num_workers if exact else 0
    xb = np.ascontiguousarray(x.data)
    check(lib().daspmm_spmm_host(d._h, kernel.index(), P, cfg.group_width, cfg.col_block,
                                 xb.ctypes.data, int(x.layout), n, y.ctypes.data,
                                 _lib.EXACT if exact else 0))
    return DenseMatrix(a.num_rows, n, Layout.RowMajor, y, x.dtype)


def spmm_auto_layout(kernel: KernelId, a, x: DenseMatrix, cfg: WorkerConfig,
                     exact: bool = False) -> DenseMatrix:
    """spmm.hpp:275-281."""
    want = Layout.ColMajor if kernel.n == 1 else Layout.RowMajor
    return spmm(kernel, a, x if x.layout == want else convert_layout(x, want), cfg, exact)


def spmm_device(kernel, a: DeviceCsr, B, C_out, P: int = 0, W: int = 8, Cb: int = 4,
                b_layout: Layout = None, exact: bool = False, stream=None):
    """Device-operand SpMM on torch tensors. B: K x N row-major tensor, or — for
    b_layout=ColMajor — an N x K tensor (the column-major buffer). C_out: M x N."""
    kid = kernel.index() if isinstance(kernel, KernelId) else int(kernel)
    if b_layout is None:
        b_layout = Layout.ColMajor if (kid >> 1) & 1 else Layout.RowMajor
    n = _check_operands(a, B, C_out, b_layout)
    check(lib().daspmm_spmm(a._h, kid, P, W, Cb, B.data_ptr(), int(b_layout), _ld(B), n,
                            C_out.data_ptr(), _ld(C_out), _lib.EXACT if exact else 0,
                            _stream_ptr(stream)))
    return C_out


def spmm_rows_to(a: DeviceCsr, B, outs, stream=None):
    """RB+RM+SR with the row epilogue replicated into every tensor of `outs` (each
    M x N row-major with the same leading dimension, fp32) — see daspmm_spmm_rows_to."""
    outs = list(outs)
    for o in outs:
        _check_operands(a, B, o, Layout.RowMajor, "spmm_rows_to")
    ldc = _ld(outs[0])
    if any(_ld(o) != ldc or tuple(o.shape) != tuple(outs[0].shape) for o in outs):
        raise InvalidArgument(_lib.ERR_DIMS, "spmm_rows_to: destinations differ in shape")
    ptrs = (C.c_void_p * len(outs))(*[o.data_ptr() for o in outs])
    check(lib().daspmm_spmm_rows_to(a._h, B.data_ptr(), _ld(B), B.shape[1], ptrs, len(outs),
                                    ldc, _stream_ptr(stream)))
    return outs[0]


def reload_env():
    """Re-read the planner's tuning environment variables (daspmm_reload_env)."""
    check(lib().daspmm_reload_env())


PLAN_VARIANTS = {0: "base", 1: "rb_window", 2: "eb_cta", 3: "eb_thread", 4: "lean", 5: "eb_tma",
                 6: "rb_tile", 7: "cm_rows"}


def plan_info(kernel, a: DeviceCsr, B, C_out, exact: bool = False, b_layout: Layout = None):
    """(variant name, parameter) of the launch daspmm_spmm would run for these device
    operands — diagnostics (see daspmm_plan_info). B as for spmm_device: K x N row-major,
    or the N x K buffer of a column-major B (the default for CM kernels)."""
    kid = kernel.index() if isinstance(kernel, KernelId) else int(kernel)
    if b_layout is None:
        b_layout = Layout.ColMajor if (kid >> 1) & 1 else Layout.RowMajor
    n = _check_operands(a, B, C_out, b_layout, "plan_info")
    v, prm = C.c_int(), C.c_int64()
    check(lib().daspmm_plan_info(a._h, kid, n, B.data_ptr(), _ld(B), C_out.data_ptr(),
                                 _ld(C_out), _lib.EXACT if exact else 0, C.byref(v),
                                 C.byref(prm)))
    return PLAN_VARIANTS[v.value], prm.value


# ------------------------------------------------------------------ features / partition
@dataclass
class FeatureVector:
    nnz: int = 0
    mat_size: int = 0
    std_row: float = 0.0
    n_cols: int = 0
    hardware_id: Optional[int] = None


def extract_features(a, n_cols: int, hardware_id: Optional[int] = None) -> FeatureVector:
    """features.hpp:21-41, on the device (std_row bit-identical to the reference)."""
    if a.num_rows == 0:
        raise InvalidArgument(_lib.ERR_INVALID_ARG,
                              "extract_features: matrix has no rows to summarize")
    d = _as_device(a)
    nnz, ms, sd = C.c_int64(), C.c_int64(), C.c_double()
    check(lib().daspmm_extract_features(d._h, n_cols, C.byref(nnz), C.byref(ms), C.byref(sd)))
    return FeatureVector(nnz.value, ms.value, sd.value, n_cols, hardware_id)


def partition_elements(a, p: int):
    """partition.hpp:45-64 via the device partition kernel. Returns
    (begin, end, row_of_chunk_start) int64 arrays."""
    if p < 1:
        raise InvalidArgument(_lib.ERR_INVALID_ARG, "partition_elements: need p >= 1")
    d = _as_device(a)
    b = np.zeros(p, np.int64)
    e = np.zeros(p, np.int64)
    r = np.zeros(p, np.int64)
    check(lib().daspmm_partition(d._h, p, b.ctypes.data, e.ctypes.data, r.ctypes.data))
    return b, e, r


# ------------------------------------------------------------------ selector
class SelectorModel:
    """load_selector result (selector.hpp:12-15, 119-132)."""

    def __init__(self, text: str):
        raw = text.encode()
        self._m = C.c_void_p()
        check(lib().daspmm_model_parse(raw, len(raw), C.byref(self._m)))
        nc, nf, nr, uh = C.c_int(), C.c_int(), C.c_int(), C.c_int()
        check(lib().daspmm_model_info(self._m, C.byref(nc), C.byref(nf), C.byref(nr), C.byref(uh)))
        self.num_classes, self.num_features, self.num_rounds = nc.value, nf.value, nr.value
        self.uses_hardware = bool(uh.value)

    def close(self):
        if self._m:
            lib().daspmm_model_destroy(self._m)
            self._m = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def load_selector(text_or_stream) -> SelectorModel:
    text = text_or_stream if isinstance(text_or_stream, str) else text_or_stream.read()
    return SelectorModel(text)


def predict_kernel(model: SelectorModel, f: FeatureVector) -> KernelId:
    """selector.hpp:62-65 (host evaluation in the reference's arithmetic)."""
    k = C.c_int()
    hw = -1 if f.hardware_id is None else int(f.hardware_id)
    check(lib().daspmm_model_predict_host(model._m, f.nnz, f.mat_size, f.std_row, f.n_cols, hw,
                                          C.byref(k)))
    return KernelId.from_index(k.value)


def select_device(a: DeviceCsr, model: SelectorModel, n_cols: int, out, hw: int = -1,
                  stream=None):
    """Device selector: writes the kernel id into ``out`` (torch int32 on the GPU)."""
    check(lib().daspmm_select(a._h, model._m, n_cols, hw, out.data_ptr(), _stream_ptr(stream)))
    return out


def spmm_selected(a: DeviceCsr, model: SelectorModel, B, C_out, b_layout=Layout.RowMajor,
                  W: int = 8, hw: int = -1, exact: bool = False, kernel_out=None, stream=None,
                  reselect: bool = False, convert_layout: bool = False):
    """DA-SpMM: device selector + on-device dispatch (graph SWITCH node). Once the
    device has published its choice for (matrix, model, N, hw), calls launch the chosen
    kernel directly; ``reselect`` forces the selector + SWITCH path on this call. A choice
    that needs the other layout of B runs its layout twin on B as given, or converts B
    first with ``convert_layout`` (the reference's spmm_auto_layout)."""
    b_layout = Layout(b_layout)
    n = _check_operands(a, B, C_out, b_layout, "spmm_selected")
    if kernel_out is not None and (not kernel_out.is_cuda or str(kernel_out.dtype) != "torch.int32"):
        raise InvalidArgument(_lib.ERR_INVALID_ARG, "spmm_selected: kernel_out must be a CUDA int32 tensor")
    kp = kernel_out.data_ptr() if kernel_out is not None else None
    flags = (_lib.EXACT if exact else 0) | (_lib.RESELECT if reselect else 0) | \
        (_lib.CONVERT_LAYOUT if convert_layout else 0)
    check(lib().daspmm_spmm_selected(a._h, model._m, hw, B.data_ptr(), int(b_layout), _ld(B), n,
                                     C_out.data_ptr(), _ld(C_out), W, flags, kp,
                                     _stream_ptr(stream)))
    return C_out


class SpmmBatch:
    """Many independent DA-SpMM calls launched as ONE CUDA graph.

    ``calls`` is a list of (DeviceCsr, B, C_out) (row-major, as spmm_selected). Each call
    runs once eagerly so the device publishes its selection; the batch is then captured
    (only the chosen kernels' launches, EB prologues included) and every ``run()`` is one
    graph launch — the per-call host path and launch latency are paid once per batch
    (small matrices: a few microseconds of kernel each). The calls are captured on
    ``branches`` parallel graph branches (forked from and joined to the capture stream),
    so small calls that each fill a fraction of the 148 SMs run side by side; calls that
    write the same C stay on one branch, in list order. Operands are bound at capture:
    refill the same B / C tensors between runs."""

    def __init__(self, calls, model: "SelectorModel", W: int = 8, hw: int = -1,
                 branches: int = 8):
        import torch

        self.calls = list(calls)
        for d, B, Cc in self.calls:
            spmm_selected(d, model, B, Cc, W=W, hw=hw)
        torch.cuda.synchronize()
        for d, B, Cc in self.calls:  # decisions are published: the direct launches
            spmm_selected(d, model, B, Cc, W=W, hw=hw)
        torch.cuda.synchronize()
        nb = max(1, min(int(branches), len(self.calls)))
        owner = {}  # C address -> branch, so writes to one C keep their order
        lanes = [[] for _ in range(nb)]
        for i, (d, B, Cc) in enumerate(self.calls):
            b = owner.setdefault(Cc.data_ptr(), len(owner) % nb)
            lanes[b].append((d, B, Cc))
        self.branches = sum(1 for ln in lanes if ln)
        self.graph = torch.cuda.CUDAGraph()
        side = torch.cuda.Stream()
        forks = [torch.cuda.Stream() for _ in range(nb)]
        side.wait_stream(torch.cuda.current_stream())
        with torch.cuda.graph(self.graph, stream=side):
            for f, ln in zip(forks, lanes):
                if not ln:
                    continue
                f.wait_stream(side)
                for d, B, Cc in ln:
                    spmm_selected(d, model, B, Cc, W=W, hw=hw, stream=f)
            for f, ln in zip(forks, lanes):
                if ln:
                    side.wait_stream(f)
        torch.cuda.current_stream().wait_stream(side)

    def run(self):
        self.graph.replay()


def selected_cache_info(a: DeviceCsr):
    """(instantiated graphs, retired graphs awaiting completion, known decisions) of the
    handle's DA-SpMM cache (daspmm_selected_cache_info)."""
    g, r, d = C.c_int64(), C.c_int64(), C.c_int64()
    check(lib().daspmm_selected_cache_info(a._h, C.byref(g), C.byref(r), C.byref(d)))
    return g.value, r.value, d.value


# ------------------------------------------------------------------ tolerance
class Tolerance:
    """spmm.hpp:283-295."""
    rtol = {np.dtype(np.float64): 1e-10, np.dtype(np.float32): 1e-3}
    atol = {np.dtype(np.float64): 1e-12, np.dtype(np.float32): 1e-6}


def tolerance_equal(y: DenseMatrix, ref: DenseMatrix, rtol=None, atol=None) -> bool:
    """spmm.hpp:298-309."""
    if y.num_rows != ref.num_rows or y.num_cols != ref.num_cols:
        return False
    rtol = Tolerance.rtol[y.dtype] if rtol is None else rtol
    atol = Tolerance.atol[y.dtype] if atol is None else atol
    a = y.logical().astype(np.float64)
    b = ref.logical().astype(np.float64)
    return bool(np.all(np.abs(a - b) <= atol + rtol * np.abs(b)))
