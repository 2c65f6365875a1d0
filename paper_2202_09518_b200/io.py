"""Matrix files of the reference's module boundary (include/oocnmf/io.hpp): PDN1 binary and
Matrix Market, read and written by the library's C++ host core (``csrc/io.cpp``).

``dtype="f32"`` writes PDN1 dtype 1 (the B200 extension in the byte the reference reserves):
half the bytes, and dense windows land directly in the f32 buffers the GPU path uploads.
"""
from __future__ import annotations

import ctypes as C
from typing import Union

import numpy as np

from . import _capi
from .nmf import CsrMatrix, ShapeError, _p, check

Matrix = Union[np.ndarray, CsrMatrix]


def _b(path) -> bytes:
    return str(path).encode()


class Pdn1File:
    """Random-access reader over a PDN1 file (reference Pdn1File, io.hpp:40-66)."""

    def __init__(self, path):
        self.path = str(path)
        kind, dtype = C.c_int32(), C.c_int32()
        rows, cols, nnz = C.c_uint64(), C.c_uint64(), C.c_uint64()
        check(_capi.lib().oocnmf_pdn1_info(_b(path), C.byref(kind), C.byref(dtype), C.byref(rows), C.byref(cols),
                                           C.byref(nnz)))
        self.kind, self.dtype = int(kind.value), int(dtype.value)
        self.rows, self.cols, self.nnz = int(rows.value), int(cols.value), int(nnz.value)

    def is_dense(self) -> bool:
        return self.kind == 0

    def read_dense_window(self, r0, r1, c0, c1, dtype=np.float64) -> np.ndarray:
        out = np.empty((r1 - r0, c1 - c0), dtype)
        fn = _capi.lib().oocnmf_pdn1_read_dense_f32 if dtype == np.float32 else _capi.lib().oocnmf_pdn1_read_dense
        check(fn(_b(self.path), r0, r1, c0, c1, _p(out, C.c_float if dtype == np.float32 else C.c_double)))
        return out

    def read_csr_rows(self, r0, r1) -> CsrMatrix:
        nnz = C.c_uint64()
        check(_capi.lib().oocnmf_pdn1_csr_rows_nnz(_b(self.path), r0, r1, C.byref(nnz)))
        rp = np.empty(r1 - r0 + 1, np.uint64)
        ci = np.empty(nnz.value, np.uint64)
        v = np.empty(nnz.value)
        check(_capi.lib().oocnmf_pdn1_read_csr_rows(_b(self.path), r0, r1, _p(rp, C.c_uint64), _p(ci, C.c_uint64),
                                                    _p(v, C.c_double)))
        return CsrMatrix(r1 - r0, self.cols, rp, ci, v)


def read_pdn1(path) -> Matrix:
    f = Pdn1File(path)
    return f.read_dense_window(0, f.rows, 0, f.cols) if f.is_dense() else f.read_csr_rows(0, f.rows)


def write_pdn1(path, a: Matrix, dtype: str = "f64") -> None:
    if dtype not in ("f64", "f32"):
        raise ShapeError("write_pdn1: dtype must be 'f64' or 'f32'")
    code = 1 if dtype == "f32" else 0
    lib = _capi.lib()
    if isinstance(a, CsrMatrix):
        check(lib.oocnmf_pdn1_write_csr(_b(path), a.rows, a.cols, _p(a.row_ptr, C.c_uint64), _p(a.col_idx, C.c_uint64),
                                        _p(a.values, C.c_double), code))
        return
    a = np.asarray(a)
    if a.ndim != 2:
        raise ShapeError("write_pdn1: 2-D input required")
    if a.dtype == np.float32 and code == 1:
        a = np.ascontiguousarray(a)
        check(lib.oocnmf_pdn1_write_dense_f32(_b(path), _p(a, C.c_float), a.shape[0], a.shape[1]))
    else:
        a = np.ascontiguousarray(a, np.float64)
        check(lib.oocnmf_pdn1_write_dense(_b(path), _p(a, C.c_double), a.shape[0], a.shape[1], code))


def read_mtx(path) -> Matrix:
    kind, rows, cols, nnz = C.c_int32(), C.c_uint64(), C.c_uint64(), C.c_uint64()
    lib = _capi.lib()
    check(lib.oocnmf_mtx_info(_b(path), C.byref(kind), C.byref(rows), C.byref(cols), C.byref(nnz)))
    m, n = int(rows.value), int(cols.value)
    if kind.value == 0:
        d = np.empty((m, n))
        check(lib.oocnmf_mtx_read(_b(path), _p(d, C.c_double), None, None, None))
        return d
    rp, ci, v = np.empty(m + 1, np.uint64), np.empty(nnz.value, np.uint64), np.empty(nnz.value)
    check(lib.oocnmf_mtx_read(_b(path), None, _p(rp, C.c_uint64), _p(ci, C.c_uint64), _p(v, C.c_double)))
    return CsrMatrix(m, n, rp, ci, v)


def write_mtx(path, a: Matrix) -> None:
    lib = _capi.lib()
    if isinstance(a, CsrMatrix):
        check(lib.oocnmf_mtx_write_csr(_b(path), a.rows, a.cols, _p(a.row_ptr, C.c_uint64), _p(a.col_idx, C.c_uint64),
                                       _p(a.values, C.c_double)))
    else:
        a = np.ascontiguousarray(a, np.float64)
        check(lib.oocnmf_mtx_write_dense(_b(path), _p(a, C.c_double), a.shape[0], a.shape[1]))


def read_matrix(path) -> Matrix:
    """Dispatch on the extension: .mtx -> Matrix Market, anything else -> PDN1."""
    return read_mtx(path) if str(path).endswith(".mtx") else read_pdn1(path)
