"""Matrix Market ingestion and the reorder pipeline through the
C-ABI of liblrspike.so (include/lrspike_io.h).  Host-side structural preprocessing ahead
of the GPU solver; CSR in, CSR out (``configs.Csr``)."""
from __future__ import annotations

import ctypes
import os

import numpy as np

from . import api
from .configs import Csr

_HERE = os.path.dirname(os.path.abspath(__file__))
_lib = None
i64, f64, i32 = ctypes.c_int64, ctypes.c_double, ctypes.c_int32


class CsrHostC(ctypes.Structure):
    _fields_ = [("n_rows", i64), ("n_cols", i64), ("nnz", i64), ("row_ptr", ctypes.POINTER(i64)),
                ("col_idx", ctypes.POINTER(i64)), ("values", ctypes.POINTER(f64))]


class IoErrorC(ctypes.Structure):
    _fields_ = [("message", ctypes.c_char * 512), ("line", i64), ("row", i64)]


def lib():
    global _lib
    if _lib is None:
        api.lib()  # liblrspike.so links liblrspike_cuda.so
        path = os.path.join(_HERE, "liblrspike.so")
        if not os.path.exists(path):
            raise ImportError(f"{path} is missing: build it with `make`")
        L = ctypes.CDLL(path)
        P = ctypes.POINTER
        for name, res, args in (
                ("lrs_io_read_mm", i32, [ctypes.c_char_p, P(CsrHostC)]),
                ("lrs_io_write_mm", i32, [ctypes.c_char_p, P(CsrHostC)]),
                ("lrs_io_free", None, [P(CsrHostC)]),
                ("lrs_reorder_rcm", i32, [P(CsrHostC), P(i64)]),
                ("lrs_reorder_strip", i32, [P(CsrHostC), P(CsrHostC), P(i64), P(i64)]),
                ("lrs_reorder_scale", i32, [P(CsrHostC), P(CsrHostC), P(f64)]),
                ("lrs_reorder_permute", i32, [P(CsrHostC), P(i64), P(i64), P(CsrHostC)]),
                ("lrs_io_last_error", i32, [P(IoErrorC)])):
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def _check(st):
    if st == 0:
        return
    e = IoErrorC()
    lib().lrs_io_last_error(ctypes.byref(e))
    msg = e.message.decode(errors="replace")
    if st == 1:
        raise api.ParseError(msg, e.line)
    if st == 4:
        raise api.SingularScalingError(msg, e.row)
    cls = api._EXC.get(st, api.Error)
    raise cls(msg)


def _to_c(a: Csr):
    rp = np.ascontiguousarray(a.row_ptr, dtype=np.int64)
    ci = np.ascontiguousarray(a.col_idx, dtype=np.int64)
    va = np.ascontiguousarray(a.values, dtype=np.float64)
    ncols = getattr(a, "n_cols", a.n)
    c = CsrHostC(a.n, ncols, va.shape[0], rp.ctypes.data_as(ctypes.POINTER(i64)),
                 ci.ctypes.data_as(ctypes.POINTER(i64)), va.ctypes.data_as(ctypes.POINTER(f64)))
    return c, (rp, ci, va)


def _from_c(c: CsrHostC) -> Csr:
    n, nnz = c.n_rows, c.nnz
    out = Csr(n, np.ctypeslib.as_array(c.row_ptr, shape=(n + 1,)).copy(),
              np.ctypeslib.as_array(c.col_idx, shape=(max(nnz, 1),))[:nnz].copy(),
              np.ctypeslib.as_array(c.values, shape=(max(nnz, 1),))[:nnz].copy())
    lib().lrs_io_free(ctypes.byref(c))
    return out


def read_matrix_market(path: str) -> Csr:
    """SPEC.md:39-47."""
    c = CsrHostC()
    _check(lib().lrs_io_read_mm(path.encode(), ctypes.byref(c)))
    return _from_c(c)


def write_matrix_market(path: str, a: Csr) -> None:
    c, keep = _to_c(a)
    _check(lib().lrs_io_write_mm(path.encode(), ctypes.byref(c)))
    del keep


def rcm_ordering(a: Csr) -> np.ndarray:
    """forward[old] = new."""
    c, keep = _to_c(a)
    fwd = np.empty(a.n, dtype=np.int64)
    _check(lib().lrs_reorder_rcm(ctypes.byref(c), fwd.ctypes.data_as(ctypes.POINTER(i64))))
    del keep
    return fwd


def strip_disconnected(a: Csr):
    """(matrix on the retained indices, removed original indices)."""
    c, keep = _to_c(a)
    out = CsrHostC()
    rem = np.empty(max(a.n, 1), dtype=np.int64)
    nrem = i64()
    _check(lib().lrs_reorder_strip(ctypes.byref(c), ctypes.byref(out),
                                   rem.ctypes.data_as(ctypes.POINTER(i64)), ctypes.byref(nrem)))
    del keep
    return _from_c(out), rem[:nrem.value].copy()


def diagonal_scale(a: Csr):
    """(D A D, d) with d = |a_ii|^-1/2."""
    c, keep = _to_c(a)
    out = CsrHostC()
    d = np.empty(a.n, dtype=np.float64)
    _check(lib().lrs_reorder_scale(ctypes.byref(c), ctypes.byref(out),
                                   d.ctypes.data_as(ctypes.POINTER(f64))))
    del keep
    return _from_c(out), d


def apply_permutation(a: Csr, row_forward, col_forward) -> Csr:
    """B[row_forward[i], col_forward[j]] = A[i, j]."""
    c, keep = _to_c(a)
    rf = np.ascontiguousarray(row_forward, dtype=np.int64)
    cf = np.ascontiguousarray(col_forward, dtype=np.int64)
    out = CsrHostC()
    _check(lib().lrs_reorder_permute(ctypes.byref(c), rf.ctypes.data_as(ctypes.POINTER(i64)),
                                     cf.ctypes.data_as(ctypes.POINTER(i64)), ctypes.byref(out)))
    del keep
    return _from_c(out)
