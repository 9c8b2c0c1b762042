"""BASELINE.json configurations c1..c5 and their seeded synthetic inputs.

The matrices come from the C generators in ``gen/lrs_gen.c`` (loaded through
ctypes from ``liblrs_gen.so``) so the CPU oracle and the CUDA path consume
bit-identical inputs.  ``scale`` shrinks the grid (or n
and b for c4) while keeping the structure; scaled variants are the parity
cases, the full sizes are the bench workloads.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None


class _Csr(ctypes.Structure):
    _fields_ = [
        ("n", ctypes.c_int64),
        ("nnz", ctypes.c_int64),
        ("row_ptr", ctypes.POINTER(ctypes.c_int64)),
        ("col_idx", ctypes.POINTER(ctypes.c_int64)),
        ("values", ctypes.POINTER(ctypes.c_double)),
    ]


def gen_lib():
    """Load liblrs_gen.so (built by ``make gen`` / ``__graft_entry__.build``)."""
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "liblrs_gen.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run `make -C {os.path.dirname(_HERE)}` first")
        lib = ctypes.CDLL(path)
        i64, f64, u64 = ctypes.c_int64, ctypes.c_double, ctypes.c_uint64
        P = ctypes.POINTER(_Csr)
        lib.lrs_gen_poisson2d.argtypes = [i64, f64, P]
        lib.lrs_gen_convdiff3d.argtypes = [i64, f64, P]
        lib.lrs_gen_hetero27.argtypes = [i64, u64, f64, P]
        lib.lrs_gen_randband.argtypes = [i64, i64, i64, u64, f64, P]
        lib.lrs_gen_feast_base.argtypes = [i64, u64, i64, f64, P]
        lib.lrs_gen_free.argtypes = [P]
        lib.lrs_gen_vector.argtypes = [ctypes.c_int, u64, i64, ctypes.c_void_p]
        lib.lrs_gen_omega.argtypes = [u64, i64, ctypes.c_int, i64, i64, ctypes.c_void_p]
        for f in ("lrs_gen_poisson2d", "lrs_gen_convdiff3d", "lrs_gen_hetero27",
                  "lrs_gen_randband", "lrs_gen_feast_base"):
            getattr(lib, f).restype = ctypes.c_int
        lib.lrs_gen_vector.restype = None
        lib.lrs_gen_omega.restype = None
        _LIB = lib
    return _LIB


@dataclass
class Csr:
    """Host CSR with int64 indices (the reference CsrMatrix layout,
    proj/core/include/lrspike/matrix.hpp:22-48)."""

    n: int
    row_ptr: np.ndarray
    col_idx: np.ndarray
    values: np.ndarray

    @property
    def nnz(self) -> int:
        return int(self.values.shape[0])

    def to_scipy(self):
        import scipy.sparse as sp

        return sp.csr_matrix((self.values, self.col_idx, self.row_ptr), shape=(self.n, self.n))


def _take(fn, *args) -> Csr:
    lib = gen_lib()
    m = _Csr()
    rc = fn(*args, ctypes.byref(m))
    if rc != 0:
        raise MemoryError("generator failed")
    try:
        n, nnz = m.n, m.nnz
        rp = np.ctypeslib.as_array(m.row_ptr, shape=(n + 1,)).copy()
        ci = np.ctypeslib.as_array(m.col_idx, shape=(nnz,)).copy()
        va = np.ctypeslib.as_array(m.values, shape=(nnz,)).copy()
    finally:
        lib.lrs_gen_free(ctypes.byref(m))
    return Csr(n, rp, ci, va)


def poisson2d(g: int, shift: float = 1e-2) -> Csr:
    return _take(gen_lib().lrs_gen_poisson2d, g, shift)


def convdiff3d(g: int, conv: float = 0.5) -> Csr:
    return _take(gen_lib().lrs_gen_convdiff3d, g, conv)


def hetero27(g: int, seed: int = 2, log10_range: float = 2.0) -> Csr:
    return _take(gen_lib().lrs_gen_hetero27, g, seed, log10_range)


def randband(n: int, b: int, m: int = 20, seed: int = 3, dom: float = 1.1) -> Csr:
    return _take(gen_lib().lrs_gen_randband, n, b, m, seed, dom)


def feast_base(g: int, seed: int = 4, pb: int | None = None, sigma: float = 0.1) -> Csr:
    if pb is None:
        pb = g * g
    return _take(gen_lib().lrs_gen_feast_base, g, seed, pb, sigma)


def vector(kind: str, seed: int, n: int, n_rhs: int = 1) -> np.ndarray:
    """Column-major n x n_rhs block (Fortran order) from the RHS stream."""
    k = {"uniform": 0, "normal": 1, "ones": 2}[kind]
    out = np.empty(n * n_rhs, dtype=np.float64)
    gen_lib().lrs_gen_vector(k, seed, n * n_rhs, out.ctypes.data)
    return out.reshape((n, n_rhs), order="F")


def omega(seed: int, partition: int, side: int, rows: int, cols: int) -> np.ndarray:
    """Gaussian test block of the randomized spike SVD."""
    out = np.empty(rows * cols, dtype=np.float64)
    gen_lib().lrs_gen_omega(seed, partition, side, rows, cols, out.ctypes.data)
    return out.reshape((rows, cols), order="F")


def shifted(A: Csr, z: complex) -> Csr:
    """The FEAST contour system z I - A of config c5 (complex128).
    Every row of the c5 base matrix holds its diagonal, so the pattern is unchanged."""
    vals = -A.values.astype(np.complex128)
    rows = np.repeat(np.arange(A.n), np.diff(A.row_ptr))
    vals[rows == A.col_idx] += z
    return Csr(A.n, A.row_ptr.copy(), A.col_idx.copy(), vals)


@dataclass
class Config:
    """One BASELINE.json configuration (possibly scaled down)."""

    name: str
    matrix: Csr
    rhs: np.ndarray
    b: int  # coupling half-bandwidth (SPEC k; SURVEY.md 0.1 calls it b)
    P: int
    r: int  # n_svd
    method: str  # "gmres" | "bicgstab"
    m: int  # GMRES restart length (0 for BiCGStab)
    tol: float
    seed: int
    shifts: list = field(default_factory=list)  # c5 only

    def system(self, j: int = 0) -> Csr:
        """The matrix of shift j (c5: z_j I - A, complex); the matrix itself otherwise."""
        return shifted(self.matrix, self.shifts[j]) if self.shifts else self.matrix


def make_config(name: str, scale: float = 1.0, P: int | None = None) -> Config:
    """Build config ``name`` in {c1..c5}.  ``scale`` < 1 shrinks the grid."""
    if name == "c1":
        g = max(8, int(round(256 * scale)))
        A = poisson2d(g, 1e-2)
        return Config("c1", A, vector("uniform", 0, A.n), g, P or 4, 8, "gmres", 30, 1e-8, 0)
    if name == "c2":
        g = max(6, int(round(64 * scale)))
        A = convdiff3d(g, 0.5)
        return Config("c2", A, vector("uniform", 1, A.n), g * g, P or 8, 16, "bicgstab", 0,
                      1e-8, 1)
    if name == "c3":
        g = max(6, int(round(96 * scale)))
        A = hetero27(g, 2, 2.0)
        return Config("c3", A, vector("ones", 2, A.n), g * g + g + 1, P or 8, 32, "gmres", 50,
                      1e-8, 2)
    if name == "c4":
        n = max(2000, int(round(2_000_000 * scale)))
        b = max(20, int(round(20_000 * scale)))
        A = randband(n, b, 20, 3, 1.1)
        return Config("c4", A, vector("normal", 3, A.n), b, P or 64, 64, "gmres", 50, 1e-8, 3)
    if name == "c5":
        g = max(6, int(round(80 * scale)))
        A = feast_base(g, 4, g * g, 0.1)
        shifts = [2.0 + 0.5 * np.exp(1j * np.pi * (2 * j + 1) / 8) for j in range(8)]
        return Config("c5", A, vector("uniform", 4, A.n, 16), g * g, P or 16, 32, "gmres", 40,
                      1e-10, 4, shifts)
    raise ValueError(name)
