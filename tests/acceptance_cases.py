"""Inputs of SPEC acceptance criteria 8 and 10, shared by the oracle
suite and the GPU tests.

Criterion 8 asks for the condition-number trend on Sherman5 "or a seeded synthetic of
matching size": Sherman5 is not available offline, so the stand-in is a 2D convection-
diffusion operator on a 42 x 39 grid (n = 1638, the size SPEC.md:179 / :615 quote,
half-bandwidth 42, central convection 0.3) partitioned in p = 3.  Criterion 10 uses the
oracle suite's random banded matrices with dominance factor d."""
import numpy as np
import scipy.sparse as sp

from paper_2504_11167_b200.configs import Csr


def convection_diffusion_2d(nx: int = 42, ny: int = 39, beta: float = 0.3) -> sp.csr_matrix:
    rows, cols, vals = [], [], []
    for j in range(ny):
        for i in range(nx):
            r = j * nx + i
            rows.append(r)
            cols.append(r)
            vals.append(4.0)
            for di, dj, c in ((1, 0, -1.0 + beta), (-1, 0, -1.0 - beta), (0, 1, -1.0), (0, -1, -1.0)):
                ii, jj = i + di, j + dj
                if 0 <= ii < nx and 0 <= jj < ny:
                    rows.append(r)
                    cols.append(jj * nx + ii)
                    vals.append(c)
    n = nx * ny
    return sp.csr_matrix((vals, (rows, cols)), shape=(n, n))


def banded(n, k, seed, dom=4.0):
    """The oracle suite's random banded matrix (tests/test_oracle.py::banded)."""
    rng = np.random.default_rng(seed)
    diags, offs = [], []
    for d in range(1, k + 1):
        diags += [rng.uniform(-1, 1, n - d), rng.uniform(-1, 1, n - d)]
        offs += [d, -d]
    M = sp.diags(diags, offs, shape=(n, n)).tocsr()
    rs = np.maximum(np.abs(M).sum(1).A1, np.abs(M).sum(0).A1)
    return (M + sp.diags(dom * rs + 1.0)).tocsr()


def to_csr(A: sp.csr_matrix) -> Csr:
    A = A.tocsr()
    A.sort_indices()
    return Csr(A.shape[0], A.indptr.astype(np.int64), A.indices.astype(np.int64), A.data.copy())


def cond2(M: np.ndarray) -> float:
    s = np.linalg.svd(M, compute_uv=False)
    return float(s[0] / s[-1])


ACC8_RANKS = (0, 4, 8, 16)
