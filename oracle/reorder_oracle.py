"""CPU restatement of the io + reorder modules -- TEST
INFRASTRUCTURE ONLY: the checker for paper_2504_11167_b200/reorder.py (C++ in
host/lrspike_reorder.cpp).  Only tests/ may import it.

Parity pinned by the SPEC examples in tests/test_reorder.py (identity / symmetric
Matrix Market files, diag(1,2,3) strip, diag(4,9) scaling, RCM on a tridiagonal and on
the 8 x 8 5-point Laplacian, reversal permutations) and cross-checked against the C++.
"""
from __future__ import annotations

from collections import deque

import numpy as np
import scipy.sparse as sp

from oracle.lrspike_oracle import Error


class ParseError(Error):
    def __init__(self, msg, line):
        super().__init__(f"{msg} (line {line})")
        self.line = line


class UnsupportedFieldError(Error):
    pass


class SingularScalingError(Error):
    def __init__(self, msg, row):
        super().__init__(msg)
        self.row = row


def read_matrix_market(path: str) -> sp.csr_matrix:
    """coordinate real / integer / pattern; general / symmetric /
    skew-symmetric expanded; duplicates summed; 0-based."""
    with open(path) as f:
        lines = f.read().split("\n")
    head = lines[0].split()
    if len(head) < 5 or head[0] != "%%MatrixMarket" or head[1].lower() != "matrix":
        raise ParseError("missing %%MatrixMarket matrix header", 1)
    fmt, field, sym = head[2].lower(), head[3].lower(), head[4].lower()
    if fmt != "coordinate":
        raise UnsupportedFieldError("only the coordinate format is supported")
    if field == "complex" or sym == "hermitian":
        raise UnsupportedFieldError("complex Matrix Market field is not supported")
    ln = 1
    size = None
    while ln < len(lines):
        s = lines[ln]
        ln += 1
        if not s or s.startswith("%"):
            continue
        size = [int(t) for t in s.split()[:3]]
        break
    if size is None:
        raise ParseError("missing size line", ln)
    nr, nc, nz = size
    r, c, v = [], [], []
    got = 0
    while got < nz and ln < len(lines):
        s = lines[ln]
        ln += 1
        if not s or s.startswith("%"):
            continue
        t = s.split()
        try:
            i, j = int(t[0]), int(t[1])
            val = 1.0 if field == "pattern" else float(t[2])
        except (ValueError, IndexError):
            raise ParseError("malformed entry", ln)
        if not (1 <= i <= nr and 1 <= j <= nc):
            raise ParseError("entry index out of range", ln)
        r.append(i - 1)
        c.append(j - 1)
        v.append(val)
        if sym != "general" and i != j:
            r.append(j - 1)
            c.append(i - 1)
            v.append(-val if sym == "skew-symmetric" else val)
        got += 1
    if got < nz:
        raise ParseError(f"expected {nz} entries, found {got}", ln + 1)
    A = sp.coo_matrix((v, (r, c)), shape=(nr, nc)).tocsr()
    A.sum_duplicates()
    A.sort_indices()
    return A


def strip_disconnected(A: sp.csr_matrix):
    """(A on the retained indices, removed indices)."""
    A = sp.csr_matrix(A)
    C = A.tocoo()
    off = C.row != C.col
    linked = np.zeros(A.shape[0], dtype=bool)
    linked[C.row[off]] = True
    linked[C.col[off]] = True
    keep = np.flatnonzero(linked)
    return A[keep][:, keep].tocsr(), np.flatnonzero(~linked)


def diagonal_scale(A: sp.csr_matrix):
    """D A D with D = diag(|a_ii|^-1/2)."""
    A = sp.csr_matrix(A)
    d = A.diagonal()
    bad = np.flatnonzero(d == 0)
    if bad.size:
        raise SingularScalingError(f"zero diagonal entry in row {bad[0]}", int(bad[0]))
    s = 1.0 / np.sqrt(np.abs(d))
    B = A.tocoo()
    B = sp.csr_matrix((s[B.row] * B.data * s[B.col], (B.row, B.col)), shape=A.shape)
    B.sort_indices()
    return B, s


def rcm_ordering(A: sp.csr_matrix) -> np.ndarray:
    """forward[old] = new.  Pattern of A + A^T without the diagonal;
    per component (by lowest vertex) a George-Liu pseudo-peripheral start (last BFS level's
    minimum (degree, index)); Cuthill-McKee visiting neighbours by (degree, index);
    the whole order reversed."""
    n = A.shape[0]
    P = (sp.csr_matrix(A) != 0).astype(np.int8)
    S = (P + P.T).tocsr()
    S.setdiag(0)
    S.eliminate_zeros()
    S.sort_indices()
    adj = [S.indices[S.indptr[i]:S.indptr[i + 1]] for i in range(n)]
    deg = np.array([len(a) for a in adj])
    key = lambda x: (deg[x], x)  # noqa: E731

    def levels(v):
        lev = {v: 0}
        comp = [v]
        h = 0
        while h < len(comp):
            u = comp[h]
            h += 1
            for w in adj[u]:
                if w not in lev:
                    lev[w] = lev[u] + 1
                    comp.append(w)
        ecc = max(lev.values())
        return ecc, [u for u in comp if lev[u] == ecc]

    placed = np.zeros(n, dtype=bool)
    order = []
    for s in range(n):
        if placed[s]:
            continue
        v = s
        ecc, last = levels(v)
        while True:
            u = min(last, key=key)
            e2, l2 = levels(u)
            if e2 <= ecc:
                break
            v, ecc, last = u, e2, l2
        q = deque([v])
        placed[v] = True
        while q:
            u = q.popleft()
            order.append(u)
            nb = sorted((w for w in adj[u] if not placed[w]), key=key)
            for w in nb:
                placed[w] = True
                q.append(w)
    order = order[::-1]
    fwd = np.empty(n, dtype=np.int64)
    fwd[np.array(order, dtype=np.int64)] = np.arange(n)
    return fwd


def apply_permutation(A: sp.csr_matrix, row_forward, col_forward) -> sp.csr_matrix:
    """B[row_forward[i], col_forward[j]] = A[i, j]."""
    C = sp.csr_matrix(A).tocoo()
    B = sp.csr_matrix((C.data, (np.asarray(row_forward)[C.row], np.asarray(col_forward)[C.col])),
                      shape=A.shape)
    B.sort_indices()
    return B


def bandwidth(A) -> int:
    C = sp.csr_matrix(A).tocoo()
    return int(np.max(np.abs(C.row - C.col))) if C.nnz else 0
