"""Inputs that drive the failure branches of SPEC.md (shared by the oracle and GPU tests).

ill_conditioned_interface(retry_succeeds): p = 2 partitions of m rows.  Each block is
tridiagonal in its interior but its k boundary rows are a decoupled diagonal, so the spikes
are exactly T_0 = [0; D^-1 B], W_1 = [D^-1 C; 0] with B = diag(b), C = diag(c): the rank-r
spike directions are the axes of the r largest entries of b (u_{T,b}) and of c (v_W), and
the interface matrix K = v_W u_{T,b} is rank-deficient -- cond_1 > 1e12
 -- whenever those axis sets share some but not all axes.
  retry_succeeds=True  (k = 4, n_svd = 2): b, c top-2 share one axis -> singular; after the
                       r-halving both top-1 axes coincide -> K = 1 x 1, fine.
  retry_succeeds=False (k = 8, n_svd = 4, rank-3 couplings): singular at r = 4 (one sigma
                       collapses; the signal block of K has rank 1) and at r = 2 (the top-2
                       axes share one) -> IllConditionedInterfaceError(0, cond).

rank_deficient_coupling(): the c1 structure (2-D 5-point Laplacian, 48 x 48, P = 4) with the
couplings between partitions cut down to 3 grid points, so every spike has rank 3 < n_svd
= 8: sigma_4..8 collapse below 1e-14 sigma_1, the flag is raised and the
solve still converges.
"""
import numpy as np

from paper_2504_11167_b200.configs import Csr


def _csr(n, rows, cols, vals):
    import scipy.sparse as sp

    A = sp.csr_matrix((vals, (rows, cols)), shape=(n, n))
    A.sum_duplicates()
    A.sort_indices()
    return Csr(n, A.indptr.astype(np.int64), A.indices.astype(np.int64), A.data.astype(np.float64))


def ill_conditioned_interface(retry_succeeds: bool, m: int = 40):
    if retry_succeeds:
        k, bv, cv = 4, [1.0, 2.0, 0.0, 0.0], [0.0, 2.0, 1.0, 0.0]
    else:
        # rank 3 couplings: at r = 4 one sigma collapses and the 3 x 3 signal block of K
        # has rank 1 (axes {0,1,2} vs {1,4,5}); at r = 2 (l = 3, exact) {0,1} vs {1,4}
        k = 8
        bv = [8.0, 7.0, 6.0, 0.0, 0.0, 0.0, 0.0, 0.0]
        cv = [0.0, 8.0, 0.0, 0.0, 7.0, 6.0, 0.0, 0.0]
    n = 2 * m
    r, c, v = [], [], []

    def add(i, j, a):
        r.append(i)
        c.append(j)
        v.append(a)

    for part in range(2):
        o = part * m
        lo_int, hi_int = (o, o + m - k) if part == 0 else (o + k, o + m)
        for i in range(o, o + m):
            add(i, i, 4.0)
            if lo_int <= i < hi_int:  # interior: tridiagonal
                if i - 1 >= lo_int:
                    add(i, i - 1, -1.0)
                if i + 1 < hi_int:
                    add(i, i + 1, -1.0)
    for t in range(k):
        if bv[t]:  # B_0: rows m-k..m-1 (bottom of partition 0), cols m..m+k-1
            add(m - k + t, m + t, bv[t])
        if cv[t]:  # C_1: rows m..m+k-1, cols m-k..m-1
            add(m + t, m - k + t, cv[t])
    return _csr(n, np.array(r), np.array(c), np.array(v)), k


def rank_deficient_coupling(g: int = 48, P: int = 4, keep: int = 3):
    from paper_2504_11167_b200 import configs

    A = configs.poisson2d(g, 1e-2).to_scipy().tolil()
    n = g * g
    size = n // P
    for q in range(1, P):
        row0 = q * size  # first row of partition q: grid line q*size/g
        for x in range(g):
            if x < keep:
                continue
            i, j = row0 + x, row0 - g + x  # the vertical edge across the cut
            A[i, j] = 0.0
            A[j, i] = 0.0
    A = A.tocsr()
    A.eliminate_zeros()
    return Csr(n, A.indptr.astype(np.int64), A.indices.astype(np.int64), A.data), g
