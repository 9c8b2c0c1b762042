"""The INT8-sliced (Ozaki) two-step LU update on the tcgen05 tensor cores (csrc/lu_i8.cu)
against the FP64 DMMA update and the oracle.  Tolerances: factor tiles within 1e-12 of
the DMMA factors (relative to the partition's largest tile entry -- the same bar as the
DMMA-vs-LAPACK kernel parity), solves at the north_star bars."""
import os

import numpy as np
import pytest

from oracle import lrspike_oracle as O
from paper_2504_11167_b200 import api, configs
from paper_2504_11167_b200.configs import Csr

pytestmark = pytest.mark.gpu


def _factor(ctx, csr, cfg, i8, quad=False, two_sm=None, sym=None):
    old = {k: os.environ.get(k) for k in ("LRS_LU_I8", "LRS_LU_QUAD", "LRS_I8_2SM", "LRS_LU_SYM")}
    os.environ["LRS_LU_I8"] = "1" if i8 else "0"
    os.environ["LRS_LU_QUAD"] = "1" if quad else "0"
    if two_sm is not None:
        os.environ["LRS_I8_2SM"] = "1" if two_sm else "0"
    if sym is not None:
        os.environ["LRS_LU_SYM"] = "1" if sym else "0"
    try:
        A = api.CsrMatrix.from_csr(ctx, csr)
        return api.factorize(ctx, A, api.SolverConfig(variant="BJ", p=cfg.P, k=cfg.b, n_svd=0))
    finally:
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def _compare(ctx, csr, cfg, quad=False):
    F8 = _factor(ctx, csr, cfg, True, quad)
    F64 = _factor(ctx, csr, cfg, False)
    assert F8.info["lu_int8"] == 1 and F64.info["lu_int8"] == 0
    if not F8.info["pivoted"]:
        assert F8.info["lu_pairs"] == (4 if quad else 2)
    worst = 0.0
    for i in range(cfg.P):
        a, b = F8.tiles(i), F64.tiles(i)
        worst = max(worst, float(np.max(np.abs(a - b)) / np.max(np.abs(b))))
    return worst


@pytest.mark.parametrize("name,scale,quad", [("c2", 0.5, False), ("c3", 24 / 96, False),
                                             ("c4", 0.05, False), ("c2", 0.5, True)])
def test_int8_2sm_update_bitwise(ctx, name, scale, quad):
    """The 2-SM bulk update (cta_group::2, M = 256: a CTA pair shares the B slices) forms
    the same integer products and the same FP64 epilogue as the 1-SM kernel: the factors
    are bitwise identical, including an odd last row pair (c3 at 24^3: 3 bulk rows)."""
    cfg = configs.make_config(name, scale)
    F2 = _factor(ctx, cfg.system(0), cfg, True, quad, two_sm=True, sym=False)
    F1 = _factor(ctx, cfg.system(0), cfg, True, quad, two_sm=False, sym=False)
    assert F2.info["lu_int8"] == 1
    for i in range(cfg.P):
        assert np.array_equal(F2.tiles(i), F1.tiles(i)), i


def test_i8_peak_positive(ctx):
    tops = ctx.i8_peak_tops()
    assert 500.0 < tops < 20000.0


@pytest.mark.parametrize("name,scale", [("c2", 0.5), ("c3", 24 / 96), ("c4", 0.05), ("c5", 0.5),
                                        ("c5", 0.3)])
def test_int8_update_matches_dmma(ctx, name, scale):
    """c5: complex128 shifted systems z I - A, the realified update (A' = [Ar Ai], B'_re =
    [Br; -Bi], B'_im = [Bi; Br]) against the 3M complex DMMA update."""
    cfg = configs.make_config(name, scale)
    assert -(-cfg.b // 128) >= 3  # the pair schedule (and so the INT8 update) is in play
    assert _compare(ctx, cfg.system(0), cfg) <= 1e-12


@pytest.mark.parametrize("name,scale", [("c2", 0.5), ("c4", 0.05)])
def test_int8_quad_update_matches_dmma(ctx, name, scale):
    """LRS_LU_QUAD=1: four steps (K = 512) per INT8 update, DMMA look-ahead inside the quad."""
    cfg = configs.make_config(name, scale)
    assert -(-cfg.b // 128) >= 8
    assert _compare(ctx, cfg.system(0), cfg, quad=True) <= 1e-12


@pytest.mark.parametrize("name,scale,quad", [("c3", 24 / 96, False), ("c3", 32 / 96, False),
                                             ("c3", 32 / 96, True), ("c3", 40 / 96, True),
                                             ("c5", 0.5, False), ("c5", 0.3, False)])
def test_symmetric_schedule_matches_full_lu(ctx, name, scale, quad):
    """Symmetric blocks (c3: A == A^T bitwise): the LU forms the lower trailing tiles only
    and takes each U panel from its L panel, U_KJ = diag(U_KK) L_JK^T.  Every band tile
    (L, U and the diagonal inverses) within 1e-12 of the full-schedule INT8 LU and of the
    DMMA LU, relative to the partition's largest entry; pairs and quads.  c5: the complex
    symmetric (not Hermitian) shifted systems z I - A, realified INT8 update."""
    cfg = configs.make_config(name, scale)
    assert -(-cfg.b // 128) >= (8 if quad else 3)
    Fs = _factor(ctx, cfg.system(0), cfg, True, quad, sym=True)
    Ff = _factor(ctx, cfg.system(0), cfg, True, quad, sym=False)
    Fd = _factor(ctx, cfg.system(0), cfg, False, sym=False)
    assert Fs.info["lu_sym"] == 1 and Ff.info["lu_sym"] == 0 and Fd.info["lu_sym"] == 0
    assert Fs.info["lu_int8"] == 1 and not Fs.info["pivoted"]
    assert Fs.info["lu_pairs"] == (4 if quad else 2)
    # the DMMA two-step kinds take the symmetric schedule too (real blocks; LRS_LU_I8=0)
    Fds = _factor(ctx, cfg.system(0), cfg, False, sym=True) if name == "c3" else None
    if Fds is not None:
        assert Fds.info["lu_sym"] == 1 and Fds.info["lu_int8"] == 0
    for i in range(cfg.P):
        a, b, d = Fs.tiles(i), Ff.tiles(i), Fd.tiles(i)
        sc = np.max(np.abs(d))
        assert np.max(np.abs(a - b)) / sc <= 1e-12, i
        assert np.max(np.abs(a - d)) / sc <= 1e-12, i
        if Fds is not None:
            assert np.max(np.abs(Fds.tiles(i) - d)) / sc <= 1e-12, i


def test_symmetric_schedule_only_for_symmetric_blocks(ctx):
    """c2 (convection: A != A^T) and a c3 matrix with one perturbed entry keep the full LU."""
    cfg = configs.make_config("c2", 0.5)
    assert _factor(ctx, cfg.system(0), cfg, True).info["lu_sym"] == 0
    cfg = configs.make_config("c3", 24 / 96)
    m = cfg.matrix
    vals = m.values.copy()
    j = int(np.flatnonzero(m.col_idx[: m.row_ptr[1]] != 0)[0])  # an off-diagonal of row 0
    vals[j] *= 1.0 + 2.0 ** -40
    F = _factor(ctx, Csr(m.n, m.row_ptr, m.col_idx, vals), cfg, True)
    assert F.info["lu_sym"] == 0 and F.info["lu_int8"] == 1


@pytest.mark.parametrize("e", [-300, 300])
def test_int8_update_far_exponents(ctx, e):
    """Uniformly scaled matrices: the per-row / per-column exponents carry the scale."""
    cfg = configs.make_config("c2", 0.5)
    m = cfg.matrix
    scaled = Csr(m.n, m.row_ptr, m.col_idx, m.values * 2.0 ** e)
    assert _compare(ctx, scaled, cfg) <= 1e-12


def test_int8_graded_rows(ctx):
    """Rows graded over 2^+-20 (a slowly varying diagonal scaling keeps dominance)."""
    cfg = configs.make_config("c2", 0.5)
    S = cfg.matrix.to_scipy().tocsr()
    n = S.shape[0]
    d = 2.0 ** np.round(20 * np.sin(np.arange(n) / 3000.0))
    import scipy.sparse as sp
    G = (sp.diags(d) @ S @ sp.diags(1.0 / d)).tocsr()
    G.sort_indices()
    csr = Csr(n, G.indptr.astype(np.int64), G.indices.astype(np.int64), G.data)
    assert _compare(ctx, csr, cfg) <= 1e-12


def test_int8_solve_parity_with_oracle(ctx):
    cfg = configs.make_config("c2", 0.5)
    S = cfg.matrix.to_scipy()
    A = api.CsrMatrix.from_csr(ctx, cfg.matrix)
    scfg = api.SolverConfig(p=cfg.P, k=cfg.b, n_svd=cfg.r, seed=cfg.seed)
    it = api.IterConfig(tol=cfg.tol, method=cfg.method, restart=cfg.m or 30, max_iters=500)
    F = api.factorize(ctx, A, scfg)
    assert F.info["lu_int8"] == 1
    x, rep, _ = api.solve(A, np.asfortranarray(cfg.rhs), it=it, F=F)
    ocfg = O.SolverConfig(p=cfg.P, k=cfg.b, n_svd=cfg.r, seed=cfg.seed)
    xo, ro, _ = O.solve(S, cfg.rhs, ocfg, O.IterConfig(tol=cfg.tol, restart=cfg.m or 30,
                                                       max_iters=500), method=cfg.method)
    assert rep.converged and rep.residual_final <= cfg.tol
    assert abs(rep.iterations - ro.iterations) <= 2
    assert np.linalg.norm(x - xo) / np.linalg.norm(xo) <= 1e-8


# ---- componentwise backward error of the factorization (|PA - LU| <= c u |L||U|) -------
def _effective_lu(F, i, n_i):
    """Dense (L, U) of partition i as the solves apply them: off-diagonal tiles as stored,
    the diagonal tiles as the exact (long double) inverses of the stored inverses
    (the solves multiply by inv(L_II), inv(U_II) directly)."""
    tl = F.tiles(i)
    nb, wl = F.info["nb"], F.info["wl"]
    T, W = tl.shape[0], tl.shape[1]
    L = np.zeros((T * nb, T * nb), dtype=np.longdouble)
    U = np.zeros((T * nb, T * nb), dtype=np.longdouble)
    for I in range(T):
        for s in range(W):
            J = I + s - wl
            if J < 0 or J >= T:
                continue
            blk = tl[I, s].astype(np.longdouble)
            r0, c0 = I * nb, J * nb
            if J < I:
                L[r0:r0 + nb, c0:c0 + nb] = blk
            elif J > I:
                U[r0:r0 + nb, c0:c0 + nb] = blk
            else:
                L[r0:r0 + nb, c0:c0 + nb] = _tri_inv(np.tril(blk, -1) + np.eye(nb), lower=True)
                U[r0:r0 + nb, c0:c0 + nb] = _tri_inv(np.triu(blk), lower=False)
    return L[:n_i, :n_i], U[:n_i, :n_i]


def _tri_inv(M, lower):
    """Inverse of a triangular long-double matrix by substitution on the identity."""
    n = M.shape[0]
    X = np.zeros_like(M)
    E = np.eye(n, dtype=M.dtype)
    rng = range(n) if lower else range(n - 1, -1, -1)
    for r in rng:
        if lower:
            X[r] = (E[r] - M[r, :r] @ X[:r]) / M[r, r]
        else:
            X[r] = (E[r] - M[r, r + 1:] @ X[r + 1:]) / M[r, r]
    return X


def _lapack_lu(Ai):
    """Dense (L, U) of LAPACK dgbtrf (no interchanges on these blocks)."""
    fo = O.factorize_block(Ai)
    assert fo.swaps == 0
    n, kl, ku = fo.n, fo.kl, fo.ku
    L = np.eye(n, dtype=np.longdouble)
    U = np.zeros((n, n), dtype=np.longdouble)
    for j in range(n):
        lo, hi = max(0, j - ku - kl), min(n, j + kl + 1)
        q = np.arange(lo, hi)
        v = fo.ab[kl + ku + q - j, j]
        low = q > j
        L[q[low], j] = v[low]
        U[q[~low], j] = v[~low]
    return L, U


def componentwise_error(Ad, L, U, rows, sym=False):
    """Backward error of A = L U over the sampled rows, in long double (64-bit mantissa: the
    residual's own rounding is ~u/2000 of the bounds below).  Returns
      scaled  max |A - LU|_ij / (max_k |L_ik| max_k |U_kj|)   -- the row / column-scaled
              bound the INT8 digit split guarantees (entries represented to 2^-54 of
              their row / column maximum)
      cw      max |A - LU|_ij / (|L||U|)_ij over entries whose (|L||U|)_ij is within
              2^-40 of the row x column scale -- componentwise (Higham's |A - LU| <=
              gamma |L||U|); the floor drops structural zeros, where the diagonal tiles'
              stored inverses re-invert to ~1e-20 instead of 0
      buckets the componentwise maximum per band of (|L||U|)_ij / scale: [2^-10, 1],
              [2^-20, 2^-10), [2^-30, 2^-20), [2^-40, 2^-30)
    sym: factors of the symmetric schedule (U = diag(U) L^T mirrored from L, the lower
    trailing tiles formed only).  An upper entry (i, j) then carries the integer-split error
    of its mirror (j, i), whose scale is max|L_j.| max|U_.i|, so the scale of an entry is the
    larger of its own and its mirror's row x column scale."""
    Lr = L[rows]
    R = np.abs(Ad[rows].astype(np.longdouble) - Lr @ U)
    B = np.abs(Lr) @ np.abs(U)
    rowL, colU = np.abs(L).max(axis=1), np.abs(U).max(axis=0)
    scale = rowL[rows][:, None] * colU[None, :]
    if sym:
        scale = np.maximum(scale, colU[rows][:, None] * rowL[None, :])
    rel = np.where(scale > 0, B / np.where(scale > 0, scale, 1), 0)
    out = {"scaled": float(np.max(R / np.where(scale > 0, scale, 1)))}
    cw = np.where(B > 0, R / np.where(B > 0, B, 1), 0)
    m = rel >= 2.0 ** -40
    out["cw"] = float(np.max(cw[m]))
    for lo, hi, tag in ((-10, 1, "b0"), (-20, -10, "b10"), (-30, -20, "b20"), (-40, -30, "b30")):
        mm = (rel >= 2.0 ** lo) & (rel < 2.0 ** hi)
        out[tag] = float(np.max(cw[mm])) if mm.any() else None
    return out


def componentwise_report(ctx, name, scale, n_rows=48, seed=0, sym=False):
    cfg = configs.make_config(name, scale)
    S = cfg.matrix.to_scipy()
    lay = O.make_layout(S.shape[0], cfg.P, cfg.b)
    blocks = O.extract_blocks(S, lay)
    F8 = _factor(ctx, cfg.matrix, cfg, True, sym=sym)
    F64 = _factor(ctx, cfg.matrix, cfg, False)
    assert F8.info["lu_int8"] == 1 and F8.info["lu_pairs"] == 2
    assert F8.info["lu_sym"] == (1 if sym else 0)
    out = {"config": name, "scale": scale, "u": float(np.finfo(np.float64).eps / 2),
           "lu_sym": int(sym)}
    rng = np.random.default_rng(seed)
    for i in (0, cfg.P // 2):
        n_i = lay.sizes[i]
        Ad = blocks.A[i].toarray()
        # rows of the bulk-update region (row tiles >= 4 see the INT8 two-step update)
        rows = np.sort(rng.choice(np.arange(min(4 * 128, n_i - 1), n_i), size=n_rows,
                                  replace=False))
        e = {}
        for tag, LU in (("int8", _effective_lu(F8, i, n_i)), ("dmma", _effective_lu(F64, i, n_i)),
                        ("lapack", _lapack_lu(blocks.A[i]))):
            e[tag] = componentwise_error(Ad, LU[0], LU[1], rows, sym=sym and tag == "int8")
        out[f"partition{i}"] = e
    return out


@pytest.mark.parametrize("name,scale,sym", [("c3", 24 / 96, False), ("c4", 0.05, False),
                                            ("c3", 24 / 96, True)])
def test_int8_componentwise_backward_error(ctx, name, scale, sym):
    """|A_i - L U| for the INT8-sliced factors on the c3 (10^4 coefficient contrast) and c4
    (random band) structures, beside the FP64 DMMA factors and LAPACK dgbtrf.

    Measured on the B200 (profiles/r02_lu_componentwise.jsonl):
      scaled (|A - LU|_ij / (max|L_i.| max|U_.j|)): INT8 8.8e-16 - 9.7e-16, DMMA the same,
        LAPACK 5e-16 - 1.2e-15 -- the INT8 update is FP64-accurate relative to the row x
        column scale;
      componentwise (/ (|L||U|)_ij): LAPACK <= 1.5e-15; DMMA <= 2.1e-12 (its panels form
        L = A inv(U) with the explicit diagonal-tile inverses); INT8 by band of
        (|L||U|)_ij / scale: <= 8e-14 in [2^-10, 1], 6.5e-11 in [2^-20, 2^-10), 4.9e-8 in
        [2^-30, 2^-20), 1.7e-5 in [2^-40, 2^-30) -- an entry 2^-e below its row x column
        scale keeps ~54 - e bits: normwise FP64, not componentwise.
    Bars: scaled <= 32 u for all three; LAPACK componentwise <= 32 u; DMMA <= 1e-11; INT8 per
    band <= 64 2^-54 / (band floor), the digit-split bound.
    sym = True: the symmetric schedule's factors (c3 is symmetric), measured against the
    symmetrized scale (componentwise_error); sym = False forces the full schedule."""
    rep = componentwise_report(ctx, name, scale, sym=sym)
    print(rep)
    u = rep["u"]
    for key, e in rep.items():
        if not key.startswith("partition"):
            continue
        for tag in ("int8", "dmma", "lapack"):
            assert e[tag]["scaled"] <= 32 * u, (tag, rep)
        assert e["lapack"]["cw"] <= 32 * u, rep
        assert e["dmma"]["cw"] <= 1e-11, rep
        for tag, floor in (("b0", -10), ("b10", -20), ("b20", -30), ("b30", -40)):
            if e["int8"][tag] is not None:
                assert e["int8"][tag] <= 64 * 2.0 ** -54 / 2.0 ** floor, (tag, rep)
