"""Matrix Market ingestion + reorder pipeline (SPEC.md:39-47,
:96-133): SPEC examples, C++ (liblrspike.so) vs the checker, properties.  CPU only."""
import os
import tempfile

import numpy as np
import pytest
import scipy.sparse as sp

from oracle import reorder_oracle as R
from paper_2504_11167_b200 import api, configs, reorder
from paper_2504_11167_b200.configs import Csr


def _csr(S):
    S = sp.csr_matrix(S)
    S.sort_indices()
    return Csr(S.shape[0], S.indptr.astype(np.int64), S.indices.astype(np.int64),
               S.data.astype(np.float64))


def _sp(a: Csr):
    return sp.csr_matrix((a.values, a.col_idx, a.row_ptr), shape=(a.n, a.n))


def _write(text):
    fd, path = tempfile.mkstemp(suffix=".mtx")
    with os.fdopen(fd, "w") as f:
        f.write(text)
    return path


def test_read_identity_and_symmetric_expansion():
    p = _write("%%MatrixMarket matrix coordinate real general\n% c\n2 2 2\n1 1 1.0\n2 2 1.0\n")
    a = reorder.read_matrix_market(p)
    assert a.n == 2 and a.nnz == 2 and np.array_equal(_sp(a).toarray(), np.eye(2))
    p = _write("%%MatrixMarket matrix coordinate real symmetric\n2 2 3\n1 1 2\n2 1 1\n2 2 2\n")
    a = reorder.read_matrix_market(p)
    assert a.nnz == 4 and np.array_equal(_sp(a).toarray(), [[2, 1], [1, 2]])
    assert np.array_equal(_sp(a).toarray(), R.read_matrix_market(p).toarray())


def test_read_errors_carry_line_numbers():
    p = _write("%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1.0\nx y z\n")
    with pytest.raises(api.ParseError) as e:
        reorder.read_matrix_market(p)
    assert e.value.line == 4
    p = _write("%%MatrixMarket matrix coordinate complex general\n1 1 1\n1 1 1 0\n")
    with pytest.raises(api.UnsupportedFieldError):
        reorder.read_matrix_market(p)
    p = _write("%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1.0\n")
    with pytest.raises(api.ParseError):
        reorder.read_matrix_market(p)


def test_write_read_roundtrip_bit_exact_and_duplicates_summed():
    S = sp.random(60, 60, density=0.1, random_state=np.random.default_rng(2), format="csr")
    S = S + sp.eye(60)
    a = _csr(S)
    fd, path = tempfile.mkstemp(suffix=".mtx")
    os.close(fd)
    reorder.write_matrix_market(path, a)
    b = reorder.read_matrix_market(path)
    assert np.array_equal(a.row_ptr, b.row_ptr) and np.array_equal(a.col_idx, b.col_idx)
    assert np.array_equal(a.values, b.values)
    p = _write("%%MatrixMarket matrix coordinate real general\n2 2 3\n1 1 1.5\n1 1 2.5\n2 2 1\n")
    assert reorder.read_matrix_market(p).values[0] == 4.0


def test_strip_disconnected():
    a, rem = reorder.strip_disconnected(_csr(sp.diags([1.0, 2.0, 3.0])))
    assert a.n == 0 and list(rem) == [0, 1, 2]
    T = sp.diags([-1.0, 2.0, -1.0], [-1, 0, 1], shape=(6, 6))
    a, rem = reorder.strip_disconnected(_csr(T))
    assert a.n == 6 and len(rem) == 0
    M = sp.block_diag([T, sp.diags([5.0, 6.0])]).tocsr()
    a, rem = reorder.strip_disconnected(_csr(M))
    B, rem_o = R.strip_disconnected(M)
    assert list(rem) == list(rem_o) == [6, 7]
    assert np.array_equal(_sp(a).toarray(), B.toarray())


def test_diagonal_scale():
    a, d = reorder.diagonal_scale(_csr(sp.diags([4.0, 9.0])))
    assert np.allclose(_sp(a).toarray(), np.eye(2), atol=0) and np.allclose(d, [0.5, 1 / 3])
    rng = np.random.default_rng(1)
    X = rng.standard_normal((10, 10))
    S = sp.csr_matrix(X @ X.T + 10 * np.eye(10))
    a, d = reorder.diagonal_scale(_csr(S))
    assert np.max(np.abs(np.abs(_sp(a).diagonal()) - 1)) <= 1e-14
    B, s = R.diagonal_scale(S)
    assert np.array_equal(d, s)
    a2, _ = reorder.diagonal_scale(a)
    assert np.max(np.abs(_sp(a2).toarray() - _sp(a).toarray())) <= 1e-14  # idempotent
    with pytest.raises(api.SingularScalingError) as e:
        reorder.diagonal_scale(_csr(sp.csr_matrix(np.array([[1.0, 1.0], [1.0, 0.0]]))))
    assert e.value.row == 1


def test_rcm_examples_and_parity_with_the_checker():
    T = sp.diags([-1.0, 2.0, -1.0], [-1, 0, 1], shape=(30, 30)).tocsr()
    f = reorder.rcm_ordering(_csr(T))
    assert R.bandwidth(R.apply_permutation(T, f, f)) <= 1
    g = 8
    L1 = sp.diags([-1.0, 2.0, -1.0], [-1, 0, 1], shape=(g, g))
    L = (sp.kron(sp.eye(g), L1) + sp.kron(L1, sp.eye(g))).tocsr()
    rng = np.random.default_rng(0)
    shuffle = rng.permutation(g * g)
    Ls = R.apply_permutation(L, shuffle, shuffle)
    f = reorder.rcm_ordering(_csr(Ls))
    assert sorted(f) == list(range(g * g))
    assert R.bandwidth(R.apply_permutation(Ls, f, f)) <= g
    assert np.array_equal(f, R.rcm_ordering(Ls))
    for seed in range(5):  # random nonsymmetric patterns with several components
        S = sp.random(200, 200, density=0.01, random_state=np.random.default_rng(seed),
                      format="csr") + sp.eye(200)
        assert np.array_equal(reorder.rcm_ordering(_csr(S)), R.rcm_ordering(S))


def test_apply_permutation_and_pipeline_on_a_config():
    S = configs.make_config("c1", 24 / 256).matrix.to_scipy()
    n = S.shape[0]
    rng = np.random.default_rng(3)
    p = rng.permutation(n)
    a = reorder.apply_permutation(_csr(S), p, p)
    assert np.array_equal(_sp(a).toarray(), R.apply_permutation(S, p, p).toarray())
    rev = np.arange(n)[::-1].copy()
    twice = reorder.apply_permutation(reorder.apply_permutation(_csr(S), rev, rev), rev, rev)
    assert np.array_equal(_sp(twice).toarray(), S.toarray())
    # strip + scale + RCM restores a narrow band of a shuffled 2D Laplacian
    shuffled = reorder.apply_permutation(_csr(S), p, p)
    b, _ = reorder.strip_disconnected(shuffled)
    b, _ = reorder.diagonal_scale(b)
    f = reorder.rcm_ordering(b)
    c = reorder.apply_permutation(b, f, f)
    assert R.bandwidth(_sp(c)) < n // 4
    assert api.CsrMatrix  # the reordered matrix feeds the GPU solver unchanged (CSR)


def test_cli_reorder_restores_the_band(tmp_path):
    from paper_2504_11167_b200 import cli

    S = configs.make_config("c1", 24 / 256).matrix.to_scipy()
    p = np.random.default_rng(5).permutation(S.shape[0])
    a = reorder.apply_permutation(_csr(S), p, p)
    src, dst, rep = tmp_path / "a.mtx", tmp_path / "b.mtx", tmp_path / "r.json"
    reorder.write_matrix_market(str(src), a)
    assert cli.main(["reorder", "--in", str(src), "--out", str(dst), "--report", str(rep)]) == 0
    import json

    r = json.load(open(rep))
    assert r["after"]["k"] < r["before"]["k"] and r["removed"] == 0
    assert reorder.read_matrix_market(str(dst)).n == S.shape[0]


def test_io_library_exports_every_declared_symbol():
    import ctypes
    import re

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    src = open(os.path.join(root, "include", "lrspike_io.h")).read()
    syms = sorted(set(re.findall(r"LRS_API\s+[\w\s\*]+?\b(lrs_\w+)\s*\(", src)))
    assert len(syms) >= 8
    lib = reorder.lib()
    for s in syms:
        assert hasattr(lib, s), s
