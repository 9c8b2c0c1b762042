"""CPU tests: golden fixtures (oracle + generators), the C-ABI library exports,
the generators' structure, and the C++ drop-in API's host logic."""
import ctypes
import json
import os
import re
import subprocess

import numpy as np
import pytest

from oracle import lrspike_oracle as O
from paper_2504_11167_b200 import configs

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = os.path.join(ROOT, "tests", "golden")


def _meta():
    with open(os.path.join(GOLD, "golden.json")) as f:
        return json.load(f)


@pytest.mark.parametrize("name", ["c1", "c2", "c3", "c4", "c5"])
def test_generators_match_golden_hash(name):
    g = _meta()["generators"][name]
    c = configs.make_config(name, g["scale"])
    import hashlib

    h = hashlib.sha256()
    for a in (c.matrix.row_ptr, c.matrix.col_idx, c.matrix.values, c.rhs):
        h.update(np.ascontiguousarray(a).tobytes())
    assert (c.matrix.n, c.matrix.nnz) == (g["n"], g["nnz"])
    assert h.hexdigest() == g["sha256"]


def test_generator_structure():
    c1 = configs.make_config("c1", 32 / 256)
    assert O.band_metrics(c1.matrix.to_scipy())[2] == 32 == c1.b
    c2 = configs.make_config("c2", 12 / 64)
    S = c2.matrix.to_scipy()
    assert O.band_metrics(S)[2] == 144 == c2.b and abs(S - S.T).max() > 0  # convection: nonsym
    c3 = configs.make_config("c3", 10 / 96)
    S3 = c3.matrix.to_scipy()
    assert O.band_metrics(S3)[2] == c3.b == 111 and abs(S3 - S3.T).max() == 0
    assert (S3.diagonal() >= np.abs(S3).sum(1).A1 - S3.diagonal() - 1e-9).all()
    c4 = configs.randband(5000, 50, 20, 3, 1.1)
    S4 = c4.to_scipy()
    assert O.band_metrics(S4)[2] <= 50 and S4.nnz == 5000 * 21
    c5 = configs.feast_base(8, 4, 64, 0.1).to_scipy()
    assert abs(c5 - c5.T).max() == 0 and O.band_metrics(c5)[2] <= 64


@pytest.mark.parametrize("key", ["c1_s48", "c2_s16"])
def test_oracle_matches_golden(key):
    case = _meta()["cases"][key]
    z = np.load(os.path.join(GOLD, f"{key}.npz"))
    c = configs.make_config(case["config"], case["scale"])
    A = c.matrix.to_scipy()
    x, rep, F = O.solve(A, c.rhs, O.SolverConfig(variant="T", p=c.P, k=c.b, n_svd=c.r, seed=c.seed),
                        O.IterConfig(tol=c.tol, restart=c.m or 30), method=case["method"])
    assert rep.iterations == case["iterations"]
    assert np.linalg.norm(x - z["x"]) / np.linalg.norm(z["x"]) < 1e-12
    assert np.linalg.norm(O.apply_precond_T(F, z["apply_in"]) - z["apply_out"]) <= \
        1e-12 * np.linalg.norm(z["apply_out"])


def _header_symbols():
    with open(os.path.join(ROOT, "include", "lrspike_capi.h")) as f:
        src = f.read()
    return sorted(set(re.findall(r"LRS_API\s+[\w\s\*]+?\b(lrs_\w+)\s*\(", src)))


def test_capi_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(os.path.join(ROOT, "paper_2504_11167_b200", "liblrspike_cuda.so"))
    syms = _header_symbols()
    assert len(syms) >= 25
    for s in syms:
        assert hasattr(lib, s), s


def test_capi_host_entry_points_without_gpu():
    from paper_2504_11167_b200 import api

    assert api.make_layout(10, 3, 2) == [4, 3, 3]
    with pytest.raises(api.LayoutError):
        api.make_layout(6, 3, 2)
    assert api.lib().lrs_status_string(6) == b"NotBlockTridiagonalError"


def test_cpp_api_host_logic():
    exe = os.path.join(ROOT, "tests", "cpp", "test_api")
    assert os.path.exists(exe), "build with `make` first"
    r = subprocess.run([exe, "cpu"], capture_output=True, text=True, timeout=120)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout


def test_product_path_does_not_import_oracle():
    """The product (package + C++ host + CUDA sources) never references the oracle."""
    pkg = os.path.join(ROOT, "paper_2504_11167_b200")
    for dirpath, _, files in os.walk(pkg):
        for fn in files:
            if fn.endswith((".py", ".cu", ".cuh", ".h", ".cpp", ".c")):
                with open(os.path.join(dirpath, fn)) as f:
                    txt = f.read()
                assert "lrspike_oracle" not in txt and "import oracle" not in txt, fn
