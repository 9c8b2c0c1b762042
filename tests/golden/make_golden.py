"""Generate the golden fixtures in tests/golden/ from the CPU oracle.

    python tests/golden/make_golden.py

Fixtures pin (a) the generators (sha256 of the CSR arrays and RHS of every
config at a test scale), and (b) the oracle's outputs on small c1 / c2 cases:
iteration counts, the solution, one preconditioner application and the leading
spike singular values.  Tests compare the oracle (CPU) and the CUDA path (GPU)
against them.  The reference itself cannot be run, so these are
oracle-generated, cross-checked against dense solves at generation time.
"""
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle import lrspike_oracle as O  # noqa: E402
from paper_2504_11167_b200 import configs  # noqa: E402

CASES = {
    "c1_s48": ("c1", 48 / 256, "gmres"),
    "c2_s16": ("c2", 16 / 64, "bicgstab"),
}
GEN_SCALES = {"c1": 48 / 256, "c2": 16 / 64, "c3": 12 / 96, "c4": 0.002, "c5": 10 / 80}


def sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def main():
    meta = {"generators": {}, "cases": {}}
    for name, sc in GEN_SCALES.items():
        c = configs.make_config(name, sc)
        m = c.matrix
        meta["generators"][name] = {"scale": sc, "n": m.n, "nnz": m.nnz,
                                    "sha256": sha(m.row_ptr, m.col_idx, m.values, c.rhs)}
    for key, (name, sc, method) in CASES.items():
        c = configs.make_config(name, sc)
        A = c.matrix.to_scipy()
        sc_o = O.SolverConfig(variant="T", p=c.P, k=c.b, n_svd=c.r, seed=c.seed)
        x, rep, F = O.solve(A, c.rhs, sc_o, O.IterConfig(tol=c.tol, restart=c.m or 30), method=method)
        xd = np.linalg.solve(A.toarray(), c.rhs)
        assert np.linalg.norm(x - xd) / np.linalg.norm(xd) < 1e-6
        f = configs.vector("uniform", 99, A.shape[0])
        y = O.apply_precond_T(F, f)
        np.savez_compressed(os.path.join(HERE, f"{key}.npz"), x=x, apply_in=f, apply_out=y,
                            sigmaT0=F.spT[0].sigma, sigmaW1=F.spW[1].sigma)
        meta["cases"][key] = {"config": name, "scale": sc, "method": method,
                              "iterations": rep.iterations, "residual_final": rep.residual_final,
                              "precond_applications": rep.precond_applications,
                              "n_svd": F.n_svd}
    with open(os.path.join(HERE, "golden.json"), "w") as fh:
        json.dump(meta, fh, indent=1, sort_keys=True)
    print(json.dumps(meta, indent=1))


if __name__ == "__main__":
    main()
