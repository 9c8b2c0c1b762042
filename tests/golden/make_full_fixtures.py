"""Full-size oracle solves of BASELINE configs c1 and c2 -> tests/golden/full_<cfg>.npz/.json.

    python tests/golden/make_full_fixtures.py c1 [c2 ...]

The CPU oracle (oracle/lrspike_oracle.py, scipy/OpenBLAS ?gbtrf/?gbtrs) runs the
whole LR-SPIKE-T solve on the full BASELINE input (c1: GMRES(30), c2: BiCGStab) and
the fixture keeps what the GPU parity tests compare against (tests/test_gpu_fullsize.py):
the iteration count, the final true residual, the preconditioner-application count,
the solution x itself (float64, compressed) and the wall time of each stage on the host
that generated it (host model and core count recorded beside it).  The inputs come from
the C generators, bit-identical on every host, so a fixture made here is valid on the
GPU box.  Test infrastructure only: nothing in the product path reads these files.
"""
import hashlib
import json
import os
import platform
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
OUT = os.environ.get("LRS_FIXTURE_DIR", HERE)  # e.g. gpurun_out/ when run on the GPU box

from oracle import lrspike_oracle as O  # noqa: E402
from paper_2504_11167_b200 import configs  # noqa: E402


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as fh:
            for line in fh:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return platform.processor() or "unknown"


def run(name: str, scale: float = 1.0, P: int | None = None, shift: int | None = None,
        nrhs: int | None = None) -> dict:
    c = configs.make_config(name, scale, P)
    A = c.system(shift).to_scipy() if shift is not None else c.matrix.to_scipy()
    rhs = c.rhs if nrhs is None else c.rhs[:, :nrhs]
    if shift is not None:
        rhs = np.asfortranarray(rhs.astype(np.complex128))
    scfg = O.SolverConfig(variant="T", p=c.P, k=c.b, n_svd=c.r, seed=c.seed)
    it = O.IterConfig(tol=c.tol, restart=c.m or 30)
    t0 = time.perf_counter()
    F = O.factorize(A, scfg)
    print(f"{name}: factorize {time.perf_counter() - t0:.1f} s", flush=True)
    t1 = time.perf_counter()
    x, rep, _ = O.solve(A, rhs, scfg, it, method=c.method, F=F)
    t2 = time.perf_counter()
    tag = f"full_{name}" if scale == 1.0 and P is None else f"{name}_s{scale:g}_P{c.P}"
    if shift is not None:
        tag += f"_z{shift}_r{rhs.shape[1]}"
    np.savez_compressed(os.path.join(OUT, f"{tag}.npz"), x=x)
    meta = {
        "config": name, "scale": scale, "P": c.P, "n": int(A.shape[0]), "nnz": int(A.nnz),
        "k": c.b, "n_svd": F.n_svd, "method": c.method, "restart": c.m, "tol": c.tol,
        "shift": shift, "nrhs": int(rhs.shape[1]),
        "iterations": rep.iterations, "residual_final": rep.residual_final,
        "converged": rep.converged, "precond_applications": rep.precond_applications,
        "matvecs": rep.matvecs, "x_norm": float(np.linalg.norm(x)),
        "x_sha256": hashlib.sha256(np.ascontiguousarray(x).tobytes()).hexdigest(),
        "host": {"cpu": cpu_model(), "cores": os.cpu_count(),
                 "openblas_threads": os.environ.get("OPENBLAS_NUM_THREADS", "default"),
                 "partition_threads": os.environ.get("LRS_ORACLE_THREADS", "1"),
                 "mem_gb": round(os.sysconf("SC_PAGE_SIZE") * os.sysconf("SC_PHYS_PAGES") / 2**30)},
        "t_factorize_s": t1 - t0, "t_solve_s": t2 - t1,
    }
    with open(os.path.join(OUT, f"{tag}.json"), "w") as fh:
        json.dump(meta, fh, indent=1, sort_keys=True)
    print(json.dumps(meta), flush=True)
    return meta


if __name__ == "__main__":
    for arg in sys.argv[1:] or ["c1"]:
        parts = arg.split(":")  # name[:scale[:P[:shift[:nrhs]]]]
        run(parts[0], float(parts[1]) if len(parts) > 1 else 1.0,
            int(parts[2]) if len(parts) > 2 else None,
            int(parts[3]) if len(parts) > 3 else None,
            int(parts[4]) if len(parts) > 4 else None)
