"""LU variants on one config: each variant (library build x environment) factorizes the
config R times in its own process; prints the median t_lu / t_factorize (library CUDA
events) and the LU's FP64-equivalent rate.

  python scripts/lu_variants.py c3 1.0 64 [R]
Variants: default, LRS_LU_QUAD=1, LRS_I8_2SM=1, both, and the builds in build/var_*/ (make variant V=...)."""
import glob
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def one(name, scale, P, R):
    import numpy as np

    from paper_2504_11167_b200 import api, configs

    cfg = configs.make_config(name, scale, P)
    ctx = api.Context(0)
    A = api.CsrMatrix.from_csr(ctx, cfg.matrix)
    scfg = api.SolverConfig(p=cfg.P, k=cfg.b, n_svd=cfg.r, seed=cfg.seed)
    lu, fa = [], []
    for _ in range(R + 1):
        F = api.factorize(ctx, A, scfg)
        lu.append(F.info["t_lu"])
        fa.append(F.info["t_factorize"])
        flops = F.info["lu_flops"]
        del F
    lu, fa = lu[1:], fa[1:]
    return {"t_lu_median": float(np.median(lu)), "t_lu_all": lu,
            "t_factorize_median": float(np.median(fa)),
            "lu_tflops_fp64_equiv": flops / float(np.median(lu)) / 1e12}


if __name__ == "__main__":
    name, scale, P = sys.argv[1], float(sys.argv[2]), int(sys.argv[3])
    R = int(sys.argv[4]) if len(sys.argv) > 4 else 3
    if os.environ.get("LRS_VARIANT_CHILD"):
        print(json.dumps(one(name, scale, P, R)), flush=True)
        sys.exit(0)
    variants = [("default", {}), ("pairs", {"LRS_LU_QUAD": "0"}), ("quad", {"LRS_LU_QUAD": "1"}),
                ("quad-mini-dmma", {"LRS_LU_QUAD": "1", "LRS_QUAD_MINI_DMMA": "1"}),
                # the full schedule on symmetric blocks (no effect on c2 / c4)
                ("sym-off", {"LRS_LU_SYM": "0"}),
                ("pairs sym-off", {"LRS_LU_QUAD": "0", "LRS_LU_SYM": "0"})]
    if os.environ.get("LRS_VARIANTS_2SM"):
        variants += [("2sm", {"LRS_I8_2SM": "1"}),
                     ("quad+2sm", {"LRS_LU_QUAD": "1", "LRS_I8_2SM": "1"})]
    for lib in sorted(glob.glob(os.path.join(ROOT, "build", "var_*", "liblrspike_cuda.so"))):
        variants.append((os.path.basename(os.path.dirname(lib)), {"LRS_LIB": lib}))
    for tag, env in variants:
        out = subprocess.run([sys.executable, __file__] + sys.argv[1:],
                             env={**os.environ, **env, "LRS_VARIANT_CHILD": "1"},
                             capture_output=True, text=True, timeout=900)
        line = out.stdout.strip().splitlines()[-1] if out.stdout.strip() else out.stderr[-500:]
        print(json.dumps({"variant": tag, "env": {k: v for k, v in env.items() if k != "LRS_LIB"},
                          "result": json.loads(line) if line.startswith("{") else line}),
              flush=True)
