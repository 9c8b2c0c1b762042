"""Locate the entry that maximises |A - LU| / (|L||U|) for the DMMA factors (c3 structure)."""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from tests import test_gpu_lu_int8 as T
from oracle import lrspike_oracle as O
from paper_2504_11167_b200 import api, configs

ctx = api.Context(0)
cfg = configs.make_config("c3", 0.25)
S = cfg.matrix.to_scipy()
lay = O.make_layout(S.shape[0], cfg.P, cfg.b)
blocks = O.extract_blocks(S, lay)
F = T._factor(ctx, cfg.matrix, cfg, False)
print(F.info)
i = 0
n_i = lay.sizes[i]
L, U = T._effective_lu(F, i, n_i)
Ad = blocks.A[i].toarray()
rows = np.arange(0, n_i, 7)
R = Ad[rows].astype(np.longdouble) - L[rows] @ U
B = np.abs(L[rows]) @ np.abs(U)
m = B > 0
rat = np.where(m, np.abs(R) / np.where(m, B, 1), 0)
for flat in np.argsort(rat.ravel())[::-1][:10]:
    a, j = np.unravel_index(flat, rat.shape)
    r = rows[a]
    print(f"row {r} col {j} d={r-j} tile ({r//128},{j//128}) A={Ad[r,j]:.3e} LU={float((L[r]@U[:,j])):.3e} "
          f"B={float(B[a,j]):.3e} ratio={float(rat[a,j]):.3e} Lrow_nz_beyond_band={int(np.sum(np.abs(L[r,:max(0,r-F.info['kl'])])>0))}")
nzL = np.abs(np.tril(L.astype(np.float64), -F.info["kl"] - 1)).max()
nzU = np.abs(np.triu(U.astype(np.float64), F.info["ku"] + 1)).max()
print("max |L| below band", nzL, "max |U| above band", nzU)
