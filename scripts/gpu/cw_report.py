"""Print the componentwise / scaled LU backward-error report (tests/test_gpu_lu_int8.py)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from tests import test_gpu_lu_int8 as T
from paper_2504_11167_b200 import api

ctx = api.Context(0)
for name, scale in (("c3", 24 / 96), ("c4", 0.05)):
    print(json.dumps(T.componentwise_report(ctx, name, scale)), flush=True)
