"""Print the componentwise / scaled LU backward-error report (tests/test_gpu_lu_int8.py)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from tests import test_gpu_lu_int8 as T
from paper_2504_11167_b200 import api

ctx = api.Context(0)
for name, scale, sym in (("c3", 24 / 96, False), ("c4", 0.05, False), ("c3", 24 / 96, True)):
    print(json.dumps(T.componentwise_report(ctx, name, scale, sym=sym)), flush=True)
