"""Per-phase cycle split of k_sym_contract_half (experiment build with
-DSKC_TRACE_CONTRACT in paper_1506_04448_b200/_lib_trace; run with
SKC_LIB_DIR=paper_1506_04448_b200/_lib_trace)."""
import ctypes as C
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1506_04448_b200 as skb  # noqa: E402
from paper_1506_04448_b200 import _lib  # noqa: E402

n, b, B, L = 400, 1 << 14, 20, 100
ctx = skb.default_context(0)
s = skb.SymTensorSketchSet(n, b, B, 5, ctx)
s.accumulate_moment(np.random.default_rng(0).normal(size=(64, n)))
ws = skb.SymContractionWorkspace(s)
U = skb.power_inits(1, n, 1, L)[0]
ws.Ivv(U)
buf = (C.c_ulonglong * 8)()
f = _lib.lib.skc_debug_contract_phases
f.argtypes = [C.POINTER(C.c_ulonglong), C.c_int]
f(buf, 1)
for _ in range(10):
    ws.Ivv(U)
f(buf, 1)
names = ["stage_zero", "scatter1", "scatter2", "dif", "pointwise", "dit", "gather"]
tot = sum(buf[i] for i in range(7))
print(json.dumps({k: round(100.0 * buf[i] / tot, 1) for i, k in enumerate(names)}))
