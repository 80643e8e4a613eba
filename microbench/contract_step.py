"""One batched T(I,u,u) power step (L restarts) on the config-1 sketch shape: the
contraction and median kernels (in-library CUDA-event scopes) and the whole Ivv call
(events on the library stream). Usage: python microbench/contract_step.py"""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1506_04448_b200 as skb  # noqa: E402

n, b, B, L = int(os.environ.get("N_", 400)), int(os.environ.get("B_", 1 << 14)), int(os.environ.get("R_", 20)), \
    int(os.environ.get("L_", 100))
ctx = skb.default_context(0)
ext = torch.cuda.ExternalStream(ctx.stream())
s = skb.SymTensorSketchSet(n, b, B, 5, ctx)
rng = np.random.default_rng(0)
X = rng.normal(size=(64, n))
s.accumulate_moment(X)
ws = skb.SymContractionWorkspace(s)
U = skb.power_inits(1, n, 1, L)[0]
for _ in range(3):
    ws.Ivv(U)
torch.cuda.synchronize()
a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record(ext)
for _ in range(10):
    ws.Ivv(U)
e.record(ext)
torch.cuda.synchronize()
call_ms = a.elapsed_time(e) / 10
ctx.profile(True)
ctx.profile_reset()
for _ in range(10):
    ws.Ivv(U)
c, _ = ctx.profile_get("sym_contract")
m, _ = ctx.profile_get("median")
ctx.profile(False)
print(json.dumps({"n": n, "b": b, "B": B, "L": L, "ivv_call_ms": call_ms, "contract_ms": c / 10, "median_ms": m / 10,
                  "us_per_restart": call_ms / L * 1e3}))
