"""Times one batched T(I,u,u) power step (L restarts) on the config-1 sketch shape with
the in-library CUDA-event profiler. Usage: SKC_CONTRACT_VARIANT=8d python microbench/contract_step.py"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1506_04448_b200 as skb  # noqa: E402

n, b, B, L = int(os.environ.get("N_", 400)), int(os.environ.get("B_", 1 << 14)), 20, int(os.environ.get("L_", 100))
ctx = skb.default_context(0)
s = skb.SymTensorSketchSet(n, b, B, 5, ctx)
rng = np.random.default_rng(0)
X = rng.normal(size=(64, n))
s.accumulate_moment(X)
ws = skb.SymContractionWorkspace(s)
U = skb.power_inits(1, n, 1, L)[0]
for _ in range(3):
    ws.Ivv(U)
ctx.profile(True)
ctx.profile_reset()
for _ in range(10):
    ws.Ivv(U)
c, _ = ctx.profile_get("sym_contract")
ctx.profile(False)
print(json.dumps({"variant": os.environ.get("SKC_CONTRACT_VARIANT", "default"), "n": n, "b": b, "L": L,
                  "contract_ms_per_step": c / 10, "us_per_restart": c / 10 / L * 1e3, "local_N": os.environ.get("SKC_LOCAL_N", "2048")}))
