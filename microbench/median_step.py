import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
import paper_1506_04448_b200 as skb
n, b, B, L = 400, 1 << 14, 20, 100
ctx = skb.default_context(0)
s = skb.SymTensorSketchSet(n, b, B, 5, ctx)
s.accumulate_moment(np.random.default_rng(0).normal(size=(64, n)))
ws = skb.SymContractionWorkspace(s)
U = skb.power_inits(1, n, 1, L)[0]
for _ in range(3): ws.Ivv(U)
ctx.profile(True); ctx.profile_reset()
for _ in range(10): ws.Ivv(U)
print({k: ctx.profile_get(k) for k in ["sym_contract", "median"]})
