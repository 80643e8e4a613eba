"""Config-0 RTPM (n=100, b=2^12, B=20, k=10, L=50, T=30) end to end through the host API:
wall time and the in-library per-kernel CUDA-event totals."""
import json
import os
import sys
import time

sys.path.insert(0, os.getcwd())
import paper_1506_04448_b200 as skb

ctx = skb.default_context(0)
T, lam, V = skb.gen_planted_tensor(100, 10, 0.01, 11)
s0 = skb.SymTensorSketchSet(100, 1 << 12, 20, 5, ctx)
s0.accumulate_dense(T, assume_symmetric=True)
base = s0.data()
cfg = skb.PowerConfig(k=10, L=50, T_iters=30, seed=3)
walls = []
for rep in range(4):
    s = skb.SymTensorSketchSet(100, 1 << 12, 20, 5, ctx)
    s.set_data(None, base)
    ctx.synchronize()
    t0 = time.perf_counter()
    d = skb.robust_tpm_fast(s, cfg)
    walls.append(time.perf_counter() - t0)
s = skb.SymTensorSketchSet(100, 1 << 12, 20, 5, ctx)
s.set_data(None, base)
ctx.profile(True)
ctx.profile_reset()
skb.robust_tpm_fast(s, cfg)
ctx.synchronize()
dev = {k: ctx.profile_get(k)[0] for k in ("sym_contract", "median", "moment", "freq_inverse", "combine", "spectrum")}
ctx.profile(False)
print(json.dumps({"rtpm_c0_wall_s": walls, "device_ms_by_scope_profiled_run": dev, "lambda0": float(d.lambda_[0])}))
