"""Full config-0 RTPM (n=100, b=2^12, B=20, k=10, L=50, T=30) on the GPU and in the
oracle (host threads) with the same seeds; prints the component-wise differences.
Test infrastructure: the oracle is the checker here (run from the repo root)."""
import json
import os
import sys
import time

_ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, _ROOT)
sys.path.insert(0, os.path.join(_ROOT, "tests"))
import numpy as np  # noqa: E402

import oracle_py as O  # noqa: E402
import paper_1506_04448_b200 as skb  # noqa: E402

n, rank, b, B, k, L, T = 100, 10, 1 << 12, 20, 10, 50, 30
Tt, lam, V = skb.gen_planted_tensor(n, rank, 0.01, 11)
ctx = skb.default_context(0)
s = skb.SymTensorSketchSet(n, b, B, 5, ctx)
s.accumulate_dense(Tt, True)
dec = skb.robust_tpm_fast(s, skb.PowerConfig(k=k, L=L, T_iters=T, seed=3))
O.lib().orc_set_num_threads(os.cpu_count() or 1)
o = O.SymSet(n, b, B, 5)
o.accumulate_dense(Tt, True)
t0 = time.perf_counter()
lo, Vo, bto = o.rtpm(k, L, T, seed=3)
cpu_s = time.perf_counter() - t0
rel = np.abs(dec.lambda_ - lo) / np.abs(lo)
vd = np.max(np.abs(dec.A - Vo), axis=0)
print(json.dumps({"lambda_gpu": dec.lambda_.tolist(), "lambda_oracle": lo.tolist(), "lambda_rel": rel.tolist(),
                  "v_maxabs": vd.tolist(), "best_tau_gpu": dec.best_tau.tolist() if dec.best_tau is not None else None,
                  "best_tau_oracle": bto.tolist(), "oracle_seconds": cpu_s}))
