"""Conditioning of the config-0 RTPM (n=100, b=2^12, B=20, k=10, L=50, T=30): run the GPU
driver on the tensor and on copies perturbed by one ulp-scale relative noise (1e-16) and
report how far the components move. Shows how much rounding-level differences (e.g. FFT
summation order) are amplified by the deflation sequence and the restart argmax."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1506_04448_b200 as skb  # noqa: E402

n, rank, b, B, k, L, T = 100, 10, 1 << 12, 20, 10, 50, 30
Tt, lam, V = skb.gen_planted_tensor(n, rank, 0.01, 11)
ctx = skb.default_context(0)


def run(tensor):
    s = skb.SymTensorSketchSet(n, b, B, 5, ctx)
    s.accumulate_dense(tensor, True)
    d = skb.robust_tpm_fast(s, skb.PowerConfig(k=k, L=L, T_iters=T, seed=3))
    return d.lambda_, d.A, d.best_tau


l0, v0, t0 = run(Tt)
out = []
rng = np.random.default_rng(1)
for trial in range(3):
    E = rng.normal(size=Tt.shape)
    E = (E + E.transpose(0, 2, 1) + E.transpose(1, 0, 2) + E.transpose(1, 2, 0) + E.transpose(2, 0, 1) +
         E.transpose(2, 1, 0)) / 6
    l1, v1, t1 = run(Tt * (1 + 1e-16 * E))
    out.append({"lambda_rel": (np.abs(l1 - l0) / np.abs(l0)).tolist(), "tau_same": (np.array(t1) == np.array(t0)).tolist()})
print(json.dumps(out))
