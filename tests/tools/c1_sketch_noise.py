"""Why RTPM cannot recover BASELINE config 1's planted components from its sketch.

Config 1 (n=400, rank 50, lambda ~ U[1,2], noise sd 0.01 per entry mirrored,
b=2^14, B=20) has ||T||_F ~ 80, so one replicate's per-coordinate error in the
sketched T(I,v,v) is about ||T||_F / sqrt(b) ~ 0.6 and the median over B leaves a
vector error comparable to lambda itself. This prints, for the first planted
components, the exact T(I,v,v) and the error of the sketched estimate (CPU oracle
sketch; the GPU sketch agrees with it to 1e-9 by the parity tests). Test
infrastructure: the oracle is the checker here. Run from the repo root.
"""
import json
import os
import sys

import numpy as np

_ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, _ROOT)
sys.path.insert(0, os.path.join(_ROOT, "tests"))
import oracle_py as O  # noqa: E402
import paper_1506_04448_b200 as skb  # noqa: E402

n, rank, sigma, seed, b, B = 400, 50, 0.01, 20150615, 1 << 14, 20
T, lam, V = skb.gen_planted_tensor(n, rank, sigma, seed)
V = np.asarray(V).reshape(rank, n).T if np.asarray(V).shape != (n, rank) else np.asarray(V)
s = O.SymSet(n, b, B, seed)
s.accumulate_dense(T, assume_symmetric=True)
rows = []
for c in range(5):
    v = V[:, c]
    exact = np.einsum("ijk,j,k->i", T, v, v)
    est = s.ivv(v)
    rows.append({"component": c, "lambda": float(lam[c]), "exact_Ivv_norm": float(np.linalg.norm(exact)),
                 "sketch_Ivv_error_norm": float(np.linalg.norm(est - exact)),
                 "exact_vvv": float(exact @ v), "sketch_vvv": float(s.vvv(v))})
print(json.dumps({"config": 1, "T_fro": float(np.linalg.norm(T)), "rows": rows}))
