"""Small shapes through every hot kernel of the round, for compute-sanitizer runs:
  compute-sanitizer --tool memcheck  python microbench/sanitize_small.py
  compute-sanitizer --tool racecheck python microbench/sanitize_small.py
Covers the class-list dense build (windows in lockstep, fp64 two limbs and fp32 one limb), the
sums pre-pass, the half-length contraction (Ivv and vvv), the paired moment kernel (local
length 2048, odd and even sample counts), the paired LDA document kernel and a short RTPM.
Checks against the oracle so a silent corruption also fails."""
import os
import sys

sys.path.insert(0, os.getcwd())
sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np

import oracle_py as O  # checker only
import paper_1506_04448_b200 as skb
from lda_fixtures import synthetic_corpus

ctx = skb.default_context(0)


def rel(a, b):
    return float(np.max(np.linalg.norm(a - b, axis=1) / np.linalg.norm(b, axis=1)))


# dense builds: n = 40, b = 2^12 (class lists, local FFT length 2048 with 2 residues)
n, b, B = 40, 4096, 3
T, lam, V = skb.gen_planted_tensor(n, 3, 0.01, 1)
s = skb.SymTensorSketchSet(n, b, B, 5, ctx)
s.accumulate_dense(T, assume_symmetric=True)
o = O.SymSet(n, b, B, 5)
o.accumulate_dense(T, True)
print("build fp64", rel(s.data(), o.data()))
assert rel(s.data(), o.data()) < 1e-9
s32 = skb.SymTensorSketchSet(n, b, B, 5, ctx)
s32.accumulate_dense(T.astype(np.float32), assume_symmetric=True)
o32 = O.SymSet(n, b, B, 5)
o32.accumulate_dense(T.astype(np.float32).astype(np.float64), True)
print("build fp32", rel(s32.data(), o32.data()))
assert rel(s32.data(), o32.data()) < 1e-4

# contractions
ws = skb.SymContractionWorkspace(s)
u = V[:, 0]
iv, oiv = ws.Ivv(u), o.ivv(u)
print("Ivv", float(np.max(np.abs(iv - oiv)) / np.max(np.abs(oiv))))
assert np.max(np.abs(iv - oiv)) <= 1e-9 * np.max(np.abs(oiv))
vv, ovv = ws.vvv(u), o.vvv(u)
assert abs(vv - ovv) <= 1e-9 * abs(ovv), (vv, ovv)

# moment (paired kernel: local length 2048), odd and even sample counts
rng = np.random.default_rng(3)
for Ns in (5, 8):
    X = rng.normal(size=(Ns, n))
    w = rng.uniform(0.5, 1.5, size=Ns) / Ns
    sm = skb.SymTensorSketchSet(n, b, B, 7, ctx)
    sm.accumulate_moment(X, w)
    om = O.SymSet(n, b, B, 7)
    for i in range(Ns):
        om.add_scaled_rank1(X[i], w[i])
    print("moment", Ns, rel(sm.data(), om.data()))
    assert rel(sm.data(), om.data()) < 1e-9

# LDA documents (paired kernel) on a tiny corpus
Vv, k = 60, 8
doc_ptr, word, count, W = synthetic_corpus(V=Vv, k=k, D=25, mean_len=9, seed=2)
sl = skb.SymTensorSketchSet(k, b, B, 9, ctx)
sl.sketch_whitened_m3(Vv, doc_ptr, word, count, W, 1.0)
ol = O.SymSet(k, b, B, 9)
ol.sketch_whitened_m3(Vv, doc_ptr, word, count, W, 1.0)
print("lda", rel(sl.data(), ol.data()))
assert rel(sl.data(), ol.data()) < 1e-9

# short RTPM (CUDA graph of the power steps, deflation)
dec = skb.robust_tpm_fast(s, skb.PowerConfig(k=2, L=4, T_iters=6, seed=3))
lam_o, V_o, _ = o.rtpm(2, 4, 6, seed=3)
assert np.allclose(dec.lambda_, lam_o, rtol=1e-9, atol=0), (dec.lambda_, lam_o)
print("sanitize_small ok")
