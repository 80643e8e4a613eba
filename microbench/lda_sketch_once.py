"""One sketch_whitened_m3 at config 4's sketch shape (k=100, b=2^14, B=10) on a synthetic
corpus (V=50000, D=20000 documents of ~150 tokens; for ncu captures of the LDA kernels)."""
import os
import sys

sys.path.insert(0, os.getcwd())
sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np

import paper_1506_04448_b200 as skb
from lda_fixtures import synthetic_corpus

V, k = 50000, 100
doc_ptr, word, count, W = synthetic_corpus(V=V, k=k, D=20000, mean_len=150, seed=3)
ctx = skb.default_context(0)
s = skb.SymTensorSketchSet(k, 1 << 14, 10, 9, ctx)
for _ in range(2):
    s.sketch_whitened_m3(V, doc_ptr, word, count, W, 1.0)
print("ok")
