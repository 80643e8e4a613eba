"""Times sketch_whitened_m3's accumulate kernels at config 4's sketch shape (k=100, b=2^14,
B=10) on a synthetic corpus of D documents (in-library CUDA-event scopes):
D_=200000 python microbench/lda_sketch_time.py"""
import json
import os
import sys

sys.path.insert(0, os.getcwd())
sys.path.insert(0, os.path.join(os.getcwd(), "tests"))

import paper_1506_04448_b200 as skb
from lda_fixtures import synthetic_corpus

V, k = 50000, 100
D = int(os.environ.get("D_", 200000))
doc_ptr, word, count, W = synthetic_corpus(V=V, k=k, D=D, mean_len=50, seed=3)
ctx = skb.default_context(0)
s = skb.SymTensorSketchSet(k, 1 << 14, 10, 9, ctx)
s.sketch_whitened_m3(V, doc_ptr, word, count, W, 1.0)
ctx.synchronize()
ctx.profile(True)
ctx.profile_reset()
s.sketch_whitened_m3(V, doc_ptr, word, count, W, 1.0)
ctx.synchronize()
out = {"D": D, "V": V}
for name in ("lda_accumulate", "lda_items", "lda_finish"):
    try:
        ms, cnt = ctx.profile_get(name)
        out[name + "_ms"] = ms
    except Exception:
        pass
ctx.profile(False)
print(json.dumps(out))
