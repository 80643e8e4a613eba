"""Config-4 whitening only (V=5e4, K=100, D=1e5 docs of Poisson(150) tokens): for
launch-list profiling of the implicit-M2 randomized eigensolver."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_1506_04448_b200 as skb  # noqa: E402

V, K, D = 50000, 100, int(os.environ.get("D_", 100000))
rng = np.random.default_rng(4)
topics = rng.dirichlet(np.full(V, 0.01), size=K)
lens = rng.poisson(150, size=D)
theta = rng.dirichlet(np.full(K, 1.0 / K), size=D)
doc_ptr, words, counts = [0], [], []
for d in range(D):
    p = theta[d] @ topics
    c = rng.multinomial(lens[d], p / p.sum())
    nz = np.nonzero(c)[0]
    words.append(nz.astype(np.int32))
    counts.append(c[nz].astype(np.int32))
    doc_ptr.append(doc_ptr[-1] + nz.size)
words, counts = np.concatenate(words), np.concatenate(counts)
ctx = skb.default_context(0)
t0 = time.perf_counter()
wm = skb.whiten_corpus(V, np.array(doc_ptr), words, counts, 1.0, K, ctx=ctx)
print("whiten seconds", time.perf_counter() - t0)
