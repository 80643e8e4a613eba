"""Small synthetic LDA corpora (CSR) and whitening maps for the a26 tests."""
import numpy as np


def synthetic_corpus(V=50, k=6, D=40, mean_len=8, seed=0):
    rng = np.random.default_rng(seed)
    topics = rng.dirichlet(np.full(V, 0.3), size=k)  # k x V
    doc_ptr, words, counts = [0], [], []
    for _ in range(D):
        theta = rng.dirichlet(np.full(k, 0.5))
        m = rng.poisson(mean_len)
        tok = rng.choice(V, size=m, p=theta @ topics) if m > 0 else np.array([], dtype=int)
        u, c = np.unique(tok, return_counts=True)
        words.extend(u.tolist())
        counts.extend(c.tolist())
        doc_ptr.append(len(words))
    W = rng.normal(size=(V, k)) / np.sqrt(V)
    return (np.array(doc_ptr, dtype=np.int64), np.array(words, dtype=np.int32), np.array(counts, dtype=np.int32), W)


def explicit_whitened_m3(V, doc_ptr, word, count, W, alpha0):
    """The tensor whose sketch sketch_whitened_m3 accumulates (lda.cpp:145-226), written
    out densely: (1/D)[sum_d s1 p^3 - 3 sum_d s2 p p q + sum_i (c1_i w_i^3 - 3 w_i w_i sumwn_i)]
    + c_m1 q^3, symmetrised."""
    k = W.shape[1]
    D = doc_ptr.size - 1
    P, S1, S2 = [], [], []
    coeff1 = np.zeros(V)
    sumwn = np.zeros((V, k))
    m1 = np.zeros(V)
    used1 = 0
    for d in range(D):
        ws = word[doc_ptr[d]:doc_ptr[d + 1]]
        cs = count[doc_ptr[d]:doc_ptr[d + 1]].astype(float)
        tot = cs.sum()
        if tot >= 1:
            m1[ws] += cs / tot
            used1 += 1
        if tot < 3:
            continue
        s1 = 1.0 / (tot * (tot - 1) * (tot - 2))
        s2 = alpha0 / ((alpha0 + 2) * tot * (tot - 1))
        p = cs @ W[ws]
        coeff1[ws] += 2 * s1 * cs
        sumwn[ws] += s1 * cs[:, None] * p[None, :]
        P.append(p)
        S1.append(s1)
        S2.append(s2)
    m1 /= used1
    q = W.T @ m1
    used = len(P)
    T = np.zeros((k, k, k))
    for p, s1, s2 in zip(P, S1, S2):
        T += s1 * np.einsum("i,j,k->ijk", p, p, p) - 3 * s2 * np.einsum("i,j,k->ijk", p, p, q)
    for i in range(V):
        T += coeff1[i] * np.einsum("i,j,k->ijk", W[i], W[i], W[i]) - 3 * np.einsum("i,j,k->ijk", W[i], W[i], sumwn[i])
    T = T / used + 2 * alpha0 ** 2 / ((alpha0 + 1) * (alpha0 + 2)) * np.einsum("i,j,k->ijk", q, q, q)
    perms = [(0, 1, 2), (0, 2, 1), (1, 0, 2), (1, 2, 0), (2, 0, 1), (2, 1, 0)]
    return sum(T.transpose(pp) for pp in perms) / 6, used, D - used
