#!/usr/bin/env python
"""Secondary measurements for every BASELINE.json config (the driver's bench.py line is
config 1). One JSON line per measurement; device times come from the library's CUDA-event
profiler or CUDA events on the library stream, CPU baselines from the oracle restatement
on the host cores (bounded samples, stated in each line).

  C0  n=100 fp64 rank 10, b=2^12 B=20: sym + asym dense build, RTPM k=10 L=50 T=30
  C1  n=400 fp64 rank 50, b=2^14 B=20: full RTPM k=50 L=100 T=30
  C2  n=1000 fp32 rank 100 (4 GB, generated on device), b=2^16 B=10: dense build
  C3  factored third moment, n=1000, K=50 Dirichlet(0.1) mixtures + 0.1 N(0,I), b=2^14 B=10:
      frequency-domain accumulation (reduced N, linear in N), then RTPM k=50 L=T=30
  C4  LDA V=50000 K=100, Dirichlet(0.01) topics, Poisson(150) docs (reduced D), b=2^14 B=10:
      whitening from the corpus M2 (implicit, randomized), sketch_whitened_m3, then RTPM
      L=100 k=100 T=30

  C5  (paper Table 4) fast ALS: n=1000 rank 10 fp32 tensor on device, asym b=2^14 B=40,
      k=10, exactly 30 sweeps

Usage: python bench_configs.py [--configs 0,1,2,3,4,5] [--quick]
"""
from __future__ import annotations

import argparse
import json
import os
import pathlib
import sys
import time

import numpy as np

ROOT = pathlib.Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "tests"))


def emit(d):
    print(json.dumps(d), flush=True)


def timed(ctx, fn, names):
    ctx.profile(True)
    ctx.profile_reset()
    t0 = time.perf_counter()
    fn()
    ctx.synchronize()
    wall = time.perf_counter() - t0
    dev = {k: ctx.profile_get(k)[0] for k in names}
    ctx.profile(False)
    return wall, dev


def c0(skb, ctx, quick):
    import oracle_py as O

    n, rank, b, B = 100, 10, 1 << 12, 20
    T, lam, V = skb.gen_planted_tensor(n, rank, 0.01, 11)
    import torch

    Td = torch.from_numpy(T).cuda()
    s = skb.SymTensorSketchSet(n, b, B, 5, ctx)
    for _ in range(3):
        s.accumulate_dense(Td, True)
    wall, dev = timed(ctx, lambda: [s.accumulate_dense(Td, True) for _ in range(20)],
                      ["build_prepass", "build_main", "build_finalize"])
    build_ms = sum(dev.values()) / 20
    a = skb.AsymTensorSketchSet(n, b, B, 5, ctx)
    a.accumulate_dense(Td)
    _, deva = timed(ctx, lambda: [a.accumulate_dense(Td) for _ in range(20)],
                    ["build_prepass", "build_main", "build_finalize"])
    s2 = skb.SymTensorSketchSet(n, b, B, 5, ctx)
    s2.accumulate_dense(Td, True)
    t0 = time.perf_counter()
    dec = skb.robust_tpm_fast(s2, skb.PowerConfig(k=10, L=50, T_iters=30, seed=3))
    rtpm_s = time.perf_counter() - t0
    match = O.greedy_match(dec.A, V)
    O.lib().orc_set_num_threads(os.cpu_count() or 1)
    o = O.SymSet(n, b, B, 5)
    t0 = time.perf_counter()
    o.accumulate_dense(T, True)
    cpu_build = time.perf_counter() - t0
    t0 = time.perf_counter()
    o.rtpm(1, 50, 30, seed=3)
    cpu_rtpm1 = time.perf_counter() - t0
    emit({"config": 0, "what": "sym dense build", "n": n, "b": b, "B": B, "device_ms": build_ms,
          "entries_per_s": n ** 3 / (build_ms * 1e-3), "cpu_oracle_ms": cpu_build * 1e3,
          "cpu_threads": O.lib().orc_num_threads()})
    emit({"config": 0, "what": "asym dense build", "device_ms": sum(deva.values()) / 20,
          "entries_per_s": n ** 3 / (sum(deva.values()) / 20 * 1e-3)})
    emit({"config": 0, "what": "RTPM k=10 L=50 T=30 (end to end, host API)", "seconds": rtpm_s,
          "lambda": dec.lambda_.tolist(), "recovered_cos_min": float(match[:, 2].min()),
          "wrong_vectors(sqdist>0.1)": int((match[:, 3] > 0.1).sum()),
          "cpu_oracle_seconds_extrapolated": cpu_rtpm1 * 10,
          "cpu_sample": "oracle RTPM of 1 component (L=50,T=30) x 10"})


def c1(skb, ctx, quick):
    import oracle_py as O

    n, rank, b, B = 400, 50, 1 << 14, 20
    k = 5 if quick else 50
    T, lam, V = skb.gen_planted_tensor(n, rank, 0.01, 20150615)
    s = skb.SymTensorSketchSet(n, b, B, 20150615, ctx)
    s.accumulate_dense(T, True)
    ctx.profile(True)
    ctx.profile_reset()
    t0 = time.perf_counter()
    dec = skb.robust_tpm_fast(s, skb.PowerConfig(k=k, L=100, T_iters=30, seed=7))
    wall = time.perf_counter() - t0
    dev = {x: ctx.profile_get(x)[0] for x in ["sym_contract", "median", "moment", "freq_inverse", "combine", "spectrum"]}
    ctx.profile(False)
    match = O.greedy_match(dec.A, V)
    O.lib().orc_set_num_threads(os.cpu_count() or 1)
    o = O.SymSet(n, b, B, 20150615)
    o.accumulate_dense(T, True)
    u = skb.power_inits(7, n, 1, 1)[0, 0]
    t0 = time.perf_counter()
    o.ivv(u)
    cpu_ivv = time.perf_counter() - t0
    emit({"config": 1, "what": f"RTPM k={k} L=100 T=30 (end to end, host API)", "seconds": wall,
          "device_ms_by_kernel": dev, "T(I,u,u)_per_s": k * 100 * 30 / wall,
          "recovered_cos_median": float(np.median(match[:, 2])),
          "wrong_vectors(sqdist>0.1)": int((match[:, 3] > 0.1).sum()),
          "cpu_oracle_one_Ivv_s": cpu_ivv, "cpu_oracle_rtpm_seconds_extrapolated": cpu_ivv * k * 100 * 31,
          "cpu_threads": O.lib().orc_num_threads()})


def c2(skb, ctx, quick):
    import torch

    n, rank, b, B = (400, 40, 1 << 16, 10) if quick else (1000, 100, 1 << 16, 10)
    Td = torch.empty(n ** 3, dtype=torch.float32, device="cuda")
    skb.gen_planted_tensor_device(ctx, n, rank, 0.01, 99, Td.data_ptr(), dtype=np.float32)
    s = skb.SymTensorSketchSet(n, b, B, 3, ctx)
    s.accumulate_dense(Td, True)
    _, dev = timed(ctx, lambda: [s.accumulate_dense(Td, True) for _ in range(3)],
                   ["build_prepass", "build_main", "build_finalize"])
    ms = sum(dev.values()) / 3
    simplex = n * (n + 1) * (n + 2) // 6
    emit({"config": 2, "what": "sym dense build fp32 (device-generated tensor)", "n": n, "b": b, "B": B,
          "device_ms": ms, "entries_per_s": n ** 3 / (ms * 1e-3), "simplex_GBps": simplex * 4 / (ms * 1e-3) / 1e9,
          "by_kernel_ms": {k: v / 3 for k, v in dev.items()}})


def c3(skb, ctx, quick):
    n, K, b, B = 1000, 50, 1 << 14, 10
    N = 1 << (14 if quick else 17)
    rng = np.random.default_rng(3)
    A, _ = np.linalg.qr(rng.normal(size=(n, K)))
    Wm = rng.dirichlet(np.full(K, 0.1), size=N)
    X = Wm @ A.T + 0.1 * rng.normal(size=(N, n))
    import torch

    Xd = torch.from_numpy(X).cuda()
    w = torch.full((N,), 1.0 / N, dtype=torch.float64, device="cuda")
    s = skb.SymTensorSketchSet(n, b, B, 4, ctx)
    s.accumulate_moment(Xd[:256], w[:256])
    _, dev = timed(ctx, lambda: s.accumulate_moment(Xd, w), ["moment", "freq_inverse", "combine"])
    ms = sum(dev.values())
    emit({"config": 3, "what": "factored moment sketch (frequency-domain accumulation)", "N": N, "n": n, "b": b,
          "B": B, "device_ms": ms, "samples_per_s": N / (ms * 1e-3),
          "extrapolated_seconds_for_N=2^22": (1 << 22) / (N / (ms * 1e-3))})
    k = 5 if quick else 50
    t0 = time.perf_counter()
    dec = skb.robust_tpm_fast(s, skb.PowerConfig(k=k, L=30, T_iters=30, seed=1))
    emit({"config": 3, "what": f"RTPM k={k} L=30 T=30 on the moment sketch", "seconds": time.perf_counter() - t0,
          "lambda_top3": dec.lambda_[:3].tolist()})


def c4(skb, ctx, quick):
    V, K, b, B = 50000, 100, 1 << 14, 10
    D = 2000 if quick else 100000
    rng = np.random.default_rng(4)
    topics = rng.dirichlet(np.full(V, 0.01), size=K)
    lens = rng.poisson(150, size=D)
    doc_ptr, words, counts = [0], [], []
    for d in range(D):
        theta = rng.dirichlet(np.full(K, 1.0 / K))
        p = theta @ topics
        c = rng.multinomial(lens[d], p / p.sum())
        nz = np.nonzero(c)[0]
        words.append(nz.astype(np.int32))
        counts.append(c[nz].astype(np.int32))
        doc_ptr.append(doc_ptr[-1] + nz.size)
    words = np.concatenate(words)
    counts = np.concatenate(counts)
    # whitening from the corpus' own second moment (lda.cpp:102-143, implicit M2 on the GPU)
    alpha0 = 1.0
    t0 = time.perf_counter()
    ctx.profile(True)
    ctx.profile_reset()
    wm = skb.whiten_corpus(V, np.array(doc_ptr), words, counts, alpha0, K, ctx=ctx)
    whiten_s = time.perf_counter() - t0
    whiten_dev = ctx.profile_get("lda_whiten")[0]
    ctx.profile(False)
    emit({"config": 4, "what": "whiten(compute_m2(corpus), K) by randomized subspace iteration on the implicit M2",
          "V": V, "K": K, "D": D, "nnz": int(words.size), "seconds": whiten_s, "device_ms": whiten_dev,
          "top_eigenvalues": wm.singular_values[:3].tolist(), "kth_eigenvalue": float(wm.singular_values[-1])})
    W = wm.W
    s = skb.SymTensorSketchSet(K, b, B, 9, ctx)
    t0 = time.perf_counter()
    ctx.profile(True)
    ctx.profile_reset()
    used, skipped = s.sketch_whitened_m3(V, np.array(doc_ptr), words, counts, W, alpha0)
    wall = time.perf_counter() - t0
    dev = {x: ctx.profile_get(x)[0] for x in ["lda_docs", "lda_vocab", "lda_accumulate"]}
    ctx.profile(False)
    emit({"config": 4, "what": "sketch_whitened_m3 given W (host CSR in, includes host transpose + H2D)", "V": V,
          "K": K, "D": D, "nnz": int(words.size), "used": used, "skipped": skipped, "seconds": wall,
          "device_ms_by_kernel": dev, "docs_per_s_device": D / (sum(dev.values()) * 1e-3)})
    k = 5 if quick else 100
    t0 = time.perf_counter()
    dec = skb.robust_tpm_fast(s, skb.PowerConfig(k=k, L=100, T_iters=30, seed=2))
    rtpm_s = time.perf_counter() - t0
    # recover_params (lda.cpp:228-248) and the recovery quality against the generating topics
    model = skb.recover_params(dec, wm, alpha0)
    Pn = model.Phi / np.linalg.norm(model.Phi, axis=0, keepdims=True)
    Tn = topics.T / np.linalg.norm(topics.T, axis=0, keepdims=True)
    cos = Pn.T @ Tn  # k x K
    best = []
    used_t = set()
    for c in np.argsort(-cos.max(axis=1)):
        order = np.argsort(-cos[c])
        t = next(t for t in order if t not in used_t)
        used_t.add(t)
        best.append(cos[c, t])
    emit({"config": 4, "what": f"RTPM k={k} L=100 T=30 on the whitened sketch + recover_params", "seconds": rtpm_s,
          "topic_cos_median": float(np.median(best)), "topic_cos_min": float(np.min(best)),
          "alpha0_recovered": float(model.alpha.sum())})


def c5(skb, ctx, quick):
    """Fast ALS at the paper's Table 4 shape: 1000-d tensor, top 10
    components, exactly T=30 sweeps, asym sketch b=2^14, B=40 (paper: 1.0 min on CPU)."""
    import torch

    n, rank, b, B = (200, 10, 1 << 12, 20) if quick else (1000, 10, 1 << 14, 40)
    Td = torch.empty(n ** 3, dtype=torch.float32, device="cuda")
    skb.gen_planted_tensor_device(ctx, n, rank, 0.01, 1234, Td.data_ptr(), dtype=np.float32)
    s = skb.AsymTensorSketchSet(n, b, B, 5, ctx)
    ctx.profile(True)
    ctx.profile_reset()
    s.accumulate_dense(Td)
    ctx.synchronize()
    build_ms = sum(ctx.profile_get(k)[0] for k in ["build_prepass", "build_main", "build_finalize"])
    ctx.profile(False)
    t0 = time.perf_counter()
    d = skb.als_fast(s, skb.AlsConfig(k=rank, max_iters=30, tol=0.0, seed=3))
    als_s = time.perf_counter() - t0
    emit({"config": "table4", "what": f"fast ALS k={rank} T=30 on the asym sketch (n={n}, b={b}, B={B})",
          "asym_build_ms": build_ms, "als_seconds": als_s, "sweeps": d.iters,
          "lambda_top3": sorted(d.lambda_.tolist(), reverse=True)[:3],
          "paper_cpu_minutes_same_b_B": 1.0})


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="0,1,2,3,4,5")
    ap.add_argument("--quick", action="store_true")
    args = ap.parse_args()
    import paper_1506_04448_b200 as skb

    ctx = skb.default_context(0)
    for c in [int(x) for x in args.configs.split(",")]:
        [c0, c1, c2, c3, c4, c5][c](skb, ctx, args.quick)


if __name__ == "__main__":
    main()
