"""Host-side breakdown of a tiny accumulate_dense (n=8): ctypes round trip, the full call
by wall clock, and the call's CUDA-event span, to size the fixed per-call overhead."""
import os
import sys
import time

sys.path.insert(0, os.getcwd())
import numpy as np
import torch

import paper_1506_04448_b200 as skb

ctx = skb.Context(0)
ext = torch.cuda.ExternalStream(ctx.stream())
for n, b, B in ((8, 1 << 14, 20), (8, 1 << 10, 2), (400, 1 << 14, 20)):
    T = torch.from_numpy(skb.gen_planted_tensor(n, 2, 0.01, 1)[0]).cuda()
    s = skb.SymTensorSketchSet(n, b, B, 3, ctx)
    for _ in range(5):
        s.accumulate_dense(T, True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(200):
        s.n()
    t_n = (time.perf_counter() - t0) / 200 * 1e6
    walls, evs = [], []
    for _ in range(50):
        torch.cuda.synchronize()
        a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        a.record(ext)
        s.accumulate_dense(T, True)
        e.record(ext)
        walls.append(time.perf_counter() - t0)
        torch.cuda.synchronize()
        evs.append(a.elapsed_time(e))
    ctx.profile(True)
    ctx.profile_reset()
    for _ in range(50):
        s.accumulate_dense(T, True)
    torch.cuda.synchronize()
    parts = {k: round(ctx.profile_get(k)[0] / max(1, ctx.profile_get(k)[1]) * 1e3, 1) for k in
             ["build_total", "build_prepass", "build_main", "build_finalize"]}
    ctx.profile(False)
    print(f"n={n} b={b} B={B}: ctypes n() {t_n:.2f} us, call wall median {np.median(walls) * 1e6:.1f} us, "
          f"event median {np.median(evs) * 1e3:.1f} us, scopes (us) {parts}")
