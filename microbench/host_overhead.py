"""Host-side cost of one accumulate_dense call: a tiny build (n=8) whose GPU work is a
few microseconds, timed by wall clock and by CUDA events around the call."""
import os
import sys
import time

sys.path.insert(0, os.getcwd())
import numpy as np
import torch

import paper_1506_04448_b200 as skb

ctx = skb.Context(0)
ext = torch.cuda.ExternalStream(ctx.stream())
for n in (8, 400):
    T = torch.from_numpy(skb.gen_planted_tensor(n, 2, 0.01, 1)[0]).cuda()
    s = skb.SymTensorSketchSet(n, 1 << 14, 20, 3, ctx)
    for _ in range(5):
        s.accumulate_dense(T, True)
    torch.cuda.synchronize()
    walls, evs = [], []
    for _ in range(50):
        a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        a.record(ext)
        s.accumulate_dense(T, True)
        e.record(ext)
        torch.cuda.synchronize()
        walls.append(time.perf_counter() - t0)
        evs.append((a, e))
    ev = [a.elapsed_time(e) for a, e in evs]
    print(f"n={n}: wall median {np.median(walls)*1e3:.4f} ms, event median {np.median(ev):.4f} ms")
    # raw pieces: python arg conversion and an empty ctypes round trip
    t0 = time.perf_counter()
    for _ in range(1000):
        skb._tensor_arg(T, n)
    print(f"  _tensor_arg {(time.perf_counter()-t0)*1e3:.4f} us/call")
