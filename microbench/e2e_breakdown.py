"""Breakdown of the end-to-end (pinned host tensor) dense build at config 1: per-kernel
times from the library profiler, plus the DMA rate of a plain pinned H2D copy of the same
byte count for comparison."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1506_04448_b200 as skb  # noqa: E402

n = 400
ctx = skb.default_context(0)
T, lam, V = skb.gen_planted_tensor(n, 50, 0.01, 20150615)
Tp = torch.from_numpy(T).pin_memory()
s = skb.SymTensorSketchSet(n, 1 << 14, 20, 20150615, ctx)
for _ in range(3):
    s.accumulate_dense(Tp.numpy(), True)
ctx.profile(True)
ctx.profile_reset()
import time  # noqa: E402

t0 = time.perf_counter()
for _ in range(5):
    s.accumulate_dense(Tp.numpy(), True)
wall = (time.perf_counter() - t0) / 5
prof = {k: ctx.profile_get(k)[0] / 5 for k in ["build_prepass", "build_main", "build_finalize", "build_pipelined"]}
ctx.profile(False)
nbytes = n * (n + 1) * (n + 2) // 6 * 8
src = torch.empty(nbytes // 8, dtype=torch.float64).pin_memory()
dst = torch.empty(nbytes // 8, dtype=torch.float64, device="cuda")
for _ in range(3):
    dst.copy_(src, non_blocking=True)
torch.cuda.synchronize()
a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
a.record()
for _ in range(5):
    dst.copy_(src, non_blocking=True)
e.record()
torch.cuda.synchronize()
dma_ms = a.elapsed_time(e) / 5
print(json.dumps({"wall_ms_per_build": wall * 1e3, "kernel_ms": prof, "simplex_bytes": nbytes,
                  "bus_GBps_over_pipelined_build": nbytes / (max(prof["build_pipelined"], 1e-9) * 1e-3) / 1e9,
                  "dma_h2d_ms_same_bytes": dma_ms, "dma_GBps": nbytes / (dma_ms * 1e-3) / 1e9}))
