"""Where the config-1 build step's time goes outside the kernels: the bench's outer
CUDA-event time per accumulate_dense call vs the in-library event spans (build_total =
first enqueue to last kernel of run_dense_build; phases inside it)."""
import os
import sys

sys.path.insert(0, os.getcwd())
import torch

import paper_1506_04448_b200 as skb

ctx = skb.Context(0)
ext = torch.cuda.ExternalStream(ctx.stream())
T, lam, V = skb.gen_planted_tensor(400, 50, 0.01, 20150615)
Td = torch.from_numpy(T).cuda()
s = skb.SymTensorSketchSet(400, 1 << 14, 20, 20150615, ctx)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for _ in range(3):
    s.accumulate_dense(Td, True)
torch.cuda.synchronize()
for flush_on in (True, False):
    ctx.profile(True)
    ctx.profile_reset()
    evs = []
    for k in range(20):
        if flush_on:
            flush.fill_(k & 0xFF)
        torch.cuda.synchronize()
        a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(ext)
        s.accumulate_dense(Td, True)
        e.record(ext)
        evs.append((a, e))
    torch.cuda.synchronize()
    outer = sum(a.elapsed_time(e) for a, e in evs) / len(evs)
    parts = {k: ctx.profile_get(k)[0] / max(1, ctx.profile_get(k)[1]) for k in
             ["build_total", "build_prepass", "build_main", "build_finalize"]}
    ctx.profile(False)
    print(f"flush={flush_on} outer {outer:.4f} ms", {k: round(v, 4) for k, v in parts.items()})
