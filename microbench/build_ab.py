"""Device-resident build time of one BASELINE config (L2 flushed before each build), and
a checksum of the sketch: python microbench/build_ab.py [c1|c2] [reps]. Used for kernel
A/B runs (each arm in its own process)."""
import hashlib
import os
import sys

sys.path.insert(0, os.getcwd())
import numpy as np
import torch

import paper_1506_04448_b200 as skb

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
ctx = skb.Context(0)
if cfg == "c1":
    n, rank, b, B, dt, tdt = 400, 50, 1 << 14, 20, np.float64, torch.float64
else:
    n, rank, b, B, dt, tdt = 1000, 100, 1 << 16, 10, np.float32, torch.float32
Td = torch.empty(n ** 3, dtype=tdt, device="cuda")
skb.gen_planted_tensor_device(ctx, n, rank, 0.01, 20150615, Td.data_ptr(), dtype=dt)
ext = torch.cuda.ExternalStream(ctx.stream())
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
s = skb.SymTensorSketchSet(n, b, B, 20150615, ctx)
for _ in range(3):
    s.accumulate_dense(Td, True)
torch.cuda.synchronize()
ms = []
for k in range(reps):
    flush.fill_(k & 0xFF)
    torch.cuda.synchronize()
    a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(ext)
    s.accumulate_dense(Td, True)
    e.record(ext)
    torch.cuda.synchronize()
    ms.append(a.elapsed_time(e))
ctx.profile(True)
ctx.profile_reset()
for k in range(reps):
    flush.fill_(k & 0xFF)
    torch.cuda.synchronize()
    s.accumulate_dense(Td, True)
torch.cuda.synchronize()
mm, mc = ctx.profile_get("build_main")
ctx.profile(False)
t = skb.SymTensorSketchSet(n, b, B, 20150615, ctx)
t.accumulate_dense(Td, True)
h = hashlib.sha1(t.data().tobytes()).hexdigest()[:16]
print(f"{cfg} env={os.environ.get('SKC_CLS_FLAT', '-')} step_ms={np.median(ms):.4f} min={min(ms):.4f} main_ms={mm / mc:.4f} sha={h}")
