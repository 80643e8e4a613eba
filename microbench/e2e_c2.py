"""End-to-end config-2 build from a pinned host tensor (the bench's e2e leg alone):
python microbench/e2e_c2.py  -> ms per build and effective bus GB/s."""
import os
import sys

sys.path.insert(0, os.getcwd())
import numpy as np
import torch

import paper_1506_04448_b200 as skb

n, b, B = 1000, 1 << 16, 10
ctx = skb.Context(0)
ext = torch.cuda.ExternalStream(ctx.stream())
Td = torch.empty(n ** 3, dtype=torch.float32, device="cuda")
skb.gen_planted_tensor_device(ctx, n, 100, 0.01, 20150615, Td.data_ptr(), dtype=np.float32)
Tp = torch.empty(n ** 3, dtype=torch.float32).pin_memory()
Tp.copy_(Td)
del Td
Tn = Tp.numpy()
s = skb.SymTensorSketchSet(n, b, B, 20150615, ctx)
for _ in range(2):
    s.accumulate_dense(Tn, True)
torch.cuda.synchronize()
ms = []
for _ in range(8):
    a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(ext)
    s.accumulate_dense(Tn, True)
    e.record(ext)
    torch.cuda.synchronize()
    ms.append(a.elapsed_time(e))
m = float(np.median(ms))
print(f"e2e build ms {m:.3f}  bus GB/s {n * (n + 1) * (n + 2) / 6 * 4 / m / 1e6:.1f}")
