"""A few device-resident builds of one BASELINE config (for ncu captures of the build
kernels): python microbench/build_once.py [c1|c2] [reps]."""
import os
import sys

sys.path.insert(0, os.getcwd())
import numpy as np
import torch

import paper_1506_04448_b200 as skb

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
ctx = skb.Context(0)
if cfg == "c1":
    n, rank, b, B, dt, tdt = 400, 50, 1 << 14, 20, np.float64, torch.float64
else:
    n, rank, b, B, dt, tdt = 1000, 100, 1 << 16, 10, np.float32, torch.float32
Td = torch.empty(n ** 3, dtype=tdt, device="cuda")
skb.gen_planted_tensor_device(ctx, n, rank, 0.01, 20150615, Td.data_ptr(), dtype=dt)
s = skb.SymTensorSketchSet(n, b, B, 20150615, ctx)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for k in range(reps):
    flush.fill_(k)
    torch.cuda.synchronize()
    s.accumulate_dense(Td, True)
torch.cuda.synchronize()
print("ok")
