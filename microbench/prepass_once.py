"""Two config-1 device-resident builds (for an ncu capture of the pre-pass / main pass)."""
import os
import sys

sys.path.insert(0, os.getcwd())
import torch

import paper_1506_04448_b200 as skb

ctx = skb.Context(0)
T, lam, V = skb.gen_planted_tensor(400, 50, 0.01, 20150615)
Td = torch.from_numpy(T).cuda()
s = skb.SymTensorSketchSet(400, 1 << 14, 20, 20150615, ctx)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for k in range(2):
    flush.fill_(k)
    torch.cuda.synchronize()
    s.accumulate_dense(Td, True)
torch.cuda.synchronize()
print("ok")
