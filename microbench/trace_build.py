import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_1506_04448_b200 as skb
ctx = skb.default_context(0)
T, lam, V = skb.gen_planted_tensor(400, 50, 0.01, 20150615)
Td = torch.from_numpy(T).cuda()
s = skb.SymTensorSketchSet(400, 1 << 14, 20, 20150615, ctx)
for _ in range(3):
    s.accumulate_dense(Td, True)
