"""Dense builds whose window count is near or above the CTA count (lockstep policy check):
N_=400 B_=65536 R_=20 python microbench/lock_many_windows.py  (G = 160 windows)
F32=1 N_=1000 B_=131072 R_=10 python microbench/lock_many_windows.py  (G = 80 windows)"""
import os, sys, time
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np, torch
import paper_1506_04448_b200 as skb
ctx = skb.default_context(0)
n, b, B = int(os.environ.get("N_", 400)), int(os.environ.get("B_", 1 << 16)), int(os.environ.get("R_", 20))
f32 = bool(os.environ.get("F32"))
Td = torch.empty(n ** 3, dtype=torch.float32 if f32 else torch.float64, device="cuda")
skb.gen_planted_tensor_device(ctx, n, 50, 0.01, 7, Td.data_ptr(), dtype=np.float32 if f32 else np.float64)
s = skb.SymTensorSketchSet(n, b, B, 11, ctx)
ext = torch.cuda.ExternalStream(ctx.stream())
for _ in range(2): s.accumulate_dense(Td, True)
torch.cuda.synchronize()
ms = []
for k in range(6):
    a, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(ext); s.accumulate_dense(Td, True); e.record(ext); torch.cuda.synchronize(); ms.append(a.elapsed_time(e))
print(f"n={n} b={b} B={B} f32={f32} build ms", np.median(ms))
if os.environ.get("CHECK"):
    import oracle_py as O
    t = skb.SymTensorSketchSet(n, b, B, 11, ctx)
    t.accumulate_dense(Td, True)
    o = O.SymSet(n, b, B, 11)
    o.accumulate_dense(Td.cpu().numpy().astype(np.float64).reshape(n, n, n), True)
    d, od = t.data(), o.data()
    print("rel err", float(np.max(np.linalg.norm(d - od, axis=1) / np.linalg.norm(od, axis=1))))
