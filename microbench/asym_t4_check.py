"""Table-4 shape asym build: class-list vs contiguous-window kernel agreement, and ALS timing."""
import os, subprocess, sys, json, time
sys.path.insert(0, os.getcwd())
code = r'''
import sys, numpy as np, torch, time
sys.path.insert(0, ".")
import paper_1506_04448_b200 as skb
ctx = skb.default_context(0)
n, rank, b, B = 1000, 10, 1 << 14, 40
Td = torch.empty(n ** 3, dtype=torch.float32, device="cuda")
skb.gen_planted_tensor_device(ctx, n, rank, 0.01, 1234, Td.data_ptr(), dtype=np.float32)
s = skb.AsymTensorSketchSet(n, b, B, 5, ctx)
s.accumulate_dense(Td)
np.save(sys.argv[1], s.data())
for rep in range(2):
    t0 = time.perf_counter()
    d = skb.als_fast(s, skb.AlsConfig(k=rank, max_iters=30, tol=0.0, seed=3))
    print("als", rep, time.perf_counter() - t0, sorted(d.lambda_.tolist(), reverse=True)[:3])
'''
for kern in ("cls", "flat"):
    env = dict(os.environ)
    if kern == "flat":
        env["SKC_BUILD_KERNEL"] = "flat"
    subprocess.run([sys.executable, "-c", code, f"/tmp/t4_{kern}.npy"], check=True, env=env)
import numpy as np
a, b = np.load("/tmp/t4_cls.npy"), np.load("/tmp/t4_flat.npy")
num = np.linalg.norm(a - b, axis=-1); den = np.linalg.norm(b, axis=-1)
print("rel per replicate max", float(np.max(num / den)))
