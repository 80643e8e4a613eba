"""Times the symmetric moment accumulation (config-3 shape: n=1000, b=2^14, B=10) on a
block of device-resident samples with the in-library CUDA-event profiler.
Usage: NS_=16384 python microbench/moment_step.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1506_04448_b200 as skb  # noqa: E402

n, b, B = int(os.environ.get("N_", 1000)), int(os.environ.get("B_", 1 << 14)), 10
Ns = int(os.environ.get("NS_", 1 << 16))
reps = int(os.environ.get("REPS_", 3))
ctx = skb.default_context(0)
s = skb.SymTensorSketchSet(n, b, B, 4, ctx)
g = torch.Generator(device="cuda").manual_seed(1)
X = torch.randn(Ns, n, generator=g, device="cuda", dtype=torch.float64)
w = torch.full((Ns,), 1.0 / Ns, device="cuda", dtype=torch.float64)
s.accumulate_moment(X, w)
ctx.synchronize()
ctx.profile(True)
ctx.profile_reset()
for _ in range(reps):
    s.accumulate_moment(X, w)
ctx.synchronize()
mom = ctx.profile_get("moment")[0] / reps
inv = ctx.profile_get("freq_inverse")[0] / reps
comb = ctx.profile_get("combine")[0] / reps
ctx.profile(False)
logb = b.bit_length() - 1
fft_flops = Ns * B * 5 * b * logb
print(json.dumps({"n": n, "b": b, "B": B, "samples": Ns, "moment_ms": mom, "freq_inverse_ms": inv, "combine_ms": comb,
                  "samples_per_s": Ns / ((mom + inv + comb) * 1e-3),
                  "fft_tflops_nominal": fft_flops / (mom * 1e-3) / 1e12}))
