"""Measure the dense TF32 tensor-core peak the same way MEASURED_PEAKS.json measures bf16:
torch.matmul on fp32 8192^3 with allow_tf32 (cuBLAS), best of 10 (burst) and back to back for 4 s
(sustained).  Prints one JSON line (used as a reference denominator beside the nominal-ratio figure)."""
import json
import time

import torch

torch.backends.cuda.matmul.allow_tf32 = True
n = 8192
a = torch.randn(n, n, device="cuda")
b = torch.randn(n, n, device="cuda")
c = torch.empty(n, n, device="cuda")
for _ in range(3):
    torch.matmul(a, b, out=c)
torch.cuda.synchronize()
best = 1e9
for _ in range(10):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    torch.matmul(a, b, out=c)
    e.record()
    torch.cuda.synchronize()
    best = min(best, s.elapsed_time(e))
flop = 2.0 * n ** 3
t0 = time.time()
s = torch.cuda.Event(enable_timing=True)
e = torch.cuda.Event(enable_timing=True)
s.record()
it = 0
while time.time() - t0 < 4.0:
    for _ in range(10):
        torch.matmul(a, b, out=c)
    it += 10
    torch.cuda.synchronize()
e.record()
torch.cuda.synchronize()
sus = flop * it / (s.elapsed_time(e) / 1e3) / 1e12
print(json.dumps({"tf32_tflops": flop / (best / 1e3) / 1e12, "tf32_tflops_sustained": sus,
                  "how": "torch.matmul fp32 8192^3 allow_tf32 (cuBLAS): best of 10 / back to back 4 s"}))
