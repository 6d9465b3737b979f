"""Sustained tensor-core throughput and SM clock under the power cap, per operand dtype.

torch.matmul (cuBLAS) [8192 x 8192] x [8192 x 8192] back to back for `secs` seconds, with
nvidia-smi clocks / power sampled during the run; data: N(0,1) (bf16) or N(0,1) scaled
by 2^12 (fp16: the shadow's scaling puts max |x| into [2^14, 2^15)).
Used to explain the fp16 vs bf16 selection-pass clock difference (profiles/r02_power_probe.txt)."""
import json
import subprocess
import sys
import time

import torch

secs = float(sys.argv[1]) if len(sys.argv) > 1 else 4.0
for name, dt, scale in (("bf16", torch.bfloat16, 1.0), ("fp16", torch.float16, 4096.0), ("fp16_unscaled", torch.float16, 1.0)):
    a = (torch.randn(8192, 8192, device="cuda") * scale).to(dt)
    b = (torch.randn(8192, 8192, device="cuda") * scale).to(dt)
    for _ in range(3):
        torch.matmul(a, b)
    torch.cuda.synchronize()
    smi = subprocess.Popen(["nvidia-smi", "--query-gpu=clocks.sm,power.draw", "--format=csv,noheader,nounits",
                            "-lms", "200"], stdout=subprocess.PIPE, text=True)
    time.sleep(0.5)
    n = 0
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.time()
    e0.record()
    while time.time() - t0 < secs:
        for _ in range(10):
            torch.matmul(a, b)
        n += 10
        torch.cuda.synchronize()
    e1.record()
    torch.cuda.synchronize()
    smi.terminate()
    lines = [l.split(",") for l in smi.stdout.read().strip().splitlines() if l.count(",") == 1]
    clk = sorted(float(x[0]) for x in lines[2:]) or [0]
    pw = sorted(float(x[1]) for x in lines[2:]) or [0]
    tf = n * 2 * 8192 ** 3 / (e0.elapsed_time(e1) / 1e3) / 1e12
    print(json.dumps({"dtype": name, "tflops": round(tf, 1), "sm_mhz_median": clk[len(clk) // 2],
                      "power_w_median": pw[len(pw) // 2]}), flush=True)
