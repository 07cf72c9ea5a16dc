"""TF32 tensor-core peak of this B200 (the roofline denominator of XKNN_PREC_FP32's 3xTF32 GEMMs),
measured the way MEASURED_PEAKS.json measures bf16: cuBLAS (torch.matmul, fp32 inputs with TF32
allowed) 8192^3, best of 10 (burst) and back to back for 4 s (sustained), CUDA events.

    python tools/measure_tf32.py > profiles/r02/tf32_peak.json
"""
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
best = 0.0
for _ in range(10):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    torch.matmul(a, b, out=c)
    e1.record()
    e1.synchronize()
    best = max(best, 2.0 * n ** 3 / (e0.elapsed_time(e1) / 1e3) / 1e12)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t0 = time.time()
e0.record()
iters = 0
while time.time() - t0 < 4.0:
    for _ in range(10):
        torch.matmul(a, b, out=c)
    iters += 10
    torch.cuda.synchronize()
e1.record()
e1.synchronize()
sus = 2.0 * n ** 3 * iters / (e0.elapsed_time(e1) / 1e3) / 1e12
print(json.dumps({"tf32_tflops": round(best, 1), "tf32_tflops_sustained": round(sus, 1),
                  "gpu": torch.cuda.get_device_name(), "torch": torch.__version__,
                  "how": "torch.matmul fp32 8192^3 with allow_tf32 (cuBLAS TF32 tensor cores): "
                         "best of 10 (burst), back to back for 4 s (sustained), CUDA events"}))
