"""Measures the roofline denominators MEASURED_PEAKS.json lacks (cuBLAS via
torch.matmul, 8192^3, best of 10 with CUDA events): FP64 DGEMM, TF32, FP32
SIMT, FP16, BF16. Writes gpurun_out/peaks.json."""
import json
import os

import torch


def bench(dtype, tf32=False, n=8192, reps=10):
    torch.backends.cuda.matmul.allow_tf32 = tf32
    a = torch.randn(n, n, device="cuda", dtype=dtype)
    b = torch.randn(n, n, device="cuda", dtype=dtype)
    for _ in range(3):
        a @ b
    best = 1e9
    for _ in range(reps):
        s, e = torch.cuda.Event(True), torch.cuda.Event(True)
        s.record(); a @ b; e.record(); e.synchronize()
        best = min(best, s.elapsed_time(e) * 1e-3)
    return 2 * n ** 3 / best / 1e12


out = {
    "fp64_dgemm_tflops": bench(torch.float64, n=8192, reps=5),
    "tf32_tflops": bench(torch.float32, tf32=True),
    "fp32_simt_tflops": bench(torch.float32, tf32=False, reps=5),
    "fp16_tflops": bench(torch.float16),
    "bf16_tflops": bench(torch.bfloat16),
    "how": "torch.matmul 8192^3 (2n^3 flops), best of 10 (5 for fp64/fp32), CUDA events",
    "gpu": torch.cuda.get_device_name(),
}
out["tf32x3_effective_tflops"] = out["tf32_tflops"] / 3
os.makedirs("gpurun_out", exist_ok=True)
json.dump(out, open("gpurun_out/peaks.json", "w"), indent=1)
print(json.dumps(out))
