"""cuBLAS fp32 SGEMM (TF32 off) on this B200: the library bar for the tuned
SIMT SGEMM family (run under gpurun).  torch.matmul -> cublasSgemm-class
kernels; CUDA events, best of 20 after warm-up.

  python tools/cublas_ref.py [--out gpurun_out/cublas_sgemm.json]
"""
import argparse
import json

import torch

ap = argparse.ArgumentParser()
ap.add_argument("--out")
a = ap.parse_args()
torch.backends.cuda.matmul.allow_tf32 = False
torch.backends.cudnn.allow_tf32 = False
res = {}
for n in (1024, 2048, 4096, 8192):
    A = torch.rand(n, n, device="cuda")
    B = torch.rand(n, n, device="cuda")
    for _ in range(3):
        C = A @ B
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(20):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        C = A @ B
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1))
    res[n] = {"ms": best, "tflops": 2 * n ** 3 / best / 1e9}
    print(f"cuBLAS fp32 {n}^3: {best:.4f} ms = {res[n]['tflops']:.1f} TFLOP/s", flush=True)
if a.out:
    open(a.out, "w").write(json.dumps(res))
