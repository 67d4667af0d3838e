"""Tensor-pipe counter calibration: a known-peak GEMM (torch.matmul bf16 8192^3,
cuBLAS) run a few times, to be profiled by ncu next to the attention kernel -- the counter whose
active fraction matches the GEMM's achieved / peak FLOP rate at the profiled clock is the one that
tracks UTCHMMA.  usage (GPU box): ncu --metrics <list> -k regex:gemm|nvjet|cutlass python tools/calib_tensor.py"""
import torch

n = 8192
a = torch.randn(n, n, dtype=torch.bfloat16, device="cuda")
b = torch.randn(n, n, dtype=torch.bfloat16, device="cuda")
for _ in range(3):
    c = a @ b
torch.cuda.synchronize()
s, e = torch.cuda.Event(True), torch.cuda.Event(True)
s.record()
for _ in range(10):
    c = a @ b
e.record()
torch.cuda.synchronize()
ms = s.elapsed_time(e) / 10
print(f"matmul bf16 {n}^3: {ms:.3f} ms  {2 * n ** 3 / ms / 1e9:.1f} TFLOP/s")
