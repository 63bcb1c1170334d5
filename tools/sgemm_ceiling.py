"""Practical FFMA ceiling on this B200: cuBLAS SGEMM (torch fp32 matmul, TF32 off) at the FP32
engine's stage shapes (C4: per task U = Φ D is 2048 × 256 × 8192, W = Φᵀ U is 8192 × 256 × 2048; 32
tasks batched) and at a large square shape.  TFLOP/s from CUDA events (median of 10 after 3 warm-up)."""
import json
import torch

torch.backends.cuda.matmul.allow_tf32 = False
torch.backends.cudnn.allow_tf32 = False


def bench(f, flop):
    for _ in range(3):
        f()
    ts = []
    for _ in range(10):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(); f(); b.record(); torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    return flop / (ts[len(ts) // 2] * 1e-3) / 1e12


out = {}
B = 32
phi = torch.randn(B, 2048, 8192, device="cuda")
D = torch.randn(B, 8192, 256, device="cuda")
U = torch.randn(B, 2048, 256, device="cuda")
out["stage1_bmm_32x(2048x8192 @ 8192x256)"] = bench(lambda: torch.bmm(phi, D), 2.0 * B * 2048 * 8192 * 256)
out["stage2_bmm_32x(8192x2048 @ 2048x256)"] = bench(lambda: torch.bmm(phi.transpose(1, 2), U), 2.0 * B * 2048 * 8192 * 256)
a = torch.randn(8192, 8192, device="cuda")
out["square_8192"] = bench(lambda: a @ a, 2.0 * 8192 ** 3)
out["ffma_peak_1965MHz"] = 148 * 128 * 2 * 1.965e9 / 1e12
print(json.dumps(out))
