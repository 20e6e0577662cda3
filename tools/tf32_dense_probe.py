#!/usr/bin/env python3
"""Measured basis for DESIGN.md's tensor-core paragraph: the time of a DENSE
GEMM of a layer's shape on the tensor cores (cuBLAS through torch.matmul: TF32,
and bf16 as the 3-pass bf16x3 / TF32x3 building block), next to the fp32
pedantic SGEMM and the sparse strict kernel's time from the per-config table.
A densified tensor-core path needs ~3 such passes for fp32-level accuracy
(3xTF32) and is never bit-exact; this only sizes it.

  python tools/tf32_dense_probe.py
"""
import torch


def t_us(fn, reps=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / reps


def main():
    shapes = [("c3 512x512 @14x14 x64", 512, 512, 64 * 196), ("MBv1 pw7 512x512 @14x14 x256", 512, 512, 256 * 196),
              ("MBv1 pw13 1024x1024 @7x7 x256", 1024, 1024, 256 * 49), ("c5 1024x1024 @7x7 x1024", 1024, 1024, 1024 * 49)]
    for name, M, K, N in shapes:
        w = torch.randn(M, K, device="cuda")
        x = torch.randn(K, N, device="cuda")
        torch.backends.cuda.matmul.allow_tf32 = False
        t32 = t_us(lambda: torch.matmul(w, x))
        torch.backends.cuda.matmul.allow_tf32 = True
        ttf = t_us(lambda: torch.matmul(w, x))
        wb, xb = w.bfloat16(), x.bfloat16()
        tbf = t_us(lambda: torch.matmul(wb, xb))
        fl = 2.0 * M * K * N
        print(f"{name}: dense fp32 {t32:7.1f} us ({fl / t32 / 1e6:6.1f} TFLOP/s)  TF32 {ttf:6.1f} us ({fl / ttf / 1e6:6.1f})  "
              f"bf16 {tbf:6.1f} us ({fl / tbf / 1e6:6.1f});  3 x TF32 = {3 * ttf:6.1f} us  -> equals a sparse kernel of "
              f"{3 * ttf:.0f} us whatever the sparsity")


if __name__ == "__main__":
    main()
