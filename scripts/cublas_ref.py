"""Comparator only: cuBLAS (torch.matmul) time for the decode GEMM shapes, L2 flushed."""
import torch

torch.manual_seed(0)
flush = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
shapes = {"qkv": (5120, 3072), "o": (3072, 3072), "gu": (16384, 3072), "down": (3072, 8192), "head": (28672, 3072)}
for N in (16, 64, 128, 224, 256):
    line = [f"N={N}"]
    for name, (M, K) in shapes.items():
        w = torch.randn(M, K, device="cuda", dtype=torch.bfloat16)
        x = torch.randn(N, K, device="cuda", dtype=torch.bfloat16)
        ts = []
        for it in range(8):
            flush.sum()  # read-only L2 flush (clean lines)
            torch.cuda.synchronize()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record()
            y = x @ w.t()
            b.record()
            torch.cuda.synchronize()
            if it > 0:
                ts.append(a.elapsed_time(b) * 1000)
        t = sorted(ts)[len(ts) // 2]
        line.append(f"{name} {t:.1f}us {2 * M * N * K / t / 1e6:.0f}TF {M * K * 2 / t / 1e3:.0f}GB/s")
    print(" | ".join(line), flush=True)
