"""Microbenchmark: tcgen05 GEMM time vs (rows N, tile BN, split-K) at Orpheus shapes (GPU)."""
import os
import sys

import numpy as np

sys.path.insert(0, '.')
sys.path.insert(0, 'baseline/_ref')
from paper_2602_00269_b200.config import tiny  # noqa: E402
from paper_2602_00269_b200.device import VoxDevice  # noqa: E402

dev = VoxDevice(tiny(max_slots=2, detok_enabled=False), 1)
rng = np.random.default_rng(0)
shapes = {"qkv": (5120, 3072), "o": (3072, 3072), "gu": (16384, 3072), "down": (3072, 8192)}
for name, (M, K) in shapes.items():
    w = rng.integers(0, 65535, size=(M, K), dtype=np.uint16) & 0x3FFF  # small finite bf16 bits
    for N in (16, 64, 256):
        x = rng.integers(0, 65535, size=(N, K), dtype=np.uint16) & 0x3FFF
        res = []
        for bn in (16, 32, 64, 128, 256):
            if bn > max(16, 1 << (N - 1).bit_length()) or bn < N // 4:
                continue
            os.environ["VOX_GEMM_BN_TEST"] = str(bn)
            for s in (1, 2, 3, 4, 6, 8, 12):
                if K // 64 // s < 2:
                    continue
                _, ms = dev.gemm_test(w, x, None, s, iters=6)
                gbs = M * K * 2 / (ms * 1e-3) / 1e9
                res.append((ms * 1000, bn, s, gbs))
        res.sort()
        print(name, "N=%d" % N, " | ".join("bn%d s%d %.1fus %.0fGB/s" % (bn, s, us, g) for us, bn, s, g in res[:6]),
              flush=True)
