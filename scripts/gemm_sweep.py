"""Microbenchmark: tcgen05 GEMM time vs (tile BN, weight sub-tiles MT, split-K) at the
Orpheus-3B decode shapes, L2 flushed before every timed launch (weights stream
from HBM as inside a decode step).  GPU only."""
import os
import sys

import numpy as np

sys.path.insert(0, '.')
sys.path.insert(0, 'baseline/_ref')
from paper_2602_00269_b200.config import tiny  # noqa: E402
from paper_2602_00269_b200.device import VoxDevice  # noqa: E402

os.environ.setdefault("VOX_GEMM_PACKED_TEST", "1")  # the decode path streams packed tiles
dev = VoxDevice(tiny(max_slots=2, detok_enabled=False), 1)
rng = np.random.default_rng(0)
shapes = {"qkv": (5120, 3072), "o": (3072, 3072), "gu": (16384, 3072), "down": (3072, 8192),
          "head": (28672, 3072)}
Ns = [int(x) for x in os.environ.get("SWEEP_N", "16,64,128,224,256").split(",")]
for name, (M, K) in shapes.items():
    w = rng.integers(0, 65535, size=(M, K), dtype=np.uint16) & 0x3FFF  # small finite bf16 bits
    for N in Ns:
        x = rng.integers(0, 65535, size=(N, K), dtype=np.uint16) & 0x3FFF
        res = []
        os.environ.pop("VOX_GEMM_BN_TEST", None)
        os.environ.pop("VOX_GEMM_MT_TEST", None)
        os.environ.pop("VOX_GEMM_SPLITS_TEST", None)
        plan = dev.gemm_plan(M, N, K) if hasattr(dev, "gemm_plan") else None
        for mt in [int(v) for v in os.environ.get("SWEEP_MT", "1,2").split(",")]:
            for bn in (16, 32, 64, 128, 256):
                if bn > max(16, 1 << (N - 1).bit_length()) or bn < N // 4:
                    continue
                os.environ["VOX_GEMM_BN_TEST"] = str(bn)
                os.environ["VOX_GEMM_MT_TEST"] = str(mt)
                for s in (1, 2, 3, 4, 6, 8, 12, 16):
                    if K // 64 // s < 2:
                        continue
                    _, ms = dev.gemm_test(w, x, None, s, iters=6)
                    gbs = M * K * 2 / (ms * 1e-3) / 1e9
                    tf = 2 * M * N * K / (ms * 1e-3) / 1e12
                    res.append((ms * 1000, bn, mt, s, gbs, tf))
        res.sort()
        print(name, "N=%d" % N, " | ".join("bn%d mt%d s%d %.1fus %.0fGB/s %.0fTF" % (bn, mt, s, us, g, t)
                                        for us, bn, mt, s, g, t in res[:5]), flush=True)
