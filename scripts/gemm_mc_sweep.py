"""Microbenchmark: cluster-multicast GEMM (gemm_mc_kernel) vs the 1-CTA kernel at the
Orpheus-3B decode shapes, L2 flushed before every timed launch.  GPU only."""
import os
import sys

import numpy as np

sys.path.insert(0, '.')
from paper_2602_00269_b200.config import tiny  # noqa: E402
from paper_2602_00269_b200.device import VoxDevice  # noqa: E402

os.environ["VOX_GEMM_PACKED_TEST"] = "1"
dev = VoxDevice(tiny(max_slots=2, detok_enabled=False), 1)
rng = np.random.default_rng(0)
shapes = {"qkv": (5120, 3072), "o": (3072, 3072), "gu": (16384, 3072), "down": (3072, 8192),
          "head": (28672, 3072)}
Ns = [int(v) for v in os.environ.get("SWEEP_N", "16,64,128,224,256").split(",")]
for name, (M, K) in shapes.items():
    w = rng.integers(0, 65535, size=(M, K), dtype=np.uint16) & 0x3FFF
    for N in Ns:
        x = rng.integers(0, 65535, size=(N, K), dtype=np.uint16) & 0x3FFF
        res = []
        for cs in (1, 2, 4, 8):
            os.environ["VOX_GEMM_CS_TEST"] = str(cs)
            os.environ.pop("VOX_GEMM_MC", None)
            for s in (1, 2, 3, 4, 5, 6, 8):
                if K // 64 // s < 2:
                    continue
                _, ms = dev.gemm_test(w, x, None, s, iters=6)
                res.append((ms * 1000, "mc cs%d s%d" % (cs, s)))
        os.environ["VOX_GEMM_MC"] = "0"
        os.environ.pop("VOX_GEMM_CS_TEST", None)
        for s in (1, 2, 3, 4, 6):
            _, ms = dev.gemm_test(w, x, None, s, iters=6)
            res.append((ms * 1000, "1cta s%d" % s))
        os.environ.pop("VOX_GEMM_MC", None)
        res.sort()
        print(name, "N=%d" % N, "ideal %.1fus |" % (M * K * 2 / 6.55e12 * 1e6),
              " | ".join("%s %.1fus %.0fGB/s" % (t, us, M * K * 2 / (us * 1e-6) / 1e9) for us, t in res[:6]),
              flush=True)
