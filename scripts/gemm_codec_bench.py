"""Codec-GEMM microbenchmark (K8 estimator shapes, 33,280 rows): persistent kernel MT 1 / 2
vs the 1-CTA kernel, L2 flushed between iterations (vox_gemm_test).  GPU only."""
import os
import sys

import numpy as np

sys.path.insert(0, '.')
from paper_2602_00269_b200.config import tiny  # noqa: E402
from paper_2602_00269_b200.device import VoxDevice  # noqa: E402

dev = VoxDevice(tiny(max_slots=2, detok_enabled=False), 1)
rng = np.random.default_rng(0)
for M, K in [(768, 256), (256, 256), (1024, 256), (256, 1024)]:
    N = 33280
    w = rng.integers(0, 65535, size=(M, K), dtype=np.uint16) & 0x3FFF
    x = rng.integers(0, 65535, size=(N, K), dtype=np.uint16) & 0x3FFF
    res = []
    for mode in ["0", "1", "2"]:
        os.environ["VOX_GEMM_PERSIST_TEST"] = mode
        _, ms = dev.gemm_test(w, x, None, 1, iters=5)
        by = (M * K + N * K) * 2 + N * M * 4
        res.append(f"{['1cta', 'persist1', 'persist2'][int(mode)]} {ms * 1e3:7.1f} us ({by / ms / 1e6:6.0f} GB/s, "
                   f"{2 * M * N * K / ms / 1e9:5.0f} TF/s)")
    print(f"M {M:5d} K {K:5d} N {N}: " + " | ".join(res), flush=True)
