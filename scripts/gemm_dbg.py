"""Per-CTA phase stamps of the decode GEMM (gemm_mc_kernel, VOX_GEMM_DBG=1). GPU only."""
import os
import sys

import numpy as np

sys.path.insert(0, '.')
from paper_2602_00269_b200.config import tiny  # noqa: E402
from paper_2602_00269_b200.device import VoxDevice  # noqa: E402

os.environ["VOX_GEMM_PACKED_TEST"] = "1"
os.environ["VOX_GEMM_DBG"] = "1"
dev = VoxDevice(tiny(max_slots=2, detok_enabled=False), 1)
rng = np.random.default_rng(0)
for name, M, K, N, s in [("gu", 16384, 3072, 224, 1), ("gu", 16384, 3072, 16, 1), ("qkv", 5120, 3072, 224, 3),
                         ("qkv", 5120, 3072, 224, 1), ("down", 3072, 8192, 224, 5), ("o", 3072, 3072, 224, 6)]:
    w = rng.integers(0, 65535, size=(M, K), dtype=np.uint16) & 0x3FFF
    x = rng.integers(0, 65535, size=(N, K), dtype=np.uint16) & 0x3FFF
    _, ms = dev.gemm_test(w, x, None, s, iters=4)
    print(name, M, K, N, "s", s, "%.1f us" % (ms * 1000), "%.0f GB/s" % (M * K * 2 / ms / 1e6),
          "%.0f TF" % (2 * M * N * K / ms / 1e9), flush=True)
