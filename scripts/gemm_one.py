"""One decode-GEMM launch (gemm_mc_kernel) at a decode shape (for ncu). GPU only."""
import os
import sys

import numpy as np

sys.path.insert(0, '.')
from paper_2602_00269_b200.config import tiny  # noqa: E402
from paper_2602_00269_b200.device import VoxDevice  # noqa: E402

os.environ.setdefault("VOX_GEMM_PACKED_TEST", "1")
M, K, N, s = (int(v) for v in os.environ.get("GEMM_SHAPE", "16384,3072,224,1").split(","))
dev = VoxDevice(tiny(max_slots=2, detok_enabled=False), 1)
rng = np.random.default_rng(0)
w = rng.integers(0, 65535, size=(M, K), dtype=np.uint16) & 0x3FFF
x = rng.integers(0, 65535, size=(N, K), dtype=np.uint16) & 0x3FFF
_, ms = dev.gemm_test(w, x, None, s, iters=2)
print("%.1f us" % (ms * 1000))
