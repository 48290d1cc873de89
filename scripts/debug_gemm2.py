"""Dev script: GEMM shapes used by the detokenizer (GPU)."""
import sys, numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'baseline/_ref')
from paper_2602_00269_b200.config import tiny
from paper_2602_00269_b200.device import VoxDevice
from oracle.weights import bf16_round
dev = VoxDevice(tiny(max_slots=2, detok_enabled=False), 1)
bits = lambda a: (bf16_round(a).view(np.uint32) >> 16).astype(np.uint16)
for (M, N, K) in [(2048, 128, 1024), (512, 128, 1024), (1024, 128, 1024), (2048, 128, 512), (2048, 64, 1024), (2048, 100, 1024), (4096, 128, 1024), (256, 128, 256), (512, 128, 512)]:
    rng = np.random.default_rng(1)
    w = bf16_round(rng.uniform(-1, 1, (M, K)).astype(np.float32)); x = bf16_round(rng.uniform(-1, 1, (N, K)).astype(np.float32))
    out, _ = dev.gemm_test(bits(w), bits(x), None, 1)
    ref = x.astype(np.float64) @ w.astype(np.float64).T
    e = np.abs(out - ref)
    print(M, N, K, 'max %.3g rms %.3g' % (e.max(), np.sqrt((e**2).mean())))
