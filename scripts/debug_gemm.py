"""Dev script: GEMM relative accuracy vs fp64 (GPU)."""
import sys, numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'baseline/_ref')
from paper_2602_00269_b200.config import tiny
from paper_2602_00269_b200.device import VoxDevice
from oracle.weights import bf16_round
dev = VoxDevice(tiny(max_slots=2, detok_enabled=False), 1)
bits = lambda a: (bf16_round(a).view(np.uint32) >> 16).astype(np.uint16)
for (M, N, K, sp) in [(128, 16, 64, 1), (128, 16, 1024, 1), (512, 128, 1024, 1), (1024, 256, 2048, 1), (256, 64, 512, 4)]:
    rng = np.random.default_rng(1)
    w = bf16_round(rng.uniform(-1, 1, (M, K)).astype(np.float32)); x = bf16_round(rng.uniform(-1, 1, (N, K)).astype(np.float32))
    out, _ = dev.gemm_test(bits(w), bits(x), None, sp)
    ref = x.astype(np.float64) @ w.astype(np.float64).T
    f32 = x @ w.T
    e = np.abs(out - ref); e2 = np.abs(f32 - ref)
    print(M, N, K, sp, 'gpu max %.3g rms %.3g | numpy-f32 max %.3g rms %.3g | scale %.3g' % (e.max(), np.sqrt((e**2).mean()), e2.max(), np.sqrt((e2**2).mean()), np.abs(ref).max()))
    # structure: which (n, m) are worst
    i = np.unravel_index(np.argmax(e), e.shape); print('   worst at', i)
