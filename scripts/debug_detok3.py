"""Dev script: isolate the detok ConvT GEMMs using the GPU's own operands (GPU)."""
import sys, ctypes as C, numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'baseline/_ref')
from paper_2602_00269_b200.config import tiny
from paper_2602_00269_b200.device import VoxDevice, Sampling
from oracle.snac import SnacOracle
cfg = tiny(max_slots=40)
dev = VoxDevice(cfg, 1234); w = SnacOracle(cfg, 1234).w
lib = dev.lib
rng = np.random.default_rng(0)
T = 28
toks = np.array([cfg.audio_base + (g % 7) * 4096 + rng.integers(0, 4096) for g in range(T)])
def run_to(stage, nf, nb):
    slot = dev.admit(stage, 4, T, Sampling()); dev.write_tokens(slot, 4, toks.tolist())
    dev._check(lib.vox_debug_detok(dev.ctx, stage, None, 0, None, 0))
    dev.detok(np.array([[slot, 1, 0, 28, 28, 0]], np.int32))
    of = np.zeros(nf, np.float32); ob = np.zeros(nb, np.uint16)
    dev._check(lib.vox_debug_detok(dev.ctx, 0, of.ctypes.data_as(C.POINTER(C.c_float)), nf, ob.ctypes.data_as(C.POINTER(C.c_uint16)), nb))
    dev.release(slot)
    return of, (ob.astype(np.uint32) << 16).view(np.float32)
# stage numbers: 1 vq, 2 in, block b: 3+8b upcat, 4+8b up, then (prep, ru) x3
n_lat = 16
for b in range(4):
    Ci, Co, s = w.ch[b], w.ch[b + 1], w.rates[b]
    up = [1, 8, 64, 256][b]
    rows = n_lat * up
    _, cat = run_to(3 + 8 * b, 1, rows * 2 * Ci)
    out, _ = run_to(4 + 8 * b, rows * s * Co, 1)
    cat = cat.reshape(rows, 2 * Ci)
    ref = (cat.astype(np.float64) @ w.up_w[b].astype(np.float64).T + w.up_b[b]).reshape(-1)
    e = np.abs(out - ref)
    print('block', b, 'rows', rows, 'K', 2 * Ci, 'M', s * Co, 'gemm max err %.3g rms %.3g' % (e.max(), np.sqrt((e**2).mean())))
    if e.max() > 1e-3:
        E = e.reshape(rows, s * Co)
        bad = np.argwhere(E > 1e-3)
        print('   bad rows', np.unique(bad[:, 0])[:20], 'bad cols', np.unique(bad[:, 1] // 128)[:20], len(bad))
