"""Dev script: streaming detok error pattern per chunk (GPU)."""
import sys, numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'baseline/_ref')
from paper_2602_00269_b200.config import tiny
from paper_2602_00269_b200.device import VoxDevice, Sampling
from paper_2602_00269_b200._ref import profiles
from oracle.snac import SnacOracle
cfg = tiny(max_slots=8)
dev = VoxDevice(cfg, 1234); orc = SnacOracle(cfg, 1234)
rng = np.random.default_rng(0)
T = 64
toks = np.array([cfg.audio_base + (g % 7) * 4096 + rng.integers(0, 4096) for g in range(T)])
ref = orc.decode_tokens(toks, T)
prof = profiles.builtin_profile('orpheus_like')
slot = dev.admit(3, 4, T, Sampling()); dev.write_tokens(slot, 4, toks.tolist())
emitted, off = 0, 0
while True:
    w = profiles.chunk_ready(T, emitted, prof, True)
    if w is None: break
    out, _ = dev.detok(np.array([[slot, w.index, w.start, w.length, w.new_tokens, int(w.final)]], np.int32))
    o = out[0]; r = ref[off:off + len(o)]; d = np.abs(o - r)
    print(w.index, len(o), 'max %.4f at %d' % (d.max(), d.argmax()), 'first64 %.4f' % d[:64].max(), 'rms %.4f' % np.sqrt((d**2).mean()), 'sig %.3f' % np.sqrt((r**2).mean()))
    off += len(o); emitted += 1
# whole sequence in one window-less decode: first window only for a fresh slot with 28 tokens
