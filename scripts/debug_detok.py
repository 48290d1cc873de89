"""Dev script: compare detok pipeline stages with the oracle (GPU)."""
import sys, ctypes as C, numpy as np
sys.path.insert(0, '.'); sys.path.insert(0, 'baseline/_ref')
from paper_2602_00269_b200.config import tiny
from paper_2602_00269_b200.device import VoxDevice, Sampling
from oracle.snac import SnacOracle, snake, causal_dwconv, codes_from_tokens
from oracle.weights import bf16_round
cfg = tiny(max_slots=40)
dev = VoxDevice(cfg, 1234)
orc = SnacOracle(cfg, 1234); w = orc.w
rng = np.random.default_rng(0)
T = 28
toks = np.array([cfg.audio_base + (g % 7) * 4096 + rng.integers(0, 4096) for g in range(T)])
codes = codes_from_tokens(toks, T, cfg)
# oracle stages
st = []
z = orc.latents(codes)
y = bf16_round(causal_dwconv(z, w.in_dw_w, w.in_dw_b, 1)); st.append(('vq', y, 'bf'))
x = y @ w.in_pw_w.T + w.in_pw_b; st.append(('in', x, 'f'))
for b in range(4):
    s_ = w.rates[b]; sx = snake(x, w.up_alpha[b])
    prev = np.concatenate([np.zeros((1, sx.shape[1]), np.float32), sx[:-1]], 0)
    cat = bf16_round(np.concatenate([sx, prev], 1)); st.append((f'upcat{b}', cat, 'bf'))
    out = cat @ w.up_w[b].T + w.up_b[b]; x = out.reshape(out.shape[0] * s_, -1); st.append((f'up{b}', x, 'f'))
    for u, dil in enumerate((1, 3, 9)):
        U = w.ru[b][u]; y1 = snake(x, U['a1']); v = causal_dwconv(y1, U['dw_w'], U['dw_b'], dil)
        y2 = bf16_round(snake(v, U['a2'])); st.append((f'ruprep{b}{u}', y2, 'bf'))
        x = (y2 @ U['pw_w'].T + U['pw_b']) + x; st.append((f'ru{b}{u}', x, 'f'))
lib = dev.lib
tab = dev.read_weight('vq_tab', 0, (3, 4096, 768), np.uint16)
print('tabs equal', np.array_equal((tab.astype(np.uint32) << 16).view(np.float32), w.tabs))
for k, (name, ref, kind) in enumerate(st):
    slot = dev.admit(7 + k, 4, T, Sampling())
    dev.write_tokens(slot, 4, toks.tolist())
    dev._check(lib.vox_debug_detok(dev.ctx, k + 1, None, 0, None, 0))
    dev.detok(np.array([[slot, 1, 0, 28, 28, 0]], np.int32))
    n = ref.size
    of = np.zeros(n, np.float32); ob = np.zeros(n, np.uint16)
    dev._check(lib.vox_debug_detok(dev.ctx, 0, of.ctypes.data_as(C.POINTER(C.c_float)), n if kind == 'f' else 0,
                                   ob.ctypes.data_as(C.POINTER(C.c_uint16)), n))
    got = of if kind == 'f' else (ob.astype(np.uint32) << 16).view(np.float32)
    got = got.reshape(ref.shape)
    err = np.abs(got - ref)
    i = np.unravel_index(np.argmax(err), err.shape)
    print(f"{name:10s} max|d|={err.max():.4g} rms|d|={np.sqrt((err**2).mean()):.3g} ref_rms={np.sqrt((ref**2).mean()):.3g} nflip={(err>0).mean():.3g}")
    dev.release(slot)
