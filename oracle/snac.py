"""Causal SNAC-24kHz-style decoder restatement (TEST INFRASTRUCTURE ONLY).

The reference detokenizer emits no audio (profiles.py:333-356; its
DetokenizerCache only records windows, model_api.py:162-174), so parity is
UNPINNED by the reference.  The architecture follows public SNAC-24kHz
([3P] hubertsiuzdak/snac, not installed here): 3 codebooks x 4096 at vq
strides [4, 2, 1] summed after projection (projected tables are the
parameters), depthwise k7 + 1x1 input convs to 1024 channels, 4 decoder
blocks (Snake, transposed conv k=2s stride s, residual units with dilations
1/3/9: Snake -> depthwise k7 -> Snake -> 1x1), Snake -> k7 conv -> tanh.
Made CAUSAL (left padding; the transposed conv keeps the first T*s outputs)
so streaming with cached left context equals a full decode — this module
decodes the whole token sequence at once and the GPU's chunked, stateful
output must match it (max-abs 2e-2, SNR >= 35 dB).  Rounding points mirror
the GPU: bf16 GEMM operands, fp32 everything else.
"""

from __future__ import annotations

import numpy as np

from .weights import DetokWeights, bf16_round

f32 = np.float32
# Orpheus 7-token frame: position k -> (codebook, sub-index)
FRAME_POS = {0: (0, 0), 1: (1, 0), 2: (2, 0), 3: (2, 1), 4: (1, 1), 5: (2, 2), 6: (2, 3)}


def snake(x: np.ndarray, a: np.ndarray) -> np.ndarray:
    s = np.sin(a * x)
    return x + (f32(1.0) / (a + f32(1e-9))) * (s * s)


def causal_dwconv(x: np.ndarray, w: np.ndarray, b: np.ndarray, dil: int) -> np.ndarray:
    """x [T, C]; y[t] = b + sum_k w[:, k] * x[t - (6-k)*dil] (zero history)."""
    T, C = x.shape
    pad = np.concatenate([np.zeros((6 * dil, C), np.float32), x], axis=0)
    y = np.broadcast_to(b, (T, C)).astype(np.float32).copy()
    for k in range(7):
        off = 6 * dil - (6 - k) * dil
        y += w[:, k] * pad[off: off + T]
    return y


def codes_from_tokens(tokens: np.ndarray, n_tokens: int, cfg) -> np.ndarray:
    """Generated audio token ids -> [F, 7] codes (partial frame padded with 0)."""
    F = -(-n_tokens // cfg.frame_tokens)
    codes = np.zeros((F, 7), np.int64)
    for g in range(F * 7):
        f, k = divmod(g, 7)
        if g < n_tokens:
            c = int(tokens[g]) - cfg.audio_base - k * cfg.codebook_size
            codes[f, k] = min(max(c, 0), cfg.codebook_size - 1)
    return codes


class SnacOracle:
    def __init__(self, cfg, seed: int, weights: DetokWeights | None = None):
        self.cfg = cfg
        self.w = weights or DetokWeights(cfg, seed)

    def latents(self, codes: np.ndarray) -> np.ndarray:
        w = self.w
        F = codes.shape[0]
        z = np.empty((4 * F, w.tabs.shape[2]), np.float32)
        for f in range(F):
            for j in range(4):
                c0 = codes[f, 0]
                c1 = codes[f, 1 if j < 2 else 4]
                c2 = codes[f, (2, 3, 5, 6)[j]]
                z[4 * f + j] = (w.tabs[0, c0] + w.tabs[1, c1]) + w.tabs[2, c2]
        return z

    def decode(self, codes: np.ndarray) -> np.ndarray:
        """Full causal decode of [F, 7] codes -> PCM [F * 2048]."""
        w = self.w
        z = self.latents(codes)
        y = bf16_round(causal_dwconv(z, w.in_dw_w, w.in_dw_b, 1))
        x = y @ w.in_pw_w.T + w.in_pw_b
        for b in range(4):
            s_ = w.rates[b]
            sx = snake(x, w.up_alpha[b])
            prev = np.concatenate([np.zeros((1, sx.shape[1]), np.float32), sx[:-1]], axis=0)
            cat = bf16_round(np.concatenate([sx, prev], axis=1))
            out = cat @ w.up_w[b].T + w.up_b[b]           # [T, s*Co]
            x = out.reshape(out.shape[0] * s_, -1)         # [T*s, Co]
            for u, dil in enumerate((1, 3, 9)):
                U = w.ru[b][u]
                y1 = snake(x, U["a1"])
                v = causal_dwconv(y1, U["dw_w"], U["dw_b"], dil)
                y2 = bf16_round(snake(v, U["a2"]))
                x = (y2 @ U["pw_w"].T + U["pw_b"]) + x
        s = snake(x, w.out_alpha)
        pcm = causal_dwconv_out(s, w.out_w, w.out_b)
        return np.tanh(pcm)

    def decode_tokens(self, tokens: np.ndarray, n_tokens: int) -> np.ndarray:
        return self.decode(codes_from_tokens(tokens, n_tokens, self.cfg))


def causal_dwconv_out(x: np.ndarray, w: np.ndarray, b) -> np.ndarray:
    """k7 causal conv C -> 1: y[t] = b + sum_{c,k} w[c,k] * x[t-6+k, c]."""
    T, C = x.shape
    pad = np.concatenate([np.zeros((6, C), np.float32), x], axis=0)
    y = np.zeros(T, np.float32)
    for k in range(7):
        y += pad[k: k + T] @ w[:, k]
    return y + f32(b)


def chunk_samples(new_tokens: int, cfg) -> int:
    """PCM samples emitted for a window with new_tokens new audio tokens."""
    return (new_tokens * cfg.frame_samples) // cfg.frame_tokens
