"""CosyVoice2-style chunked detokenizer restatement (TEST INFRASTRUCTURE ONLY).

The reference's detokenizer is a stub (profiles.py:333-356: it records windows and
returns a playback duration), so the algorithm is the public CosyVoice2 token2wav
([3P] FunAudioLLM/CosyVoice ``CausalMaskedDiffWithXvec`` flow + ``HiFTGenerator``,
NOT installed here -- parity UNPINNED by a third-party run; restated from the
published architecture) at the config of
``paper_2602_00269_b200.config.CosyDetokConfig``:

  per call (VoxServe's chunking; profiles.py:135 ref_window_tokens=50):
    tokens = [50 reference tokens of the request | the chunk's new tokens]  (T rows)
    h   = Emb[tokens]; enc_layers x pre-LN transformer (full attention, RoPE);
    mu  = LN(h) W_mu + b  repeated x2 -> 2T mel frames (50 Hz)
    x0  = seeded noise (request seed, call index); n_steps Euler steps on the cosine
          schedule t_i = 1 - cos(pi/2 * i/N) of  dx/dt = (1+l) v(x, mu, spk, cond, t) - l v(x, 0, 0, 0, t)
          (classifier-free guidance l = cfg_rate); v = estimator: [x|mu|spk|cond] W_in + b_in
          + temb(t) -> est_layers transformer -> LN -> W_out;  cond = reference mel on the
          first 2 * ref_tokens frames, 0 after
    mel = x_N of the 2 * new frames
  vocoder (STATEFUL across a request's calls; causal, so chunked == whole sequence):
    k7 conv 80 -> 512; per ratio 8/5/3: LReLU(0.1), ConvT(k 2r, stride r) halving
    channels, residual block LReLU-k3-LReLU-k3 (+x); LReLU, k7 conv -> 9 log-magnitudes +
    9 phase logits; causal iSTFT (periodic Hann 16, hop 4, overlap-add of the last 4
    frames / 1.5): 480 samples per mel frame.

``exact=False`` mirrors the device's rounding points (bf16 GEMM operands); the GPU
must match within max-abs 2e-2 / SNR >= 35 dB on the PCM.
"""

from __future__ import annotations

import math

import numpy as np

from .weights import CosyDetokWeights, bf16_round, cosy_noise, cosy_request_tensors

f32 = np.float32


def _ln(x, w, b, eps):
    m = x.mean(axis=1, keepdims=True, dtype=np.float64).astype(f32)
    xc = x - m
    v = (xc.astype(np.float64) ** 2).mean(axis=1, keepdims=True).astype(f32)
    return (xc / np.sqrt(v + f32(eps)) * w + b).astype(f32)


def _gelu(x):
    from scipy.special import erf

    return (f32(0.5) * x * (f32(1.0) + erf(x / f32(math.sqrt(2.0))).astype(f32))).astype(f32)


def _lrelu(x, s):
    return np.where(x > 0, x, f32(s) * x).astype(f32)


def t_schedule(n: int) -> np.ndarray:
    return np.array([1.0 - math.cos(math.pi / 2 * i / n) for i in range(n + 1)], dtype=np.float32)


def timestep_embedding(w: CosyDetokWeights, t: float) -> np.ndarray:
    ds = w.cfg.d_est
    half = ds // 2
    fr = np.exp(-math.log(10000.0) * np.arange(half, dtype=np.float32) / f32(half)).astype(f32)
    arg = (f32(1000.0) * f32(t) * fr).astype(f32)
    e = np.concatenate([np.sin(arg), np.cos(arg)]).astype(f32)
    a = (w.t1 @ e + w.t1b).astype(f32)
    a = (a / (f32(1.0) + np.exp(-a))).astype(f32)
    return (w.t2 @ a + w.t2b).astype(f32)


class CosyDetokOracle:
    def __init__(self, cfg, seed: int, weights: CosyDetokWeights | None = None):
        self.cfg = cfg
        self.w = weights or CosyDetokWeights(cfg, seed)

    def _gemm(self, x, w, exact):
        if not exact:
            x = bf16_round(x)
        return (x.astype(f32) @ w.T.astype(f32)).astype(f32)

    def _rope(self, x, heads):
        T, D = x.shape
        hd = D // heads
        inv = (1.0 / (self.cfg.rope_theta ** (np.arange(0, hd, 2, dtype=np.float32) / hd))).astype(f32)
        fr = np.arange(T, dtype=np.float32)[:, None] * inv[None, :]
        emb = np.concatenate([fr, fr], axis=1)
        cos, sin = np.cos(emb)[:, None, :], np.sin(emb)[:, None, :]
        x = x.reshape(T, heads, hd)
        h = hd // 2
        rot = np.concatenate([-x[..., h:], x[..., :h]], axis=-1)
        return (x * cos + rot * sin).astype(f32)

    def _xf(self, h, L, heads, exact):
        cfg = self.cfg
        T, D = h.shape
        hd = D // heads
        x = _ln(h, L["ln1w"], L["ln1b"], cfg.eps)
        qkv = self._gemm(x, L["qkv"], exact)
        q, k = self._rope(qkv[:, :D], heads), self._rope(qkv[:, D:2 * D], heads)
        v = qkv[:, 2 * D:].reshape(T, heads, hd)
        s = np.einsum("qhd,khd->hqk", q, k).astype(f32) * f32(1.0 / math.sqrt(hd))
        s = s - s.max(axis=-1, keepdims=True)
        p = np.exp(s).astype(f32)
        p = p / p.sum(axis=-1, keepdims=True)
        o = np.einsum("hqk,khd->qhd", p, v).reshape(T, D).astype(f32)
        h = (h + self._gemm(o, L["o"], exact)).astype(f32)
        x = _ln(h, L["ln2w"], L["ln2b"], cfg.eps)
        return (h + self._gemm(_gelu(self._gemm(x, L["fc1"], exact)), L["fc2"], exact)).astype(f32)

    # ------------------------------------------------------------------ flow
    def flow(self, req_seed: int, call: int, new_tokens: np.ndarray, exact: bool = True) -> np.ndarray:
        """One call's new mel frames [2 * len(new_tokens), mel]."""
        cfg, w = self.cfg, self.w
        ref, spk, rmel = cosy_request_tensors(cfg, req_seed)
        tok = np.concatenate([ref, np.asarray(new_tokens, np.int64)])
        T = len(tok)
        h = w.emb[tok].astype(f32)
        for L in w.enc:
            h = self._xf(h, L, cfg.enc_heads, exact)
        mu_t = (self._gemm(_ln(h, w.elnf_w, w.elnf_b, cfg.eps), w.mu, exact) + w.mu_b).astype(f32)
        mu = np.repeat(mu_t, 2, axis=0)
        R = 2 * T
        cond = np.zeros((R, cfg.mel), f32)
        cond[:2 * cfg.ref_tokens] = rmel
        x = cosy_noise(cfg, req_seed, call, R)
        ts = t_schedule(cfg.n_steps)
        lam = f32(cfg.cfg_rate)
        inp_c = np.concatenate([x, mu, np.broadcast_to(spk, (R, cfg.mel)), cond], axis=1)
        for i in range(cfg.n_steps):
            bias = (w.b_in + timestep_embedding(w, float(ts[i]))).astype(f32)
            vs = []
            for branch in (0, 1):
                inp = np.concatenate([x, mu, np.broadcast_to(spk, (R, cfg.mel)), cond], axis=1) if branch == 0 else \
                    np.concatenate([x, np.zeros((R, 3 * cfg.mel), f32)], axis=1)
                z = (self._gemm(inp, w.w_in, exact) + bias).astype(f32)
                for L in w.est:
                    z = self._xf(z, L, cfg.est_heads, exact)
                vs.append((self._gemm(_ln(z, w.oln_w, w.oln_b, cfg.eps), w.w_out, exact) + w.b_out).astype(f32))
            v = ((f32(1.0) + lam) * vs[0] - lam * vs[1]).astype(f32)
            x = (x + (ts[i + 1] - ts[i]) * v).astype(f32)
        del inp_c
        return x[2 * cfg.ref_tokens:]

    # ------------------------------------------------------------------ vocoder
    def _conv(self, x, w, b, k, act, exact):
        R, C = x.shape
        a = _lrelu(x, self.cfg.slope) if act else x
        pad = np.concatenate([np.zeros((k - 1, C), f32), a], axis=0)
        col = np.concatenate([pad[j:j + R] for j in range(k)], axis=1)
        if col.shape[1] < w.shape[1]:
            col = np.concatenate([col, np.zeros((R, w.shape[1] - col.shape[1]), f32)], axis=1)
        return (self._gemm(col, w, exact) + b).astype(f32)

    def vocoder(self, mel: np.ndarray, exact: bool = True) -> np.ndarray:
        """mel [F, 80] (a request's whole new-mel sequence) -> PCM [F * samples_per_mel]."""
        cfg, w = self.cfg, self.w
        x = self._conv(mel.astype(f32), w.vpre, w.vpre_b, cfg.voc_kernel, False, exact)
        for b, s in enumerate(cfg.ratios):
            B = w.blocks[b]
            R, C = x.shape
            a = _lrelu(x, cfg.slope)
            prev = np.concatenate([np.zeros((1, C), f32), a[:-1]], axis=0)
            y = self._gemm(np.concatenate([prev, a], axis=1), B["upw"], exact)
            Co = B["upw"].shape[0] // s
            x = (y.reshape(R * s, Co) + B["upb"]).astype(f32)
            r = self._conv(x, B["r1w"], B["r1b"], cfg.res_kernel, True, exact)
            x = (x + self._conv(r, B["r2w"], B["r2b"], cfg.res_kernel, True, exact)).astype(f32)
        y = self._conv(x, w.vpost, w.vpost_b, cfg.post_kernel, True, exact)
        return istft(y, cfg)

    def decode(self, req_seed: int, chunks, exact: bool = True) -> np.ndarray:
        """A request's calls (lists of new tokens, in order) -> its whole PCM stream."""
        mel = np.concatenate([self.flow(req_seed, c, t, exact) for c, t in enumerate(chunks)], axis=0)
        return self.vocoder(mel, exact)


def istft(y: np.ndarray, cfg) -> np.ndarray:
    """Causal iSTFT of conv_post rows y [J, 2 * nb]: log-magnitudes, phase logits."""
    n, hop = cfg.n_fft, cfg.hop
    nb = n // 2 + 1
    mag = np.minimum(np.exp(y[:, :nb].astype(np.float64)), 100.0)
    ph = np.sin(y[:, nb:].astype(np.float64))
    re, im = mag * np.cos(ph), mag * np.sin(ph)
    t = np.arange(n)
    kk = np.arange(1, nb - 1)
    frames = (re[:, :1] + re[:, nb - 1:nb] * ((-1.0) ** t)[None, :]
              + 2 * (re[:, 1:nb - 1] @ np.cos(2 * np.pi * np.outer(kk, t) / n)
                     - im[:, 1:nb - 1] @ np.sin(2 * np.pi * np.outer(kk, t) / n))) / n
    win = 0.5 - 0.5 * np.cos(2 * np.pi * t / n)
    wf = frames * win[None, :]
    J = y.shape[0]
    out = np.zeros(J * hop)
    q = n // hop
    env = (win ** 2).reshape(q, hop).sum(axis=0)  # = 1.5 for every phase (periodic Hann, hop n/4)
    for j in range(J):
        for a in range(q):
            if j - a >= 0:
                out[j * hop:(j + 1) * hop] += wf[j - a, a * hop:(a + 1) * hop]
    return (out / np.tile(env, J)).astype(f32)
