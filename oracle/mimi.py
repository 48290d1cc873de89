"""Mimi-style streaming decoder restatement (TEST INFRASTRUCTURE ONLY).

The reference's detokenizer emits no audio (profiles.py:333-356), so the
algorithm is the public one it stands for: [3P] transformers 5.5.0
``MimiModel.decode`` (models/mimi/modeling_mimi.py:1613-1680):

  * ``MimiSplitResidualVectorQuantizer.decode`` (:1340-1350): semantic codebooks
    and acoustic codebooks are each summed (``MimiResidualVectorQuantizer.decode``
    :1282-1294, embed = embed_sum / cluster_usage :1192-1195) and projected by
    their own 1x1 ``output_proj`` (256 -> 512), then added;
  * ``upsample`` = ``MimiConvTranspose1d`` depthwise (groups 512, k 4, stride 2,
    right-trimmed: :354-410) -> 25 Hz;
  * ``decoder_transformer`` = ``MimiTransformerModel`` (:996-1140): per layer
    LayerNorm -> q/k/v -> RoPE (rotate-half, theta 1e4) -> causal attention over
    the last ``sliding_window`` = 250 positions (masking_utils.py:90-99:
    kv > q - window) -> o_proj -> x + layer_scale * . ; LayerNorm -> fc1 -> GELU
    (erf) -> fc2 -> x + layer_scale * .  (:926-993);
  * ``MimiDecoder`` (:1143-1173): causal ``MimiConv1d`` (left pad k-1, :331-351)
    k7 512 -> 1024; per ratio r in 8/6/5/4: ELU, ConvT(k 2r, stride r, trimmed
    right, :403-410), ``MimiResnetBlock`` (:412-451: ELU, k3 conv C -> C/2, ELU,
    k1 conv C/2 -> C, + identity); ELU, k3 conv 64 -> 1.

PINNED: tests/test_mimi_oracle.py loads the same weights into transformers'
``MimiModel`` and requires ``decode`` == ``MimiOracle.decode(exact=True)`` (fp32).
``exact=False`` mirrors the device's rounding points (bf16 GEMM operands,
projected codebook tables, fp32 everything else) -- the GPU's chunked, stateful
decode must match the full-sequence decode within max-abs 2e-2 / SNR >= 35 dB.
"""

from __future__ import annotations

import math

import numpy as np

from .weights import MimiWeights, bf16_round

f32 = np.float32


def _elu(x: np.ndarray) -> np.ndarray:
    return np.where(x > 0, x, np.expm1(np.minimum(x, 0))).astype(f32)


def _gelu(x: np.ndarray) -> np.ndarray:
    from scipy.special import erf

    return (f32(0.5) * x * (f32(1.0) + erf(x / f32(math.sqrt(2.0))).astype(f32))).astype(f32)


def _ln(x: np.ndarray, w: np.ndarray, b: np.ndarray, eps: float) -> np.ndarray:
    m = x.mean(axis=1, keepdims=True, dtype=np.float64).astype(f32)
    xc = x - m
    v = (xc.astype(np.float64) ** 2).mean(axis=1, keepdims=True).astype(f32)
    return (xc / np.sqrt(v + f32(eps)) * w + b).astype(f32)


class MimiOracle:
    def __init__(self, cfg, seed: int, weights: MimiWeights | None = None):
        self.cfg = cfg
        self.w = weights or MimiWeights(cfg, seed)
        hd = cfg.head_dim
        self.inv_freq = (1.0 / (cfg.rope_theta ** (np.arange(0, hd, 2, dtype=np.int64).astype(np.float32) / hd))).astype(f32)

    # ------------------------------------------------------------------ pieces
    def _gemm(self, x: np.ndarray, w: np.ndarray, exact: bool) -> np.ndarray:
        """x [R, K] @ w[M, K]^T with fp32 accumulation; bf16 operands unless exact."""
        if not exact:
            x = bf16_round(x)
        return (x.astype(f32) @ w.T.astype(f32)).astype(f32)

    def _conv(self, x: np.ndarray, w: np.ndarray, b: np.ndarray, k: int, exact: bool, elu: bool = True) -> np.ndarray:
        """Causal conv (left pad k-1 zeros) as im2col GEMM, W[o, j*C + c]."""
        R, C = x.shape
        a = _elu(x) if elu else x
        pad = np.concatenate([np.zeros((k - 1, C), f32), a], axis=0)
        col = np.concatenate([pad[j:j + R] for j in range(k)], axis=1)
        return self._gemm(col, w, exact) + b

    def _convt(self, x: np.ndarray, blk: dict, s: int, exact: bool) -> np.ndarray:
        R, C = x.shape
        a = _elu(x)
        prev = np.concatenate([np.zeros((1, C), f32), a[:-1]], axis=0)
        y = self._gemm(np.concatenate([prev, a], axis=1), blk["upw"], exact)  # [R, s*Co]
        Co = blk["upw"].shape[0] // s
        return (y.reshape(R * s, Co) + blk["upb"]).astype(f32)

    def embed(self, codes: np.ndarray, exact: bool = True) -> np.ndarray:
        """codes [F, n_q] -> [F, hidden] (quantizer.decode)."""
        cfg, w = self.cfg, self.w
        if exact:  # transformers: sum per group, then project
            sem = sum(w.emb[q][codes[:, q]] for q in range(cfg.n_semantic)).astype(f32)
            ac = sum(w.emb[q][codes[:, q]] for q in range(cfg.n_semantic, cfg.n_q)).astype(f32)
            return (sem @ w.psem.T + ac @ w.pac.T).astype(f32)
        # device: projected per-codebook tables, summed in codebook order
        out = np.zeros((codes.shape[0], cfg.hidden), f32)
        for q in range(cfg.n_q):
            P = w.psem if q < cfg.n_semantic else w.pac
            out += (w.emb[q][codes[:, q]] @ P.T).astype(f32)
        return out

    def upsample(self, x: np.ndarray) -> np.ndarray:
        F, D = x.shape
        prev = np.concatenate([np.zeros((1, D), f32), x[:-1]], axis=0)
        y = np.empty((2 * F, D), f32)
        y[0::2] = x * self.w.up[:, 0] + prev * self.w.up[:, 2]
        y[1::2] = x * self.w.up[:, 1] + prev * self.w.up[:, 3]
        return y

    def _rope(self, x: np.ndarray, pos: np.ndarray) -> np.ndarray:
        """x [R, H, hd]; HF rotate-half convention."""
        fr = pos[:, None].astype(f32) * self.inv_freq[None, :]
        emb = np.concatenate([fr, fr], axis=1)
        cos, sin = np.cos(emb)[:, None, :].astype(f32), np.sin(emb)[:, None, :].astype(f32)
        h = x.shape[-1] // 2
        rot = np.concatenate([-x[..., h:], x[..., :h]], axis=-1)
        return (x * cos + rot * sin).astype(f32)

    def transformer(self, h: np.ndarray, exact: bool = True) -> np.ndarray:
        cfg = self.cfg
        T, D = h.shape
        H, hd, W = cfg.n_heads, cfg.head_dim, cfg.window
        pos = np.arange(T)
        qi, ki = np.meshgrid(pos, pos, indexing="ij")
        mask = (ki <= qi) & (ki > qi - W)
        h = h.copy()
        for L in self.w.layers:
            x = _ln(h, L["ln1w"], L["ln1b"], cfg.eps)
            qkv = self._gemm(x, L["qkv"], exact)
            q = self._rope(qkv[:, :D].reshape(T, H, hd), pos)
            k = self._rope(qkv[:, D:2 * D].reshape(T, H, hd), pos)
            v = qkv[:, 2 * D:].reshape(T, H, hd)
            s = np.einsum("qhd,khd->hqk", q, k).astype(f32) * f32(1.0 / math.sqrt(hd))
            s = np.where(mask[None], s, -np.inf)
            s = s - s.max(axis=-1, keepdims=True)
            p = np.exp(s).astype(f32)
            p = p / p.sum(axis=-1, keepdims=True)
            o = np.einsum("hqk,khd->qhd", p, v).reshape(T, D).astype(f32)
            h = (h + L["ls1"] * self._gemm(o, L["o"], exact)).astype(f32)
            x = _ln(h, L["ln2w"], L["ln2b"], cfg.eps)
            a = _gelu(self._gemm(x, L["fc1"], exact))
            h = (h + L["ls2"] * self._gemm(a, L["fc2"], exact)).astype(f32)
        return h

    def seanet(self, h: np.ndarray, exact: bool = True) -> np.ndarray:
        cfg, w = self.cfg, self.w
        x = self._conv(h, w.c0w, w.c0b, cfg.kernel, exact, elu=False)
        for b, s in enumerate(cfg.ratios):
            B = w.blocks[b]
            x = self._convt(x, B, s, exact)
            r = self._conv(x, B["r1w"], B["r1b"], cfg.res_kernel, exact)
            x = (x + self._conv(r, B["r2w"], B["r2b"], 1, exact)).astype(f32)
        # final ELU + k3 conv to one channel (fp32 on the device too)
        R, C = x.shape
        a = _elu(x)
        lk = cfg.last_kernel
        pad = np.concatenate([np.zeros((lk - 1, C), f32), a], axis=0)
        col = np.concatenate([pad[j:j + R] for j in range(lk)], axis=1)
        return (col @ w.outw + w.outb).astype(f32)

    def decode(self, codes: np.ndarray, exact: bool = True) -> np.ndarray:
        """codes [F, n_q] int -> PCM [F * frame_samples] float32 (whole stream, zero history)."""
        codes = np.asarray(codes, np.int64)
        x = self.upsample(self.embed(codes, exact))
        return self.seanet(self.transformer(x, exact), exact)
