"""CPU restatement of the decode step (TEST INFRASTRUCTURE ONLY).

The reference's LM forward is a hash stub (profiles.py:318-331), so this
backbone follows the public Llama architecture ([3P] transformers 5.5.0
models/llama/modeling_llama.py: LlamaRMSNorm :53, rotate_half RoPE :73,
LlamaMLP :171, LlamaAttention :225 with GQA) -- and, with cfg.qkv_bias, its
Qwen2 variant (q/k/v projections with bias: [3P] models/qwen2/modeling_qwen2.py
Qwen2Attention) -- and mirrors the GPU rounding points exactly: bf16 weights,
fp32 residual stream, bf16 GEMM inputs (normalised x, attention output,
SiLU*up), fp32 accumulation, fp32 logits.
Parity status: no LM arithmetic in the reference; pinned to transformers'
LlamaForCausalLM / Qwen2ForCausalLM on shared weights (tests/test_llama_oracle.py:
1.1e-6 max-relative with the rounding points off) and checked against the device
path by tests/test_gpu_lm.py, test_gpu_config2_parity.py and test_gpu_cosy.py.
"""

from __future__ import annotations

import numpy as np

from .weights import BackboneWeights, bf16_round

f32 = np.float32


def rmsnorm_bf16(h: np.ndarray, w: np.ndarray, eps: float) -> np.ndarray:
    """lm_kernels.cu:embed_norm_kernel / resid_norm_kernel."""
    h = h.astype(np.float32)
    ss = np.sum(h * h, axis=-1, dtype=np.float32, keepdims=True)
    inv = f32(1.0) / np.sqrt(ss / f32(h.shape[-1]) + f32(eps))
    return bf16_round((h * inv) * w)


def rope(x: np.ndarray, pos: np.ndarray, inv_freq: np.ndarray) -> np.ndarray:
    """rotate_half RoPE; x [n, heads, hd]; angle=float32(pos)*inv_freq, sin/cos in fp64."""
    half = x.shape[-1] // 2
    ang = pos.astype(np.float32)[:, None] * inv_freq[None, :]
    c = np.cos(ang.astype(np.float64)).astype(np.float32)[:, None, :]
    s = np.sin(ang.astype(np.float64)).astype(np.float32)[:, None, :]
    x1, x2 = x[..., :half], x[..., half:]
    return np.concatenate([x1 * c - x2 * s, x2 * c + x1 * s], axis=-1)


class LlamaOracle:
    """Per-request contiguous KV (the paged layout is checked via oracle/paging.py)."""

    def __init__(self, cfg, seed: int, weights: BackboneWeights | None = None, lazy_emb: bool = False):
        self.cfg = cfg
        self.w = weights or BackboneWeights(cfg, seed, lazy_emb=lazy_emb)
        self.k = {}  # rid -> [L, T, KV, hd]
        self.v = {}

    def _layer_kv(self, rid):
        if rid not in self.k:
            c = self.cfg
            self.k[rid] = np.zeros((c.n_layers, c.max_ctx, c.n_kv_heads, c.head_dim), np.float32)
            self.v[rid] = np.zeros_like(self.k[rid])
        return self.k[rid], self.v[rid]

    def embed(self, tokens: np.ndarray, ext: np.ndarray | None = None) -> np.ndarray:
        """lm_kernels.cu:embed_norm_kernel input rows, fp32.

        tokens [n] or [n, C] (CSM-style frame: the sum of the embedding rows of all
        ids, codebook order, -1 = absent); an id of -2 in column 0 takes ext[i]."""
        t = np.asarray(tokens)
        if t.ndim == 1:
            t = t[:, None]
        h = np.zeros((t.shape[0], self.cfg.d_model), np.float32)
        for i in range(t.shape[0]):
            if t[i, 0] == -2:
                h[i] = ext[i]
                continue
            acc = self.w.emb_rows([t[i, 0]])[0].astype(np.float32)
            for cb in range(1, t.shape[1]):
                if t[i, cb] >= 0:
                    acc = acc + self.w.emb_rows([t[i, cb]])[0]
            h[i] = acc
        return h

    def project(self, xf: np.ndarray) -> np.ndarray:
        """vox_project_ext: bf16 source hidden rows x the bf16 input projector, fp32."""
        return (xf.astype(np.float32) @ self.w.proj.T).astype(np.float32)

    def forward(self, rid, tokens: np.ndarray, positions: np.ndarray, want_logits: bool = True,
                ext: np.ndarray | None = None, head: tuple | None = None):
        """Run tokens [n] (or CSM frames [n, C]) at positions [n] (ascending) of request rid.

        Returns logits [n, vocab] fp32 of every row (or None; `head`=(lo, hi) limits
        them to vocabulary rows lo..hi-1) and the final normalised hidden rows xf
        [n, d] (bf16 values)."""
        n = len(tokens)
        return self.forward_rows([rid] * n, tokens, positions, want_logits, ext, head)

    def forward_rows(self, rids, tokens: np.ndarray, positions: np.ndarray, want_logits: bool = True,
                     ext: np.ndarray | None = None, head: tuple | None = None):
        """One mixed batch as the device runs it (vox_forward): row i feeds tokens[i] of
        request rids[i] at positions[i]; rows of one request are causal among
        themselves (every row's K/V is appended before attention reads the cache)."""
        c, w = self.cfg, self.w
        H, KV, hd = c.n_heads, c.n_kv_heads, c.head_dim
        G = H // KV
        n = len(tokens)
        positions = np.asarray(positions)
        h = self.embed(tokens, ext)  # fp32 residual
        x = rmsnorm_bf16(h, w.layers[0]["norm_attn"], c.rms_eps)
        scale = f32(1.0) / np.sqrt(f32(hd))
        groups: dict = {}
        for i, r in enumerate(rids):
            groups.setdefault(r, []).append(i)
        for l, L in enumerate(w.layers):
            qkv = x @ L["qkv"].T
            if "qkv_bias" in L:  # Qwen2 q|k|v bias, added after the projection (lm_kernels.cu)
                qkv = qkv + L["qkv_bias"]
            q = qkv[:, : H * hd].reshape(n, H, hd)
            k = qkv[:, H * hd: (H + KV) * hd].reshape(n, KV, hd)
            v = qkv[:, (H + KV) * hd:].reshape(n, KV, hd)
            q = bf16_round(rope(q, positions, w.inv_freq))
            k = bf16_round(rope(k, positions, w.inv_freq))
            v = bf16_round(v)
            out = np.empty((n, H, hd), np.float32)
            for rid, idx in groups.items():
                K, V = self._layer_kv(rid)
                K[l, positions[idx]] = k[idx]
                V[l, positions[idx]] = v[idx]
                pos = positions[idx]
                T = int(pos.max()) + 1
                kk = K[l, :T]  # [T, KV, hd]
                vv = V[l, :T]
                qg = q[idx].reshape(len(idx), KV, G, hd)
                s_ = np.einsum("nkgd,tkd->nkgt", qg, kk).astype(np.float32) * scale
                s_ = np.where(np.arange(T)[None, None, None, :] <= pos[:, None, None, None], s_, -np.inf)
                m = s_.max(axis=-1, keepdims=True)
                p = np.exp(s_ - m).astype(np.float32)
                o = np.einsum("nkgt,tkd->nkgd", p, vv).astype(np.float32)
                out[idx] = (o / p.sum(axis=-1, dtype=np.float32, keepdims=True)).reshape(len(idx), H, hd)
            a = bf16_round(out.reshape(n, H * hd))
            h = h + a @ L["o"].T
            x = rmsnorm_bf16(h, L["norm_mlp"], c.rms_eps)
            gu = x @ L["gu"].T
            g_, u_ = gu[:, : c.d_ff], gu[:, c.d_ff:]
            act = bf16_round((g_ / (f32(1.0) + np.exp(-g_))) * u_)
            h = h + act @ L["down"].T
            nw = w.layers[l + 1]["norm_attn"] if l + 1 < len(w.layers) else w.norm_final
            x = rmsnorm_bf16(h, nw, c.rms_eps)
        logits = None
        if want_logits:
            lo, hi = head if head is not None else (0, c.vocab)
            logits = (x @ w.emb_slice(lo, hi).T).astype(np.float32)
        return logits, x

    def release(self, rid):
        self.k.pop(rid, None)
        self.v.pop(rid, None)


def audio_range(cfg, step: int):
    """Orpheus frame-slot codebook-offset mask for generated token `step`."""
    if cfg.audio_base < 0:
        return 0, cfg.vocab
    k = step % cfg.frame_tokens
    lo = cfg.audio_base + k * cfg.codebook_size
    return lo, lo + cfg.codebook_size


def masked(logits_row: np.ndarray, lo: int, hi: int) -> np.ndarray:
    out = np.full(logits_row.shape, -np.inf, dtype=np.float64)
    out[lo:hi] = logits_row[lo:hi]
    return out
