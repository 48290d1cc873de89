"""Bit-exact CPU mirror of the device random-init (TEST INFRASTRUCTURE ONLY).

Mirrors paper_2602_00269_b200/csrc/init.cu (w = bf16_rn(unit_pm1(mix64(key+i)) * scale))
and the tensor-key / scale choices of csrc/vox_api.cu (create_backbone,
create_detok).  splitmix64 is the reference's mixer (model_api.py:39-51).
"""

from __future__ import annotations

import numpy as np

MASK64 = (1 << 64) - 1
GOLDEN = 0x9E3779B97F4A7C15

# tensor ids (csrc/vox_api.cu: TensorId)
T_EMB, T_NORM_ATTN, T_NORM_MLP, T_NORM_FINAL = 1, 2, 3, 4
T_QKV, T_O, T_GU, T_DOWN, T_QKV_BIAS, T_PROJ = 5, 6, 7, 8, 9, 10
T_VQ_TAB, T_IN_DW_W, T_IN_DW_B, T_IN_PW_W, T_IN_PW_B = 20, 21, 22, 23, 24
T_UP_ALPHA, T_UP_W, T_UP_B = 30, 34, 38
T_RU_A1, T_RU_DW_W, T_RU_DW_B, T_RU_A2, T_RU_PW_W, T_RU_PW_B = 50, 70, 90, 110, 130, 150
T_OUT_ALPHA, T_OUT_W, T_OUT_B = 170, 171, 172


def mix64(x: int) -> int:
    """splitmix64 finalizer (model_api.py:39-44)."""
    x = (x + GOLDEN) & MASK64
    x = ((x ^ (x >> 30)) * 0xBF58476D1CE4E5B9) & MASK64
    x = ((x ^ (x >> 27)) * 0x94D049BB133111EB) & MASK64
    return x ^ (x >> 31)


def mix64_arr(x: np.ndarray) -> np.ndarray:
    """Vectorised splitmix64 (model_api.py:47-51)."""
    with np.errstate(over="ignore"):
        x = x + np.uint64(GOLDEN)
        x = (x ^ (x >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        x = (x ^ (x >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return x ^ (x >> np.uint64(31))


def tensor_key(seed: int, tid: int, layer: int) -> int:
    a = mix64((seed ^ ((tid * 0xD1B54A32D192ED03) & MASK64)) & MASK64)
    return mix64(a ^ ((layer * 0x8CB92BA72F3D8DD7) & MASK64))


def bf16_round(x: np.ndarray) -> np.ndarray:
    """float32 -> nearest-even bfloat16, returned as float32 (no NaN inputs)."""
    b = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    b = (b + np.uint64(0x7FFF) + ((b >> np.uint64(16)) & np.uint64(1))) & np.uint64(0xFFFF0000)
    return b.astype(np.uint32).view(np.float32)


def unit_pm1(n: int, key: int, start: int = 0) -> np.ndarray:
    i = np.arange(start, start + n, dtype=np.uint64)
    with np.errstate(over="ignore"):
        h = mix64_arr(np.uint64(key) + i)
    return (h >> np.uint64(40)).astype(np.int32).astype(np.float32) * np.float32(1.0 / 8388608.0) - np.float32(1.0)


def init_bf16(n: int, key: int, scale, chunk: int = 1 << 24, start: int = 0) -> np.ndarray:
    """csrc/init.cu:init_bf16_kernel, as float32 values (elements start .. start+n)."""
    out = np.empty(n, dtype=np.float32)
    s = np.float32(scale)
    for a in range(0, n, chunk):
        m = min(chunk, n - a)
        out[a: a + m] = bf16_round(unit_pm1(m, key, start + a) * s)
    return out


def init_f32(n: int, key: int, scale, offset) -> np.ndarray:
    """csrc/init.cu:init_f32_kernel."""
    u = unit_pm1(n, key)
    return bf16_round(u * np.float32(scale) + np.float32(offset))


def f32(x) -> np.float32:
    return np.float32(x)


class BackboneWeights:
    """All backbone tensors as float32 arrays holding bf16 values."""

    def __init__(self, cfg, seed: int, layers=None, lazy_emb: bool = False):
        """lazy_emb: generate embedding rows on demand (config-2 sizes: the full
        [156,940 x 3072] table is 1.9 GB of fp32; tests touch only the prompt rows
        and the audio-row slice of the tied head)."""
        d, hd, H, KV, dff, V = cfg.d_model, cfg.head_dim, cfg.n_heads, cfg.n_kv_heads, cfg.d_ff, cfg.vocab
        self.cfg = cfg
        k = lambda tid, l=0: tensor_key(seed, tid, l)  # noqa: E731
        self._emb_key = k(T_EMB)
        self._emb_cache: dict = {}
        self._emb = None if lazy_emb else init_bf16(V * d, self._emb_key, f32(cfg.embed_half_width)).reshape(V, d)
        nqkv = (H + 2 * KV) * hd
        self.layers = []
        for l in range(cfg.n_layers if layers is None else layers):
            L = {}
            L["norm_attn"] = init_f32(d, k(T_NORM_ATTN, l), 0.25, 1.0)
            L["norm_mlp"] = init_f32(d, k(T_NORM_MLP, l), 0.25, 1.0)
            L["qkv"] = init_bf16(nqkv * d, k(T_QKV, l), np.sqrt(f32(3.0) / f32(d))).reshape(nqkv, d)
            L["o"] = init_bf16(d * H * hd, k(T_O, l), np.sqrt(f32(3.0) / f32(H * hd))).reshape(d, H * hd)
            L["gu"] = init_bf16(2 * dff * d, k(T_GU, l), np.sqrt(f32(3.0) / f32(d))).reshape(2 * dff, d)
            L["down"] = init_bf16(d * dff, k(T_DOWN, l), np.sqrt(f32(3.0) / f32(dff))).reshape(d, dff)
            if getattr(cfg, "qkv_bias", False):  # Qwen2-style (vox_api.cu: T_QKV_BIAS)
                L["qkv_bias"] = init_f32(nqkv, k(T_QKV_BIAS, l), 0.5, 0.0)
            self.layers.append(L)
        self.norm_final = init_f32(d, k(T_NORM_FINAL), 0.25, 1.0)
        ext = getattr(cfg, "ext_dim", 0)
        if ext:  # input projector of external hidden rows (vox_api.cu: T_PROJ)
            self.proj = init_bf16(d * ext, k(T_PROJ), np.sqrt(f32(3.0) / f32(ext))).reshape(d, ext)
        self.inv_freq = np.array(
            [np.float32(1.0 / (float(cfg.rope_theta) ** ((2.0 * i) / hd))) for i in range(hd // 2)],
            dtype=np.float32,
        )


    @property
    def emb(self) -> np.ndarray:
        if self._emb is None:
            raise AttributeError("lazy embedding: use emb_rows() / emb_slice()")
        return self._emb

    def emb_rows(self, ids) -> np.ndarray:
        """Rows `ids` of the (tied) embedding table, float32 [n, d] of bf16 values."""
        ids = np.asarray(ids, dtype=np.int64).reshape(-1)
        if self._emb is not None:
            return self._emb[ids]
        d = self.cfg.d_model
        out = np.empty((len(ids), d), np.float32)
        for j, i in enumerate(ids):
            i = int(i)
            if i not in self._emb_cache:
                self._emb_cache[i] = init_bf16(d, self._emb_key, f32(self.cfg.embed_half_width), start=i * d)
            out[j] = self._emb_cache[i]
        return out

    def emb_slice(self, lo: int, hi: int) -> np.ndarray:
        """Rows [lo, hi) of the embedding table (the head's vocabulary slice), cached."""
        if self._emb is not None:
            return self._emb[lo:hi]
        key = ("slice", lo, hi)
        if key not in self._emb_cache:
            d = self.cfg.d_model
            self._emb_cache[key] = init_bf16((hi - lo) * d, self._emb_key, f32(self.cfg.embed_half_width),
                                             start=lo * d).reshape(hi - lo, d)
        return self._emb_cache[key]


class DetokWeights:
    """Causal SNAC-style decoder tensors (csrc/vox_api.cu:create_detok)."""

    def __init__(self, cfg, seed: int):
        k = lambda tid, l=0: tensor_key(seed, tid, l)  # noqa: E731
        L, D0, cb = cfg.latent_dim, cfg.decoder_dim, cfg.codebook_size
        self.tabs = init_bf16(3 * cb * L, k(T_VQ_TAB), 0.866).reshape(3, cb, L)
        self.in_dw_w = init_f32(7 * L, k(T_IN_DW_W), np.sqrt(f32(3.0) / f32(7.0)), 0.0).reshape(L, 7)
        self.in_dw_b = init_f32(L, k(T_IN_DW_B), 0.05, 0.0)
        self.in_pw_w = init_bf16(D0 * L, k(T_IN_PW_W), np.sqrt(f32(3.0) / f32(L))).reshape(D0, L)
        self.in_pw_b = init_f32(D0, k(T_IN_PW_B), 0.05, 0.0)
        ch = [D0]
        for _ in range(4):
            ch.append(ch[-1] // 2)
        self.ch = ch
        self.rates = list(cfg.rates)
        self.up_alpha, self.up_w, self.up_b = [], [], []
        self.ru = []
        for b in range(4):
            Ci, Co, s = ch[b], ch[b + 1], self.rates[b]
            self.up_alpha.append(init_f32(Ci, k(T_UP_ALPHA + b), 0.5, 1.0))
            self.up_w.append(init_bf16(s * Co * 2 * Ci, k(T_UP_W + b),
                                       np.sqrt(f32(3.0) / (f32(2.0) * f32(Ci)))).reshape(s * Co, 2 * Ci))
            small = init_f32(Co, k(T_UP_B + b), 0.05, 0.0)
            self.up_b.append(np.tile(small, s))
            units = []
            for u in range(3):
                li = b * 3 + u
                units.append(dict(
                    a1=init_f32(Co, k(T_RU_A1, li), 0.5, 1.0),
                    a2=init_f32(Co, k(T_RU_A2, li), 0.5, 1.0),
                    dw_w=init_f32(7 * Co, k(T_RU_DW_W, li), np.sqrt(f32(3.0) / f32(7.0)), 0.0).reshape(Co, 7),
                    dw_b=init_f32(Co, k(T_RU_DW_B, li), 0.05, 0.0),
                    pw_w=init_bf16(Co * Co, k(T_RU_PW_W, li), f32(0.25) * np.sqrt(f32(3.0) / f32(Co))).reshape(Co, Co),
                    pw_b=init_f32(Co, k(T_RU_PW_B, li), 0.05, 0.0),
                ))
            self.ru.append(units)
        C4 = ch[4]
        self.out_alpha = init_f32(C4, k(T_OUT_ALPHA), 0.5, 1.0)
        self.out_w = init_f32(7 * C4, k(T_OUT_W), f32(0.15) * np.sqrt(f32(3.0) / (f32(7.0) * f32(C4))),
                              0.0).reshape(C4, 7)
        self.out_b = init_f32(1, k(T_OUT_B), 0.05, 0.0)[0]


# Mimi-style decoder (csrc/mimi.cu: mimi_create) -- tensor ids 300.., layer = codebook /
# transformer layer / SEANet block.  GEMM weights are generated directly in the device's
# GEMM layout ([out, taps * in] with tap-major K); MimiWeights.torch_layout() turns them
# into the PyTorch Conv1d / ConvTranspose1d / Linear layouts transformers uses.
T_MI_EMB, T_MI_PSEM, T_MI_PAC, T_MI_UP = 300, 301, 302, 303
T_MI_LN1W, T_MI_LN1B, T_MI_LN2W, T_MI_LN2B = 310, 311, 312, 313
T_MI_QKV, T_MI_O, T_MI_FC1, T_MI_FC2, T_MI_LS1, T_MI_LS2 = 314, 315, 316, 317, 318, 319
T_MI_C0W, T_MI_C0B, T_MI_UPW, T_MI_UPB = 330, 331, 332, 333
T_MI_R1W, T_MI_R1B, T_MI_R2W, T_MI_R2B, T_MI_OUTW, T_MI_OUTB = 334, 335, 336, 337, 338, 339


class MimiWeights:
    """All Mimi tensors as float32 arrays holding bf16-representable values."""

    def __init__(self, cfg, seed: int):
        k = lambda tid, l=0: tensor_key(seed, tid, l)  # noqa: E731
        D, cd, cb, F = cfg.hidden, cfg.cb_dim, cfg.cb_size, cfg.ffn
        self.cfg = cfg
        self.emb = [init_f32(cb * cd, k(T_MI_EMB, q), np.sqrt(f32(3.0) / f32(cfg.n_q)), 0.0).reshape(cb, cd)
                    for q in range(cfg.n_q)]
        self.psem = init_bf16(D * cd, k(T_MI_PSEM), np.sqrt(f32(3.0) / f32(cd))).reshape(D, cd)
        self.pac = init_bf16(D * cd, k(T_MI_PAC), np.sqrt(f32(3.0) / f32(cd))).reshape(D, cd)
        self.up = init_f32(D * 4, k(T_MI_UP), 0.5, 0.0).reshape(D, 4)
        self.layers = []
        for l in range(cfg.n_layers):
            self.layers.append(dict(
                ln1w=init_f32(D, k(T_MI_LN1W, l), 0.25, 1.0), ln1b=init_f32(D, k(T_MI_LN1B, l), 0.05, 0.0),
                ln2w=init_f32(D, k(T_MI_LN2W, l), 0.25, 1.0), ln2b=init_f32(D, k(T_MI_LN2B, l), 0.05, 0.0),
                qkv=init_bf16(3 * D * D, k(T_MI_QKV, l), np.sqrt(f32(3.0) / f32(D))).reshape(3 * D, D),
                o=init_bf16(D * D, k(T_MI_O, l), np.sqrt(f32(3.0) / f32(D))).reshape(D, D),
                fc1=init_bf16(F * D, k(T_MI_FC1, l), np.sqrt(f32(3.0) / f32(D))).reshape(F, D),
                fc2=init_bf16(D * F, k(T_MI_FC2, l), np.sqrt(f32(3.0) / f32(F))).reshape(D, F),
                ls1=init_f32(D, k(T_MI_LS1, l), 0.05, 0.1), ls2=init_f32(D, k(T_MI_LS2, l), 0.05, 0.1),
            ))
        ch = cfg.channels
        kk = cfg.kernel
        self.c0w = init_bf16(ch[0] * kk * D, k(T_MI_C0W), np.sqrt(f32(3.0) / f32(kk * D))).reshape(ch[0], kk * D)
        self.c0b = init_f32(ch[0], k(T_MI_C0B), 0.05, 0.0)
        self.blocks = []
        rk = cfg.res_kernel
        for b, s in enumerate(cfg.ratios):
            Ci, Co = ch[b], ch[b + 1]
            h = Co // cfg.compress
            self.blocks.append(dict(
                upw=init_bf16(s * Co * 2 * Ci, k(T_MI_UPW, b), np.sqrt(f32(3.0) / (f32(2.0) * f32(Ci)))).reshape(s * Co, 2 * Ci),
                upb=init_f32(Co, k(T_MI_UPB, b), 0.05, 0.0),
                r1w=init_bf16(h * rk * Co, k(T_MI_R1W, b), np.sqrt(f32(3.0) / f32(rk * Co))).reshape(h, rk * Co),
                r1b=init_f32(h, k(T_MI_R1B, b), 0.05, 0.0),
                r2w=init_bf16(Co * h, k(T_MI_R2W, b), f32(0.5) * np.sqrt(f32(3.0) / f32(h))).reshape(Co, h),
                r2b=init_f32(Co, k(T_MI_R2B, b), 0.05, 0.0),
            ))
        lk, C4 = cfg.last_kernel, ch[-1]
        self.outw = init_f32(lk * C4, k(T_MI_OUTW), np.sqrt(f32(3.0) / f32(lk * C4)), 0.0).reshape(lk * C4)
        self.outb = init_f32(1, k(T_MI_OUTB), 0.05, 0.0)[0]

    def torch_layout(self) -> dict:
        """name -> np.ndarray in transformers MimiModel parameter layout (modeling_mimi.py)."""
        cfg, D = self.cfg, self.cfg.hidden
        out = {}
        for q in range(cfg.n_q):
            if q < cfg.n_semantic:
                pre = f"quantizer.semantic_residual_vector_quantizer.layers.{q}.codebook"
            else:
                pre = f"quantizer.acoustic_residual_vector_quantizer.layers.{q - cfg.n_semantic}.codebook"
            out[pre + ".embed_sum"] = self.emb[q]
            out[pre + ".cluster_usage"] = np.ones(cfg.cb_size, np.float32)
        out["quantizer.semantic_residual_vector_quantizer.output_proj.weight"] = self.psem[:, :, None]
        out["quantizer.acoustic_residual_vector_quantizer.output_proj.weight"] = self.pac[:, :, None]
        out["upsample.conv.weight"] = self.up[:, None, :]
        for l, L in enumerate(self.layers):
            p = f"decoder_transformer.layers.{l}."
            out[p + "input_layernorm.weight"], out[p + "input_layernorm.bias"] = L["ln1w"], L["ln1b"]
            out[p + "post_attention_layernorm.weight"], out[p + "post_attention_layernorm.bias"] = L["ln2w"], L["ln2b"]
            out[p + "self_attn.q_proj.weight"] = L["qkv"][:D]
            out[p + "self_attn.k_proj.weight"] = L["qkv"][D:2 * D]
            out[p + "self_attn.v_proj.weight"] = L["qkv"][2 * D:]
            out[p + "self_attn.o_proj.weight"] = L["o"]
            out[p + "mlp.fc1.weight"], out[p + "mlp.fc2.weight"] = L["fc1"], L["fc2"]
            out[p + "self_attn_layer_scale.scale"], out[p + "mlp_layer_scale.scale"] = L["ls1"], L["ls2"]
        ch, kk, rk = cfg.channels, cfg.kernel, cfg.res_kernel
        # GEMM layout W[o, j*Cin + c] (tap j reads x[t-(k-1)+j]) -> Conv1d weight[o, c, j]
        conv = lambda w, k, ci: w.reshape(w.shape[0], k, ci).transpose(0, 2, 1)  # noqa: E731
        out["decoder.layers.0.conv.weight"] = conv(self.c0w, kk, D)
        out["decoder.layers.0.conv.bias"] = self.c0b
        for b, s in enumerate(cfg.ratios):
            B = self.blocks[b]
            Ci, Co = ch[b], ch[b + 1]
            h = Co // cfg.compress
            # GEMM row j*Co + o, cols [x_{t-1} | x_t]: out[t*s + j] = x_t w[:, :, j] + x_{t-1} w[:, :, j + s]
            w4 = B["upw"].reshape(s, Co, 2, Ci)
            wt = np.empty((Ci, Co, 2 * s), np.float32)
            wt[:, :, :s] = w4[:, :, 1, :].transpose(2, 1, 0)
            wt[:, :, s:] = w4[:, :, 0, :].transpose(2, 1, 0)
            i = 1 + 3 * b
            out[f"decoder.layers.{i + 1}.conv.weight"] = wt
            out[f"decoder.layers.{i + 1}.conv.bias"] = B["upb"]
            out[f"decoder.layers.{i + 2}.block.1.conv.weight"] = conv(B["r1w"], rk, Co)
            out[f"decoder.layers.{i + 2}.block.1.conv.bias"] = B["r1b"]
            out[f"decoder.layers.{i + 2}.block.3.conv.weight"] = conv(B["r2w"], 1, h)
            out[f"decoder.layers.{i + 2}.block.3.conv.bias"] = B["r2b"]
        n = 2 + 3 * len(cfg.ratios)
        out[f"decoder.layers.{n}.conv.weight"] = conv(self.outw[None, :], cfg.last_kernel, ch[-1])
        out[f"decoder.layers.{n}.conv.bias"] = np.array([self.outb], np.float32)
        return out


# CosyVoice2-style detokenizer (csrc/cosy_detok.cu: cd_create) -- tensor ids 400..;
# per-request tensors (reference tokens / speaker embedding / reference mel / ODE noise)
# are keyed by the REQUEST seed instead of the weight seed.
T_CD_EMB = 400
T_CD_ENC = 401          # + 0..7: ln1w ln1b ln2w ln2b qkv o fc1 fc2 (layer = encoder layer)
T_CD_ELNFW, T_CD_ELNFB, T_CD_MU, T_CD_MUB = 409, 410, 411, 412
T_CD_SPK, T_CD_REFTOK, T_CD_REFMEL, T_CD_NOISE = 413, 414, 415, 416
T_CD_IN, T_CD_INB, T_CD_T1, T_CD_T1B, T_CD_T2, T_CD_T2B = 420, 421, 422, 423, 424, 425
T_CD_EST = 430          # + 0..7 as T_CD_ENC (layer = estimator layer)
T_CD_OLNW, T_CD_OLNB, T_CD_OUT, T_CD_OUTB = 438, 439, 440, 441
T_CD_VPRE, T_CD_VPREB, T_CD_UPW, T_CD_UPB = 450, 451, 452, 453
T_CD_R1W, T_CD_R1B, T_CD_R2W, T_CD_R2B, T_CD_VPOST, T_CD_VPOSTB = 454, 455, 456, 457, 458, 459


def _xf_layer(k, base, l, d, ffn):
    return dict(
        ln1w=init_f32(d, k(base + 0, l), 0.25, 1.0), ln1b=init_f32(d, k(base + 1, l), 0.05, 0.0),
        ln2w=init_f32(d, k(base + 2, l), 0.25, 1.0), ln2b=init_f32(d, k(base + 3, l), 0.05, 0.0),
        qkv=init_bf16(3 * d * d, k(base + 4, l), np.sqrt(f32(3.0) / f32(d))).reshape(3 * d, d),
        o=init_bf16(d * d, k(base + 5, l), f32(0.5) * np.sqrt(f32(3.0) / f32(d))).reshape(d, d),
        fc1=init_bf16(ffn * d, k(base + 6, l), np.sqrt(f32(3.0) / f32(d))).reshape(ffn, d),
        fc2=init_bf16(d * ffn, k(base + 7, l), f32(0.5) * np.sqrt(f32(3.0) / f32(ffn))).reshape(d, ffn),
    )


def _pad_k(w: np.ndarray) -> np.ndarray:
    K = w.shape[1]
    Kp = (K + 63) // 64 * 64
    return w if Kp == K else np.concatenate([w, np.zeros((w.shape[0], Kp - K), np.float32)], axis=1)


class CosyDetokWeights:
    """All CosyVoice2-style detokenizer tensors (float32 arrays of bf16-representable values)."""

    def __init__(self, cfg, seed: int):
        k = lambda tid, l=0: tensor_key(seed, tid, l)  # noqa: E731
        de, ds, M = cfg.d_enc, cfg.d_est, cfg.mel
        self.cfg = cfg
        self.emb = init_f32(cfg.vocab * de, k(T_CD_EMB), 1.0, 0.0).reshape(cfg.vocab, de)
        self.enc = [_xf_layer(k, T_CD_ENC, l, de, cfg.enc_ffn) for l in range(cfg.enc_layers)]
        self.elnf_w, self.elnf_b = init_f32(de, k(T_CD_ELNFW), 0.25, 1.0), init_f32(de, k(T_CD_ELNFB), 0.05, 0.0)
        self.mu = init_bf16(M * de, k(T_CD_MU), np.sqrt(f32(3.0) / f32(de))).reshape(M, de)
        self.mu_b = init_f32(M, k(T_CD_MUB), 0.05, 0.0)
        self.w_in = init_bf16(ds * 4 * M, k(T_CD_IN), np.sqrt(f32(3.0) / f32(4 * M))).reshape(ds, 4 * M)
        self.b_in = init_f32(ds, k(T_CD_INB), 0.05, 0.0)
        self.t1 = init_f32(ds * ds, k(T_CD_T1), np.sqrt(f32(3.0) / f32(ds)), 0.0).reshape(ds, ds)
        self.t1b = init_f32(ds, k(T_CD_T1B), 0.05, 0.0)
        self.t2 = init_f32(ds * ds, k(T_CD_T2), np.sqrt(f32(3.0) / f32(ds)), 0.0).reshape(ds, ds)
        self.t2b = init_f32(ds, k(T_CD_T2B), 0.05, 0.0)
        self.est = [_xf_layer(k, T_CD_EST, l, ds, cfg.est_ffn) for l in range(cfg.est_layers)]
        self.oln_w, self.oln_b = init_f32(ds, k(T_CD_OLNW), 0.25, 1.0), init_f32(ds, k(T_CD_OLNB), 0.05, 0.0)
        self.w_out = init_bf16(M * ds, k(T_CD_OUT), np.sqrt(f32(3.0) / f32(ds))).reshape(M, ds)
        self.b_out = init_f32(M, k(T_CD_OUTB), 0.05, 0.0)
        ch, vk, rk = cfg.voc_channels, cfg.voc_kernel, cfg.res_kernel
        self.vpre = _pad_k(init_bf16(ch[0] * vk * M, k(T_CD_VPRE), np.sqrt(f32(3.0) / f32(vk * M))).reshape(ch[0], vk * M))
        self.vpre_b = init_f32(ch[0], k(T_CD_VPREB), 0.05, 0.0)
        self.blocks = []
        for b, s in enumerate(cfg.ratios):
            Ci, Co = ch[b], ch[b + 1]
            self.blocks.append(dict(
                upw=init_bf16(s * Co * 2 * Ci, k(T_CD_UPW, b), np.sqrt(f32(3.0) / (f32(2.0) * f32(Ci)))).reshape(s * Co, 2 * Ci),
                upb=init_f32(Co, k(T_CD_UPB, b), 0.05, 0.0),
                r1w=init_bf16(Co * rk * Co, k(T_CD_R1W, b), np.sqrt(f32(3.0) / f32(rk * Co))).reshape(Co, rk * Co),
                r1b=init_f32(Co, k(T_CD_R1B, b), 0.05, 0.0),
                r2w=init_bf16(Co * rk * Co, k(T_CD_R2W, b), f32(0.5) * np.sqrt(f32(3.0) / f32(rk * Co))).reshape(Co, rk * Co),
                r2b=init_f32(Co, k(T_CD_R2B, b), 0.05, 0.0),
            ))
        nb = cfg.n_fft // 2 + 1
        pk = cfg.post_kernel
        self.vpost = _pad_k(init_bf16(2 * nb * pk * ch[-1], k(T_CD_VPOST), np.sqrt(f32(3.0) / f32(pk * ch[-1]))).reshape(2 * nb, pk * ch[-1]))
        self.vpost_b = init_f32(2 * nb, k(T_CD_VPOSTB), 0.05, 0.0)


def cosy_request_tensors(cfg, req_seed: int):
    """Per-request reference tokens [ref_tokens], speaker embedding [mel], reference mel
    [2 * ref_tokens, mel] (csrc/cosy_detok.cu: vox_cosy_open)."""
    k = lambda tid, l=0: tensor_key(req_seed, tid, l)  # noqa: E731
    i = np.arange(cfg.ref_tokens, dtype=np.uint64)
    with np.errstate(over="ignore"):
        h = mix64_arr(np.uint64(k(T_CD_REFTOK)) + i)
    ref = (h % np.uint64(cfg.vocab)).astype(np.int64)
    spk = init_f32(cfg.mel, k(T_CD_SPK), 1.0, 0.0)
    rmel = init_f32(2 * cfg.ref_tokens * cfg.mel, k(T_CD_REFMEL), 1.0, 0.0).reshape(2 * cfg.ref_tokens, cfg.mel)
    return ref, spk, rmel


def cosy_noise(cfg, req_seed: int, chunk: int, rows: int) -> np.ndarray:
    """x0 of the flow ODE for call `chunk` of a request: unit-variance uniform noise."""
    return init_f32(rows * cfg.mel, tensor_key(req_seed, T_CD_NOISE, chunk), np.sqrt(f32(3.0)), 0.0).reshape(rows, cfg.mel)
