"""Model + capacity configurations (BASELINE.json configs 1 and 2).

Backbone dims follow public Llama-3.2 shapes (Orpheus-3B is a Llama-3.2-3B
fine-tune; [3P] transformers LlamaConfig); the detokenizer follows the public
SNAC-24kHz decoder dims (decoder_dim 1024, rates [8,8,4,2], 3 codebooks of 4096,
vq strides [4,2,1]), made causal.  Weights are random-init
from a counter RNG (oracle/weights.py reproduces them bit-for-bit).
"""

from __future__ import annotations

import math
from dataclasses import asdict, dataclass, field, replace

# Orpheus token layout: 128256 Llama-3 text ids + 10 special ids, then
# 7 x 4096 audio ids (frame slot k uses [base + k*4096, base + (k+1)*4096)).
ORPHEUS_AUDIO_BASE = 128266
ORPHEUS_VOCAB = 156940
ORPHEUS_TEXT_VOCAB = 128000


@dataclass(frozen=True)
class ModelConfig:
    name: str
    n_layers: int
    d_model: int
    n_heads: int
    n_kv_heads: int
    head_dim: int
    d_ff: int
    vocab: int = ORPHEUS_VOCAB
    rope_theta: float = 500000.0
    rms_eps: float = 1e-5
    text_vocab: int = ORPHEUS_TEXT_VOCAB
    audio_base: int = ORPHEUS_AUDIO_BASE
    codebook_size: int = 4096
    frame_tokens: int = 7
    # capacity
    page_size: int = 16
    max_slots: int = 64
    max_ctx: int = 1024
    n_pages: int = 0          # 0 -> max_slots * ceil(max_ctx / page_size)
    max_rows: int = 512
    # detokenizer
    detok_enabled: bool = True
    latent_dim: int = 768
    decoder_dim: int = 1024
    rates: tuple = (8, 8, 4, 2)
    max_detok_frames: int = 256
    embed_scale: float = 0.0  # 0 -> logit std ~2.5 (see embed_half_width)
    qkv_bias: bool = False    # Qwen2-style q|k|v bias (CosyVoice2's LM)
    n_codebooks: int = 1      # CSM-style frames: embedding = sum over the frame's codebook ids
    ext_dim: int = 0          # > 0: token -2 rows take a projected external hidden (CSM depth pos 0)

    @property
    def embed_half_width(self) -> float:
        if self.embed_scale > 0:
            return self.embed_scale
        return 2.5 * math.sqrt(3.0) / math.sqrt(self.d_model)

    @property
    def pages(self) -> int:
        if self.n_pages > 0:
            return self.n_pages
        return self.max_slots * ((self.max_ctx + self.page_size - 1) // self.page_size)

    @property
    def hop(self) -> int:
        h = 1
        for r in self.rates:
            h *= r
        return h

    @property
    def frame_samples(self) -> int:
        """PCM samples per 7-token frame (4 latent frames x hop)."""
        return 4 * self.hop

    @property
    def weight_bytes(self) -> int:
        """bf16 backbone bytes streamed per decode step (tied embedding/head counted once)."""
        d, hd = self.d_model, self.head_dim
        per_layer = (self.n_heads + 2 * self.n_kv_heads) * hd * d + d * self.n_heads * hd
        per_layer += 3 * d * self.d_ff
        return 2 * (self.n_layers * per_layer + self.vocab * d)

    @property
    def kv_bytes_per_token(self) -> int:
        return 2 * 2 * self.n_layers * self.n_kv_heads * self.head_dim

    def with_capacity(self, **kw) -> "ModelConfig":
        return replace(self, **kw)

    def to_dict(self) -> dict:
        d = asdict(self)
        d["rates"] = list(self.rates)
        return d


def detok_role(lm: ModelConfig, **kw) -> ModelConfig:
    """The detokenizer-side context of a disaggregated deployment: the
    same token layout and detokenizer as `lm`, with a 1-layer d=64 placeholder backbone
    that is never run (the context only needs the token store, slots and the SNAC-style
    decoder; a few MB instead of the LM's weights and KV pool)."""
    return replace(lm, name=lm.name + "-detok", n_layers=1, d_model=64, n_heads=1, n_kv_heads=1, head_dim=64,
                   d_ff=64, detok_enabled=True, **kw)


def tiny(**kw) -> ModelConfig:
    """Config 1: 2-layer Llama backbone, d=256 (runs on the CPU oracle)."""
    base = ModelConfig(
        name="tiny-orpheus", n_layers=2, d_model=256, n_heads=4, n_kv_heads=2, head_dim=64,
        d_ff=1024, max_slots=32, max_ctx=1024, max_rows=512, max_detok_frames=256,
    )
    return replace(base, **kw)


# Greedy-parity init (config 1, SURVEY.md section 7 "Hard parts"): the same tiny
# backbone with the tied embedding's half-width x400.  RMSNorm makes every GEMM
# input scale-free, so the attention/MLP contributions keep their size while the
# token embedding carries more of the residual stream; device/oracle differences
# (tensor-core vs CPU fp32 summation order -> 1-ulp bf16 flips) then rarely reach
# the final hidden state (median |dlogit| ~1e-3 at logit std ~1000, measured on
# B200) while the decisions still depend on the layers: with weight seed 2024,
# zeroing the attention output changes 81 of config 1's 256 greedy tokens and
# zeroing attention + MLP 157 (tests/test_oracle_greedy.py).
# tests/test_gpu_lm.py asserts, at every decision, that the oracle's penalised
# top-2 margin exceeds 10x that step's measured device/oracle logit error before
# demanding bit-exact token streams.
PLANTED_EMBED_MULT = 400.0
PLANTED_WEIGHT_SEED = 2024


def tiny_planted(**kw) -> ModelConfig:
    """Config 1 with the planted-margin init (greedy token streams bit-exact)."""
    base = tiny(**kw)
    return replace(base, name="tiny-orpheus-planted", embed_scale=PLANTED_EMBED_MULT * base.embed_half_width)


def orpheus3b(**kw) -> ModelConfig:
    """Config 2: Orpheus-3B-style (Llama-3.2-3B backbone + SNAC-24k-style decoder)."""
    base = ModelConfig(
        name="orpheus-3b", n_layers=28, d_model=3072, n_heads=24, n_kv_heads=8, head_dim=128,
        d_ff=8192, max_slots=512, max_ctx=768, max_rows=1024, max_detok_frames=1024,
    )
    return replace(base, **kw)


# CosyVoice2's LM is Qwen2.5-0.5B ([3P] Qwen2.5-0.5B config: hidden 896, 24 layers,
# 14 q / 2 kv heads of 64, FFN 4864, rope theta 1e6, rms eps 1e-6, tied embeddings,
# q|k|v bias).  Token layout: 151,936 Qwen ids, then the 6,561 + 3 speech tokens
# (FSQ codes + sos/eos/task, CosyVoice2 llm_decoder width); speech positions may
# only emit speech ids (the same range mask as Orpheus's frame slots, one slot).
COSY_TEXT_VOCAB = 151643
COSY_SPEECH_BASE = 151936
COSY_SPEECH_TOKENS = 6564


def cosyvoice2(**kw) -> ModelConfig:
    """Config 4 (LM): CosyVoice2-style Qwen2.5-0.5B backbone over speech tokens."""
    base = ModelConfig(
        name="cosyvoice2-0.5b", n_layers=24, d_model=896, n_heads=14, n_kv_heads=2, head_dim=64,
        d_ff=4864, vocab=COSY_SPEECH_BASE + COSY_SPEECH_TOKENS, rope_theta=1e6, rms_eps=1e-6,
        text_vocab=COSY_TEXT_VOCAB, audio_base=COSY_SPEECH_BASE, codebook_size=COSY_SPEECH_TOKENS,
        frame_tokens=1, qkv_bias=True, detok_enabled=False, max_slots=256, max_ctx=1024, max_rows=1024,
    )
    return replace(base, **kw)


def tiny_cosy(**kw) -> ModelConfig:
    """CPU-oracle-sized CosyVoice2-style LM: 2 layers, same head geometry (G = 7, hd 64) + bias."""
    return cosyvoice2(**{"name": "tiny-cosyvoice2", "n_layers": 2, "d_model": 448, "d_ff": 1024,
                         "max_slots": 16, "max_ctx": 512, "max_rows": 512, **kw})


# CSM-1B ([3P] transformers CsmConfig defaults, configuration_csm.py:55-157): Llama-1B
# backbone (16 layers, d 2048, 32 q / 8 kv heads of 64, FFN 8192) over frames of 32
# codebooks, and a depth decoder (4 layers, d 1024, 8 q / 2 kv heads of 128, FFN 8192)
# that fills codebooks 1..31 of each frame from the backbone's last hidden state.
# Codebooks are 2048 codes here (CSM's 2051 carries 3 specials; 2048 keeps every
# codebook slice a whole number of 128-row weight tiles).  Backbone rows: 128,256 text
# ids, then codebook c at [base + c*2048, base + (c+1)*2048); the codebook-0 head is
# tied to its embedding rows.  Depth rows: codebook c at [c*2048, (c+1)*2048), tied
# input/output table (HF CSM unties the depth head; one table keeps the id of a
# sampled codebook-k code equal to its input row at the next depth position).
CSM_TEXT_VOCAB = 128256
CSM_CODES = 2048


def csm_backbone(**kw) -> ModelConfig:
    """Config 3 backbone: CSM-1B-style Llama-1B over 32-codebook frames (codebook-0 head)."""
    nc = kw.pop("n_codebooks", 32)
    base = ModelConfig(
        name="csm-1b-backbone", n_layers=16, d_model=2048, n_heads=32, n_kv_heads=8, head_dim=64,
        d_ff=8192, vocab=CSM_TEXT_VOCAB + nc * CSM_CODES, text_vocab=CSM_TEXT_VOCAB,
        audio_base=CSM_TEXT_VOCAB, codebook_size=CSM_CODES, frame_tokens=1, n_codebooks=nc,
        detok_enabled=False, max_slots=256, max_ctx=512, max_rows=512,
    )
    return replace(base, **kw)


def csm_depth(**kw) -> ModelConfig:
    """Config 3 depth decoder: position 0 = projected backbone state, position k >= 1 =
    the frame's codebook k-1 code; position k samples codebook k (frame slot k-1)."""
    nc = kw.pop("n_codebooks", 32)
    ext = kw.pop("ext_dim", 2048)
    base = ModelConfig(
        name="csm-1b-depth", n_layers=4, d_model=1024, n_heads=8, n_kv_heads=2, head_dim=128,
        d_ff=8192, vocab=nc * CSM_CODES, text_vocab=CSM_CODES, audio_base=CSM_CODES,
        codebook_size=CSM_CODES, frame_tokens=nc - 1, ext_dim=ext, detok_enabled=False,
        max_slots=256, max_ctx=48, max_rows=512,
    )
    return replace(base, **kw)


def tiny_csm(n_codebooks: int = 8):
    """CPU-oracle-sized CSM-style pair (same head geometries, 8 codebooks)."""
    bb = csm_backbone(name="tiny-csm-backbone", n_layers=2, d_model=256, n_codebooks=n_codebooks,
                      max_slots=8, max_ctx=256, max_rows=256)
    dp = csm_depth(name="tiny-csm-depth", n_layers=2, d_model=256, n_heads=4, n_kv_heads=1,
                   d_ff=1024, n_codebooks=n_codebooks, ext_dim=256, max_slots=8, max_rows=256)
    return bb, dp


@dataclass(frozen=True)
class MimiConfig:
    """Config 3 detokenizer: Mimi-style 12.5 Hz streaming decoder ([3P] transformers 5.5.0
    ``MimiConfig`` defaults, configuration_mimi.py:86-123; ``MimiModel.decode``
    modeling_mimi.py:1613-1680): split RVQ (1 semantic + n_q-1 acoustic codebooks of
    2048 x 256, each group summed then projected 256 -> 512), depthwise ConvT x2 to 25 Hz,
    an 8-layer sliding-window (250) transformer (LayerNorm, GELU MLP, layer scale, RoPE),
    and the causal SEANet decoder (k7 conv 512 -> 1024; per ratio 8/6/5/4: ELU,
    ConvT(k = 2r, stride r) halving channels, one residual block ELU-k3-ELU-k1; ELU, k3
    conv -> 1 channel).  1920 samples per 12.5 Hz frame at 24 kHz."""

    name: str = "mimi-12.5hz"
    n_q: int = 32
    n_semantic: int = 1
    cb_size: int = 2048
    cb_dim: int = 256
    hidden: int = 512
    n_layers: int = 8
    n_heads: int = 8
    ffn: int = 2048
    window: int = 250
    rope_theta: float = 10000.0
    eps: float = 1e-5
    filters: int = 64
    ratios: tuple = (8, 6, 5, 4)
    kernel: int = 7
    last_kernel: int = 3
    res_kernel: int = 3
    compress: int = 2
    max_slots: int = 64
    max_frames: int = 256     # 12.5 Hz frames per decode call (all requests)

    @property
    def head_dim(self) -> int:
        return self.hidden // self.n_heads

    @property
    def hop(self) -> int:
        """samples per 25 Hz transformer position"""
        h = 1
        for r in self.ratios:
            h *= r
        return h

    @property
    def frame_samples(self) -> int:
        return 2 * self.hop

    @property
    def channels(self) -> list:
        """SEANet channels: 2^len(ratios) * filters halving per ratio (1024 .. 64)"""
        c = [self.filters * (1 << len(self.ratios))]
        for _ in self.ratios:
            c.append(c[-1] // 2)
        return c

    def with_capacity(self, **kw) -> "MimiConfig":
        return replace(self, **kw)


def mimi(**kw) -> MimiConfig:
    return MimiConfig(**kw)


def tiny_mimi(**kw) -> MimiConfig:
    """CPU-test-sized Mimi: production conv/transformer dims, 2 transformer layers, 4 codebooks."""
    return MimiConfig(**{"name": "tiny-mimi", "n_q": 4, "n_layers": 2, "max_slots": 8, "max_frames": 64, **kw})


@dataclass(frozen=True)
class CosyDetokConfig:
    """Config 4 detokenizer: CosyVoice2-style chunked token-to-mel flow matching + HiFT-style
    vocoder (public CosyVoice2 architecture [3P] FunAudioLLM/CosyVoice, not installed here;
    PAPER.md:102 'flow-matching module built on Transformer layers and a HiFi-GAN vocoder'),
    as VoxServe runs it: each call consumes the request's reference tokens
    (ref_tokens = 50, profiles.py:135 ref_window_tokens) plus the chunk's new tokens.

    flow:    speech-token embedding -> enc_layers pre-LN transformer (full attention over
             the call's tokens, RoPE) -> LN -> x2 upsample to 50 Hz mel frames -> linear to
             80 = mu;  n_steps Euler steps of the conditional flow ODE (cosine t schedule)
             with classifier-free guidance (cfg_rate): the estimator is in-proj of
             [x | mu | spk | prompt-mel] + timestep embedding -> est_layers transformer ->
             LN -> linear to 80;
    vocoder: causal HiFT-style: k7 conv 80 -> voc_ch, per ratio LeakyReLU + ConvT(k 2r,
             stride r) halving channels + residual block (LReLU-k3-LReLU-k3), LReLU, k7 conv
             to n_fft/2+1 log-magnitudes + phases, causal iSTFT (Hann, n_fft 16, hop 4):
             480 samples per mel frame, 960 per token at 24 kHz.  Stateful per request
             (conv histories + iSTFT overlap tail) across chunks."""

    name: str = "cosyvoice2-detok"
    vocab: int = 6561
    ref_tokens: int = 50
    d_enc: int = 512
    enc_layers: int = 6
    enc_heads: int = 8
    enc_ffn: int = 2048
    mel: int = 80
    d_est: int = 256
    est_layers: int = 8
    est_heads: int = 4
    est_ffn: int = 1024
    n_steps: int = 10
    cfg_rate: float = 0.7
    rope_theta: float = 10000.0
    eps: float = 1e-5
    voc_ch: int = 512
    ratios: tuple = (8, 5, 3)
    voc_kernel: int = 7
    res_kernel: int = 3
    post_kernel: int = 7
    n_fft: int = 16
    hop: int = 4
    slope: float = 0.1
    max_slots: int = 128
    max_tokens: int = 2048    # new tokens per call over all requests
    max_chunk: int = 64       # new tokens per request per call

    @property
    def mel_per_token(self) -> int:
        return 2

    @property
    def samples_per_mel(self) -> int:
        h = self.hop
        for r in self.ratios:
            h *= r
        return h

    @property
    def samples_per_token(self) -> int:
        return self.mel_per_token * self.samples_per_mel

    @property
    def voc_channels(self) -> list:
        c = [self.voc_ch]
        for _ in self.ratios:
            c.append(c[-1] // 2)
        return c

    def with_capacity(self, **kw) -> "CosyDetokConfig":
        return replace(self, **kw)


def tiny_cosy_detok(**kw) -> CosyDetokConfig:
    """CPU-test-sized: 2 encoder / 2 estimator layers, 4 ODE steps, production vocoder."""
    return CosyDetokConfig(**{"name": "tiny-cosy-detok", "enc_layers": 2, "est_layers": 2, "n_steps": 4,
                              "max_slots": 8, "max_tokens": 256, **kw})


CONFIGS = {"tiny": tiny, "tiny_planted": tiny_planted, "orpheus3b": orpheus3b, "cosyvoice2": cosyvoice2, "tiny_cosy": tiny_cosy,
           "csm_backbone": csm_backbone, "csm_depth": csm_depth}
