"""CPU baseline: the oracle port of one serving step, timed on host cores.

TEST/BENCH INFRASTRUCTURE ONLY (bench.py cpu_baseline and --impl reference).
Same arithmetic as the GPU step at config 2 (Orpheus-3B-style): decode rows
through the Llama backbone (oracle/llama.py), the full-vocab LM head, the
restated reference sampler (oracle/sampler.py == model_api.sample) with the
Orpheus parameters (profiles.py:192-194), and the causal SNAC-style decoder
for the chunk due that step (oracle/snac.py).  numpy/BLAS uses every host
core.  Bounded sample: B_s = 8 streams at context 394 (7 decode rows + 1
detok window per iteration, as the GPU step at 256 streams), nothing
extrapolated.  Weights are fast random fills of the right shapes (values do
not change the work).
"""

from __future__ import annotations

import os
import time

import numpy as np

from . import sampler as osamp
from .llama import rmsnorm_bf16, rope
from .snac import SnacOracle
from .weights import bf16_round


def _cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def time_cpu_step(budget_s: float = 20.0, steps: int = 20, warmup: int = 1, B_s: int = 8, ctx: int = 394,
                  weight_sets: int = 2):
    """One steady-state serving iteration of B_s streams on the host, the GPU bench's
    step structure (scheduler.py:152-156: a stream selected for detok sits out that
    iteration's LM batch): B_s - 1 decode rows through ALL 28 layers (weight arrays
    cycled over `weight_sets` distinct sets -- every layer's GEMMs and attention are
    executed, each streaming its full weights from DRAM), the full-vocab head, the
    reference sampler per row, and one 7-token detok window (2048 samples) with the
    causal SNAC-style decoder.  audio-s/s = (B_s - 1)/86 per step / step time."""
    from paper_2602_00269_b200.config import orpheus3b

    cfg = orpheus3b()
    rng = np.random.default_rng(0)
    d, H, KV, hd, dff, V = cfg.d_model, cfg.n_heads, cfg.n_kv_heads, cfg.head_dim, cfg.d_ff, cfg.vocab
    n_dec = B_s - 1

    def rnd(*shape, scale=0.02):
        return ((rng.random(shape, dtype=np.float32) - np.float32(0.5)) * np.float32(2 * scale))

    sets = [dict(qkv=rnd((H + 2 * KV) * hd, d), o=rnd(d, H * hd), gu=rnd(2 * dff, d), down=rnd(d, dff),
                 na=np.ones(d, np.float32), nm=np.ones(d, np.float32)) for _ in range(weight_sets)]
    emb = rnd(V, d)
    Ks = [rnd(n_dec, ctx, KV, hd, scale=1.0) for _ in range(cfg.n_layers)]
    Vs = [rnd(n_dec, ctx, KV, hd, scale=1.0) for _ in range(cfg.n_layers)]
    inv = np.array([1.0 / (cfg.rope_theta ** (2 * i / hd)) for i in range(hd // 2)], np.float32)
    snac = SnacOracle(cfg, 1)
    G = H // KV
    scale = np.float32(1.0 / np.sqrt(hd))
    windows = [osamp.RingWindow(64, V) for _ in range(n_dec)]
    rngs = [osamp.request_rng(0, i) for i in range(n_dec)]

    def one_step(t):
        tt = {}
        t0 = time.perf_counter()
        h = emb[rng.integers(0, V, n_dec)].copy()
        x = rmsnorm_bf16(h, sets[0]["na"], cfg.rms_eps)
        pos = np.full(n_dec, ctx - 1)
        for l in range(cfg.n_layers):
            L = sets[l % weight_sets]
            qkv = x @ L["qkv"].T
            q = bf16_round(rope(qkv[:, : H * hd].reshape(n_dec, H, hd), pos, inv))
            qg = q.reshape(n_dec, KV, G, hd)
            s_ = np.einsum("nkgd,ntkd->nkgt", qg, Ks[l]) * scale
            p = np.exp(s_ - s_.max(axis=-1, keepdims=True))
            out = np.einsum("nkgt,ntkd->nkgd", p, Vs[l]) / p.sum(axis=-1, keepdims=True)
            h = h + bf16_round(out.reshape(n_dec, -1).astype(np.float32)) @ L["o"].T
            x = rmsnorm_bf16(h, L["nm"], cfg.rms_eps)
            gu = x @ L["gu"].T
            g_, u_ = gu[:, :dff], gu[:, dff:]
            h = h + bf16_round((g_ / (1 + np.exp(-g_))) * u_) @ L["down"].T
            x = rmsnorm_bf16(h, L["na"], cfg.rms_eps)
        tt["layers"] = time.perf_counter() - t0
        t1 = time.perf_counter()
        logits = (x @ emb.T).astype(np.float32)
        tt["head"] = time.perf_counter() - t1
        t2 = time.perf_counter()
        for i in range(n_dec):
            k = (t + i) % 7
            lo = cfg.audio_base + k * cfg.codebook_size
            row = np.full(V, -np.inf)
            row[lo: lo + cfg.codebook_size] = logits[i, lo: lo + cfg.codebook_size]
            osamp.sample(row, 0.6, None, 0.8, 1.3, windows[i], rngs[i])
        tt["sample"] = time.perf_counter() - t2
        t3 = time.perf_counter()
        codes = rng.integers(0, cfg.codebook_size, size=(1, 7))
        snac.decode(codes)
        tt["detok"] = time.perf_counter() - t3
        return tt

    for w in range(warmup):
        one_step(w)
    tot = []
    parts = []
    t_start = time.perf_counter()
    for s in range(steps):
        tt = one_step(100 + s)
        parts.append(tt)
        tot.append(sum(tt.values()))
        if time.perf_counter() - t_start > budget_s:
            break
    ms = float(np.mean(tot)) * 1000
    audio = n_dec / 86.0  # each decoded token = 1/86 s of audio (profiles.py:183)
    return {
        "audio_s_per_s": audio / (ms / 1000),
        "ms_per_step": ms,
        "cores": _cores(),
        "steps": len(tot),
        "sample": f"steady-state iteration of {B_s} streams at ctx {ctx} (the GPU step's structure at B={B_s} "
                  f"instead of 256): {n_dec} decode rows through all 28 layers ({weight_sets} weight sets cycled), "
                  f"full-vocab head, reference sampler (T .6, top-p .8, rp 1.3), one 7-token detok window; "
                  f"{len(tot)} steps; breakdown ms " +
                  ", ".join(f"{k}={np.mean([p[k] for p in parts]) * 1000:.1f}" for k in parts[0]),
    }
