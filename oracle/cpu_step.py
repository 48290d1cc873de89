"""CPU baseline: the oracle port of one serving step, timed on host cores.

TEST/BENCH INFRASTRUCTURE ONLY (bench.py cpu_baseline and --impl reference).
Same arithmetic as the GPU step at config 2 (Orpheus-3B-style): decode rows
through the Llama backbone (oracle/llama.py), the full-vocab LM head, the
restated reference sampler (oracle/sampler.py == model_api.sample) with the
Orpheus parameters (profiles.py:192-194), and the causal SNAC-style decoder
for the chunks due that step (oracle/snac.py).  numpy/BLAS uses every host
core.  Bounded sample: B_s = 4 streams at context 394, 2 of the 28 layers
timed and scaled x14, one 7-token detok frame per 8 stream-steps (the
steady-state chunk rate).  Weights are fast random fills of the right
shapes (values do not change the work).
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


def time_cpu_step(budget_s: float = 20.0, steps: int = 2, warmup: int = 1, B_s: int = 4, ctx: int = 394,
                  layers_timed: int = 2):
    from paper_2602_00269_b200.config import orpheus3b

    cfg = orpheus3b()
    rng = np.random.default_rng(0)
    d, H, KV, hd, dff, V = cfg.d_model, cfg.n_heads, cfg.n_kv_heads, cfg.head_dim, cfg.d_ff, cfg.vocab

    def rnd(*shape, scale=0.02):
        return (rng.standard_normal(shape, dtype=np.float32) * np.float32(scale))

    layers = [dict(qkv=rnd((H + 2 * KV) * hd, d), o=rnd(d, H * hd), gu=rnd(2 * dff, d), down=rnd(d, dff),
                   na=np.ones(d, np.float32), nm=np.ones(d, np.float32)) for _ in range(layers_timed)]
    emb = rnd(V, d)
    Ks = [rnd(B_s, ctx, KV, hd, scale=1.0) for _ in range(layers_timed)]
    Vs = [rnd(B_s, ctx, KV, hd, scale=1.0) for _ in range(layers_timed)]
    inv = np.array([1.0 / (cfg.rope_theta ** (2 * i / hd)) for i in range(hd // 2)], np.float32)
    snac = SnacOracle(cfg, 1)
    G = H // KV
    scale = np.float32(1.0 / np.sqrt(hd))
    windows = [osamp.RingWindow(64, V) for _ in range(B_s)]
    rngs = [osamp.request_rng(0, i) for i in range(B_s)]

    def one_step(t):
        tt = {}
        t0 = time.perf_counter()
        h = emb[rng.integers(0, V, B_s)].copy()
        x = rmsnorm_bf16(h, layers[0]["na"], cfg.rms_eps)
        pos = np.full(B_s, ctx - 1)
        for l, L in enumerate(layers):
            qkv = x @ L["qkv"].T
            q = bf16_round(rope(qkv[:, : H * hd].reshape(B_s, H, hd), pos, inv))
            out = np.empty((B_s, H, hd), np.float32)
            for i in range(B_s):
                for hh in range(H):
                    s = (Ks[l][i, :, hh // G, :] @ q[i, hh]) * scale
                    p = np.exp(s - s.max())
                    out[i, hh] = (p @ Vs[l][i, :, hh // G, :]) / p.sum()
            h = h + bf16_round(out.reshape(B_s, -1)) @ L["o"].T
            x = rmsnorm_bf16(h, L["nm"], cfg.rms_eps)
            gu = x @ L["gu"].T
            g_, u_ = gu[:, :dff], gu[:, dff:]
            h = h + bf16_round((g_ / (1 + np.exp(-g_))) * u_) @ L["down"].T
            x = rmsnorm_bf16(h, L["na"], cfg.rms_eps)
        tt["layers"] = (time.perf_counter() - t0) * (cfg.n_layers / layers_timed)
        t1 = time.perf_counter()
        logits = (x @ emb.T).astype(np.float32)
        tt["head"] = time.perf_counter() - t1
        t2 = time.perf_counter()
        for i in range(B_s):
            k = (t + i) % 7
            lo = cfg.audio_base + k * cfg.codebook_size
            row = np.full(V, -np.inf)
            row[lo: lo + cfg.codebook_size] = logits[i, lo: lo + cfg.codebook_size]
            osamp.sample(row, 0.6, None, 0.8, 1.3, windows[i], rngs[i])
        tt["sample"] = time.perf_counter() - t2
        t3 = time.perf_counter()
        codes = rng.integers(0, cfg.codebook_size, size=(1, 7))
        snac.decode(codes)
        tt["detok"] = (time.perf_counter() - t3) * (B_s / 8.0)
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
    audio = B_s / 86.0  # each decoded token = 1/86 s of audio (profiles.py:183)
    return {
        "audio_s_per_s": audio / (ms / 1000),
        "ms_per_step": ms,
        "cores": _cores(),
        "sample": f"{B_s} streams x 1 decode step at ctx {ctx}: {layers_timed}/28 layers timed (x14), full-vocab "
                  f"head, reference sampler (T .6, top-p .8, rp 1.3), 1/8 detok frame per stream; "
                  f"{len(tot)} steps; breakdown ms " +
                  ", ".join(f"{k}={np.mean([p[k] for p in parts]) * 1000:.1f}" for k in parts[0]),
    }
