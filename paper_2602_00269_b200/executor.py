"""B200Executor: the reference ``Executor`` Protocol backed by the C-ABI library.

Drop-in for ``SyntheticExecutor`` (profiles.py:308-362) behind the unchanged
model-execution interface (model_api.py:199-226):

    engine = speechserve.engine.SimEngine(profile, policy, pipeline, seed)
    engine.executor = B200Executor(profile, model_cfg, weight_seed=0)

``forward`` runs the real backbone (prefill / decode rows) and returns masked
fp32 logits as float64 [B, codebooks, vocab] with the measured latency;
the reference ``sample()`` then picks tokens on the host exactly as before
(engine.py:294-303).  ``detokenize_windows`` runs the causal streaming
detokenizer with the request's cached left context and returns
``PcmChunkOut`` (an ``AudioChunkOut`` carrying the PCM).  The fused fast path
used by the serving engine (device-side sampling, async streams) is
``engine.StreamingEngine``.
"""

from __future__ import annotations

import time
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from ._ref import errors, model_api
from .config import ModelConfig
from .device import Sampling, VoxDevice


@dataclass(frozen=True)
class PcmChunkOut(model_api.AudioChunkOut):
    """AudioChunkOut (model_api.py:229-235) plus the decoded 24 kHz PCM."""

    pcm: Optional[np.ndarray] = field(default=None, repr=False, compare=False)


class B200Executor:
    """Implements speechserve.model_api.Executor on one B200 (one VoxDevice)."""

    def __init__(self, profile, model_cfg: ModelConfig, weight_seed: int = 0, device: int = 0,
                 dev: Optional[VoxDevice] = None):
        if profile.codebooks != 1:
            raise errors.CodebookMismatch("the Orpheus-style path is single-codebook")
        if profile.vocab_size != model_cfg.vocab:
            raise ValueError(f"profile vocab {profile.vocab_size} != model vocab {model_cfg.vocab}")
        self.profile = profile
        self.cfg = model_cfg
        self.dev = dev or VoxDevice(model_cfg, weight_seed, device)
        self.sampling = Sampling.from_ref(profile.sampling_defaults)
        self._slot: dict[int, int] = {}
        self._prompt: dict[int, int] = {}

    # ------------------------------------------------------------------ helpers
    def _slot_for(self, rid: int) -> int:
        try:
            return self._slot[rid]
        except KeyError:
            raise errors.CacheMissing(f"request {rid} has no device slot (not prefilled)") from None

    def release(self, rid: int) -> None:
        slot = self._slot.pop(rid, None)
        self._prompt.pop(rid, None)
        if slot is not None:
            self.dev.release(slot)

    # ------------------------------------------------------------------ Protocol
    def forward(self, batch: model_api.StageBatch) -> tuple[np.ndarray, float]:
        """Prefill/decode (model_api.py:209-211, lm_forward :278-294)."""
        n = len(batch)
        V = self.cfg.vocab
        t0 = time.perf_counter()
        if batch.kind is model_api.StageKind.PREFILL:
            rows = []
            for i, rid in enumerate(batch.request_ids):
                P = int(batch.prompt_tokens[i])
                if rid not in self._slot:
                    # the reference Protocol carries no target length: reserve the context
                    target = self.cfg.max_ctx - P - 1
                    if target < 1:
                        raise errors.PromptTooLong(f"prompt of {P} tokens exceeds context capacity")
                    self._slot[rid] = self.dev.admit(batch.seeds[i], P, target, self.sampling)
                    self._prompt[rid] = P
                rows += [[self._slot[rid], p, -1, 0] for p in range(P - 1)]
            if rows:
                self.dev.forward(np.asarray(rows, np.int32), sample=False, sync=True)
            logits = np.zeros((n, 1, V), np.float64)  # the engine discards prefill logits (engine.py:251)
            return logits, time.perf_counter() - t0
        if batch.kind is not model_api.StageKind.DECODE:
            raise ValueError(f"forward got {batch.kind}")
        rows = []
        for i, rid in enumerate(batch.request_ids):
            slot = self._slot_for(rid)
            step = int(batch.steps[i])
            pos = self._prompt[rid] - 1 + step
            # step 0 consumes the last prompt token; later steps the host-sampled id
            tok = -1 if step == 0 else int(batch.frames[i].ids[0, 0])
            rows.append([slot, pos, tok, 1])
        _, lg = self.dev.forward(np.asarray(rows, np.int32), sample=False, full_logits=True, sync=True)
        out = np.full((n, 1, V), -np.inf, np.float64)
        for i, step in enumerate(batch.steps):
            lo, hi = self.audio_range(int(step))
            out[i, 0, lo:hi] = lg[i, lo:hi]
        return out, time.perf_counter() - t0

    def audio_range(self, step: int) -> tuple[int, int]:
        c = self.cfg
        if c.audio_base < 0:
            return 0, c.vocab
        lo = c.audio_base + (step % c.frame_tokens) * c.codebook_size
        return lo, lo + c.codebook_size

    def detokenize_windows(self, batch, specs: Sequence, windows: Sequence[np.ndarray],
                           caches: Sequence[model_api.DetokenizerCache]):
        """Chunk-wise streaming detokenization (model_api.py:213-220, profiles.py:333-356)."""
        t0 = time.perf_counter()
        rows = []
        for spec, win, cache in zip(specs, windows, caches):
            slot = self._slot_for(spec.request)
            # the host engine sampled these ids: make the device token store authoritative
            P = self._prompt[spec.request]
            self.dev.write_tokens(slot, P + spec.start, np.asarray(win)[:, 0].astype(np.int32).tolist())
            rows.append([slot, spec.index, spec.start, spec.length, spec.new_tokens, int(spec.final)])
        pcms, _ = self.dev.detok(np.asarray(rows, np.int32), sync=True)
        outs = []
        for spec, win, cache, pcm in zip(specs, windows, caches, pcms):
            cache.window_ids = np.array(win, copy=True)
            cache.calls += 1
            cache.bytes_held = 4 * pcm.size
            from ._ref import core

            outs.append(PcmChunkOut(request=spec.request, new_tokens=spec.new_tokens,
                                    playback_us=core.playback_us_for(spec.new_tokens, self.profile.token_rate),
                                    pcm=pcm))
            if spec.final:
                self.release(spec.request)
        return outs, time.perf_counter() - t0

    def depth_logits(self, seed: int, step: int, codebook: int) -> np.ndarray:
        raise errors.DepthStageUnsupported("the Orpheus-style path has no depth stage")

    def depth_latency(self, batch_size: int) -> float:
        raise errors.DepthStageUnsupported("the Orpheus-style path has no depth stage")
