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
                 dev: Optional[VoxDevice] = None, detokenizer=None):
        """detokenizer: None -> the ctx's SNAC-style decoder (Orpheus, config 2); a
        ``cosy_detok.CosyDetokenizer`` -> the CosyVoice2-style flow + vocoder (config 4)."""
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
        self.detokenizer = detokenizer
        self._dslot: dict[int, int] = {}

    # ------------------------------------------------------------------ helpers
    def _slot_for(self, rid: int) -> int:
        try:
            return self._slot[rid]
        except KeyError:
            raise errors.CacheMissing(f"request {rid} has no device slot (not prefilled)") from None

    def _admit(self, seed: int, P: int) -> int:
        # the reference Protocol carries no target length: reserve the rest of the context
        target = self.cfg.max_ctx - P - 1
        if target < 1:
            raise errors.PromptTooLong(f"prompt of {P} tokens exceeds context capacity {self.cfg.max_ctx}")
        try:
            return self.dev.admit(seed, P, target, self.sampling)
        except MemoryError as e:
            raise MemoryError(
                f"{e}: this executor holds at most {self.cfg.max_slots} live requests (ModelConfig.max_slots); "
                "set PolicyConfig.max_live_requests <= max_slots") from None

    def release(self, rid: int) -> None:
        slot = self._slot.pop(rid, None)
        self._prompt.pop(rid, None)
        if slot is not None:
            self.dev.release(slot)
        ds = self._dslot.pop(rid, None)
        if ds is not None:
            self.detokenizer.release(ds)

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
                    self._slot[rid] = self._admit(batch.seeds[i], P)
                    self._prompt[rid] = P
                    if self.detokenizer is not None:
                        self._dslot[rid] = self.detokenizer.open(int(batch.seeds[i]))
                rows += [[self._slot[rid], p, -1, 0] for p in range(P - 1)]
            # prompts of many requests can exceed one forward's row capacity: split
            # at max_rows (positions of one request stay in order, so the causal
            # K/V of a later chunk is already appended)
            cap = self.cfg.max_rows
            for a in range(0, len(rows), cap):
                self.dev.forward(np.asarray(rows[a:a + cap], np.int32), sample=False, sync=True)
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
        # logits only (VOX_FWD_SAMPLE clear): the host's sample() decides (engine.py:294-303)
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
        if self.detokenizer is not None:
            return self._detok_cosy(specs, windows, caches)
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

    def _detok_cosy(self, specs, windows, caches):
        """CosyVoice2-style: each window's new speech tokens (ids - audio_base; the LM's
        3 special ids past the 6,561 codes clamp to the last code) through the flow +
        stateful vocoder of the request's stream."""
        from ._ref import core

        t0 = time.perf_counter()
        c = self.cfg
        slots, toks = [], []
        for spec, win in zip(specs, windows):
            if spec.request not in self._dslot:
                raise errors.CacheMissing(f"request {spec.request} has no detokenizer stream")
            w = np.asarray(win)[:, 0]
            ids = w[w.shape[0] - spec.new_tokens:] - max(c.audio_base, 0)
            slots.append(self._dslot[spec.request])
            toks.append(np.clip(ids, 0, self.detokenizer.cfg.vocab - 1).astype(np.int32))
        pcms = self.detokenizer.decode(slots, toks) if slots else []
        outs = []
        for spec, win, cache, pcm in zip(specs, windows, caches, pcms):
            cache.window_ids = np.array(win, copy=True)
            cache.calls += 1
            cache.bytes_held = 4 * pcm.size
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


class CsmExecutor:
    """The reference ``Executor`` Protocol for a depth-stage profile (CSM-1B-style, BASELINE
    config 3; ``profiles.py:214-231`` depth_like shape) on two device contexts.

    The reference engine drives one backbone forward per frame (engine.py:258-273), then
    ``depth_forward`` (model_api.py:438-458) asks ``depth_logits(seed, step, codebook)``
    for codebooks 1..C-1 and samples each on the host, and only then samples codebook 0
    from ``forward``'s logits (engine.py:294-303).  A real depth decoder conditions
    codebook k on codebooks 0..k-1 of the same frame, which the Protocol never passes
    back.  So ``forward`` runs the whole frame on the device -- backbone (codebook 0 by
    K1) then the depth decoder's C-1 positions (each codebook by K1) -- and serves the
    logits K1 decided from:

    * greedy profiles with repetition penalty 1 ("logits" mode): the real logits of
      every codebook, read back exactly as K1 consumed them; the host's greedy
      ``sample()`` picks the same codes (K1 greedy is bit-exact to it), so host and
      device histories agree, which ``forward`` checks on the next frame
      (``mismatches``);
    * otherwise ("decided" mode): a one-hot row (0 at the device's code, -inf
      elsewhere), so the host's ``sample()`` returns the device's draw -- the Protocol's
      logits cannot carry a conditional depth distribution whose host draw the
      device could follow.

    The host's previous frame (``batch.frames``) is written into the device token /
    frame stores before each backbone step, so the device always continues the
    history the engine recorded.  Latencies are measured wall time of the device work.
    """

    def __init__(self, profile, bcfg: ModelConfig, dcfg: ModelConfig, weight_seed: int = 0, device: int = 0,
                 mimi_cfg=None):
        from .config import MimiConfig
        from .csm import CsmFrames
        from .mimi import MimiDecoder

        if not profile.has_depth_stage:
            raise errors.DepthStageUnsupported(f"profile {profile.name} has no depth stage")
        if profile.codebooks != bcfg.n_codebooks or profile.vocab_size != bcfg.codebook_size:
            raise errors.CodebookMismatch("profile codebooks/vocab must match the backbone's frames")
        self.profile = profile
        self.bcfg, self.dcfg = bcfg, dcfg
        self.bb = VoxDevice(bcfg, weight_seed, device)
        self.dp = VoxDevice(dcfg, weight_seed + 1, device)
        self.pipe = CsmFrames(self.bb, self.dp)
        p = profile.sampling_defaults
        self.sampling = Sampling.from_ref(p)
        self.decided = p.temperature > 0 or p.repetition_penalty != 1.0
        self.C, self.cs, self.base = bcfg.n_codebooks, bcfg.codebook_size, bcfg.audio_base
        self._slot: dict[int, tuple[int, int, int]] = {}  # rid -> (bslot, dslot, prompt)
        self._frames: dict[tuple[int, int], np.ndarray] = {}  # (seed, step) -> [C, cs] logits
        self._codes: dict[int, np.ndarray] = {}  # rid -> device codes of its last frame
        self._depth_s = 0.0
        self.mismatches = 0
        self.frames_run = 0
        # K7: the Mimi-style streaming detokenizer over this profile's codebooks
        mc = mimi_cfg or MimiConfig(max_slots=bcfg.max_slots, max_frames=max(64, profile.max_detok_batch *
                                                                            profile.chunk_size))
        if mc.n_q != self.C or mc.cb_size != self.cs:
            from dataclasses import replace as _replace

            mc = _replace(mc, n_q=self.C, cb_size=self.cs)
        self.mimi = MimiDecoder(mc, weight_seed + 2, device)
        self._mslot: dict[int, int] = {}
        self._covered: dict[int, int] = {}

    def close(self) -> None:
        self.bb.close()
        self.dp.close()
        self.mimi.close()

    def release(self, rid: int) -> None:
        s = self._slot.pop(rid, None)
        self._codes.pop(rid, None)
        self._covered.pop(rid, None)
        if s is not None:
            self.bb.release(s[0])
            self.dp.release(s[1])
        ms = self._mslot.pop(rid, None)
        if ms is not None:
            self.mimi.release(ms)

    def _rows_logits(self, dev: VoxDevice, n: int) -> np.ndarray:
        lg, _ = dev.read_logits()
        assert lg.shape == (n, self.cs)
        return lg

    def forward(self, batch: model_api.StageBatch) -> tuple[np.ndarray, float]:
        n, V, C = len(batch), self.profile.vocab_size, self.C
        t0 = time.perf_counter()
        if batch.kind is model_api.StageKind.PREFILL:
            rows = []
            for i, rid in enumerate(batch.request_ids):
                P = int(batch.prompt_tokens[i])
                if rid not in self._slot:
                    target = self.bcfg.max_ctx - P - 1
                    if target < 1:
                        raise errors.PromptTooLong(f"prompt of {P} tokens exceeds context capacity")
                    st = self.pipe.admit(batch.seeds[i], P, target, self.sampling, self.sampling)
                    self._slot[rid] = (st.bslot, st.dslot, P)
                    self._mslot[rid] = self.mimi.open()
                    self._covered[rid] = 0
                rows += [[self._slot[rid][0], p, -1, 0] for p in range(P - 1)]
            for a in range(0, len(rows), self.bcfg.max_rows):
                self.bb.forward(np.asarray(rows[a:a + self.bcfg.max_rows], np.int32), sample=False, sync=True)
            return np.zeros((n, C, V), np.float64), time.perf_counter() - t0
        if batch.kind is not model_api.StageKind.DECODE:
            raise ValueError(f"forward got {batch.kind}")
        rows = []
        for i, rid in enumerate(batch.request_ids):
            if rid not in self._slot:
                raise errors.CacheMissing(f"request {rid} has no device slot (not prefilled)")
            bslot, dslot, P = self._slot[rid]
            step = int(batch.steps[i])
            pos = P - 1 + step
            tok = -1
            if step > 0:  # the host's previous frame becomes this position's input
                ids = np.asarray(batch.frames[i].ids[0], np.int64)
                prev = self._codes.get(rid)
                if prev is not None and not np.array_equal(prev, ids):
                    self.mismatches += 1
                tok = int(self.base + ids[0])
                self.bb.write_frame(bslot, pos, (self.base + np.arange(1, C) * self.cs + ids[1:])[None, :])
            rows.append([bslot, pos, tok, 1])
        rows = np.asarray(rows, np.int32)
        c0, _ = self.bb.forward(rows, want_tokens=True)
        lg0 = self._rows_logits(self.bb, n)
        t1 = time.perf_counter()
        # depth decoder: position 0 = projected backbone state, 1 = c0, k samples codebook k
        dsl = [self._slot[rid][1] for rid in batch.request_ids]
        self.dp.project_ext(self.bb, n)
        self.dp.link_tokens(self.bb, np.array([[d, 1, b, p + 1] for d, (b, p) in
                                               zip(dsl, [(r[0], r[1]) for r in rows])], np.int32), -self.base, 0)
        logits = np.empty((n, C, V), np.float64)
        logits[:, 0] = lg0
        drows = np.array([[d, 0, -2, 0] for d in dsl] + [[d, 1, -1, 1] for d in dsl], np.int32)
        self.dp.forward(drows, want_tokens=False)
        logits[:, 1] = self._rows_logits(self.dp, n)
        for k in range(2, C):
            self.dp.forward(np.array([[d, k, -1, 1] for d in dsl], np.int32))
            logits[:, k] = self._rows_logits(self.dp, n)
        codes = np.zeros((n, C), np.int64)
        codes[:, 0] = np.asarray(c0) - self.base
        for i, d in enumerate(dsl):
            codes[i, 1:] = self.dp.read_tokens(d, 2, C - 1) - np.arange(1, C) * self.cs
        self._depth_s = time.perf_counter() - t1
        if self.decided:
            logits[:] = -np.inf
            for i in range(n):
                logits[i, np.arange(C), codes[i]] = 0.0
        for i, rid in enumerate(batch.request_ids):
            self._codes[rid] = codes[i]
            self._frames[(int(batch.seeds[i]), int(batch.steps[i]))] = logits[i]
        self.frames_run += n
        return logits, t1 - t0

    def depth_logits(self, seed: int, step: int, codebook: int) -> np.ndarray:
        """Codebook `codebook` of frame `step` (model_api.py:222-223), computed by forward."""
        try:
            row = self._frames[(int(seed), int(step))]
        except KeyError:
            raise errors.CacheMissing(f"no depth frame for seed {seed} step {step}") from None
        if codebook == self.C - 1:
            self._frames.pop((int(seed), int(step)))
        return row[codebook].copy()

    def depth_latency(self, batch_size: int) -> float:
        return self._depth_s

    def detokenize_windows(self, batch, specs: Sequence, windows: Sequence[np.ndarray],
                           caches: Sequence[model_api.DetokenizerCache]):
        """Stateful Mimi decode of each window's new frames (model_api.py:213-220;
        profiles.py:333-356 is the stub it replaces): the request's stream on the K7
        context continues from its cached history, so the chunks concatenate to the
        full-sequence decode."""
        from ._ref import core

        t0 = time.perf_counter()
        slots, codes = [], []
        for spec, win in zip(specs, windows):
            if spec.request not in self._mslot:
                raise errors.CacheMissing(f"request {spec.request} has no detokenizer stream")
            w = np.asarray(win)
            g0 = spec.start + spec.length - spec.new_tokens
            if g0 != self._covered[spec.request]:
                raise errors.WindowRuleViolation("the stateful Mimi decoder needs in-order windows")
            slots.append(self._mslot[spec.request])
            codes.append(w[w.shape[0] - spec.new_tokens:])
        pcms = self.mimi.decode(slots, codes) if slots else []
        outs = []
        for spec, win, cache, pcm in zip(specs, windows, caches, pcms):
            cache.window_ids = np.array(win, copy=True)
            cache.calls += 1
            cache.bytes_held = 4 * pcm.size
            self._covered[spec.request] += spec.new_tokens
            outs.append(PcmChunkOut(request=spec.request, new_tokens=spec.new_tokens,
                                    playback_us=core.playback_us_for(spec.new_tokens, self.profile.token_rate),
                                    pcm=pcm))
            if spec.final:
                self.release(spec.request)
        return outs, time.perf_counter() - t0
