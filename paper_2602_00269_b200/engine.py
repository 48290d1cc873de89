"""StreamingEngine: wall-clock serving loop over the fused B200 path.

Same loop shape as the reference's virtual-clock ``SimEngine.run``
(engine.py:364-404) and ``run_iteration`` (engine.py:204-360), with the
reference's own ``preprocess`` (model_api.py:238), ``chunk_ready``
(profiles.py:235) and streaming-aware ``schedule`` (scheduler.py:218) called
unchanged; what changes is the execution underneath:

* one ``vox_forward`` per iteration runs prefill and decode rows as ONE mixed
  batch through a per-bucket CUDA graph; tokens are sampled on the device
  (K1) and written straight into the device token store — no logits or
  token ids cross PCIe on the hot path;
* ``vox_detok`` runs on a second stream ordered after the forward that
  produced each window's last token (the data-ready rule of engine.py:311-314)
  so detokenization overlaps the next LM steps (asynchronous pipeline,
  PipelineMode.ASYNCHRONOUS, engine.py:355-360);
* the host prepares iteration k+1 while the GPU runs k (the scheduler only
  needs token COUNTS, which are known without a device round trip); run-ahead
  is bounded to ``max_inflight`` forwards;
* chunk availability ``t_i`` is the CUDA-event time at which the chunk's PCM
  has landed in pinned host memory, on the same clock as arrivals.

The resulting ``Trace`` feeds the reference metrics (core.py:300-333)
unchanged: TTFA, pooled viability, percentiles, inverse RTF.
"""

from __future__ import annotations

import gc
import time
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from ._ref import core, model_api, profiles, scheduler
from .device import Sampling, VoxDevice


@dataclass
class _Run:
    req: core.Request
    state: model_api.SamplingState
    cache: model_api.DetokenizerCache
    slot: int
    pending_chunks: int = 0
    dslot: int = -1  # slot on the detokenizer context (disaggregated mode)


@dataclass
class EngineStats:
    iterations: int = 0
    lm_rows: int = 0
    decode_rows: int = 0
    decode_ctx: int = 0  # sum over decode rows of the context each attends (pos + 1)
    prefill_rows: int = 0
    detok_calls: int = 0
    detok_windows: int = 0
    pcm_samples: int = 0
    host_s: float = 0.0
    wait_s: float = 0.0  # host time blocked on the device (run-ahead bound)
    decisions: list = field(default_factory=list)


class StreamingEngine:
    def __init__(self, dev: VoxDevice, profile, policy, seed: int, max_inflight: int = 2,
                 delivery_overhead_us: int = 0, keep_pcm: bool = False, detok_dev: Optional[VoxDevice] = None):
        """detok_dev: disaggregated LM -> detok (reference engine.py:119-123,150-156,
        PAPER.md:300): the LM runs on `dev`, detokenization on `detok_dev` (another GPU,
        a ``config.detok_role`` context with the same detokenizer weights); each window's
        tokens cross over vox_copy_tokens (NVLink peer copy) ordered after the forward
        that produced them."""
        if profile.vocab_size != dev.cfg.vocab:
            raise ValueError("profile vocab must equal the model vocab")
        self.dev = dev
        self.profile = profile
        self.policy = policy
        self.seed = seed
        self.max_inflight = max_inflight
        self.delivery_overhead_us = delivery_overhead_us
        self.sampling = Sampling.from_ref(profile.sampling_defaults)
        self.ddev = detok_dev or dev
        self.disaggregated = detok_dev is not None
        self.live: dict[int, _Run] = {}
        self.trace = core.Trace()
        self.stats = EngineStats()
        self.keep_pcm = keep_pcm
        self.pcm: dict[int, list[np.ndarray]] = {}
        self._tickets: list[tuple[int, list[tuple[_Run, object, int, int]]]] = []
        self._fwd_seqs: list[int] = []
        self._t0 = 0.0
        # on_chunk(request_id, chunk_index, available_us, playback_us, pcm or None, final):
        # called from the engine loop when a chunk's PCM has landed (serve.py streams it)
        self.on_chunk = None

    # ------------------------------------------------------------------ clock
    def now_us(self) -> int:
        return int((time.perf_counter() - self._t0) * 1e6)

    # ------------------------------------------------------------------ lifecycle
    def admit(self, rid: int, spec) -> None:
        req, cache, state = model_api.preprocess(
            prompt_tokens=spec.prompt_tokens, profile=self.profile, seed=self.seed, request_id=rid,
            arrival_us=spec.arrival_us, target_output_tokens=spec.target_output_tokens)
        slot = self.dev.admit(state.seed, spec.prompt_tokens, spec.target_output_tokens, self.sampling)
        dslot = -1
        if self.disaggregated:
            dslot = self.ddev.admit(state.seed, spec.prompt_tokens, spec.target_output_tokens, self.sampling)
        self.live[rid] = _Run(req=req, state=state, cache=cache, slot=slot, dslot=dslot)

    def _snapshot(self) -> list:
        out = []
        for run in self.live.values():
            r = run.req
            win = profiles.chunk_ready(r.tokens_generated, r.chunks_emitted, self.profile,
                                       stream_ended=r.done_generating, request=r.id)
            if r.done_generating:
                lm = None
            elif not r.prefilled:
                lm = model_api.StageKind.PREFILL
            else:
                lm = model_api.StageKind.DECODE
            out.append(scheduler.QueueEntry(request=r, ready_window=win, lm_work=lm))
        return out

    # ------------------------------------------------------------------ one iteration
    def run_iteration(self, decision) -> None:
        st = self.stats
        st.iterations += 1
        rows = []
        for e in decision.lm:
            run = self.live[e.request]
            r = run.req
            if e.kind is model_api.StageKind.PREFILL:
                rows += [[run.slot, p, -1, 0] for p in range(r.prompt_tokens - 1)]
                st.prefill_rows += r.prompt_tokens - 1
                r.prefilled = True
            else:
                rows.append([run.slot, r.prompt_tokens - 1 + r.tokens_generated, -1, 1])
                st.decode_ctx += r.prompt_tokens + r.tokens_generated
                r.tokens_generated += 1
                st.decode_rows += 1
        if rows:
            # bound host run-ahead: at most max_inflight forwards on the device
            if len(self._fwd_seqs) >= self.max_inflight:
                w0 = time.perf_counter()
                self.dev.forward_wait(self._fwd_seqs.pop(0))
                st.wait_s += time.perf_counter() - w0
            cap = self.dev.cfg.max_rows
            for a in range(0, len(rows), cap):
                self.dev.forward(np.asarray(rows[a:a + cap], np.int32))
            self._fwd_seqs.append(self.dev.forward_seq())
            st.lm_rows += len(rows)
        if decision.detok:
            self._issue_detok(decision.detok)
        st.decisions.append((len(decision.lm), len(decision.detok)))

    def _issue_detok(self, specs: Sequence) -> None:
        cfg = self.ddev.cfg
        batches, cur, frames = [], [], 0
        for w in specs:
            f = 4 * -(-w.new_tokens // cfg.frame_tokens)
            if cur and frames + f > cfg.max_detok_frames:
                batches.append(cur)
                cur, frames = [], 0
            cur.append(w)
            frames += f
        if cur:
            batches.append(cur)
        for b in batches:
            # a ticket is valid for VOX_TICKET_RING (32) calls: retire old ones first
            while len(self._tickets) >= 24:
                self._poll(block=True)
            if self.disaggregated:
                spans = []
                for w in b:
                    run = self.live[w.request]
                    p0 = run.req.prompt_tokens + w.start
                    spans.append([run.dslot, p0, run.slot, p0, w.length])
                self.ddev.copy_tokens(self.dev, np.asarray(spans, np.int32))
                arr = np.asarray([[self.live[w.request].dslot, w.index, w.start, w.length, w.new_tokens,
                                   int(w.final)] for w in b], np.int32)
            else:
                arr = np.asarray([[self.live[w.request].slot, w.index, w.start, w.length, w.new_tokens,
                                   int(w.final)] for w in b], np.int32)
            ns, ticket = self.ddev.detok(arr, sync=False)
            items = []
            off = 0
            for w, n in zip(b, ns):
                run = self.live[w.request]
                r = run.req
                pb = core.playback_us_for(w.new_tokens, self.profile.token_rate)
                # reference bookkeeping happens at issue time (engine.py:339-342)
                r.chunks_emitted += 1
                r.covered_tokens += w.new_tokens
                r.playback_emitted_us += pb
                run.pending_chunks += 1
                items.append((run, w, pb, (off, int(n))))
                off += int(n)
            self._tickets.append((ticket, items))
            self.stats.detok_calls += 1
            self.stats.detok_windows += len(b)

    def _poll(self, block: bool = False) -> int:
        """Retire completed detok tickets (block=True: wait for at least one)."""
        done = 0
        while self._tickets:
            ticket, items = self._tickets[0]
            ok, t_ms = self.ddev.ticket_done(ticket)
            if not ok:
                if not block or done > 0:
                    break
                self.ddev.ticket_pcm(ticket)  # waits for the ticket's event
                ok, t_ms = self.ddev.ticket_done(ticket)
            self._tickets.pop(0)
            pcm = self.ddev.ticket_pcm(ticket) if (self.keep_pcm or self.on_chunk is not None) else None
            avail = int(t_ms * 1000) + self.delivery_overhead_us
            for run, w, pb, (off, n) in items:
                r = run.req
                self.trace.chunks.append(core.ChunkEvent(request=r.id, index=w.index, available_us=avail,
                                                         playback_us=pb, new_tokens=w.new_tokens))
                self.stats.pcm_samples += n
                if pcm is not None and self.keep_pcm:
                    self.pcm.setdefault(r.id, []).append(pcm[off:off + n].copy())
                if self.on_chunk is not None:
                    self.on_chunk(r.id, w.index, avail, pb, pcm[off:off + n].copy(), bool(w.final))
                run.pending_chunks -= 1
                if r.first_chunk_us is None:
                    r.first_chunk_us = avail
                    r.phase = core.Phase.STEADY_STATE
                if r.done_generating and r.covered_tokens >= r.target_output_tokens and run.pending_chunks == 0:
                    r.phase = core.Phase.FINISHED
                    self.dev.release(run.slot)
                    if self.disaggregated:
                        self.ddev.release(run.dslot)
                    self.trace.requests.append(self.live.pop(r.id).req)
            done += 1
        return done

    def shutdown(self) -> None:
        """Drain in-flight work and release every live slot (abandoned requests)."""
        while self._tickets:
            self._poll(block=True)
        self.dev.synchronize()
        self.ddev.synchronize()
        for run in list(self.live.values()):
            self.dev.release(run.slot)
            if self.disaggregated:
                self.ddev.release(run.dslot)
        self.live.clear()

    # ------------------------------------------------------------------ full run
    def run(self, arrivals: Sequence[tuple[int, object]], max_wall_s: Optional[float] = None) -> core.Trace:
        """Serve (request_id, ArrivalSpec) pairs in real time; returns the trace."""
        pending = sorted(arrivals, key=lambda p: (p[1].arrival_us, p[0]))
        idx = 0
        # The host loop must keep one step queued ahead of the GPU: a cyclic-GC
        # pass over the engine's objects stalls it for tens of ms (measured:
        # 3.5 -> 5.8 ms/step bench swings).  Collect now, freeze the survivors,
        # and defer collection until the run ends.
        gc_on = gc.isenabled()
        gc.collect()
        gc.freeze()
        gc.disable()
        self.dev.clock_reset()
        if self.disaggregated:
            self.ddev.clock_reset()
        self._t0 = time.perf_counter()
        t_host = 0.0
        while idx < len(pending) or self.live:
            now = self.now_us()
            if max_wall_s is not None and now > max_wall_s * 1e6:
                break
            cap = min(self.policy.max_live_requests, self.dev.cfg.max_slots)
            while idx < len(pending) and pending[idx][1].arrival_us <= now:
                if len(self.live) >= cap:  # the rest waits on the host (counts toward TTFA)
                    break
                self.admit(*pending[idx])
                idx += 1
            self._poll()
            if not self.live:
                if idx < len(pending):
                    time.sleep(max(0.0, (pending[idx][1].arrival_us - self.now_us()) / 1e6))
                continue
            h0 = time.perf_counter()
            snap = self._snapshot()
            decision = scheduler.schedule(snap, now, self.policy)
            t_host += time.perf_counter() - h0
            if decision.empty:
                # waiting on in-flight chunks or the next arrival
                if self._tickets:
                    self._poll(block=True)
                elif idx < len(pending):
                    time.sleep(max(0.0, min(0.001, (pending[idx][1].arrival_us - self.now_us()) / 1e6)))
                else:
                    raise RuntimeError(f"engine stall with {len(self.live)} live requests")
                continue
            self.run_iteration(decision)
        while self._tickets:
            self._poll(block=True)
        self.dev.synchronize()
        self.ddev.synchronize()
        gc.unfreeze()
        if gc_on:
            gc.enable()
        self.stats.host_s = t_host
        self.trace.requests.extend(run.req for run in self.live.values())
        self.trace.requests.sort(key=lambda r: r.id)
        self.trace.chunks.sort(key=lambda c: (c.available_us, c.request, c.index))
        return self.trace


    # ------------------------------------------------------------------ online serving
    def serve(self, inbox, stop, idle_s: float = 0.0005) -> None:
        """Online twin of ``run``: arrivals come from ``inbox`` (a queue.Queue of
        (request_id, prompt_tokens, output_tokens)) while the loop runs, each stamped with
        the engine clock when it is admitted; chunks are delivered through ``on_chunk``.
        Returns when ``stop`` is set and no request is live (graceful drain)."""
        import queue as _queue

        from ._ref import workload

        gc_on = gc.isenabled()
        gc.collect()
        gc.freeze()
        gc.disable()
        self.dev.clock_reset()
        if self.disaggregated:
            self.ddev.clock_reset()
        self._t0 = time.perf_counter()
        waiting: list = []
        try:
            while True:
                while True:
                    try:
                        waiting.append(inbox.get_nowait())
                    except _queue.Empty:
                        break
                if stop.is_set() and not self.live and not waiting and not self._tickets:
                    break
                now = self.now_us()
                cap = min(self.policy.max_live_requests, self.dev.cfg.max_slots)
                while waiting and len(self.live) < cap:
                    rid, P, T = waiting.pop(0)
                    self.admit(rid, workload.ArrivalSpec(arrival_us=now, prompt_tokens=P, target_output_tokens=T))
                self._poll()
                if not self.live:
                    time.sleep(idle_s)
                    continue
                decision = scheduler.schedule(self._snapshot(), now, self.policy)
                if decision.empty:
                    if self._tickets:
                        self._poll(block=True)
                    else:
                        time.sleep(idle_s)
                    continue
                self.run_iteration(decision)
            self.dev.synchronize()
        finally:
            gc.unfreeze()
            if gc_on:
                gc.enable()


def orpheus_profile(max_batch: int = 256):
    """orpheus_like (profiles.py:180-196) at the real Orpheus vocabulary and batch cap."""
    from dataclasses import replace

    from .config import ORPHEUS_VOCAB

    return replace(profiles.builtin_profile("orpheus_like"), vocab_size=ORPHEUS_VOCAB,
                   max_lm_batch=max_batch, max_detok_batch=max_batch)
