"""CPU: StreamingEngine host logic (scheduling, chunk bookkeeping, slot lifecycle) with a fake device.

The fake device does no compute; it records what the engine asks for so the
host side can be checked against the reference's own rules: every request's
chunk sequence (index, new_tokens) equals what chunk_ready yields
(profiles.py:235-290), audio is conserved (SPEC AC2), windows reach the
device in order, and every slot is released exactly once.
"""

import time
from dataclasses import dataclass

import numpy as np

from paper_2602_00269_b200._ref import core, profiles, scheduler, workload
from paper_2602_00269_b200.engine import StreamingEngine, orpheus_profile


@dataclass
class _Cfg:
    vocab: int = 156940
    max_rows: int = 1024
    max_detok_frames: int = 256
    frame_tokens: int = 7
    max_slots: int = 64


class FakeDevice:
    def __init__(self):
        self.cfg = _Cfg()
        self.free = list(range(self.cfg.max_slots))
        self.live = {}
        self.rows = []
        self.windows = []
        self.released = []
        self._tickets = {}
        self._next = 0
        self._seq = 0
        self.t0 = time.perf_counter()

    def clock_reset(self):
        self.t0 = time.perf_counter()

    def admit(self, seed, P, T, sampling):
        s = self.free.pop(0)
        self.live[s] = dict(P=P, T=T, pos=[], covered=0)
        return s

    def release(self, slot):
        assert slot in self.live
        del self.live[slot]
        self.released.append(slot)
        self.free.append(slot)

    def forward(self, rows, **kw):
        self._seq += 1
        for s, pos, tok, samp in rows:
            self.live[int(s)]["pos"].append(int(pos))
        self.rows.append(np.array(rows))
        return None, None

    def forward_seq(self):
        return self._seq

    def forward_wait(self, seq):
        pass

    def detok(self, arr, sync=False):
        ns = []
        for slot, index, start, length, new, final in arr:
            st = self.live[int(slot)]
            assert start + length - new == st["covered"], "windows must arrive in order"
            st["covered"] += int(new)
            self.windows.append((int(slot), int(index), int(start), int(length), int(new), int(final)))
            ns.append(int(new) * 2048 // 7)
        t = self._next
        self._next += 1
        self._tickets[t] = (time.perf_counter() - self.t0) * 1000 + 5.0
        return np.array(ns), t

    def ticket_done(self, t):
        return True, self._tickets[t]

    def ticket_pcm(self, t):
        return np.zeros(1, np.float32)

    def synchronize(self):
        pass


def _expected_chunks(T, prof):
    out, emitted = [], 0
    while True:
        # streaming readiness while generating, flush once the stream ended
        w = profiles.chunk_ready(T, emitted, prof, stream_ended=True)
        if w is None:
            return out
        out.append((w.index, w.new_tokens))
        emitted += 1


def test_engine_chunks_match_reference_rules():
    dev = FakeDevice()
    prof = orpheus_profile(max_batch=32)
    policy = scheduler.PolicyConfig(max_lm_batch=32, max_detok_batch=32)
    spec = workload.WorkloadSpec(rate=200.0, duration_s=0.1, prompt_dist=workload.fixed(12),
                                 output_dist=workload.uniform_int(1, 80), seed=3)
    arr = list(enumerate(workload.build_workload(spec)))
    eng = StreamingEngine(dev, prof, policy, seed=3)
    tr = eng.run(arr)
    assert len(tr.requests) == len(arr)
    assert all(r.phase is core.Phase.FINISHED for r in tr.requests)
    assert sorted(dev.released) == sorted(set(dev.released)) and len(dev.released) == len(arr)
    for rid, a in arr:
        got = [(c.index, c.new_tokens) for c in tr.chunks_for(rid)]
        assert got == _expected_chunks(a.target_output_tokens, prof), rid
        assert sum(n for _, n in got) == a.target_output_tokens  # audio conservation
    # every decode row consumed the next position; prefill covered prompt[:-1]
    rep = core.build_report(tr)
    assert rep.requests_completed == len(arr) and rep.viability_fraction > 0


def test_engine_positions_are_contiguous():
    dev = FakeDevice()
    prof = orpheus_profile(max_batch=16)
    policy = scheduler.PolicyConfig(max_lm_batch=16, max_detok_batch=16)
    arr = [(i, workload.ArrivalSpec(arrival_us=0, prompt_tokens=5, target_output_tokens=30)) for i in range(5)]
    eng = StreamingEngine(dev, prof, policy, seed=0)
    seen = {}
    orig = dev.forward

    def spy(rows, **kw):
        for s, pos, tok, samp in rows:
            seen.setdefault(int(s), []).append(int(pos))
        return orig(rows, **kw)

    dev.forward = spy
    eng.run(arr)
    for s, pos in seen.items():
        assert pos == list(range(5 - 1 + 30)), (s, pos)  # prompt[:-1] then 30 decode positions
