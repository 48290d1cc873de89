"""CPU: the streaming wire format and the HTTP frontend's protocol.

The frontend runs here over a stand-in engine (same serve()/on_chunk contract as
engine.StreamingEngine, synthetic audio); the GPU test drives the real engine."""

import asyncio
import threading
import time
from types import SimpleNamespace

import numpy as np
from hypothesis import given, settings
from hypothesis import strategies as st

from paper_2602_00269_b200._ref import core
from paper_2602_00269_b200.serve import ChunkFrame, VoxServer, generate, load_test, pcm16


@settings(max_examples=200, deadline=None)
@given(st.integers(0, 2**64 - 1), st.integers(0, 2**32 - 1), st.integers(0, 2**64 - 1), st.integers(0, 2**32 - 1),
       st.binary(max_size=300), st.booleans(), st.booleans())
def test_frame_round_trip(rid, idx, at, pb, payload, fin, err):
    f = ChunkFrame(rid, idx, at, pb, payload, fin, err)
    data = f.encode()
    assert len(data) == 4 + 28 + len(payload)
    got, rest = ChunkFrame.decode_stream(data + data[:7])
    assert got == [f] and rest == data[:7]


def test_pcm16_scaling():
    x = np.array([0.0, 0.5, -1.0, 2.0], np.float32)
    assert np.frombuffer(pcm16(x), "<i2").tolist() == [0, 16384, -32767, 32767]


class FakeEngine:
    """serve(inbox, stop) + on_chunk: emits ceil(T / 7) chunks of 2048 samples per request."""

    def __init__(self, chunk_ms=2.0):
        self.policy = SimpleNamespace(max_live_requests=4)
        self.dev = SimpleNamespace(cfg=SimpleNamespace(max_slots=4, max_ctx=1024))
        self.trace = core.Trace()
        self.on_chunk = None
        self._t0 = 0.0
        self.chunk_ms = chunk_ms

    def serve(self, inbox, stop):
        self._t0 = time.perf_counter()
        while not stop.is_set() or not inbox.empty():
            try:
                rid, P, T = inbox.get(timeout=0.01)
            except Exception:
                continue
            n = -(-T // 7)
            for k in range(1, n + 1):
                time.sleep(self.chunk_ms / 1e3)
                now = int((time.perf_counter() - self._t0) * 1e6)
                self.on_chunk(rid, k, now, 85333, np.full(2048, 0.25 * k / n, np.float32), k == n)


def test_http_protocol_and_load_client():
    async def main():
        srv = await VoxServer(FakeEngine()).start()
        st200, arr, frames = await generate("127.0.0.1", srv.port, 21, 10, time.perf_counter())
        assert st200 == 200 and [f.chunk_index for _, f in frames] == [1, 2, 3] and frames[-1][1].is_final
        assert all(len(f.payload) == 4096 and f.playback_ms == 85 for _, f in frames)
        st400, _, _ = await generate("127.0.0.1", srv.port, 0, 10)
        assert st400 == 400
        from paper_2602_00269_b200._ref import workload

        spec = workload.WorkloadSpec(rate=50.0, duration_s=0.2, prompt_dist=workload.fixed(8),
                                     output_dist=workload.fixed(14), seed=3)
        res = await load_test("127.0.0.1", srv.port, spec)
        assert not res["errors"] and res["report"]["requests_completed"] + res["rejected"] == res["requests"]
        assert max(res["client_minus_server_ttfa_ms"]) < 20.0  # SPEC.md:720 delivery-overhead bound
        srv.draining = True
        st503, _, _ = await generate("127.0.0.1", srv.port, 7, 10)
        assert st503 == 503
        await srv.shutdown(5.0)

    asyncio.run(main())


def test_429_beyond_live_cap():
    async def main():
        eng = FakeEngine(chunk_ms=30.0)
        srv = await VoxServer(eng, max_live=1).start()
        t0 = time.perf_counter()
        a = asyncio.create_task(generate("127.0.0.1", srv.port, 14, 4, t0))
        await asyncio.sleep(0.01)
        st, _, _ = await generate("127.0.0.1", srv.port, 7, 4, t0)
        assert st == 429
        assert (await a)[0] == 200
        await srv.shutdown(5.0)

    asyncio.run(main())
