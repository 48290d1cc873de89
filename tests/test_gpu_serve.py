"""GPU: the HTTP streaming frontend (serve.py) over the real StreamingEngine (tiny config):
a Poisson load test from the built-in client; every request streams its frames to the
final flag, the PCM payloads are the engine's audio (== the SNAC oracle of the tokens
the device generated), and client TTFA exceeds server TTFA only by delivery overhead
(< 20 ms on localhost)."""

import asyncio
from dataclasses import replace

import numpy as np
import pytest

from oracle.snac import SnacOracle
from paper_2602_00269_b200._ref import profiles, scheduler, workload

pytestmark = pytest.mark.gpu


def test_http_streaming_load_test(tiny_dev, tiny_cfg):
    from paper_2602_00269_b200.engine import StreamingEngine
    from paper_2602_00269_b200.serve import VoxServer, load_test

    prof = replace(profiles.builtin_profile("orpheus_like"), vocab_size=156940, max_lm_batch=64, max_detok_batch=64)
    eng = StreamingEngine(tiny_dev, prof, scheduler.PolicyConfig(max_lm_batch=64, max_detok_batch=64), seed=2)
    toks = {}
    orig_release = tiny_dev.release

    def grab(slot):
        run = next(r for r in eng.live.values() if r.slot == slot)
        toks[run.req.id] = tiny_dev.read_tokens(slot, run.req.prompt_tokens, run.req.target_output_tokens)
        orig_release(slot)

    tiny_dev.release = grab
    spec = workload.WorkloadSpec(rate=30.0, duration_s=0.3, prompt_dist=workload.fixed(16),
                                 output_dist=workload.uniform_int(20, 50), seed=5)

    async def main():
        srv = await VoxServer(eng).start()
        try:
            return await load_test("127.0.0.1", srv.port, spec)
        finally:
            await srv.shutdown(30.0)

    try:
        res = asyncio.run(main())
    finally:
        tiny_dev.release = orig_release
    assert not res["errors"] and res["rejected"] == 0
    rep = res["report"]
    assert rep["requests_completed"] == res["requests"] > 0
    gaps = res["client_minus_server_ttfa_ms"]
    print(f"serve: {res['requests']} requests, client p90 TTFA {rep['ttfa_p90'] * 1e3:.1f} ms, viability "
          f"{rep['viability_fraction']:.3f}, client-server TTFA gap max {max(gaps):.2f} ms")
    assert max(gaps) < 20.0
    # payloads: each request's streamed PCM == the SNAC oracle of the tokens the device generated
    snac = SnacOracle(tiny_cfg, 1234)
    assert set(res["audio"]) == set(toks)
    for rid in sorted(res["audio"])[:3]:
        pcm = res["audio"][rid].astype(np.float32) / 32767.0
        ref = snac.decode_tokens(toks[rid], len(toks[rid]))[: len(pcm)]
        assert len(pcm) == len(ref) and np.abs(pcm - ref).max() <= 2e-2 + 2.0 / 32767, rid
