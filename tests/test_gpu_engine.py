"""GPU: the drop-in executor under the UNMODIFIED reference SimEngine, and the
fused StreamingEngine, on the tiny config."""

from dataclasses import replace

import numpy as np
import pytest

from oracle.snac import SnacOracle
from paper_2602_00269_b200._ref import core, profiles, ref_engine, scheduler, workload
from paper_2602_00269_b200.engine import StreamingEngine

pytestmark = pytest.mark.gpu


def _prof(max_batch=64):
    return replace(profiles.builtin_profile("orpheus_like"), vocab_size=156940, max_lm_batch=max_batch,
                   max_detok_batch=max_batch,
                   sampling_defaults=profiles.builtin_profile("orpheus_like").sampling_defaults)


def test_reference_simengine_with_b200_executor(tiny_dev, tiny_cfg):
    """engine.executor = B200Executor(...) is the whole integration (engine.py:146)."""
    from paper_2602_00269_b200.executor import B200Executor, PcmChunkOut

    prof = replace(_prof(), sampling_defaults=replace(_prof().sampling_defaults, temperature=0.0))
    eng = ref_engine.SimEngine(prof, scheduler.PolicyConfig(max_lm_batch=64, max_detok_batch=64),
                               ref_engine.PipelineMode.ASYNCHRONOUS, seed=0)
    ex = B200Executor(prof, tiny_cfg, dev=tiny_dev)
    eng.executor = ex
    seen = []
    orig = ex.detokenize_windows

    def spy(batch, specs, windows, caches):
        outs, lat = orig(batch, specs, windows, caches)
        seen.extend(outs)
        return outs, lat

    ex.detokenize_windows = spy
    arr = [(i, workload.ArrivalSpec(arrival_us=0, prompt_tokens=20, target_output_tokens=35)) for i in range(3)]
    tr = eng.run(arr)
    rep = core.build_report(tr)
    assert rep.requests_completed == 3
    assert all(isinstance(o, PcmChunkOut) and o.pcm is not None and np.isfinite(o.pcm).all() for o in seen)
    # the host-sampled ids (reference sample()) are in the masked Orpheus ranges
    assert not ex._slot  # every slot released on its final window


def test_streaming_engine_serves_and_pcm_matches_oracle(tiny_dev, tiny_cfg):
    prof = _prof()
    policy = scheduler.PolicyConfig(max_lm_batch=64, max_detok_batch=64)
    spec = workload.WorkloadSpec(rate=40.0, duration_s=0.3, prompt_dist=workload.fixed(16),
                                 output_dist=workload.uniform_int(20, 60), seed=1)
    arr = list(enumerate(workload.build_workload(spec)))
    eng = StreamingEngine(tiny_dev, prof, policy, seed=1, keep_pcm=True)
    # keep the generated ids for the oracle check: read them before release
    released = {}
    orig_release = tiny_dev.release

    def grab(slot):
        run = next(r for r in eng.live.values() if r.slot == slot)
        n = run.req.target_output_tokens
        released[run.req.id] = tiny_dev.read_tokens(slot, run.req.prompt_tokens, n)
        orig_release(slot)

    tiny_dev.release = grab
    try:
        tr = eng.run(arr)
    finally:
        tiny_dev.release = orig_release
    rep = core.build_report(tr)
    assert rep.requests_completed == len(arr)
    snac = SnacOracle(tiny_cfg, 1234)
    for rid, a in arr[:3]:
        pcm = np.concatenate(eng.pcm[rid])
        assert len(pcm) == sum((c.new_tokens * 2048) // 7 for c in tr.chunks_for(rid))
        ref = snac.decode_tokens(released[rid], a.target_output_tokens)[: len(pcm)]
        assert np.abs(pcm - ref).max() <= 2e-2
