"""GPU: the opt-in spatial LM / detok split (VOX_DETOK_SMS, green contexts in
vox_create): the detok stream runs on its own SM partition, the LM stream on the
rest, grids and split-K plans follow the LM partition -- and a served workload's
PCM still matches the oracle decode of the generated ids."""

from dataclasses import replace

import numpy as np
import pytest

from oracle.snac import SnacOracle
from paper_2602_00269_b200._ref import core, profiles, scheduler, workload
from paper_2602_00269_b200.engine import StreamingEngine

pytestmark = pytest.mark.gpu


def test_partitioned_streams_serve_and_match_oracle(tiny_cfg, monkeypatch):
    from paper_2602_00269_b200.device import VoxDevice

    monkeypatch.setenv("VOX_DETOK_SMS", "16")
    dev = VoxDevice(tiny_cfg, weight_seed=1234)
    try:
        prof = replace(profiles.builtin_profile("orpheus_like"), vocab_size=156940, max_lm_batch=64,
                       max_detok_batch=64)
        policy = scheduler.PolicyConfig(max_lm_batch=64, max_detok_batch=64)
        spec = workload.WorkloadSpec(rate=40.0, duration_s=0.3, prompt_dist=workload.fixed(16),
                                     output_dist=workload.uniform_int(20, 60), seed=3)
        arr = list(enumerate(workload.build_workload(spec)))
        eng = StreamingEngine(dev, prof, policy, seed=3, keep_pcm=True)
        released = {}
        orig_release = dev.release

        def grab(slot):
            run = next(r for r in eng.live.values() if r.slot == slot)
            released[run.req.id] = dev.read_tokens(slot, run.req.prompt_tokens, run.req.target_output_tokens)
            orig_release(slot)

        dev.release = grab
        try:
            tr = eng.run(arr)
        finally:
            dev.release = orig_release
        assert core.build_report(tr).requests_completed == len(arr)
        snac = SnacOracle(tiny_cfg, 1234)
        for rid, a in arr[:3]:
            pcm = np.concatenate(eng.pcm[rid])
            ref = snac.decode_tokens(released[rid], a.target_output_tokens)[: len(pcm)]
            assert np.abs(pcm - ref).max() <= 2e-2
    finally:
        dev.close()
