"""GPU: disaggregated LM -> detok (reference engine.py:119-123,150-156,
PAPER.md:300).  The LM context decodes; a separate detokenizer context (config.detok_role:
same token layout and SNAC-style decoder weights, placeholder backbone) receives every
window's tokens through vox_copy_tokens and detokenizes on its own streams.  On this
1-GPU box both contexts share device 0 (the copy takes the peer-access kernel path it
also takes between NVLink peers).  Every request's audio == the SNAC oracle of the
tokens the LM context generated."""

from dataclasses import replace

import numpy as np
import pytest

from oracle.snac import SnacOracle
from paper_2602_00269_b200._ref import core, profiles, scheduler, workload

pytestmark = pytest.mark.gpu


def test_disaggregated_engine(tiny_dev, tiny_cfg):
    from paper_2602_00269_b200.config import detok_role
    from paper_2602_00269_b200.device import VoxDevice
    from paper_2602_00269_b200.engine import StreamingEngine

    ddev = VoxDevice(detok_role(tiny_cfg), weight_seed=1234, device=0)
    prof = replace(profiles.builtin_profile("orpheus_like"), vocab_size=156940, max_lm_batch=64, max_detok_batch=64)
    eng = StreamingEngine(tiny_dev, prof, scheduler.PolicyConfig(max_lm_batch=64, max_detok_batch=64), seed=7,
                          keep_pcm=True, detok_dev=ddev)
    spec = workload.WorkloadSpec(rate=40.0, duration_s=0.25, prompt_dist=workload.fixed(16),
                                 output_dist=workload.uniform_int(20, 60), seed=2)
    arr = list(enumerate(workload.build_workload(spec)))
    toks = {}
    orig = tiny_dev.release

    def grab(slot):
        run = next(r for r in eng.live.values() if r.slot == slot)
        toks[run.req.id] = tiny_dev.read_tokens(slot, run.req.prompt_tokens, run.req.target_output_tokens)
        orig(slot)

    tiny_dev.release = grab
    try:
        tr = eng.run(arr)
    finally:
        tiny_dev.release = orig
    rep = core.build_report(tr)
    assert rep.requests_completed == len(arr)
    snac = SnacOracle(tiny_cfg, 1234)
    for rid, a in arr:
        pcm = np.concatenate(eng.pcm[rid])
        assert len(pcm) == sum((c.new_tokens * 2048) // 7 for c in tr.chunks_for(rid))
        ref = snac.decode_tokens(toks[rid], a.target_output_tokens)[: len(pcm)]
        assert np.abs(pcm - ref).max() <= 2e-2, rid
    print(f"disaggregated: {len(arr)} requests, p90 TTFA {rep.ttfa_p90 * 1e3:.1f} ms, viability "
          f"{rep.viability_fraction:.3f}")
    ddev.close()
