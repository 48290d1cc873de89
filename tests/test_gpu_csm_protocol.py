"""The UNMODIFIED reference SimEngine drives a depth-stage profile through CsmExecutor.

profiles.py:214-231 (depth_like) reshaped to the CSM-style geometry (8 codebooks of
2048 codes, greedy): the engine calls lm_forward -> CsmExecutor.forward
(engine.py:258-273), depth_forward -> depth_logits / depth_latency for codebooks
1..7 (model_api.py:438-458, engine.py:277-292), samples codebook 0 on the host
(engine.py:294-303) and detokenizes windows of all codebooks (engine.py:305-347).
Every code the host sampled must be the code the device decided (no history
mismatch), and the frames equal a direct device pipeline run (csm.CsmFrames) of the
same requests, which tests/test_gpu_csm.py checks against the CPU oracle.
"""

from dataclasses import replace

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("temperature", [0.0, 0.8])
def test_reference_engine_drives_depth_stage(temperature):
    from paper_2602_00269_b200._ref import ref_engine as r_engine
    from paper_2602_00269_b200._ref import model_api, profiles, scheduler, workload
    from oracle.mimi import MimiOracle
    from paper_2602_00269_b200.config import tiny_csm, tiny_mimi
    from paper_2602_00269_b200.csm import CsmFrames
    from paper_2602_00269_b200.device import Sampling
    from paper_2602_00269_b200.executor import CsmExecutor

    bcfg, dcfg = tiny_csm()
    params = model_api.SamplingParams(temperature=temperature, top_p=0.95 if temperature else 1.0,
                                      repetition_penalty=1.0)
    prof = replace(profiles.builtin_profile("depth_like"), codebooks=bcfg.n_codebooks,
                   vocab_size=bcfg.codebook_size, sampling_defaults=params)
    mcfg = tiny_mimi(n_q=bcfg.n_codebooks, max_slots=8, max_frames=64)
    ex = CsmExecutor(prof, bcfg, dcfg, weight_seed=31, mimi_cfg=mcfg)
    assert ex.decided == (temperature > 0)
    seen: dict = {}
    pcm: dict = {}
    orig = ex.detokenize_windows

    def spy(batch, specs, windows, caches):
        for sp, w in zip(specs, windows):
            seen.setdefault(sp.request, {})[sp.start] = np.asarray(w)
        outs, lat = orig(batch, specs, windows, caches)
        for sp, o in zip(specs, outs):
            assert o.pcm.shape == (sp.new_tokens * mcfg.frame_samples,)
            pcm.setdefault(sp.request, []).append(o.pcm)
        return outs, lat

    ex.detokenize_windows = spy
    eng = r_engine.SimEngine(prof, scheduler.PolicyConfig(), r_engine.PipelineMode.ASYNCHRONOUS, seed=5)
    eng.executor = ex
    P, T, R = 12, 14, 3
    arr = [(r, workload.ArrivalSpec(arrival_us=r * 1000, prompt_tokens=P, target_output_tokens=T))
           for r in range(R)]
    tr = eng.run(arr)
    assert len(tr.requests) == R and all(r.tokens_generated == T for r in tr.requests)
    assert ex.frames_run == R * T and ex.mismatches == 0
    host = {}
    for rid, wins in seen.items():
        toks = np.zeros((T, bcfg.n_codebooks), np.int64)
        for start, w in wins.items():
            toks[start:start + len(w)] = w
        host[rid] = toks
    # K7: every request's streamed audio == the Mimi oracle's full decode of its frames
    orc = MimiOracle(mcfg, 31 + 2)
    for rid, toks in host.items():
        got = np.concatenate(pcm[rid])
        ref = orc.decode(toks, exact=True)
        snr = 10 * np.log10((ref ** 2).sum() / ((got - ref) ** 2).sum())
        assert got.shape == ref.shape and np.abs(got - ref).max() < 2e-2 and snr >= 35, (rid, snr)
    if temperature > 0:
        ex.close()
        return
    # the same requests through the device pipeline directly
    pipe = CsmFrames(ex.bb, ex.dp)
    g = Sampling(temperature=0.0, repetition_penalty=1.0)
    streams = [pipe.admit(model_api.request_seed(5, r), P, T + 1, g, g) for r in range(R)]
    pipe.prefill(streams)
    for _ in range(T):
        pipe.step(streams)
    for r, s in enumerate(streams):
        direct = np.stack([pipe.frame(s, P + t) for t in range(T)])
        assert np.array_equal(direct, host[r]), r
        pipe.release(s)
    ex.close()
