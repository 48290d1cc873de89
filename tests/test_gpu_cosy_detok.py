"""K8 CosyVoice2-style detokenizer (csrc/cosy_detok.cu) vs oracle/cosy_detok.py.

Each call = flow matching over [reference tokens | chunk tokens] (the same function of
the call's inputs on device and oracle), then the stateful causal vocoder: a request's
chunks must concatenate to the oracle's whole-sequence vocoder output of its new mel.
Bar: max-abs 2e-2 and SNR >= 35 dB (BASELINE north_star audio tolerance).
"""

import numpy as np
import pytest

from oracle.cosy_detok import CosyDetokOracle
from paper_2602_00269_b200.config import tiny_cosy_detok

pytestmark = pytest.mark.gpu


def _snr(ref, got):
    return 10 * np.log10((ref.astype(np.float64) ** 2).sum() / max(((got - ref).astype(np.float64) ** 2).sum(), 1e-30))


def test_chunks_vs_oracle():
    from paper_2602_00269_b200.cosy_detok import CosyDetokenizer

    cfg = tiny_cosy_detok()
    dec = CosyDetokenizer(cfg, weight_seed=7)
    orc = CosyDetokOracle(cfg, 7)
    rng = np.random.default_rng(0)
    seeds = [1001, 2002, 3003]
    plans = [[15, 15, 9], [5, 15, 15], [15, 1, 20]]
    toks = [[rng.integers(0, cfg.vocab, c) for c in p] for p in plans]
    slots = [dec.open(s) for s in seeds]
    out = [[] for _ in seeds]
    for call in range(3):
        pcms = dec.decode(slots, [toks[i][call] for i in range(3)])
        for i, p in enumerate(pcms):
            assert p.shape == (len(toks[i][call]) * cfg.samples_per_token,)
            out[i].append(p)
    for i, s in enumerate(seeds):
        got = np.concatenate(out[i])
        ref = orc.decode(s, toks[i], exact=True)
        snr = _snr(ref, got)
        print(f"cosy detok request {i}: max-abs {np.abs(got - ref).max():.2e}, SNR {snr:.1f} dB, "
              f"rms {np.sqrt((ref ** 2).mean()):.3f}")
        assert got.shape == ref.shape
        assert np.abs(got - ref).max() < 2e-2 and snr >= 35
    assert dec.launch_count() > 0
    for s in slots:
        dec.release(s)
    dec.close()


def test_flow_is_per_call_and_vocoder_is_stateful():
    """The same tokens decoded by a fresh stream and by a stream with history give the
    same flow but different vocoder left context: the first samples differ, the
    request's whole-stream output equals the oracle's."""
    from paper_2602_00269_b200.cosy_detok import CosyDetokenizer

    cfg = tiny_cosy_detok()
    dec = CosyDetokenizer(cfg, weight_seed=3)
    t = np.arange(15) * 37 % cfg.vocab
    a = dec.open(55)
    b = dec.open(55)
    first = dec.decode([a], [t])[0]
    dec.decode([b], [t])
    second = dec.decode([b], [t])[0]  # call index 1: new noise, history present
    assert not np.allclose(first, second)
    dec.close()


def test_errors():
    from paper_2602_00269_b200._ref import errors
    from paper_2602_00269_b200.cosy_detok import CosyDetokenizer

    cfg = tiny_cosy_detok(max_slots=2, max_tokens=32, max_chunk=20)
    dec = CosyDetokenizer(cfg, weight_seed=1)
    with pytest.raises(errors.CacheMissing):
        dec.decode([0], [np.zeros(3, np.int32)])
    s = dec.open(1)
    with pytest.raises(ValueError):
        dec.decode([s], [np.array([cfg.vocab])])
    with pytest.raises(errors.BatchTooLarge):
        dec.decode([s], [np.zeros(21, np.int32)])
    dec.open(2)
    with pytest.raises(MemoryError):
        dec.open(3)
    dec.close()


def test_reference_simengine_drives_cosy_lm_and_detok():
    """The UNMODIFIED reference SimEngine on a cosy_like profile (profiles.py:163-179, chunk
    15, greedy here) drives B200Executor: the CosyVoice2-style LM (config 4 geometry, tiny)
    decodes on the device, the host samples with the reference sample(), and
    detokenize_windows runs K8 per chunk; every request's streamed PCM equals the
    oracle's flow + vocoder over the tokens the engine sampled."""
    from dataclasses import replace

    from paper_2602_00269_b200._ref import profiles, ref_engine, scheduler, workload
    from paper_2602_00269_b200.config import tiny_cosy
    from paper_2602_00269_b200.cosy_detok import CosyDetokenizer
    from paper_2602_00269_b200.executor import B200Executor

    lm = tiny_cosy(max_slots=8)
    dcfg = tiny_cosy_detok()
    base = profiles.builtin_profile("cosy_like")
    prof = replace(base, vocab_size=lm.vocab, sampling_defaults=replace(base.sampling_defaults, temperature=0.0))
    ex = B200Executor(prof, lm, weight_seed=9, detokenizer=CosyDetokenizer(dcfg, weight_seed=10))
    seen: dict = {}
    orig = ex.detokenize_windows

    def spy(batch, specs, windows, caches):
        outs, lat = orig(batch, specs, windows, caches)
        for sp, w, o in zip(specs, windows, outs):
            ids = np.asarray(w)[:, 0]
            seen.setdefault(sp.request, []).append((ids[len(ids) - sp.new_tokens:] - lm.audio_base, o.pcm))
        return outs, lat

    ex.detokenize_windows = spy
    eng = ref_engine.SimEngine(prof, scheduler.PolicyConfig(max_lm_batch=16, max_detok_batch=16),
                               ref_engine.PipelineMode.ASYNCHRONOUS, seed=4)
    eng.executor = ex
    arr = [(i, workload.ArrivalSpec(arrival_us=i * 500, prompt_tokens=12, target_output_tokens=40)) for i in range(3)]
    tr = eng.run(arr)
    assert len(tr.requests) == 3 and all(r.tokens_generated == 40 for r in tr.requests)
    from paper_2602_00269_b200._ref import model_api

    orc = CosyDetokOracle(dcfg, 10)
    for rid, chunks in seen.items():
        toks = [np.clip(t, 0, dcfg.vocab - 1) for t, _ in chunks]
        got = np.concatenate([p for _, p in chunks])
        ref = orc.decode(model_api.request_seed(4, rid), toks, exact=True)
        assert got.shape == ref.shape and np.abs(got - ref).max() < 2e-2 and _snr(ref, got) >= 35, rid
    assert not ex._dslot
    ex.detokenizer.close()
