"""K4 streaming detokenizer (causal SNAC-style, cached left context) vs the CPU oracle."""

import numpy as np
import pytest

from oracle.snac import SnacOracle
from oracle.workload import request_seed
from paper_2602_00269_b200._ref import profiles
from paper_2602_00269_b200.device import Sampling

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def snac(tiny_cfg):
    return SnacOracle(tiny_cfg, 1234)


def _profile():
    p = profiles.builtin_profile("orpheus_like")
    return p


def _generate(dev, slot, P, T):
    dev.forward(np.array([[slot, p, -1, 0] for p in range(P - 1)], np.int32), sample=False)
    for s in range(T):
        dev.forward(np.array([[slot, P - 1 + s, -1, 1]], np.int32))
    return dev.read_tokens(slot, P, T)


def _windows(T, rid=0):
    prof = _profile()
    out, emitted = [], 0
    while True:
        w = profiles.chunk_ready(T, emitted, prof, stream_ended=True, request=rid)
        if w is None:
            return out
        out.append(w)
        emitted += 1


def _snr_db(ref, got):
    return 10 * np.log10(np.sum(ref.astype(np.float64) ** 2) / max(np.sum((ref - got).astype(np.float64) ** 2), 1e-30))


@pytest.mark.parametrize("T", [64, 30])
def test_streaming_equals_full_decode(tiny_dev, tiny_cfg, snac, T):
    c = tiny_cfg
    P = 12
    slot = tiny_dev.admit(request_seed(5, T), P, T, Sampling(temperature=0.9, top_p=0.9, repetition_penalty=1.3))
    toks = _generate(tiny_dev, slot, P, T)
    pcm = []
    for w in _windows(T):
        out, _ = tiny_dev.detok(np.array([[slot, w.index, w.start, w.length, w.new_tokens, int(w.final)]], np.int32))
        assert len(out[0]) == (w.new_tokens * c.frame_samples) // c.frame_tokens
        pcm.append(out[0])
    got = np.concatenate(pcm)
    ref = snac.decode_tokens(toks, T)[: len(got)]
    assert np.abs(got - ref).max() <= 2e-2
    assert _snr_db(ref, got) >= 35.0
    tiny_dev.release(slot)


def test_batched_ragged_windows(tiny_dev, tiny_cfg, snac):
    """Mixed first (28-token) and steady (7-token) windows in one detok call."""
    P = 8
    T = 42
    slots = [tiny_dev.admit(request_seed(9, r), P, T, Sampling(temperature=1.0)) for r in range(3)]
    toks = [_generate(tiny_dev, s, P, T) for s in slots]
    wins = _windows(T)
    # request 0 goes one chunk ahead so the batch mixes first and steady windows
    w0 = wins[0]
    out0, _ = tiny_dev.detok(np.array([[slots[0], w0.index, w0.start, w0.length, w0.new_tokens, 0]], np.int32))
    pcm = {0: [out0[0]], 1: [], 2: []}
    idx = {0: 1, 1: 0, 2: 0}
    while any(idx[r] < len(wins) for r in range(3)):
        batch, who = [], []
        for r in range(3):
            if idx[r] < len(wins):
                w = wins[idx[r]]
                batch.append([slots[r], w.index, w.start, w.length, w.new_tokens, int(w.final)])
                who.append(r)
                idx[r] += 1
        outs, _ = tiny_dev.detok(np.array(batch, np.int32))
        for r, o in zip(who, outs):
            pcm[r].append(o)
    for r in range(3):
        got = np.concatenate(pcm[r])
        ref = snac.decode_tokens(toks[r], T)[: len(got)]
        assert np.abs(got - ref).max() <= 2e-2 and _snr_db(ref, got) >= 35.0
        tiny_dev.release(slots[r])


def test_window_rules(tiny_dev):
    from paper_2602_00269_b200._ref import errors

    slot = tiny_dev.admit(request_seed(1, 1), 4, 28, Sampling())
    with pytest.raises(errors.WindowRuleViolation):  # steady window before the first
        tiny_dev.detok(np.array([[slot, 2, 0, 28, 7, 0]], np.int32))
    with pytest.raises(errors.CacheMissing):
        tiny_dev.detok(np.array([[31, 1, 0, 28, 28, 0]], np.int32))
    tiny_dev.release(slot)
