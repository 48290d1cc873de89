"""CPU: the sampling restatement is pinned to the reference (golden vectors + SPEC examples)."""

from pathlib import Path

import numpy as np
import pytest
from scipy import stats

from oracle import sampler as osamp

GOLDEN = Path(__file__).resolve().parent / "golden" / "sampling_golden.npz"


def _run_case(g, i):
    x = g["logits"][i]
    t, k, p, pen = g["params"][i]
    win = osamp.RingWindow(64, len(x))
    for tok in g["windows"][i][: g["window_len"][i]]:
        win.append(int(tok))
    rng = osamp.request_rng(int(g["run_seed"][i]), int(g["request_id"][i]))
    return osamp.sample(x, float(t), int(k) or None, float(p), float(pen), win, rng)


def test_golden_vectors_reproduced():
    g = np.load(GOLDEN)
    n = len(g["expected"])
    assert n >= 600
    got = [_run_case(g, i) for i in range(n)]
    assert got == g["expected"].tolist()


def test_spec_known_answers():
    V = 3
    w = osamp.RingWindow(64, V)
    assert osamp.sample(np.array([2.0, 1.0, 0.0]), 0.0, None, 1.0, 1.0, w, None) == 0
    w = osamp.RingWindow(64, 2)
    w.append(0)
    assert osamp.sample(np.array([1.0, 0.95]), 0.0, None, 1.0, 1.3, w, None) == 1
    rng = np.random.default_rng(0)
    for _ in range(2000):
        w = osamp.RingWindow(64, 3)
        assert osamp.sample(np.log([0.5, 0.3, 0.2]), 1.0, None, 0.7, 1.0, w, rng) != 2
    x = np.random.default_rng(1).normal(size=17)
    for _ in range(50):
        w = osamp.RingWindow(64, 17)
        assert osamp.sample(x, 0.7, 1, 1.0, 1.0, w, rng) == int(np.argmax(x))


def test_ring_window_and_penalty_semantics():
    # capacity 2 after 0,1,2 -> buf [2,1], pos 1, counts [0,1,1,0]
    w = osamp.RingWindow(2, 4)
    for t in (0, 1, 2):
        w.append(t)
    assert w.buf == [2, 1] and w.pos == 1 and w.counts.tolist() == [0, 1, 1, 0]
    assert w.recent() == [1, 2]
    # penalty on [2,0,-1,5] with window {0,1,2}, p=2 -> [1,0,-2,5]
    w = osamp.RingWindow(8, 4)
    for t in (0, 1, 2, 2):
        w.append(t)
    out = osamp.apply_repetition_penalty(np.array([2.0, 0.0, -1.0, 5.0]), 2.0, w)
    assert out.tolist() == [1.0, 0.0, -2.0, 5.0]
    # greedy ties -> lowest id
    assert osamp.sample(np.array([1.0, 3.0, 3.0]), 0.0, None, 1.0, 1.0, osamp.RingWindow(4, 3), None) == 1


def test_errors():
    with pytest.raises(ValueError):
        osamp.sample(np.array([np.nan, 1.0]), 0.0, None, 1.0, 1.0, osamp.RingWindow(4, 2), None)
    with pytest.raises(osamp.DegenerateDistribution):
        osamp.sample(np.array([-np.inf, -np.inf]), 0.0, None, 1.0, 1.0, osamp.RingWindow(4, 2), None)


def test_softmax_fidelity_chi_square():
    lg = np.array([0.3, -1.0, 1.2, 0.0])
    rng = np.random.default_rng(5)
    n = 20000
    toks = [osamp.sample(lg, 1.0, None, 1.0, 1.0, osamp.RingWindow(0, 4), rng) for _ in range(n)]
    p = np.exp(lg) / np.exp(lg).sum()
    assert stats.chisquare(np.bincount(toks, minlength=4), p * n).pvalue > 0.01


def test_against_live_reference_when_importable():
    model_api = pytest.importorskip("speechserve.model_api")
    rng = np.random.default_rng(11)
    for case in range(100):
        x = rng.normal(size=64).astype(np.float32) * 2
        w_ref = model_api._RingWindow(64, 64)
        w_orc = osamp.RingWindow(64, 64)
        for t in rng.integers(0, 64, size=int(rng.integers(0, 70))):
            w_ref.append(int(t))
            w_orc.append(int(t))
        params = model_api.SamplingParams(temperature=0.6, top_p=0.8, repetition_penalty=1.3)
        st = model_api.SamplingState(seed=0, rng=osamp.request_rng(9, case), windows=[w_ref])
        a = model_api.sample(x.astype(np.float64), params, st)
        b = osamp.sample(x, 0.6, None, 0.8, 1.3, w_orc, osamp.request_rng(9, case))
        assert a == b
