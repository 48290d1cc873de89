"""K1 fused sampler vs the reference sample() (model_api.py:311-381) on the GPU."""

import numpy as np
import pytest
from scipy import stats

from oracle import sampler as osamp
from paper_2602_00269_b200._ref import errors, model_api
from paper_2602_00269_b200.device import Sampling

pytestmark = pytest.mark.gpu

V = 156940


def _hash_logits(n, seed=7):
    seeds = [model_api.request_seed(seed, i) for i in range(n)]
    return model_api.synthetic_logits_batch(seeds, list(range(n)), 0, V).astype(np.float32), seeds


def _ref_greedy(row32, window, penalty, lo=None, hi=None):
    arr = row32.astype(np.float64)
    if lo is not None:
        m = np.full_like(arr, -np.inf)
        m[lo:hi] = arr[lo:hi]
        arr = m
    w = model_api._RingWindow(64, V)
    for t in window:
        w.append(int(t))
    # the reference itself, on identical fp32-valued logits
    state = model_api.SamplingState(seed=0, rng=np.random.default_rng(0), windows=[w])
    p = model_api.SamplingParams(temperature=0.0, repetition_penalty=penalty)
    return model_api.sample(arr, p, state)


@pytest.mark.parametrize("masked", [False, True])
def test_greedy_bit_exact_full_vocab(tiny_dev, masked):
    n = 48
    logits, seeds = _hash_logits(n)
    rng = np.random.default_rng(0)
    windows, lo, hi = [], [], []
    for i in range(n):
        k = i % 7
        l0, h0 = (128266 + k * 4096, 128266 + (k + 1) * 4096) if masked else (0, V)
        lo.append(l0)
        hi.append(h0)
        top = np.argsort(-logits[i, l0:h0], kind="stable")[:40] + l0  # penalise likely winners
        windows.append(list(rng.choice(top, size=int(rng.integers(0, 64)), replace=True)))
    params = [Sampling(temperature=0.0, repetition_penalty=1.3)] * n
    got = tiny_dev.sample_logits(logits, params, windows, seeds, list(range(n)), lo, hi)
    for i in range(n):
        exp = _ref_greedy(logits[i], windows[i], 1.3, lo[i] if masked else None, hi[i] if masked else None)
        assert got[i] == exp, (i, got[i], exp)


def test_spec_examples(tiny_dev):
    # SPEC.md:231-235
    g = Sampling(temperature=0.0)
    assert tiny_dev.sample_logits(np.array([[2.0, 1.0, 0.0]], np.float32), [g], [[]], [1], [0])[0] == 0
    pen = Sampling(temperature=0.0, repetition_penalty=1.3)
    assert tiny_dev.sample_logits(np.array([[1.0, 0.95]], np.float32), [pen], [[0]], [1], [0])[0] == 1
    # top_p 0.7 over probs [.5,.3,.2] never yields token 2
    lg = np.log(np.array([0.5, 0.3, 0.2], np.float32))
    n = 4000
    tp = tiny_dev.sample_logits(np.tile(lg, (n, 1)), [Sampling(temperature=1.0, top_p=0.7)] * n,
                                [[]] * n, [5] * n, list(range(n)))
    assert set(np.unique(tp)) <= {0, 1}
    # top_k 1 == greedy for any T > 0
    x = np.random.default_rng(3).normal(size=(64, 33)).astype(np.float32)
    a = tiny_dev.sample_logits(x, [Sampling(temperature=0.7, top_k=1)] * 64, [[]] * 64, [9] * 64, list(range(64)))
    assert np.array_equal(a, np.argmax(x, axis=1))


def test_ties_lowest_id(tiny_dev):
    x = np.array([[1.0, 3.0, 3.0], [0.0, 0.0, 0.0]], np.float32)
    out = tiny_dev.sample_logits(x, [Sampling(temperature=0.0)] * 2, [[], []], [0, 0], [0, 1])
    assert list(out) == [1, 0]


def test_softmax_chi_square(tiny_dev):
    # SPEC.md:268 / AC8: 1e5 draws on a 4-token vocab at alpha = 0.01
    lg = np.array([0.3, -1.0, 1.2, 0.0], np.float32)
    n = 100_000
    toks = tiny_dev.sample_logits(np.tile(lg, (n, 1)), [Sampling(temperature=1.0)] * n, [[]] * n,
                                  [11] * n, list(range(n)))
    p = np.exp(lg.astype(np.float64))
    p /= p.sum()
    obs = np.bincount(toks, minlength=4)
    assert stats.chisquare(obs, p * n).pvalue > 0.01


def test_topk_topp_kept_set_and_frequencies(tiny_dev):
    # full-vocab hash logits, cosy-like params: every draw must lie in the
    # reference's kept set, and the within-set distribution must match.
    logits, seeds = _hash_logits(1)
    row = logits[0]
    prm = Sampling(temperature=0.8, top_k=50, top_p=0.95, repetition_penalty=1.1)
    win = osamp.RingWindow(64, V)
    order, probs = osamp.kept_set(row, 0.8, 50, 0.95, 1.1, win)
    n = 20_000
    toks = tiny_dev.sample_logits(np.tile(row, (n, 1)), [prm] * n, [[]] * n, [seeds[0]] * n, list(range(n)))
    assert set(np.unique(toks)) <= set(order.tolist())
    cnt = np.array([np.sum(toks == t) for t in order])
    assert stats.chisquare(cnt, probs * n).pvalue > 0.001


def test_orpheus_params_top_p_only(tiny_dev):
    logits, seeds = _hash_logits(1, seed=3)
    row = logits[0]
    win = osamp.RingWindow(64, V)
    for t in np.argsort(-row)[:20]:
        win.append(int(t))
    order, probs = osamp.kept_set(row, 0.6, None, 0.8, 1.3, win)
    n = 4000
    toks = tiny_dev.sample_logits(np.tile(row, (n, 1)), [Sampling(0.6, None, 0.8, 1.3)] * n,
                                  [win.recent()] * n, [seeds[0]] * n, list(range(n)))
    assert set(np.unique(toks)) <= set(order.tolist())


def test_errors(tiny_dev):
    with pytest.raises(ValueError):
        tiny_dev.sample_logits(np.array([[np.nan, 1.0]], np.float32), [Sampling(0.0)], [[]], [0], [0])
    with pytest.raises(ValueError):
        tiny_dev.sample_logits(np.array([[np.inf, 1.0]], np.float32), [Sampling(1.0)], [[]], [0], [0])
    with pytest.raises(errors.DegenerateDistribution):
        tiny_dev.sample_logits(np.array([[-np.inf, -np.inf]], np.float32), [Sampling(0.0)], [[]], [0], [0])
