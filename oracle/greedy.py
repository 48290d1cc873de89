"""Config-1 greedy token streams on the CPU oracle (TEST INFRASTRUCTURE ONLY).

The decode loop of the reference engine for one request (engine.py:258-303):
the first decode consumes the last prompt token, every later decode the token
sampled one step earlier; each sampling row is masked to the Orpheus frame
slot's codebook range (-inf elsewhere, which sample() treats as masked:
model_api.py:366-367) and decided by greedy sample() with the repetition
penalty over the request's ring window (model_api.py:124-150, 342-381).
`decide(row, window)` is that sample() call -- the reference's own function
when it is importable (tests/golden/make_greedy_golden.py), else the pinned
restatement oracle/sampler.py.
"""

from __future__ import annotations

import numpy as np

from . import sampler as osamp
from .llama import LlamaOracle, audio_range, masked
from .workload import prompt_ids, request_seed


def penalised_margin(row: np.ndarray, lo: int, hi: int, penalty: float, window) -> float:
    """Top-2 gap of the penalised candidates [lo, hi) (what argmax decides on)."""
    pen = osamp.apply_repetition_penalty(row, penalty, window)
    srt = np.sort(pen[lo:hi])[::-1]
    return float(srt[0] - srt[1])


def greedy_streams(cfg, weight_seed: int, run_seed: int, n_req: int, prompt: int, n_tok: int, penalty: float,
                   decide=None, window_factory=None, oracle: LlamaOracle | None = None):
    """Free-running greedy streams: (tokens [R, T], penalised margins [R, T], prompts [R, P])."""
    orc = oracle or LlamaOracle(cfg, weight_seed)
    if decide is None:
        def decide(row, window):
            return osamp.sample(row, 0.0, None, 1.0, penalty, window, None)
    if window_factory is None:
        def window_factory():
            return osamp.RingWindow(64, cfg.vocab)
    toks = np.zeros((n_req, n_tok), np.int64)
    margins = np.zeros((n_req, n_tok), np.float64)
    prompts = np.zeros((n_req, prompt), np.int64)
    for r in range(n_req):
        seed = request_seed(run_seed, r)
        pr = np.array(prompt_ids(seed, prompt, cfg.text_vocab))
        prompts[r] = pr
        rid = ("greedy", r)
        orc.forward(rid, pr[:-1], np.arange(prompt - 1), want_logits=False)
        win = window_factory()
        tok = int(pr[-1])
        for s in range(n_tok):
            lg, _ = orc.forward(rid, np.array([tok]), np.array([prompt - 1 + s]))
            lo, hi = audio_range(cfg, s)
            row = masked(lg[0], lo, hi)
            margins[r, s] = penalised_margin(row, lo, hi, penalty, win)
            tok = decide(row, win)
            toks[r, s] = tok
        orc.release(rid)
    return toks, margins, prompts
