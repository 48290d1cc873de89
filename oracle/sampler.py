"""Restatement of the reference sampling path (TEST INFRASTRUCTURE ONLY).

Follows /root/reference/pkg/src/speechserve/model_api.py:
  RingWindow            :124-150 (_RingWindow: capacity, FIFO overwrite, counts>0 mask)
  apply_repetition_penalty :342-352 (x>0 -> x/p else x*p on DISTINCT window ids)
  truncate_and_sample   :311-339 (stable descending argsort, top-k, max-shift
                         softmax, top-p minimal prefix with cum >= p, renorm,
                         rng.random(), searchsorted right)
  sample                :355-381 (NaN/+inf rejection, T=0 -> argmax)
The rng is numpy PCG64 seeded like preprocess() (model_api.py:256-259), so
this restatement reproduces the reference's stochastic draws exactly; tests pin
it against the reference's own sample() (tests/golden/sampling_golden.npz).
"""

from __future__ import annotations

import numpy as np

MASK64 = (1 << 64) - 1


class DegenerateDistribution(Exception):
    pass


class RingWindow:
    def __init__(self, capacity: int, vocab: int):
        self.capacity = capacity
        self.buf: list[int] = []
        self.pos = 0
        self.counts = np.zeros(vocab, dtype=np.int32)

    def append(self, token: int) -> None:
        if self.capacity == 0:
            return
        if len(self.buf) < self.capacity:
            self.buf.append(token)
        else:
            self.counts[self.buf[self.pos]] -= 1
            self.buf[self.pos] = token
            self.pos = (self.pos + 1) % self.capacity
        self.counts[token] += 1

    def __len__(self):
        return len(self.buf)

    def recent(self) -> list[int]:
        """Window contents oldest-first (what the device reads from its token store)."""
        if len(self.buf) < self.capacity:
            return list(self.buf)
        return self.buf[self.pos:] + self.buf[: self.pos]


def request_rng(run_seed: int, request_id: int) -> np.random.Generator:
    return np.random.Generator(np.random.PCG64(np.random.SeedSequence([run_seed & MASK64, request_id])))


def apply_repetition_penalty(logits: np.ndarray, penalty: float, window: RingWindow) -> np.ndarray:
    if penalty == 1.0 or len(window) == 0:
        return logits
    mask = window.counts > 0
    out = logits.copy()
    pos = mask & (out > 0)
    neg = mask & ~(out > 0)
    out[pos] = out[pos] / penalty
    out[neg] = out[neg] * penalty
    return out


def truncate_and_sample(scaled: np.ndarray, top_k, top_p: float, rng) -> int:
    order = np.argsort(-scaled, kind="stable")
    if top_k is not None:
        order = order[:top_k]
    kept = scaled[order]
    fin = np.isfinite(kept)
    if not fin.any():
        raise DegenerateDistribution("all -inf")
    probs = np.exp(kept - kept[fin].max())
    total = probs.sum()
    if total <= 0:
        raise DegenerateDistribution("mass vanished")
    probs = probs / total
    if top_p < 1.0:
        cum = np.cumsum(probs)
        cut = min(int(np.searchsorted(cum, top_p, side="left")) + 1, len(order))
        order = order[:cut]
        probs = probs[:cut]
        probs = probs / probs.sum()
    r = rng.random()
    idx = int(np.searchsorted(np.cumsum(probs), r, side="right"))
    return int(order[min(idx, len(order) - 1)])


def sample(logits: np.ndarray, temperature: float, top_k, top_p: float, penalty: float,
           window: RingWindow, rng) -> int:
    arr = np.asarray(logits, dtype=np.float64)
    if np.isnan(arr).any() or np.isposinf(arr).any():
        raise ValueError("logits must not contain NaN or +inf")
    arr = apply_repetition_penalty(arr, penalty, window)
    if temperature == 0:
        if not np.isfinite(arr).any():
            raise DegenerateDistribution("all -inf")
        tok = int(np.argmax(arr))
    else:
        tok = truncate_and_sample(arr / temperature, top_k, top_p, rng)
    window.append(tok)
    return tok


def kept_set(logits: np.ndarray, temperature: float, top_k, top_p: float, penalty: float,
             window: RingWindow) -> tuple[np.ndarray, np.ndarray]:
    """The candidate ids and renormalised probabilities sample() draws from."""
    arr = apply_repetition_penalty(np.asarray(logits, np.float64), penalty, window) / temperature
    order = np.argsort(-arr, kind="stable")
    if top_k is not None:
        order = order[:top_k]
    kept = arr[order]
    fin = np.isfinite(kept)
    probs = np.exp(kept - kept[fin].max())
    probs = probs / probs.sum()
    if top_p < 1.0:
        cum = np.cumsum(probs)
        cut = min(int(np.searchsorted(cum, top_p, side="left")) + 1, len(order))
        order, probs = order[:cut], probs[:cut]
        probs = probs / probs.sum()
    return order, probs
