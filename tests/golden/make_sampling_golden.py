"""Generate tests/golden/sampling_golden.npz by running the REFERENCE sample().

Run in the build container (needs the reference importable):
    PYTHONPATH=/root/reference/pkg/src python tests/golden/make_sampling_golden.py
Each case: fp32 logits (vocab 64, the reference default, profiles.py:97, or a
hash row at the Orpheus vocab), SamplingParams, a recent-token window and a
per-case rng stream SeedSequence([run_seed, request_id]) (model_api.py:259);
the expected token is what speechserve.model_api.sample() returns.
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

try:
    from speechserve import model_api
except ImportError:  # pragma: no cover
    sys.path.insert(0, "/root/reference/pkg/src")
    from speechserve import model_api

OUT = Path(__file__).resolve().parent / "sampling_golden.npz"
PARAM_SETS = [
    # (temperature, top_k or 0, top_p, penalty)
    (0.0, 0, 1.0, 1.0),
    (0.0, 0, 1.0, 1.3),
    (1.0, 0, 1.0, 1.0),
    (0.6, 0, 0.8, 1.3),      # orpheus_like (profiles.py:192-194)
    (0.8, 50, 0.95, 1.1),    # cosy_like (profiles.py:175-177)
    (0.7, 0, 0.9, 1.05),     # step_audio_like
    (0.5, 5, 1.0, 1.0),
    (1.3, 1, 1.0, 1.2),
]


def main() -> None:
    rng = np.random.default_rng(20260217)
    V = 64
    rows, prm, wins, wlen, seeds, rids, exp = [], [], [], [], [], [], []
    for case in range(640):
        t, k, p, pen = PARAM_SETS[case % len(PARAM_SETS)]
        kind = case % 5
        if kind == 0:
            x = rng.normal(size=V) * 2.0
        elif kind == 1:
            x = np.round(rng.normal(size=V) * 2.0, 1)          # many ties
        elif kind == 2:
            x = rng.normal(size=V) * 2.0
            x[rng.random(V) < 0.7] = -np.inf                    # masked entries
        elif kind == 3:
            x = model_api.synthetic_logits(model_api.request_seed(case, 3), case, 0, V)
        else:
            x = rng.normal(size=V) * 0.3
        x = x.astype(np.float32)
        wl = int(rng.integers(0, 65))
        w = rng.choice(np.argsort(-x)[:12], size=wl) if wl else np.zeros(0, np.int64)
        run_seed, rid = int(rng.integers(0, 2**32)), case
        params = model_api.SamplingParams(temperature=t, top_k=(k or None), top_p=p, repetition_penalty=pen)
        win = model_api._RingWindow(64, V)
        for tok in w:
            win.append(int(tok))
        state = model_api.SamplingState(
            seed=0,
            rng=np.random.Generator(np.random.PCG64(np.random.SeedSequence([run_seed, rid]))),
            windows=[win],
        )
        tok = model_api.sample(x.astype(np.float64), params, state)
        rows.append(x)
        prm.append([t, k, p, pen])
        pad = np.zeros(64, np.int64)
        pad[:wl] = w
        wins.append(pad)
        wlen.append(wl)
        seeds.append(run_seed)
        rids.append(rid)
        exp.append(tok)
    np.savez_compressed(
        OUT, logits=np.array(rows), params=np.array(prm), windows=np.array(wins), window_len=np.array(wlen),
        run_seed=np.array(seeds, np.uint64), request_id=np.array(rids), expected=np.array(exp),
    )
    print(OUT, len(exp))


if __name__ == "__main__":
    main()
