"""Generate tests/golden/greedy_config1.npz: config 1's greedy token streams.

Config 1 (BASELINE.json configs[0]): tiny Orpheus-style backbone (planted-margin
init, paper_2602_00269_b200/config.py:tiny_planted, weight seed 2024), 4
concurrent greedy requests (run seed 0, request ids 0..3), prompt 50, 64 audio
tokens each, repetition penalty 1.3 over a 64-token window.

Every decision is taken by the REFERENCE's own sample() (model_api.py:355-381)
on the CPU oracle's logits with the Orpheus frame-slot range mask applied as
-inf (sample treats -inf as masked: model_api.py:366-367), and the reference's
_RingWindow carries the penalty window (model_api.py:124-150).  The stored
margins are the penalised top-2 gaps the GPU parity test relies on.

Run in the build container (reference importable):
    python tests/golden/make_greedy_golden.py
"""

from __future__ import annotations

import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[2]
sys.path.insert(0, str(ROOT))
try:
    from speechserve import model_api
except ImportError:  # pragma: no cover
    sys.path.insert(0, "/root/reference/pkg/src")
    from speechserve import model_api

from oracle.greedy import greedy_streams  # noqa: E402
from paper_2602_00269_b200.config import PLANTED_WEIGHT_SEED, tiny_planted  # noqa: E402

OUT = Path(__file__).resolve().parent / "greedy_config1.npz"
WEIGHT_SEED, RUN_SEED, R, P, T, PENALTY = PLANTED_WEIGHT_SEED, 0, 4, 50, 64, 1.3


def reference_decide(row: np.ndarray, window) -> int:
    params = model_api.SamplingParams(temperature=0.0, repetition_penalty=PENALTY, penalty_window=64)
    state = model_api.SamplingState(seed=0, rng=np.random.default_rng(0), windows=[window])
    return int(model_api.sample(row, params, state))


def main() -> None:
    cfg = tiny_planted()
    toks, margins, prompts = greedy_streams(cfg, WEIGHT_SEED, RUN_SEED, R, P, T, PENALTY, decide=reference_decide,
                                            window_factory=lambda: model_api._RingWindow(64, cfg.vocab))
    np.savez_compressed(OUT, tokens=toks, margins=margins, prompts=prompts,
                        meta=np.array([WEIGHT_SEED, RUN_SEED, R, P, T], np.int64),
                        penalty=np.float64(PENALTY), embed_scale=np.float64(cfg.embed_half_width))
    print(OUT, "min margin", margins.min())


if __name__ == "__main__":
    main()
