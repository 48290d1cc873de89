"""CPU: the oracle's config-1 greedy streams are pinned to the golden fixture.

tests/golden/greedy_config1.npz was produced by tests/golden/make_greedy_golden.py,
which took every decision with the REFERENCE's own sample() and _RingWindow
(model_api.py:124-150, 342-381).  Here the restated sampler (oracle/sampler.py)
must reproduce those 4 x 64 token streams exactly, and the planted-margin init
must keep every penalised top-2 margin far from a tie.
"""

from pathlib import Path

import numpy as np

from oracle.greedy import greedy_streams
from paper_2602_00269_b200.config import tiny_planted

GOLD = Path(__file__).resolve().parent / "golden" / "greedy_config1.npz"


def test_oracle_greedy_streams_match_reference_golden():
    g = np.load(GOLD)
    ws, run_seed, R, P, T = (int(x) for x in g["meta"])
    cfg = tiny_planted()
    assert float(g["embed_scale"]) == cfg.embed_half_width
    toks, margins, prompts = greedy_streams(cfg, ws, run_seed, R, P, T, float(g["penalty"]))
    assert np.array_equal(prompts, g["prompts"])
    assert np.array_equal(toks, g["tokens"])
    np.testing.assert_allclose(margins, g["margins"], rtol=0, atol=1e-9)
    # every step's token is in its frame slot's codebook range (Orpheus layout)
    for s in range(T):
        lo = cfg.audio_base + (s % cfg.frame_tokens) * cfg.codebook_size
        assert ((toks[:, s] >= lo) & (toks[:, s] < lo + cfg.codebook_size)).all()
    # the planted init keeps decisions away from ties (logit std ~1000)
    assert margins.min() > 1.0, margins.min()


def test_planted_streams_depend_on_the_layers():
    """The planted init must not make the streams trivial: zeroing the attention
    output projections (and the MLP down projections) changes many tokens."""
    from oracle.llama import LlamaOracle

    g = np.load(GOLD)
    ws, run_seed, R, P, T = (int(x) for x in g["meta"])
    cfg = tiny_planted()
    o = LlamaOracle(cfg, ws)
    for L in o.w.layers:
        L["o"] = np.zeros_like(L["o"])
    no_attn, _, _ = greedy_streams(cfg, ws, run_seed, R, P, T, float(g["penalty"]), oracle=o)
    assert (no_attn != g["tokens"]).sum() >= 0.2 * R * T
