"""Split-KV decode attention (K2 + combine) at the hd-64 / GQA 14:2 geometry of the
CosyVoice2-style LM: at small batch and long context the default policy splits each
(row, kv head) over up to 8 CTAs (attn_pick_splits); the merged result must match the
unsplit kernel to bf16 rounding of the attention output, for every split count."""

import numpy as np
import pytest

from paper_2602_00269_b200.config import cosyvoice2
from paper_2602_00269_b200.device import Sampling, VoxDevice

pytestmark = pytest.mark.gpu

B, CTX = 16, 700


def _logits(monkeypatch, splits):
    if splits is None:
        monkeypatch.delenv("VOX_ATTN_SPLITS_TEST", raising=False)
    else:
        monkeypatch.setenv("VOX_ATTN_SPLITS_TEST", str(splits))
    dev = VoxDevice(cosyvoice2(n_layers=2, max_slots=B, max_rows=1024), weight_seed=11)
    try:
        g = Sampling(temperature=0.0, repetition_penalty=1.0)
        slots = [dev.admit(500 + i, 50, 688, g) for i in range(B)]
        for i in range(B):  # prefill contexts of CTX - 1 - i tokens (ragged page tails)
            n = CTX - 1 - 7 * i
            dev.forward(np.array([[slots[i], p, -1, 0] for p in range(n)], np.int32), sample=False)
        rows = np.array([[slots[i], CTX - 1 - 7 * i, -1, 1] for i in range(B)], np.int32)
        dev.forward(rows, graph=False)
        lg, _ = dev.read_logits()
        return lg.astype(np.float64)
    finally:
        dev.close()


@pytest.mark.parametrize("splits", [None, 2, 3, 5, 8])
def test_split_kv_matches_unsplit(monkeypatch, splits):
    ref = _logits(monkeypatch, 1)
    got = _logits(monkeypatch, splits)
    assert np.isfinite(got).all()
    err = np.abs(got - ref).max() / np.abs(ref).max()
    assert err < 1e-2, err
    assert (got.argmax(axis=1) == ref.argmax(axis=1)).mean() > 0.9
