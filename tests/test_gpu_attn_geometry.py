"""Paged decode attention at the Orpheus-3B head geometry (24 q : 8 kv heads, hd 128,
GQA group 3) — the shape the bench runs — vs the CPU oracle, teacher-forced.

The tiny config (4:2 heads, hd 64) covers the G=2 / hd=64 instantiation; this
covers G=3 / hd=128 with a batch of rows at different context lengths (ragged
page counts, partial last pages, split-KV at small batch, one CTA-persistent
pass at larger batch)."""

import numpy as np
import pytest

from oracle.llama import LlamaOracle
from oracle.workload import prompt_ids, request_seed
from paper_2602_00269_b200.config import tiny
from paper_2602_00269_b200.device import Sampling, VoxDevice

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def geo():
    cfg = tiny(n_heads=24, n_kv_heads=8, head_dim=128, max_slots=16, max_ctx=512, detok_enabled=False)
    dev = VoxDevice(cfg, weight_seed=99)
    orc = LlamaOracle(cfg, 99)
    yield cfg, dev, orc
    dev.close()


@pytest.mark.parametrize("splits1", [False, True])
@pytest.mark.parametrize("lens", [(37,), (5, 16, 17, 63, 130, 200), tuple(range(20, 330, 31))])
def test_decode_logits_ragged_batch(geo, monkeypatch, lens, splits1):
    # splits1: every GEMM unsplit -> the gate|up GEMM runs the fused SiLU(gate)*up
    # epilogue (the decode path at large batch) instead of partials + silu kernel
    if splits1:
        monkeypatch.setenv("VOX_GEMM_SPLITS_TEST", "1")
    cfg, dev, orc = geo
    slots, prompts = [], []
    for i, P in enumerate(lens):
        seed = request_seed(5 + int(splits1), 100 * len(lens) + i)
        slot = dev.admit(seed, P, 8, Sampling(temperature=0.0))
        prompt = np.array(prompt_ids(seed, P, cfg.text_vocab))
        dev.forward(np.array([[slot, p, -1, 0] for p in range(P - 1)], np.int32), sample=False, sync=True,
                    graph=False)
        orc.forward(("g", i, len(lens), splits1), prompt[:-1], np.arange(P - 1), want_logits=False)
        slots.append(slot)
        prompts.append(prompt)
    rows = np.array([[s, P - 1, -1, 1] for s, P in zip(slots, lens)], np.int32)
    _, lg = dev.forward(rows, sample=False, full_logits=True, sync=True)
    for i, P in enumerate(lens):
        ol, _ = orc.forward(("g", i, len(lens), splits1), prompts[i][-1:], np.array([P - 1]))
        err = np.abs(lg[i] - ol[0]).max()
        assert err < 2e-2 * max(1.0, np.abs(ol[0]).max()), (i, P, err)
    for s in slots:
        dev.release(s)
