"""K6 layer chain (csrc/layer_chain.cu) == the per-kernel decode path, bit for bit.

The chain runs each decoder layer's O / gate|up / down / next-layer q|k|v
projections, both residual+RMSNorms and the q|k|v RoPE + KV append as one
persistent launch.  It keeps the per-kernel path's split-K factors, k-block
rotation and reduction orders, so the logits K1 consumes, the sampled tokens
and the appended K/V must be IDENTICAL to VOX_CHAIN=0 on the same weights and
rows.  Together with the per-kernel path's oracle parity
(test_gpu_config2_parity.py, test_gpu_lm.py) this carries parity to the chain.
Covered: the bench geometry (d 3072, 24:8 x 128, FFN 8192, 3 layers) at the
224- and 256-row buckets and small buckets, the Qwen2-style q|k|v bias (cosy
geometry), prefill rows of one slot at many positions, and padding rows.
"""

import os

import numpy as np
import pytest

from oracle.workload import request_seed
from paper_2602_00269_b200.config import cosyvoice2, orpheus3b
from paper_2602_00269_b200.device import Sampling, VoxDevice

pytestmark = pytest.mark.gpu


def _dev(cfg, ws, chain):
    old = os.environ.get("VOX_CHAIN")
    os.environ["VOX_CHAIN"] = "1" if chain else "0"  # the chain is opt-in
    try:
        return VoxDevice(cfg, weight_seed=ws)
    finally:
        if old is None:
            del os.environ["VOX_CHAIN"]
        else:
            os.environ["VOX_CHAIN"] = old


@pytest.fixture(scope="module", params=["orpheus", "cosy"])
def pair(request):
    if request.param == "orpheus":
        cfg = orpheus3b(n_layers=3, max_slots=264, max_ctx=96, max_rows=1024, detok_enabled=False)
    else:
        cfg = cosyvoice2(n_layers=3, max_slots=264, max_ctx=96, max_rows=1024)
    a = _dev(cfg, 99, chain=False)
    b = _dev(cfg, 99, chain=True)
    yield cfg, a, b
    a.close()
    b.close()


def _run(dev, cfg, n, P, steps, graph):
    sp = Sampling(temperature=0.0, repetition_penalty=1.3)
    slots = [dev.admit(request_seed(5, 100 * n + i), P, 64, sp) for i in range(n)]
    out_tok, out_lg = [], []
    try:
        # prefill: up to 200 rows per forward (many positions of a few slots)
        pre = np.array([[s, p, -1, 0] for s in slots for p in range(P - 1)], np.int32)
        for i in range(0, len(pre), 200):
            dev.forward(pre[i:i + 200], sample=False, graph=graph)
        for t in range(steps):
            rows = np.array([[s, P - 1 + t, -1, 1] for s in slots], np.int32)
            tok, _ = dev.forward(rows, want_tokens=True, graph=graph)
            lg, base = dev.read_logits()
            out_tok.append(tok.copy())
            out_lg.append(lg.copy())
        kv = [dev.read_kv(layer, slots[-1], P - 1 + steps - 1) for layer in range(cfg.n_layers)]
    finally:
        for s in slots:
            dev.release(s)
    return out_tok, out_lg, kv


@pytest.mark.parametrize("n,graph", [(1, True), (7, False), (50, True), (200, True), (224, True), (256, True)])
def test_chain_bit_identical(pair, n, graph):
    cfg, a, b = pair
    P, steps = 6, 3
    ta, la, kva = _run(a, cfg, n, P, steps, graph)
    tb, lb, kvb = _run(b, cfg, n, P, steps, graph)
    for t in range(steps):
        assert np.array_equal(ta[t], tb[t]), f"step {t}: tokens differ"
        assert la[t].shape == lb[t].shape
        diff = np.abs(la[t] - lb[t]).max()
        assert np.array_equal(la[t], lb[t]), f"step {t}: logits differ (max {diff})"
    for (ka, va), (kb, vb) in zip(kva, kvb):
        assert np.array_equal(ka, kb) and np.array_equal(va, vb)


def test_chain_launch_count(pair):
    """One chain launch per layer (+1 for layer 0's q|k|v): the step issues L + 1
    chains, L attention launches, the embed norm, LM head and sampler."""
    cfg, a, b = pair
    sp = Sampling(temperature=0.0)
    s = b.admit(request_seed(6, 1), 4, 16, sp)
    b.forward(np.array([[s, p, -1, 0] for p in range(3)], np.int32), sample=False)
    b.synchronize()
    c0 = b.launch_count()
    b.forward(np.array([[s, 3, -1, 1]], np.int32), graph=False)
    b.synchronize()
    assert b.launch_count() - c0 == 2 * cfg.n_layers + 1 + 3
    b.release(s)
