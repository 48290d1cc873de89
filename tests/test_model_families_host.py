"""CPU: configuration and oracle host logic of the config-3 (CSM-style) and config-4
(CosyVoice2-style) model families."""

from types import SimpleNamespace

import numpy as np
import pytest

from oracle.llama import LlamaOracle
from paper_2602_00269_b200.config import (COSY_SPEECH_BASE, COSY_SPEECH_TOKENS, CSM_CODES, CSM_TEXT_VOCAB,
                                          cosyvoice2, csm_backbone, csm_depth, tiny_cosy, tiny_csm)


def test_csm_token_layouts():
    bb, dp = csm_backbone(), csm_depth()
    assert bb.vocab == CSM_TEXT_VOCAB + 32 * CSM_CODES and bb.audio_base == CSM_TEXT_VOCAB
    assert bb.n_codebooks == 32 and bb.frame_tokens == 1            # head = codebook-0 rows
    assert dp.vocab == 32 * CSM_CODES and dp.audio_base == CSM_CODES  # outputs = codebooks 1..31
    assert dp.frame_tokens == 31 and dp.ext_dim == bb.d_model
    assert CSM_CODES % 128 == 0                                      # one-slot head = whole tiles
    assert dp.max_ctx >= 2 + 31                                      # ext, c0, codebooks 1..31
    for c in (bb, dp):
        assert c.d_model % 64 == 0 and c.d_ff % 64 == 0 and c.n_heads % c.n_kv_heads == 0
        assert c.n_heads // c.n_kv_heads <= 8 and (c.n_heads // c.n_kv_heads) * c.head_dim <= 512


def test_cosy_token_layout():
    c = cosyvoice2()
    assert c.vocab == COSY_SPEECH_BASE + COSY_SPEECH_TOKENS and c.audio_base == COSY_SPEECH_BASE
    assert c.frame_tokens == 1 and c.qkv_bias and c.n_heads // c.n_kv_heads == 7 and c.head_dim == 64
    t = tiny_cosy()
    assert (t.n_heads, t.n_kv_heads, t.head_dim, t.qkv_bias) == (c.n_heads, c.n_kv_heads, c.head_dim, True)


def test_oracle_frame_embedding_and_ext_rows():
    bcfg, dcfg = tiny_csm()
    bb = LlamaOracle(bcfg, 5)
    ids = bcfg.audio_base + np.arange(bcfg.n_codebooks) * bcfg.codebook_size + 7
    h = bb.embed(ids[None, :])[0]
    ref = bb.w.emb[ids[0]].astype(np.float32)
    for i in ids[1:]:
        ref = ref + bb.w.emb[i]
    assert np.array_equal(h, ref)
    partial = ids.copy()
    partial[3:] = -1  # absent codebooks contribute nothing
    assert np.array_equal(bb.embed(partial[None, :])[0], bb.w.emb[ids[0]] + bb.w.emb[ids[1]] + bb.w.emb[ids[2]])
    dp = LlamaOracle(dcfg, 6)
    xf = np.ones((1, bcfg.d_model), np.float32)
    ext = dp.project(xf)
    assert ext.shape == (1, dcfg.d_model)
    assert np.allclose(ext[0], dp.w.proj.sum(axis=1), rtol=1e-5, atol=1e-5)
    assert np.array_equal(dp.embed(np.array([-2]), ext)[0], ext[0])


def test_cosy_oracle_has_bias():
    o = LlamaOracle(tiny_cosy(n_layers=1), 3)
    nq = (o.cfg.n_heads + 2 * o.cfg.n_kv_heads) * o.cfg.head_dim
    assert o.w.layers[0]["qkv_bias"].shape == (nq,) and np.abs(o.w.layers[0]["qkv_bias"]).max() > 0


def test_csm_pipeline_rejects_mismatched_geometry():
    from paper_2602_00269_b200.csm import CsmFrames

    bcfg, dcfg = tiny_csm()
    fake = lambda c: SimpleNamespace(cfg=c)  # noqa: E731
    CsmFrames(fake(bcfg), fake(dcfg))
    with pytest.raises(ValueError):
        CsmFrames(fake(bcfg), fake(tiny_csm(4)[1]))
