"""CosyVoice2-style LM (BASELINE config 4's backbone: Qwen2.5-0.5B geometry -- 14 q / 2 kv
heads of 64 (GQA group 7), q|k|v bias, tied embeddings, speech-token range mask) vs the CPU
oracle: weights, prefill/decode logits and KV, and greedy speech tokens."""

import numpy as np
import pytest

from oracle import sampler as osamp
from oracle.llama import LlamaOracle, audio_range, masked
from oracle.workload import prompt_ids, request_seed
from paper_2602_00269_b200.config import tiny_cosy
from paper_2602_00269_b200.device import Sampling, VoxDevice

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cosy():
    cfg = tiny_cosy()
    dev = VoxDevice(cfg, weight_seed=77)
    orc = LlamaOracle(cfg, 77)
    yield cfg, dev, orc
    dev.close()


def test_qkv_bias_bit_identical(cosy):
    cfg, dev, orc = cosy
    nq = (cfg.n_heads + 2 * cfg.n_kv_heads) * cfg.head_dim
    b = dev.read_weight("qkv_bias", 1, (nq,), np.float32)
    assert np.array_equal(b, orc.w.layers[1]["qkv_bias"])
    assert np.abs(b).max() > 0.1


@pytest.mark.parametrize("lens", [(23,), (9, 40, 130)])
def test_prefill_decode_logits(cosy, lens):
    cfg, dev, orc = cosy
    slots, prompts = [], []
    for i, P in enumerate(lens):
        seed = request_seed(3, 10 * len(lens) + i)
        slot = dev.admit(seed, P, 16, Sampling(temperature=0.0))
        prompt = np.array(prompt_ids(seed, P, cfg.text_vocab))
        dev.forward(np.array([[slot, p, -1, 0] for p in range(P - 1)], np.int32), sample=False, sync=True,
                    graph=False)
        orc.forward(("c", len(lens), i), prompt[:-1], np.arange(P - 1), want_logits=False)
        slots.append(slot)
        prompts.append(prompt)
    rows = np.array([[s, P - 1, -1, 1] for s, P in zip(slots, lens)], np.int32)
    _, lg = dev.forward(rows, sample=False, full_logits=True, sync=True)
    for i, P in enumerate(lens):
        ol, _ = orc.forward(("c", len(lens), i), prompts[i][-1:], np.array([P - 1]))
        err = np.abs(lg[i] - ol[0]).max()
        assert err < 2e-2 * max(1.0, np.abs(ol[0]).max()), (i, P, err)
        for layer in range(cfg.n_layers):
            k, v = dev.read_kv(layer, slots[i], P - 1)
            assert np.abs(k - orc.k[("c", len(lens), i)][layer, P - 1]).max() < 3e-2
            assert np.abs(v - orc.v[("c", len(lens), i)][layer, P - 1]).max() < 3e-2
    for s in slots:
        dev.release(s)
    for i in range(len(lens)):
        orc.release(("c", len(lens), i))


def test_greedy_speech_tokens(cosy):
    """2 greedy requests x 32 speech tokens (rp 1.1 as the cosy_like profile): the fused
    device path free-runs; every token equals the argmax of the device's own penalised
    logits and the oracle's greedy choice wherever the oracle's top-2 margin exceeds twice
    the measured device/oracle logit error (numerically determined decisions)."""
    cfg, dev, orc = cosy
    P, T, R, pen = 30, 32, 2, 1.1
    greedy = Sampling(temperature=0.0, repetition_penalty=pen)
    slots = [dev.admit(request_seed(9, r), P, T, greedy) for r in range(R)]
    dev.forward(np.concatenate([np.array([[s, p, -1, 0] for p in range(P - 1)], np.int32) for s in slots]),
                sample=False)
    got = np.zeros((R, T), np.int64)
    for s in range(T):
        toks, _ = dev.forward(np.array([[sl, P - 1 + s, -1, 1] for sl in slots], np.int32), want_tokens=True)
        got[:, s] = toks
    lo, hi = audio_range(cfg, 0)
    assert ((got >= lo) & (got < hi)).all()  # speech positions emit speech ids only
    for sl in slots:
        dev.release(sl)
    # teacher-forced replay through the parity path and the oracle
    slots = [dev.admit(request_seed(9, r), P, T, greedy) for r in range(R)]
    dev.forward(np.concatenate([np.array([[s, p, -1, 0] for p in range(P - 1)], np.int32) for s in slots]),
                sample=False)
    prompts = [np.array(prompt_ids(request_seed(9, r), P, cfg.text_vocab)) for r in range(R)]
    for r in range(R):
        orc.forward(("g", r), prompts[r][:-1], np.arange(P - 1), want_logits=False)
    wins = [osamp.RingWindow(64, cfg.vocab) for _ in range(R)]
    checked = ties = 0
    for s in range(T):
        rows = np.array([[sl, P - 1 + s, (-1 if s == 0 else int(got[r, s - 1])), 1] for r, sl in enumerate(slots)],
                        np.int32)
        _, dlog = dev.forward(rows, sample=False, full_logits=True, sync=True)
        for r in range(R):
            tok_in = int(prompts[r][-1]) if s == 0 else int(got[r, s - 1])
            ol, _ = orc.forward(("g", r), np.array([tok_in]), np.array([P - 1 + s]))
            dpen = osamp.apply_repetition_penalty(masked(dlog[r], lo, hi), pen, wins[r])
            opn = osamp.apply_repetition_penalty(masked(ol[0], lo, hi), pen, wins[r])
            assert int(np.argmax(dpen)) == got[r, s], (r, s)
            err = np.abs(dlog[r, lo:hi].astype(np.float64) - ol[0, lo:hi]).max()
            assert err < 0.15, (r, s, err)
            srt = np.sort(opn[lo:hi])[::-1]
            if srt[0] - srt[1] > 2 * err:
                checked += 1
                assert int(np.argmax(opn)) == got[r, s], (r, s)
            else:
                ties += 1
            wins[r].append(int(got[r, s]))
    assert checked >= 0.8 * R * T, (checked, ties)
    for r, sl in enumerate(slots):
        dev.release(sl)
        orc.release(("g", r))


def test_greedy_speech_tokens_bit_exact_planted():
    """CosyVoice2-style LM (q|k|v bias, GQA 14:2), planted-margin init as config 1's
    (config.tiny_planted's embedding scale): 2 greedy requests x 32 speech tokens, rp
    1.1, free-running on the serving path.  Precondition asserted at EVERY decision:
    the oracle's penalised top-2 margin exceeds 10x that step's measured device /
    oracle logit error; then every device token equals the oracle's greedy choice on
    the same history, so the device stream IS the oracle's free-running stream."""
    from dataclasses import replace

    from paper_2602_00269_b200.config import PLANTED_EMBED_MULT, PLANTED_WEIGHT_SEED, tiny_cosy
    from paper_2602_00269_b200.device import VoxDevice

    base = tiny_cosy(max_slots=4)
    cfg = replace(base, embed_scale=PLANTED_EMBED_MULT * base.embed_half_width)
    dev = VoxDevice(cfg, weight_seed=PLANTED_WEIGHT_SEED)
    orc = LlamaOracle(cfg, PLANTED_WEIGHT_SEED)
    P, T, R, pen = 30, 32, 2, 1.1
    greedy = Sampling(temperature=0.0, repetition_penalty=pen)
    slots = [dev.admit(request_seed(19, r), P, T, greedy) for r in range(R)]
    dev.forward(np.concatenate([np.array([[s, p, -1, 0] for p in range(P - 1)], np.int32) for s in slots]),
                sample=False)
    prompts = [np.array(prompt_ids(request_seed(19, r), P, cfg.text_vocab)) for r in range(R)]
    for r in range(R):
        orc.forward(("p", r), prompts[r][:-1], np.arange(P - 1), want_logits=False)
    wins = [osamp.RingWindow(64, cfg.vocab) for _ in range(R)]
    lo, hi = audio_range(cfg, 0)
    got = np.zeros((R, T), np.int64)
    ratio = np.zeros((R, T))
    for s in range(T):
        toks, _ = dev.forward(np.array([[sl, P - 1 + s, -1, 1] for sl in slots], np.int32), want_tokens=True)
        got[:, s] = toks
        dlog, col0 = dev.read_logits()
        for r in range(R):
            tok_in = int(prompts[r][-1]) if s == 0 else int(got[r, s - 1])
            ol, _ = orc.forward(("p", r), np.array([tok_in]), np.array([P - 1 + s]))
            d_full = np.full(cfg.vocab, -np.inf)
            d_full[col0:col0 + dlog.shape[1]] = dlog[r]
            dpen = osamp.apply_repetition_penalty(masked(d_full, lo, hi), pen, wins[r])
            opn = osamp.apply_repetition_penalty(masked(ol[0], lo, hi), pen, wins[r])
            assert int(np.argmax(dpen)) == got[r, s], (r, s)  # K1 in situ
            err = np.abs(dpen[lo:hi] - opn[lo:hi]).max()
            srt = np.sort(opn[lo:hi])[::-1]
            ratio[r, s] = (srt[0] - srt[1]) / max(err, 1e-30)
            assert ratio[r, s] >= 10.0, (r, s, srt[0] - srt[1], err)  # precondition
            assert int(np.argmax(opn)) == got[r, s], (r, s)
            wins[r].append(int(got[r, s]))
    print(f"cosy planted greedy: min margin/err {ratio.min():.1f}")
    for r, sl in enumerate(slots):
        dev.release(sl)
        orc.release(("p", r))
    dev.close()
