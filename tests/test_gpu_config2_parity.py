"""Config-2 dims parity: the bench's decode step vs the CPU oracle.

Orpheus-3B-style geometry (d 3072, 24 q / 8 kv heads x 128, FFN 8192, vocab
156,940, tied head) with 2 of the 28 layers, one mixed batch of 200 or 256
decode rows -- the 224- and 256-row graph buckets the serving bench runs, and
273 / 300 rows (decode plus a prefill burst: one GEMM n-tile of 288 / 320 rows) --
through the DEFAULT serving path: CUDA-graph-captured step with PDL, the mc
tcgen05 GEMM with its split-K fp32 planes for QKV / O / down and the fused
SiLU(gate)*up epilogue on gate|up, paged attention, the packed audio-row LM
head and K1 greedy.  Rows sit at 11 different generation steps (so the frame
slots differ and the head covers all 28,672 audio rows) over contexts of
3..29 tokens.

Checked against oracle/llama.py on the same random-init weights:
  * the head logits K1 consumed (vox_read_logits), every row, every audio id;
  * K/V appended at the decode position, every layer (sampled rows);
  * K1 in situ: every token = argmax of the device's own penalised, masked
    logits (bit-exact), and = the oracle's greedy choice wherever the oracle's
    top-2 margin exceeds twice that row's measured logit error.  At this
    (bench) init the logit std is ~2.5 and the device/oracle error ~1e-2
    (fp32 summation order -> bf16 flips), so ~12% of 4096-way decisions are
    numerically undetermined; exact stream equality is shown on the
    planted-margin init (tests/test_gpu_lm.py::test_greedy_tokens_bit_exact_config1).
"""

import numpy as np
import pytest

from oracle import sampler as osamp
from oracle.llama import LlamaOracle
from oracle.workload import prompt_ids, request_seed
from paper_2602_00269_b200.config import orpheus3b
from paper_2602_00269_b200.device import Sampling, VoxDevice

pytestmark = pytest.mark.gpu

WS = 4321
PEN = 1.3


@pytest.fixture(scope="module")
def c2():
    cfg = orpheus3b(n_layers=2, max_slots=320, max_ctx=64, max_rows=1024, detok_enabled=False)
    dev = VoxDevice(cfg, weight_seed=WS)
    orc = LlamaOracle(cfg, WS, lazy_emb=True)
    yield cfg, dev, orc
    dev.close()


def _plan(cfg, n, salt):
    rng = np.random.default_rng(1000 + n + salt)
    reqs = []
    for r in range(n):
        P = 3 + (r * 5) % 17
        s = (r * 3 + salt) % 11
        gen = [cfg.audio_base + (k % cfg.frame_tokens) * cfg.codebook_size + int(rng.integers(cfg.codebook_size))
               for k in range(s)]
        reqs.append((request_seed(77, 1000 * n + r + salt), P, s, gen))
    return reqs


@pytest.mark.parametrize("n", [200, 256, 273, 300])
def test_config2_dims_decode_step(c2, n):
    cfg, dev, orc = c2
    reqs = _plan(cfg, n, 0)
    greedy = Sampling(temperature=0.0, repetition_penalty=PEN)
    slots = [dev.admit(seed, P, 16, greedy) for seed, P, s, gen in reqs]
    try:
        _check_step(cfg, dev, orc, n, reqs, slots)
    finally:
        for sl in slots:
            dev.release(sl)
        for r in range(n):
            orc.release((n, r))


def _check_step(cfg, dev, orc, n, reqs, slots):
    # history: prompt[:-1] (+ prompt[-1] and the first s-1 generated ids when s >= 1)
    pre, o_rid, o_tok, o_pos = [], [], [], []
    for r, ((seed, P, s, gen), sl) in enumerate(zip(reqs, slots)):
        prompt = prompt_ids(seed, P, cfg.text_vocab)
        hist = prompt[:-1] + ([prompt[-1]] + gen[: s - 1] if s >= 1 else [])
        for p, t in enumerate(hist):
            pre.append([sl, p, -1 if p < P else t, 0])
            o_rid.append((n, r))
            o_tok.append(t)
            o_pos.append(p)
    pre = np.asarray(pre, np.int32)
    for a in range(0, len(pre), cfg.max_rows):
        dev.forward(pre[a:a + cfg.max_rows], sample=False)
    for a in range(0, len(o_tok), 1024):
        orc.forward_rows(o_rid[a:a + 1024], np.array(o_tok[a:a + 1024]), np.array(o_pos[a:a + 1024]),
                         want_logits=False)
    # the decode step: one sampling row per request (graph bucket 224 or 256)
    rows, d_tok = [], []
    for (seed, P, s, gen), sl in zip(reqs, slots):
        tok = prompt_ids(seed, P, cfg.text_vocab)[-1] if s == 0 else gen[s - 1]
        rows.append([sl, P - 1 + s, -1 if s == 0 else tok, 1])
        d_tok.append(tok)
    rows = np.asarray(rows, np.int32)
    # first call of a bucket: eager pass + capture; the second replays the captured
    # graph (the step is idempotent: same K/V rewritten, same token sampled)
    dev.forward(rows, want_tokens=False)
    got, _ = dev.forward(rows, want_tokens=True)
    dlog, base = dev.read_logits()
    A = cfg.frame_tokens * cfg.codebook_size
    assert base == cfg.audio_base and dlog.shape == (n, A)
    ol, _ = orc.forward_rows([(n, r) for r in range(n)], np.array(d_tok), rows[:, 1], head=(base, base + A))
    # logits: every row, every audio id
    d = dlog.astype(np.float64) - ol
    rel_rms = np.sqrt((d ** 2).mean(axis=1)) / np.sqrt((ol.astype(np.float64) ** 2).mean(axis=1))
    assert rel_rms.max() < 1e-2, rel_rms.max()
    assert (np.abs(d).max(axis=1) < 2e-2 * np.maximum(1.0, np.abs(ol).max(axis=1))).all()
    # K/V appended at the decode position
    for r in range(0, n, 7):
        seed, P, s, gen = reqs[r]
        for layer in range(cfg.n_layers):
            k, v = dev.read_kv(layer, slots[r], P - 1 + s)
            ko, vo = orc.k[(n, r)][layer, P - 1 + s], orc.v[(n, r)][layer, P - 1 + s]
            assert np.abs(k - ko).max() < 3e-2 * max(1.0, np.abs(ko).max()), (r, layer)
            assert np.abs(v - vo).max() < 3e-2 * max(1.0, np.abs(vo).max()), (r, layer)
    # tokens: K1 in situ (bit-exact) and the oracle's decision where it is determined
    checked = 0
    for r in range(n):
        seed, P, s, gen = reqs[r]
        k = s % cfg.frame_tokens
        lo, hi = k * cfg.codebook_size, (k + 1) * cfg.codebook_size  # columns of the audio head
        win = osamp.RingWindow(64, A)
        for t in gen:
            win.append(t - base)
        dpen = osamp.apply_repetition_penalty(dlog[r].astype(np.float64), PEN, win)[lo:hi]
        open_ = osamp.apply_repetition_penalty(ol[r].astype(np.float64), PEN, win)[lo:hi]
        assert int(np.argmax(dpen)) + lo + base == got[r], r
        e = np.abs(dpen - open_).max()
        srt = np.sort(open_)[::-1]
        if srt[0] - srt[1] > 2 * e:
            checked += 1
            assert int(np.argmax(open_)) + lo + base == got[r], (r, srt[0] - srt[1], e)
    print(f"config-2 step n={n}: max rel-rms logit error {rel_rms.max():.2e}, determined decisions {checked}/{n}")
    assert checked >= 0.8 * n, checked
    for r, ((seed, P, s, gen), sl) in enumerate(zip(reqs, slots)):
        assert dev.read_tokens(sl, P + s, 1)[0] == got[r]
