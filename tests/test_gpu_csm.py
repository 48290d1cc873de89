"""CSM-style multi-codebook frames (BASELINE config 3 structure):
backbone over summed codebook embeddings + depth decoder conditioned on the projected
backbone state, with device-side hand-overs -- vs the CPU oracle (tiny geometry,
8 codebooks)."""

import numpy as np
import pytest

from oracle.llama import LlamaOracle
from oracle.workload import prompt_ids, request_seed
from paper_2602_00269_b200.config import tiny_csm
from paper_2602_00269_b200.csm import CsmFrames
from paper_2602_00269_b200.device import Sampling, VoxDevice

pytestmark = pytest.mark.gpu
GREEDY = Sampling(temperature=0.0, repetition_penalty=1.0)


@pytest.fixture(scope="module")
def csm():
    bcfg, dcfg = tiny_csm()
    bb, dp = VoxDevice(bcfg, weight_seed=31), VoxDevice(dcfg, weight_seed=32)
    yield bcfg, dcfg, bb, dp, LlamaOracle(bcfg, 31), LlamaOracle(dcfg, 32)
    bb.close()
    dp.close()


def test_frame_embedding_sum(csm):
    """A position's input is the sum of its codebook embeddings (frame store)."""
    bcfg, _, bb, _, bo, _ = csm
    C, cs, base = bcfg.n_codebooks, bcfg.codebook_size, bcfg.audio_base
    P = 10
    seed = request_seed(2, 1)
    slot = bb.admit(seed, P, 8, GREEDY)
    prompt = np.array(prompt_ids(seed, P, bcfg.text_vocab))
    rng = np.random.default_rng(0)
    codes = rng.integers(0, cs, size=C)
    ids = base + np.arange(C) * cs + codes
    bb.write_tokens(slot, P, [int(ids[0])])
    bb.write_frame(slot, P, ids[1:][None, :])
    assert np.array_equal(bb.read_frame(slot, P, 1)[0], ids[1:])
    bb.forward(np.array([[slot, p, -1, 0] for p in range(P)], np.int32), sample=False, sync=True, graph=False)
    _, lg = bb.forward(np.array([[slot, P, -1, 1]], np.int32), sample=False, full_logits=True, sync=True)
    bo.forward("e", prompt, np.arange(P), want_logits=False)
    ol, _ = bo.forward("e", ids[None, :], np.array([P]))
    err = np.abs(lg[0] - ol[0]).max()
    assert err < 2e-2 * max(1.0, np.abs(ol[0]).max()), err
    bb.release(slot)
    bo.release("e")


def test_greedy_frames_vs_oracle(csm):
    """2 streams x 3 frames, greedy.  The device pipeline free-runs; the oracle replays
    it teacher-forced and every code must be the oracle's argmax wherever the oracle's
    top-2 margin exceeds 0.15 (bf16 noise is ~0.03-0.06, see test_gpu_lm.py)."""
    bcfg, dcfg, bb, dp, bo, do = csm
    C, cs, base = bcfg.n_codebooks, bcfg.codebook_size, bcfg.audio_base
    pipe = CsmFrames(bb, dp)
    P, F, R = 12, 3, 2
    streams = [pipe.admit(request_seed(4, r), P, F + 1, GREEDY, GREEDY) for r in range(R)]
    pipe.prefill(streams)
    for _ in range(F):
        pipe.step(streams)
    frames = np.array([[pipe.frame(s, P + f) for f in range(F)] for s in streams])  # [R, F, C]
    assert frames.shape == (R, F, C) and ((frames >= 0) & (frames < cs)).all()
    checked = ties = 0
    for r in range(R):
        prompt = np.array(prompt_ids(request_seed(4, r), P, bcfg.text_vocab))
        bo.forward(("b", r), prompt[:-1], np.arange(P - 1), want_logits=False)
        inp = np.array([prompt[-1]] + [-1] * (C - 1))
        for f in range(F):
            lg, xf = bo.forward(("b", r), inp[None, :], np.array([P - 1 + f]))
            row = lg[0, base:base + cs]
            srt = np.sort(row)[::-1]
            if srt[0] - srt[1] > 0.15:
                checked += 1
                assert int(np.argmax(row)) == frames[r, f, 0], ("c0", r, f)
            else:
                ties += 1
            # depth decoder on the device's codes (teacher forcing)
            ext = do.project(xf)
            dl, _ = do.forward(("d", r, f), np.array([-2, int(frames[r, f, 0])]), np.array([0, 1]), ext=np.vstack([ext, ext]))
            for k in range(1, C):
                if k > 1:
                    tok = (k - 1) * cs + int(frames[r, f, k - 1])
                    dl, _ = do.forward(("d", r, f), np.array([tok]), np.array([k]))
                drow = dl[-1, k * cs:(k + 1) * cs]
                srt = np.sort(drow)[::-1]
                if srt[0] - srt[1] > 0.15:
                    checked += 1
                    assert int(np.argmax(drow)) == frames[r, f, k], ("depth", r, f, k)
                else:
                    ties += 1
            do.release(("d", r, f))
            inp = base + np.arange(C) * cs + frames[r, f]
        bo.release(("b", r))
    assert checked >= 0.75 * R * F * C, (checked, ties)
    for s in streams:
        pipe.release(s)


def test_stochastic_frames_deterministic_and_in_range(csm):
    """Sampled (T 0.9, top-k 50) frames: every code lies in its codebook's range, and the
    same seeds reproduce the same frames (counter-based RNG keyed by request seed/step)."""
    bcfg, dcfg, bb, dp, _, _ = csm
    pipe = CsmFrames(bb, dp)
    prm = Sampling(temperature=0.9, top_k=50, repetition_penalty=1.0)
    runs = []
    for _ in range(2):
        streams = [pipe.admit(request_seed(8, r), 10, 4, prm, prm) for r in range(2)]
        pipe.prefill(streams)
        for _ in range(2):
            pipe.step(streams)
        runs.append(np.array([[pipe.frame(s, 10 + f) for f in range(2)] for s in streams]))
        for s in streams:
            pipe.release(s)
    assert ((runs[0] >= 0) & (runs[0] < bcfg.codebook_size)).all()
    assert np.array_equal(runs[0], runs[1])
    assert len(np.unique(runs[0])) > 4  # not collapsed onto one code
