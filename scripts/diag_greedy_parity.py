"""Diagnostic (GPU): config-1 greedy parity vs the planted-margin embedding multiplier.

For each multiplier: device free-running (fused graph path + K1), oracle teacher-forced
on the device's history; prints the margin / logit-error distribution, the number of
decisions with margin < 10x error, whether the streams equal the oracle's free-running
streams, and the fraction of K/V elements that differ bit-wise (layer 1, all positions).
"""
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "baseline" / "_ref"))

from oracle import sampler as osamp  # noqa: E402
from oracle.greedy import greedy_streams  # noqa: E402
from oracle.llama import LlamaOracle, audio_range  # noqa: E402
from oracle.workload import prompt_ids, request_seed  # noqa: E402
from paper_2602_00269_b200.config import tiny  # noqa: E402
from paper_2602_00269_b200.device import Sampling, VoxDevice  # noqa: E402


class Shift:
    def __init__(self, win, lo, hi):
        self.counts = win.counts[lo:hi]
        self._n = len(win)

    def __len__(self):
        return self._n


def run(mult, ws, R=4, P=50, T=64, pen=1.3):
    base = tiny(max_slots=8)
    c = tiny(max_slots=8, embed_scale=base.embed_half_width * mult)
    dev = VoxDevice(c, weight_seed=ws)
    orc = LlamaOracle(c, ws)
    slots = [dev.admit(request_seed(0, r), P, T, Sampling(temperature=0.0, repetition_penalty=pen)) for r in range(R)]
    dev.forward(np.array([[s, p, -1, 0] for s in slots for p in range(P - 1)], np.int32), sample=False)
    prompts = [np.array(prompt_ids(request_seed(0, r), P, c.text_vocab)) for r in range(R)]
    for r in range(R):
        orc.forward(r, prompts[r][:-1], np.arange(P - 1), want_logits=False)
    wins = [osamp.RingWindow(64, c.vocab) for _ in range(R)]
    got = np.zeros((R, T), np.int64)
    err = np.zeros((R, T))
    margin = np.zeros((R, T))
    agree = 0
    for s in range(T):
        toks, _ = dev.forward(np.array([[sl, P - 1 + s, -1, 1] for sl in slots], np.int32), want_tokens=True)
        got[:, s] = toks
        dlog, base_col = dev.read_logits()
        lo, hi = audio_range(c, s)
        for r in range(R):
            tok_in = int(prompts[r][-1]) if s == 0 else int(got[r, s - 1])
            ol, _ = orc.forward(r, np.array([tok_in]), np.array([P - 1 + s]), head=(lo, hi))
            dpen = osamp.apply_repetition_penalty(dlog[r].astype(np.float64), pen, Shift(wins[r], lo, hi))
            opn = osamp.apply_repetition_penalty(ol[0].astype(np.float64), pen, Shift(wins[r], lo, hi))
            err[r, s] = np.abs(dpen - opn).max()
            srt = np.sort(opn)[::-1]
            margin[r, s] = srt[0] - srt[1]
            agree += int(np.argmax(opn)) + lo == got[r, s]
            wins[r].append(int(got[r, s]))
    # K/V bit agreement, layer L-1, all positions of request 0
    diff = tot = 0
    for pos in range(P - 1 + T):
        k, v = dev.read_kv(c.n_layers - 1, slots[0], pos)
        ko, vo = orc.k[0][c.n_layers - 1, pos], orc.v[0][c.n_layers - 1, pos]
        diff += int((k != ko).sum() + (v != vo).sum())
        tot += k.size + v.size
    ref, om, _ = greedy_streams(c, ws, 0, R, P, T, pen)
    ratio = margin / np.maximum(err, 1e-30)
    print(f"mult {mult:7.0f} ws {ws}: logit std ~{np.std(dlog):.1f} min margin {margin.min():.4g} "
          f"max err {err.max():.4g} median err {np.median(err):.3g} steps ratio<10 {(ratio < 10).sum()} "
          f"ratio<2 {(ratio < 2).sum()} agree {agree}/{R*T} stream==oracle free-run {np.array_equal(got, ref)} "
          f"(first diff {np.argwhere(got != ref)[:1].tolist()}) KV bits differ {diff / tot:.4f}", flush=True)
    dev.close()


if __name__ == "__main__":
    mults = [float(x) for x in sys.argv[1].split(",")] if len(sys.argv) > 1 else [1, 100, 1000, 10000]
    seeds = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [1234, 7]
    for mult in mults:
        for ws in seeds:
            run(mult, ws)
