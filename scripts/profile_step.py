"""Profiling driver: eager Orpheus-3B-style decode steps at batch B, context ctx.

Used under ncu (one GPU):  ncu ... python scripts/profile_step.py --batch 256 --ctx 394
The KV cache is filled by prefill forwards first; then --steps eager decode
steps (no CUDA graph, so every kernel is a separate launch) and one detok
call per 8 streams (steady-state chunk rate) run back to back.
"""

import argparse
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "baseline" / "_ref"))

from paper_2602_00269_b200.config import orpheus3b  # noqa: E402
from paper_2602_00269_b200.device import Sampling, VoxDevice  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=256)
    ap.add_argument("--ctx", type=int, default=394)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--detok", type=int, default=32)
    a = ap.parse_args()
    dev = VoxDevice(orpheus3b(max_slots=max(a.batch, 8)), 0)
    prm = Sampling(temperature=0.6, top_p=0.8, repetition_penalty=1.3)
    P = 50
    slots = [dev.admit(1000 + i, P, 688, prm) for i in range(a.batch)]
    per = max(1, 1000 // (a.ctx - 1))
    for i in range(0, a.batch, per):
        rows = np.array([[s, p, -1, 0] for s in slots[i:i + per] for p in range(a.ctx - 1)], np.int32)
        dev.forward(rows, sample=False)
    dev.synchronize()
    print("kv filled", flush=True)
    for step in range(a.steps):
        rows = np.array([[s, a.ctx - 1 + step, -1, 1] for s in slots], np.int32)
        dev.forward(rows, graph=False)
    dev.synchronize()
    # detok: first windows need >= 28 generated tokens; generate into a few slots
    k = min(a.detok, a.batch)
    for step in range(a.steps, 28):
        rows = np.array([[s, a.ctx - 1 + step, -1, 1] for s in slots[:k]], np.int32)
        dev.forward(rows)
    dev.synchronize()
    # (the windows index generated tokens; decode rows started at ctx-1, so
    #  generated index g lives at position P + g: make the store consistent)
    w = np.array([[s, 1, 0, 28, 28, 0] for s in slots[:k]], np.int32)
    dev.detok(w)
    dev.synchronize()
    print("done", flush=True)


if __name__ == "__main__":
    main()
