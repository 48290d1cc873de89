"""Profiling driver: eager Orpheus-3B-style decode steps at batch B, context ctx.

Used under ncu (one GPU), with the profiled region bracketed by
cudaProfilerStart/Stop so the KV-fill prefill passes are not captured:

  ncu --profile-from-start off --metrics gpu__time_duration.sum ... \
      python scripts/profile_step.py --batch 224 --ctx 394

The KV cache is filled by prefill forwards first; then --steps eager decode
steps (no CUDA graph, so every kernel is a separate launch) and, with
--detok N, one steady-state detok call over N streams run inside the range.
"""

import argparse
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "baseline" / "_ref"))

from paper_2602_00269_b200.config import CONFIGS  # noqa: E402
from paper_2602_00269_b200.device import Sampling, VoxDevice  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=224)
    ap.add_argument("--ctx", type=int, default=394)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--detok", type=int, default=32)
    ap.add_argument("--graph", action="store_true", help="graph-captured decode steps")
    ap.add_argument("--config", default="orpheus3b", help="orpheus3b | cosyvoice2 (no SNAC detok: --detok 0)")
    a = ap.parse_args()
    import torch

    dev = VoxDevice(CONFIGS[a.config](max_slots=max(a.batch, 8)), 0)
    prm = (Sampling(temperature=0.8, top_p=0.95, top_k=50, repetition_penalty=1.1) if "cosy" in a.config
           else Sampling(temperature=0.6, top_p=0.8, repetition_penalty=1.3))
    P = 50
    slots = [dev.admit(1000 + i, P, 688, prm) for i in range(a.batch)]
    per = max(1, 1000 // (a.ctx - 1))
    for i in range(0, a.batch, per):
        rows = np.array([[s, p, -1, 0] for s in slots[i:i + per] for p in range(a.ctx - 1)], np.int32)
        dev.forward(rows, sample=False)
    # tokens for a detok window (first chunk: 28 generated tokens) in the first k slots
    k = min(a.detok, a.batch)
    for step in range(35 if k > 0 else 0):
        rows = np.array([[s, a.ctx - 1 + step, -1, 1] for s in slots[:k]], np.int32)
        dev.forward(rows)
    if k > 0:  # first window outside the profiled range; the profiled one is a steady 7-token window
        dev.detok(np.array([[s, 1, 0, 28, 28, 0] for s in slots[:k]], np.int32))
    rows = np.array([[s, a.ctx - 1 + 35, -1, 1] for s in slots], np.int32)
    dev.forward(rows, graph=a.graph)  # warm
    dev.synchronize()
    print("kv filled", flush=True)
    torch.cuda.profiler.start()
    for step in range(a.steps):
        rows = np.array([[s, a.ctx - 1 + 36 + step, -1, 1] for s in slots], np.int32)
        dev.forward(rows, graph=a.graph)
    if k > 0:
        dev.detok(np.array([[s, 2, 7, 28, 7, 0] for s in slots[:k]], np.int32))
    dev.synchronize()
    torch.cuda.profiler.stop()
    print("done", flush=True)


if __name__ == "__main__":
    main()
