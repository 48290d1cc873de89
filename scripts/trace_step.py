"""In-graph timeline of steady-state decode steps (vox_trace_*): per-launch spans,
gaps and overlap between consecutive LM-stream kernels.  GPU only.

  python scripts/trace_step.py --batch 224 --ctx 394 --steps 3 [--detok 32]
"""
import argparse
import collections
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2602_00269_b200.config import CONFIGS  # noqa: E402
from paper_2602_00269_b200.device import Sampling, VoxDevice  # noqa: E402

from paper_2602_00269_b200.trace import NAMES, launches  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=224)
    ap.add_argument("--ctx", type=int, default=394)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--config", default="orpheus3b")
    a = ap.parse_args()
    dev = VoxDevice(CONFIGS[a.config](max_slots=max(a.batch, 8)), 0)
    prm = (Sampling(temperature=0.8, top_p=0.95, top_k=50, repetition_penalty=1.1) if "cosy" in a.config
           else Sampling(temperature=0.6, top_p=0.8, repetition_penalty=1.3))
    P = 50
    slots = [dev.admit(1000 + i, P, 688, prm) for i in range(a.batch)]
    per = max(1, 1000 // (a.ctx - 1))
    for i in range(0, a.batch, per):
        rows = np.array([[s, p, -1, 0] for s in slots[i:i + per] for p in range(a.ctx - 1)], np.int32)
        dev.forward(rows, sample=False)
    for w in range(8):  # >= 7: one graph per head frame slot when every row shares it
        rows = np.array([[s, a.ctx - 8 + w, -1, 1] for s in slots], np.int32)
        dev.forward(rows)
    dev.synchronize()
    import time
    t = time.perf_counter()
    for step in range(a.steps):
        rows = np.array([[s, a.ctx + step, -1, 1] for s in slots], np.int32)
        dev.forward(rows)
    dev.synchronize()
    print(f"untraced wall {(time.perf_counter() - t) * 1e3 / a.steps:.3f} ms/step")
    dev.trace_arm()
    for step in range(a.steps):
        rows = np.array([[s, a.ctx + a.steps + step, -1, 1] for s in slots], np.int32)
        dev.forward(rows)
    dev.synchronize()
    rec = dev.trace_read()
    ls = launches(rec)
    t_start = ls[0]["t0"]
    t_end = max(l["t1max"] for l in ls)
    print(f"{len(rec)} CTA records, {len(ls)} launches, {a.steps} steps, span {(t_end - t_start) / 1e3:.1f} us "
          f"= {(t_end - t_start) / 1e3 / a.steps:.1f} us/step")
    per_kind = collections.defaultdict(lambda: [0, 0.0])
    gaps = collections.defaultdict(float)
    prev = None
    for l in ls:
        name = NAMES.get(l["tag"] & 255, "?") + f"[{l['tag'] >> 8}]"
        dur = (l["t1max"] - l["t0"]) / 1e3
        per_kind[name][0] += 1
        per_kind[name][1] += dur
        if prev is not None:
            gaps[prev[0] + " -> " + name] += (l["t0"] - prev[1]) / 1e3
        prev = (name, l["t1max"])
    print("per kernel (launch span = first CTA start -> last CTA end):")
    for k, (n, t) in sorted(per_kind.items(), key=lambda x: -x[1][1]):
        print(f"  {k:24s} {n:5d} launches {t / a.steps:9.1f} us/step {t / n:7.2f} us/launch")
    print("boundaries (next first-CTA start - prev last-CTA end; negative = PDL overlap), us/step:")
    for k, t in sorted(gaps.items(), key=lambda x: -abs(x[1])):
        print(f"  {k:48s} {t / a.steps:8.1f}")
    # exposed time: end(k) - end(k-1) along the LM stream (the critical path)
    exp = collections.defaultdict(float)
    prev_end = None
    for l in ls:
        name = NAMES.get(l["tag"] & 255, "?") + f"[{l['tag'] >> 8}]"
        if prev_end is not None:
            exp[name] += (l["t1max"] - prev_end) / 1e3
        prev_end = max(prev_end or 0, l["t1max"])
    print("exposed time per kernel (end - previous end), us/step:")
    for k, t in sorted(exp.items(), key=lambda x: -x[1]):
        print(f"  {k:24s} {t / a.steps:9.1f}")
    busy = sum(t for _, t in per_kind.values())
    print(f"sum of launch spans {busy / a.steps:.1f} us/step vs wall {(t_end - t_start) / 1e3 / a.steps:.1f}")


if __name__ == "__main__":
    main()
