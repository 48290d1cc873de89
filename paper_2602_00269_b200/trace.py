"""Host-side analysis of the in-graph kernel tracer (vox_trace_arm / vox_trace_read).

Records are one per CTA: {tag = kernel id | (grid CTAs << 8), smid, t0, t1} on
%globaltimer.  `launches` groups them into kernel launches; `exposed` charges each
launch the time it adds to the LM stream's critical path (its last-CTA end minus
the previous launch's), which is what a kernel costs inside a PDL-chained graph.
"""

from __future__ import annotations

import collections

import numpy as np

NAMES = {1: "gemm1cta", 2: "gemm_mc", 3: "attn", 4: "attn_comb", 5: "qkv_rope", 6: "resid_norm",
         7: "embed_norm", 8: "silu", 9: "sampler", 10: "detok", 11: "chain"}
# kernel -> class of the eager per-class CUDA-event timing (vox_timing_read)
CLASS = {"chain": "chain", "gemm1cta": "gemm", "gemm_mc": "gemm", "attn": "attn", "attn_comb": "attn",
         "qkv_rope": "qkv_rope", "resid_norm": "norm", "embed_norm": "norm", "silu": "silu",
         "sampler": "sampler", "detok": "detok"}


def launches(rec: np.ndarray) -> list[dict]:
    """Group per-CTA records into launches: a maximal run (by start time) of one tag,
    at most the launch's CTA count long."""
    rec = np.sort(rec[(rec["tag"] & 255) < 32], order="t0")  # >= 32: layer-chain event marks
    out: list[dict] = []
    open_: dict[int, dict] = {}
    for r in rec:
        tag = int(r["tag"])
        cur = open_.get(tag)
        if cur is not None and r["t0"] <= cur["t1max"] + 500 and cur["n"] < (tag >> 8):
            cur["n"] += 1
            cur["t1max"] = max(cur["t1max"], int(r["t1"]))
            continue
        cur = {"tag": tag, "t0": int(r["t0"]), "t1max": int(r["t1"]), "n": 1}
        open_[tag] = cur
        out.append(cur)
    return out


def name_of(tag: int) -> str:
    return NAMES.get(tag & 255, "?")


def exposed(ls: list[dict], key=lambda tag: name_of(tag)) -> dict[str, float]:
    """Critical-path time (ns) per key: end(launch) - max end of the launches before it."""
    out: dict[str, float] = collections.defaultdict(float)
    prev_end = None
    for launch in ls:
        if name_of(launch["tag"]) == "detok":  # second stream
            continue
        if prev_end is not None:
            out[key(launch["tag"])] += max(0, launch["t1max"] - prev_end)
        prev_end = max(prev_end or 0, launch["t1max"])
    return dict(out)
