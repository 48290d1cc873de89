"""Data-parallel serving: request-sharded full replicas, one process per GPU.

Routing follows the reference exactly (engine.py:110-116, 476-494): a router
rng ``PCG64(SeedSequence([seed, 3]))`` and ``route_dp`` per request in arrival
order, so every rank derives the same assignment locally (no communication).
Each rank serves its share with its own StreamingEngine; there is no
collective on the serving path.  At the end one gather (NCCL over NVLink on
GPUs, gloo in CPU tests) pools the per-request metrics so the merged report
equals ``core.build_report(merge_traces(...))`` (engine.py:447-457).
"""

from __future__ import annotations

from typing import Sequence

import numpy as np

from ._ref import core, ref_engine


def route(arrivals: Sequence, n_instances: int, seed: int) -> list[list[tuple[int, object]]]:
    """Split [(rid, spec)] into per-instance lists with the reference router."""
    router = np.random.Generator(np.random.PCG64(np.random.SeedSequence([seed & (2**64 - 1), 3])))
    out: list[list[tuple[int, object]]] = [[] for _ in range(n_instances)]
    for rid, spec in arrivals:
        out[ref_engine.route_dp(rid, n_instances, router)].append((rid, spec))
    return out


def local_summary(trace: core.Trace) -> dict:
    """Per-rank quantities whose pooled combination gives the merged report.

    Same values as ``core.ttfa_samples`` and the per-request ``_ontime_flags`` over
    ``trace.chunks_for`` (core.py:118-120, 200-223, 290-297), with the chunks grouped
    by request once: ``chunks_for`` scans every chunk per request, which at a 60 s
    load test (~5k requests x ~96 chunks) made the report take 75-90 s per run."""
    by_req: dict = {}
    for c in trace.chunks:
        by_req.setdefault(c.request, []).append(c)
    ttfa = []
    ontime = total = 0
    for req in trace.requests:
        ch = by_req.get(req.id)
        if ch:
            ch.sort(key=lambda c: c.index)  # stable, as chunks_for's sorted()
            ttfa.append(core.to_seconds(ch[0].available_us - req.arrival_us))
            flags = core._ontime_flags(ch)
            ontime += sum(flags)
            total += len(flags)
    return {
        "ttfa": ttfa,
        "ontime": ontime,
        "total": total,
        "audio_us": sum(c.playback_us for c in trace.chunks),
        "makespan_us": trace.makespan_us(),
        "completed": sum(1 for r in trace.requests if r.phase is core.Phase.FINISHED),
        "requests": len(trace.requests),
    }


def pool(summaries: Sequence[dict]) -> dict:
    """Combine rank summaries (viability pooled over chunks, nearest-rank percentiles)."""
    ttfa = [t for s in summaries for t in s["ttfa"]]
    ontime = sum(s["ontime"] for s in summaries)
    total = sum(s["total"] for s in summaries)
    makespan = max(s["makespan_us"] for s in summaries)
    audio = sum(s["audio_us"] for s in summaries)
    return {
        "ttfa_p50": core.percentile(ttfa, 50) if ttfa else float("nan"),
        "ttfa_p90": core.percentile(ttfa, 90) if ttfa else float("nan"),
        "ttfa_p99": core.percentile(ttfa, 99) if ttfa else float("nan"),
        "viability": ontime / total if total else 1.0,
        "audio_s": audio / 1e6,
        "inverse_rtf": audio / makespan if makespan else 0.0,
        "completed": sum(s["completed"] for s in summaries),
        "requests": sum(s["requests"] for s in summaries),
    }


def gather_pool(summary: dict, world_size: int) -> dict:
    """All-gather the rank summaries (the run's only collective) and pool them."""
    if world_size == 1:
        return pool([summary])
    import torch.distributed as dist

    objs: list = [None] * world_size
    dist.all_gather_object(objs, summary)
    return pool(objs)
