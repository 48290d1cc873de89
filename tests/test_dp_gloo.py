"""CPU, world_size 2 (gloo): request routing and the end-of-run metric reduction.

The pooled report gathered across ranks must equal the reference's own
build_report over merge_traces(...) of the per-rank traces.
"""

import os
import socket

import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2602_00269_b200 import dp
from paper_2602_00269_b200._ref import core, ref_engine, workload


def _fake_trace(arrivals, rank):
    """Deterministic per-request chunk timelines (no GPU): synthetic but reference-typed."""
    tr = core.Trace()
    for rid, spec in arrivals:
        req = core.Request(id=rid, arrival_us=spec.arrival_us, prompt_tokens=spec.prompt_tokens,
                           target_output_tokens=spec.target_output_tokens, phase=core.Phase.FINISHED)
        t = spec.arrival_us + 150_000 + 1_000 * (rid % 7)
        for i in range(1, 6):
            pb = 81_395
            late = 5_000 if (rid % 5 == 0 and i == 3) else 0
            tr.chunks.append(core.ChunkEvent(request=rid, index=i, available_us=t + late, playback_us=pb, new_tokens=7))
            t += pb - 1_000
        tr.requests.append(req)
    return tr


def _worker(rank, ws, port, out):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(ws))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    spec = workload.WorkloadSpec(rate=20.0, duration_s=3.0, seed=5)
    arr = list(enumerate(workload.build_workload(spec)))
    mine = dp.route(arr, ws, seed=5)[rank]
    pooled = dp.gather_pool(dp.local_summary(_fake_trace(mine, rank)), ws)
    if rank == 0:
        out.put(pooled)
    dist.destroy_process_group()


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_route_matches_reference_run_scenario_split():
    spec = workload.WorkloadSpec(rate=30.0, duration_s=4.0, seed=11)
    arr = list(enumerate(workload.build_workload(spec)))
    parts = dp.route(arr, 4, seed=11)
    # the reference's own split (engine.py:476-482)
    import numpy as np

    router = np.random.Generator(np.random.PCG64(np.random.SeedSequence([11, 3])))
    ref = [[] for _ in range(4)]
    for rid, s in arr:
        ref[ref_engine.route_dp(rid, 4, router)].append(rid)
    assert [[rid for rid, _ in p] for p in parts] == ref
    assert sorted(r for p in parts for r, _ in p) == [r for r, _ in arr]


def test_gloo_world2_pool_equals_reference_merge():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    pooled = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    spec = workload.WorkloadSpec(rate=20.0, duration_s=3.0, seed=5)
    arr = list(enumerate(workload.build_workload(spec)))
    parts = dp.route(arr, 2, seed=5)
    merged = ref_engine.merge_traces([_fake_trace(parts[r], r) for r in range(2)])
    rep = core.build_report(merged)
    assert pooled["ttfa_p90"] == rep.ttfa_p90 and pooled["ttfa_p50"] == rep.ttfa_p50
    assert pooled["viability"] == pytest.approx(rep.viability_fraction)
    assert pooled["completed"] == rep.requests_completed
    assert pooled["audio_s"] == pytest.approx(rep.audio_seconds_generated)
