"""dp.local_summary (chunks grouped by request once) equals the reference's own
per-request functions over Trace.chunks_for (core.py:118-120, 200-223, 290-297) on
a random trace: chunks appended out of order, requests without chunks, ties."""

import numpy as np

from paper_2602_00269_b200 import dp
from paper_2602_00269_b200._ref import core


def test_local_summary_matches_reference():
    rng = np.random.default_rng(7)
    tr = core.Trace()
    for rid in range(60):
        tr.requests.append(core.Request(id=rid, arrival_us=int(rng.integers(0, 10**6)), prompt_tokens=10,
                                        target_output_tokens=100, phase=core.Phase.FINISHED))
        if rid % 7 == 3:
            continue  # no chunk delivered
        n = int(rng.integers(1, 12))
        t = tr.requests[-1].arrival_us + int(rng.integers(1000, 900000))
        for i in range(1, n + 1):
            t += int(rng.integers(0, 400000))
            tr.chunks.append(core.ChunkEvent(request=rid, index=i, available_us=t,
                                             playback_us=int(rng.choice([83333, 291666])), new_tokens=7))
    rng.shuffle(tr.chunks)
    got = dp.local_summary(tr)
    ref_ttfa = core.ttfa_samples(tr)
    ontime = total = 0
    for req in tr.requests:
        ch = tr.chunks_for(req.id)
        if ch:
            f = core._ontime_flags(ch)
            ontime += sum(f)
            total += len(f)
    assert got["ttfa"] == ref_ttfa
    assert (got["ontime"], got["total"]) == (ontime, total)
