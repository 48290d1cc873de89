"""Timeline of CSM-style frames (backbone + 31 depth forwards per frame): GPU busy vs
idle on each ctx's LM stream (host-bound or device-bound?).  GPU only."""
import sys
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2602_00269_b200.config import csm_backbone, csm_depth  # noqa: E402
from paper_2602_00269_b200.csm import CsmFrames  # noqa: E402
from paper_2602_00269_b200.device import Sampling, VoxDevice  # noqa: E402

B = int(sys.argv[1]) if len(sys.argv) > 1 else 64
bb = VoxDevice(csm_backbone(max_slots=B + 4, max_ctx=128), 1)
dp = VoxDevice(csm_depth(max_slots=B + 4), 2)
pipe = CsmFrames(bb, dp)
g = Sampling(temperature=0.0, repetition_penalty=1.0)
streams = [pipe.admit(100 + i, 50, 32, g, g) for i in range(B)]
for a in range(0, B, 8):
    pipe.prefill(streams[a:a + 8])
for _ in range(2):
    pipe.step(streams)
bb.synchronize()
dp.synchronize()
bb.trace_arm()  # one tracer buffer per process-wide kernel set: arm via either ctx
t0 = time.perf_counter()
for _ in range(4):
    pipe.step(streams)
dp.synchronize()
bb.synchronize()
wall = (time.perf_counter() - t0) / 4
rec = bb.trace_read()
iv = sorted(zip(rec["t0"].astype(np.int64), rec["t1"].astype(np.int64)))
busy, cs, ce = 0, None, None
for a, b in iv:
    if cs is None or a > ce:
        if cs is not None:
            busy += ce - cs
        cs, ce = a, b
    else:
        ce = max(ce, b)
busy += ce - cs
span = iv[-1][1] - iv[0][0]
print(f"B={B}: wall {wall * 1e3:.2f} ms/frame; GPU span {span / 4e6:.2f} ms/frame, busy {busy / 4e6:.2f} ms/frame")
from paper_2602_00269_b200 import trace  # noqa: E402

ls = trace.launches(rec)
per = {}
for l in ls:
    k = trace.name_of(l["tag"]) + f"[{l['tag'] >> 8}]"
    n, t = per.get(k, (0, 0))
    per[k] = (n + 1, t + l["t1max"] - l["t0"])
print("per kernel (launch span), us/frame:")
for k, (n, t) in sorted(per.items(), key=lambda kv: -kv[1][1])[:20]:
    print(f"  {k:24s} {n / 4:7.1f} launches/frame {t / 4e3:9.1f} us/frame {t / n / 1e3:7.2f} us/launch")
ex = trace.exposed(ls)
print("exposed per kernel, us/frame:")
for k, v in sorted(ex.items(), key=lambda kv: -kv[1])[:12]:
    print(f"  {k:24s} {v / 4e3:9.1f}")
