"""Timeline of K6 layer-chain launches (vox_trace event marks): for one steady
decode step, per job of the middle layers: when its inputs were ready at the
producers, when its MMAs ran and when its epilogue / rows finished, relative to
the launch's first CTA entry (us; min / median / max over CTAs).  GPU only.

  python scripts/trace_chain.py --batch 224 --ctx 394
"""
import argparse
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
from paper_2602_00269_b200.config import CONFIGS  # noqa: E402
from paper_2602_00269_b200.device import Sampling, VoxDevice  # noqa: E402

JOBS = ["O", "norm1", "gate|up", "down", "norm2", "qkv", "rope"]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--batch", type=int, default=224)
    ap.add_argument("--ctx", type=int, default=394)
    ap.add_argument("--config", default="orpheus3b")
    ap.add_argument("--layers", default="5,14")
    a = ap.parse_args()
    dev = VoxDevice(CONFIGS[a.config](max_slots=max(a.batch, 8)), 0)
    prm = Sampling(temperature=0.6, top_p=0.8, repetition_penalty=1.3)
    P = 50
    slots = [dev.admit(1000 + i, P, 688, prm) for i in range(a.batch)]
    per = max(1, 1000 // (a.ctx - 1))
    for i in range(0, a.batch, per):
        rows = np.array([[s, p, -1, 0] for s in slots[i:i + per] for p in range(a.ctx - 1)], np.int32)
        dev.forward(rows, sample=False)
    for w in range(8):
        dev.forward(np.array([[s, a.ctx - 8 + w, -1, 1] for s in slots], np.int32))
    dev.synchronize()
    dev.trace_arm()
    dev.forward(np.array([[s, a.ctx, -1, 1] for s in slots], np.int32))
    dev.synchronize()
    rec = dev.trace_read()
    tag = rec["tag"] & 255
    cta = rec["tag"] >> 8
    ent = rec[tag == 11]
    ent = np.sort(ent, order="t0")
    # launches: clusters of chain CTA entries
    starts = ent["t0"].astype(np.int64)
    cut = np.where(np.diff(starts) > 3000)[0]
    bounds = [starts[0]] + [starts[c + 1] for c in cut]
    ends = []
    for i, b0 in enumerate(bounds):
        b1 = bounds[i + 1] if i + 1 < len(bounds) else 1 << 62
        m = (starts >= b0) & (starts < b1)
        ends.append(int(ent["t1"][m].max()))
    print(f"{len(bounds)} chain launches; span per launch (us):",
          [round((e - b) / 1e3, 1) for b, e in zip(bounds, ends)][:30])
    ev = rec[(tag >= 32) & (tag < 56)]
    wts = rec[tag >= 56]
    for li in [int(x) for x in a.layers.split(",")]:
        L0 = li + 1  # launch 0 is layer 0's q|k|v chain
        if L0 >= len(bounds):
            continue
        b0, b1 = bounds[L0], ends[L0]
        m = (ev["t0"].astype(np.int64) >= b0 - 1000) & (ev["t1"].astype(np.int64) <= b1 + 1000)
        e = ev[m]
        mw = (wts["t0"].astype(np.int64) >= b0 - 1000) & (wts["t0"].astype(np.int64) <= b1 + 1000)
        wl = wts[mw]
        wlt = wl["tag"] & 255
        et = e["tag"] & 255
        print(f"\nlayer {li}: span {(b1 - b0) / 1e3:.1f} us")
        print(f"{'job':8s} {'dep ready (min/med/max)':>26s} {'mma start min':>14s} {'mma end max':>12s} "
              f"{'epi start min':>14s} {'epi end max':>12s} {'units':>6s} {'mma us/unit':>12s}")
        for j, name in enumerate(JOBS):
            def sel(k):
                return e[et == k + j]
            dp, mm, ep = sel(32), sel(40), sel(48)
            f = lambda x: (x.astype(np.int64) - b0) / 1e3  # noqa: E731
            dps = f(dp["t1"]) if len(dp) else np.array([np.nan])
            s = (f"{name:8s} {np.nanmin(dps):8.1f}/{np.nanmedian(dps):7.1f}/{np.nanmax(dps):7.1f}   "
                 f"{(f(mm['t0']).min() if len(mm) else np.nan):14.1f} {(f(mm['t1']).max() if len(mm) else np.nan):12.1f} "
                 f"{(f(ep['t0']).min() if len(ep) else np.nan):14.1f} {(f(ep['t1']).max() if len(ep) else np.nan):12.1f} "
                 f"{len(mm) if len(mm) else len(ep):6d} "
                 f"{(np.median((mm['t1'].astype(np.int64) - mm['t0'].astype(np.int64)) / 1e3) if len(mm) else np.nan):12.2f}")
            print(s)
            wt = wl[wlt == 56 + j]
            if len(wt):
                packed = wt["t1"].astype(np.uint64)
                ww = (packed >> np.uint64(32)).astype(np.int64) / 1e3
                wx = (packed & np.uint64(0xFFFFFFFF)).astype(np.int64) / 1e3
                print(f"{'':8s}   MMA stalls per unit (us, median/max): waiting W {np.median(ww):.2f}/{ww.max():.2f}"
                      f"  waiting X {np.median(wx):.2f}/{wx.max():.2f}")
            if len(ep):
                st, en = f(ep["t0"]), f(ep["t1"])
                pct = lambda x: "/".join(f"{v:.1f}" for v in np.percentile(x, [10, 50, 90, 100]))  # noqa: E731
                print(f"{'':8s}   epi start p10/50/90/max {pct(st)}   end {pct(en)}   "
                      f"dur med {np.median(en - st):.1f} max {np.max(en - st):.1f}")


if __name__ == "__main__":
    main()
