#!/usr/bin/env python
"""Benchmark: Orpheus-3B-style streaming TTS serving on B200 (BASELINE.json config 2).

Headline metric (BASELINE.json): req/s at >=99% streaming viability and p90
TTFA <= 500 ms; audio-seconds per second per B200.

* A "step" is one serving iteration of the StreamingEngine in steady state
  over B concurrent streams (default B=256): the reference streaming-aware
  scheduler's decision (scheduler.py:119-175) executed as one fused decode
  step for the LM batch (tcgen05 GEMMs + paged attention + K1 sampler, CUDA
  graph) plus the detokenization of that iteration's ready chunks (causal
  SNAC-style decoder with cached left context) on the overlapped detok stream.
* value = audio seconds represented by the tokens decoded in the timed
  region / device time (CUDA events on both streams, max over ranks).
* e2e  = the same metric on the host wall clock of the same steps, which
  include every step's H2D row upload from pinned memory and the D2H of the
  sampled ids and of the emitted PCM.
* slo  = the paper's serving metric from a short Poisson load test through
  the same engine: the highest offered rate whose pooled viability >= 0.99
  and p90 TTFA <= 0.5 s (reference core.py metrics, unchanged).
* --impl reference: the reference CPU path timed on this host (the oracle
  port of the same arithmetic, numpy/BLAS on all cores; bounded sample).
"""

from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))
if (ROOT / "baseline" / "_ref").exists():
    sys.path.insert(0, str(ROOT / "baseline" / "_ref"))

import numpy as np  # noqa: E402

METRIC = "req/s at >=99% streaming viability & p90 TTFA; audio-sec/sec per B200"
UNIT = "audio-s/s"


def _peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return d.get("hbm_gbs", 6650.0), d.get("bf16_tflops_sustained", 1400.0), "measured"
    return 6650.0, 1590.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    def __init__(self, index: int = 0):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._th = None

    def __enter__(self):
        def loop():
            q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
                 "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
            while not self._stop.is_set():
                try:
                    out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                         timeout=5).stdout.strip()
                    if out:
                        self.rows.append([x.strip() for x in out.split(",")])
                except Exception:
                    pass
                self._stop.wait(0.2)

        self._th = threading.Thread(target=loop, daemon=True)
        self._th.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        if self._th:
            self._th.join(timeout=6)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 2 + i and "Active" in r[2 + i]
                          and "Not" not in r[2 + i]})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


# ---------------------------------------------------------------------------- distributed
def dist_setup(backend: str):
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1:
        import torch.distributed as dist

        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        if backend == "nccl":
            import torch

            n_dev = max(torch.cuda.device_count(), 1)
            if n_dev < ws:
                # more ranks than GPUs (functional testing of the multi-rank path on one
                # device): NCCL refuses duplicate devices, so reduce metrics over gloo
                backend = "gloo"
            local = local % n_dev
            torch.cuda.set_device(local)
        dist.init_process_group(backend=backend)
        global _DIST_DEVICE
        _DIST_DEVICE = None if backend == "gloo" else "cuda"
    return ws, rank, local


_DIST_DEVICE = "cuda"


def reduce_max(x: float, ws: int, device=None) -> float:
    if ws == 1:
        return x
    import torch
    import torch.distributed as dist

    t = torch.tensor([x], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def reduce_sum(xs, ws: int, device=None):
    if ws == 1:
        return list(xs)
    import torch
    import torch.distributed as dist

    t = torch.tensor(list(xs), dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return [float(v) for v in t.tolist()]


# ---------------------------------------------------------------------------- our arm
def steady_state_steps(dev, B: int, steps: int, warmup: int, prompt: int, seed: int):
    """Closed-loop serving of B concurrent 688-token streams, timed in steady state.

    Streams are admitted at a uniform rate over one stream lifetime (688 tokens at
    8 iterations per 7 tokens: a stream selected for detok sits out that LM batch,
    scheduler.py:152-156), then every finished stream is replaced at once, so the
    streams' ages -- and contexts -- are spread uniformly over the lifetime (mean
    context ~ prompt + 344) and every timed iteration carries
    the prefills of newly admitted streams as well as decode rows and detok windows."""
    import torch

    from paper_2602_00269_b200._ref import scheduler, workload
    from paper_2602_00269_b200.engine import StreamingEngine, orpheus_profile

    prof = orpheus_profile(max_batch=B)
    policy = scheduler.PolicyConfig(max_lm_batch=B, max_detok_batch=B, startup_concurrency_limit=B,
                                    max_live_requests=4 * B)
    eng = StreamingEngine(dev, prof, policy, seed)
    target = 688
    rid = 0
    dev.clock_reset()
    eng._t0 = time.perf_counter()

    def admit_one():
        nonlocal rid
        eng.admit(rid, workload.ArrivalSpec(arrival_us=eng.now_us(), prompt_tokens=prompt,
                                            target_output_tokens=target))
        rid += 1

    def one_iter(refill: bool):
        if refill:
            while len(eng.live) < B:
                admit_one()
        snap = eng._snapshot()
        dec = scheduler.schedule(snap, eng.now_us(), policy)
        if not dec.empty:
            eng.run_iteration(dec)
        eng._poll()

    ramp = (target * 8) // 7 + 8  # iterations of one stream lifetime
    for it in range(ramp):
        while rid < ((it + 1) * B) // ramp:
            admit_one()
        one_iter(False)
    for _ in range(warmup):
        one_iter(True)
    dev.synchronize()
    lm_s, dt_s = dev.streams()
    s_lm = torch.cuda.ExternalStream(lm_s)
    s_dt = torch.cuda.ExternalStream(dt_s)
    ev0 = torch.cuda.Event(enable_timing=True)
    ev_lm = torch.cuda.Event(enable_timing=True)
    ev_dt = torch.cuda.Event(enable_timing=True)
    st0 = eng.stats
    dec0, chunks0, pcm0 = st0.decode_rows, len(eng.trace.chunks), st0.pcm_samples
    ctx0, pre0 = st0.decode_ctx, st0.prefill_rows
    rows0, dcalls0, wait0 = st0.lm_rows, st0.detok_calls, st0.wait_s
    launches0 = dev.launch_count()
    import gc

    gc.collect()  # before the first event: a full collection takes tens of ms
    gc.freeze()
    gc.disable()  # as StreamingEngine.run: no cyclic-GC stalls of the host loop while timed
    ev0.record(s_lm)
    s_dt.wait_event(ev0)
    t0 = time.perf_counter()
    trace_from = 0 if (os.environ.get("VOX_BENCH_TRACE") and steps >= 8) else steps + 1
    it_ms = []
    for i_step in range(steps):
        if i_step == trace_from:
            dev.trace_arm(1 << 23)
        t_it = time.perf_counter()
        one_iter(True)
        it_ms.append((time.perf_counter() - t_it) * 1e3)
        if i_step == 0:
            ev1 = torch.cuda.Event(enable_timing=True)
            ev1.record(s_lm)
    ev_lm.record(s_lm)
    ev_dt.record(s_dt)
    torch.cuda.synchronize()
    if os.environ.get("VOX_BENCH_TRACE"):
        a = np.array(it_ms)
        print(f"ev0->ev1 (first iteration) {ev0.elapsed_time(ev1):.2f} ms; host iteration ms: first {a[0]:.2f} "
              f"median {np.median(a):.2f} max {a.max():.2f} top5 {np.sort(a)[-5:].round(2).tolist()} "
              f"sum {a.sum():.1f}", file=sys.stderr)
    while eng._tickets:
        eng._poll(block=True)
    t_wall = time.perf_counter() - t0
    gc.unfreeze()
    gc.enable()
    dev_ms = max(ev0.elapsed_time(ev_lm), ev0.elapsed_time(ev_dt))
    if trace_from < steps:
        _trace_summary(dev.trace_read(1 << 23))
    st = eng.stats
    decoded = st.decode_rows - dec0
    chunks = len(eng.trace.chunks) - chunks0
    pcm = st.pcm_samples - pcm0
    rows = st.lm_rows - rows0
    out = dict(decoded=decoded, chunks=chunks, pcm_samples=pcm, dev_ms=dev_ms, wall_s=t_wall,
               mean_ctx=(st.decode_ctx - ctx0) / max(decoded, 1), prefill_rows=st.prefill_rows - pre0,
               launches=dev.launch_count() - launches0, rows=rows, detok_calls=st.detok_calls - dcalls0,
               token_rate=prof.token_rate, live=len(eng.live), wait_s=st.wait_s - wait0)
    # pure device time of one graph-captured LM step at this batch (no host in the loop)
    live = list(eng.live.values())[: max(1, args_batch_decode(B))]
    rows_np = np.asarray([[r.slot, r.req.prompt_tokens - 1 + r.req.tokens_generated - 1, -1, 1] for r in live],
                         np.int32)
    for _ in range(3):
        dev.forward(rows_np)
    ea = torch.cuda.Event(enable_timing=True)
    eb = torch.cuda.Event(enable_timing=True)
    ea.record(s_lm)
    for _ in range(10):
        dev.forward(rows_np)
    eb.record(s_lm)
    torch.cuda.synchronize()
    out["lm_graph_step_ms"] = ea.elapsed_time(eb) / 10
    out["lm_graph_rows"] = len(live)
    eng.shutdown()
    return out


def _trace_summary(rec):
    """Diagnostics (VOX_BENCH_TRACE=1): LM vs detok kernel activity over the traced steps."""
    rec = np.sort(rec, order="t0")
    t0 = int(rec["t0"].min())
    det = rec[(rec["tag"] & 255) == 10]
    lm = rec[(rec["tag"] & 255) != 10]
    span = (int(rec["t1"].max()) - t0) / 1e3

    def busy(r):  # union of CTA intervals
        iv = sorted(zip(r["t0"].astype(np.int64), r["t1"].astype(np.int64)))
        tot, cs, ce = 0, None, None
        for a, b in iv:
            if cs is None or a > ce:
                if cs is not None:
                    tot += ce - cs
                cs, ce = a, b
            else:
                ce = max(ce, b)
        return (tot + (ce - cs if cs is not None else 0)) / 1e3

    print(f"trace: span {span:.1f} us; LM busy {busy(lm):.1f} us; detok busy {busy(det):.1f} us; "
          f"detok CTAs {len(det)}, first {(int(det['t0'].min()) - t0) / 1e3 if len(det) else -1:.1f} us, "
          f"last end {(int(det['t1'].max()) - t0) / 1e3 if len(det) else -1:.1f} us; "
          f"LM last end {(int(lm['t1'].max()) - t0) / 1e3:.1f} us", file=sys.stderr)
    # per-step detok windows relative to the LM step boundaries (sampler CTAs end a step)
    # LM-stream idle gaps (no LM CTA running): host not keeping up
    iv = sorted(zip(lm["t0"].astype(np.int64), lm["t1"].astype(np.int64)))
    gaps, ce = [], iv[0][1]
    for a, b in iv[1:]:
        if a > ce:
            gaps.append(a - ce)
        ce = max(ce, b)
    gaps = np.array(gaps) / 1e3
    print(f"trace: LM idle gaps: n={len(gaps)} total {gaps.sum():.1f} us, >50us: {int((gaps > 50).sum())}, "
          f"largest {np.sort(gaps)[-5:].round(1).tolist() if len(gaps) else []}", file=sys.stderr)
    samp = np.sort(lm[(lm["tag"] & 255) == 9]["t1"].astype(np.int64))
    print("trace: sampler ends (us):", [round((int(x) - t0) / 1e3, 1) for x in samp[:: max(1, len(samp) // 8)]],
          file=sys.stderr)
    if len(det):
        dd = np.sort(det["t0"].astype(np.int64))
        gaps = np.where(np.diff(dd) > 100000)[0]
        starts = [dd[0]] + [dd[g + 1] for g in gaps]
        print("trace: detok burst starts (us):", [round((int(x) - t0) / 1e3, 1) for x in starts], file=sys.stderr)


def args_batch_decode(B: int) -> int:
    """Decode rows of a steady-state iteration: 7 of every 8 streams (1 in 8 is detokenizing)."""
    return B - B // 8


def kernel_roofline(dev, B: int, prompt: int, seed: int, hbm: float, tflops: float):
    """Per-kernel-class CUDA-event timing of eager decode steps at batch B (timing mode)."""
    from paper_2602_00269_b200.device import Sampling

    cfg = dev.cfg
    ctx = prompt + 344  # mid-stream context (average over a 688-token request)
    slots = []
    for i in range(B):
        slots.append(dev.admit(seed + i, prompt, 688, Sampling(temperature=0.6, top_p=0.8, repetition_penalty=1.3)))
    # fill KV for `ctx` positions with one big prefill-like pass per slot group
    for a in range(0, B, 2):
        rows = np.array([[s, p, -1, 0] for s in slots[a:a + 2] for p in range(ctx - 1)], np.int32)
        dev.forward(rows, sample=False)
    dev.synchronize()
    # the decode rows of one serving iteration at B streams (1 in 8 is detokenizing)
    rows = np.array([[s, ctx - 1, -1, 1] for s in slots[:args_batch_decode(B)]], np.int32)
    dev.forward(rows, graph=False)  # warm
    dev.synchronize()
    dev.timing(True)
    n = 3
    for _ in range(n):
        dev.forward(rows, graph=False)
    dev.synchronize()
    classes = {}
    for cls in ("gemm", "attn", "qkv_rope", "norm", "silu", "lm_head", "sampler"):
        ms, cnt, by = dev.timing_read(cls)
        classes[cls] = dict(ms=ms / n, launches=cnt // n, bytes=by / n)
    dev.timing(False)
    in_graph = traced_classes(dev, rows, classes)
    sweep = batch_sweep(dev, slots, ctx, hbm, tflops)
    for s in slots:
        dev.release(s)
    step_ms = sum(v["ms"] for v in classes.values())
    return classes, step_ms, ctx, sweep, in_graph, len(rows)


def traced_classes(dev, rows, classes, steps: int = 4):
    """Diagnostic: per-class time on the LM critical path INSIDE the graph-captured step
    (vox_trace per-CTA spans; a class's exposed time = end - previous end, so work that
    PDL overlaps with its predecessor is not counted).  This is a share of the step,
    NOT a kernel roofline (the roofline uses whole launch durations)."""
    from paper_2602_00269_b200 import trace

    for _ in range(8):  # graphs for every head frame slot (rows share one position)
        dev.forward(rows)
    dev.synchronize()
    dev.trace_arm()
    for _ in range(steps):
        dev.forward(rows)
    dev.synchronize()
    rec = dev.trace_read()
    ls = trace.launches(rec)
    ex = trace.exposed(ls, key=lambda tag: trace.CLASS.get(trace.name_of(tag), "?"))
    span = (max(l["t1max"] for l in ls) - min(l["t0"] for l in ls)) / 1e6 / steps
    out = {"step_ms": round(span, 4), "classes": {}}
    for cls, ns in sorted(ex.items(), key=lambda kv: -kv[1]):
        out["classes"][cls] = {"exposed_ms_per_step": round(ns / 1e6 / steps, 4)}
    return out


def batch_sweep(dev, slots, ctx: int, hbm: float, tflops: float):
    """Config 2 batch sweep: graph-captured decode step (head + sampler
    included) over the first b of the filled slots at context ctx, CUDA events on the LM
    stream; HBM roofline bytes = serving weights + b * ctx * KV bytes per token."""
    import torch

    cfg = dev.cfg
    d, hd = cfg.d_model, cfg.head_dim
    proj = 2 * cfg.n_layers * ((cfg.n_heads + 2 * cfg.n_kv_heads) * hd * d + d * cfg.n_heads * hd + 3 * d * cfg.d_ff)
    # every row sits at the same frame position, so the LM head reads one frame slot's
    # codebook (vox_forward's one-slot rule), not all frame_tokens x codebook_size rows
    head = 2 * cfg.codebook_size * d
    flops_tok = proj + head  # 2 FLOP per bf16 weight (2 bytes) per row
    lm_s, _ = dev.streams()
    st = torch.cuda.ExternalStream(lm_s)
    out = []
    for b in [1, 2, 4, 8, 16, 32, 64, 128, 192, 224, 256]:
        if b > len(slots):
            break
        rows = np.array([[s, ctx - 1, -1, 1] for s in slots[:b]], np.int32)
        for _ in range(2):
            dev.forward(rows)
        ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ea.record(st)
        for _ in range(10):
            dev.forward(rows)
        eb.record(st)
        torch.cuda.synchronize()
        ms = ea.elapsed_time(eb) / 10
        by = proj + head + b * ctx * cfg.kv_bytes_per_token
        out.append({"batch": b, "ms_per_step": round(ms, 4), "tokens_per_s": round(b / ms * 1e3, 1),
                    "audio_s_per_s": round(b / ms * 1e3 / 86.0, 1), "hbm_gbs": round(by / ms / 1e6, 1),
                    "hbm_frac": round(by / ms / 1e6 / hbm, 4),
                    "tflops": round(flops_tok * b / ms / 1e9, 1)})
    return out


def step_work(cfg, rows: int, ctx_sum: float, head_slots: int | None = None):
    """Algorithmic work of one decode step per kernel class: what the
    math must move / compute, independent of how the kernels split it (no split-K
    partial planes, no re-reads).  head_slots = distinct frame slots among the sampled
    rows (the LM head reads head_slots x codebook_size weight rows; default: all
    frame_tokens).  Returns {class: (flops, bytes)} for the whole step."""
    d, H, KV, hd, dff, L = cfg.d_model, cfg.n_heads, cfg.n_kv_heads, cfg.head_dim, cfg.d_ff, cfg.n_layers
    nqkv, Hhd, R = (H + 2 * KV) * hd, H * hd, rows
    w_layer = nqkv * d + d * Hhd + 2 * dff * d + d * dff
    A = (cfg.frame_tokens if head_slots is None else head_slots) * cfg.codebook_size
    return {
        # 4 projections per layer: bf16 weights + bf16 inputs + outputs (fp32 q|k|v, O and
        # down results; bf16 SiLU(gate)*up from the fused epilogue)
        "gemm": (2.0 * R * L * w_layer,
                 2.0 * L * w_layer + L * R * 2.0 * (d + Hhd + d + dff) + L * R * (4.0 * nqkv + 4.0 * d + 2.0 * dff
                                                                                + 4.0 * d)),
        # paged K/V of every row's context (bf16) + q in, output out
        "attn": (4.0 * ctx_sum * L * H * hd, 4.0 * ctx_sum * L * KV * hd + 4.0 * L * R * Hhd),
        # q|k|v fp32 in, RoPE'd q out, K/V appended (bf16)
        "qkv_rope": (0.0, L * R * (4.0 * nqkv + 2.0 * Hhd + 4.0 * KV * hd)),
        # embed + 2L residual+RMSNorm: h and the delta in (fp32), h out (fp32), x out (bf16)
        "norm": (0.0, R * d * (2.0 + 4.0 + 2.0) + 2 * L * R * d * 14.0),
        "silu": (0.0, 0.0),
        "lm_head": (2.0 * R * A * d, 2.0 * A * d + 2.0 * R * d + 4.0 * R * A),
        "sampler": (0.0, 4.0 * R * cfg.codebook_size),
    }


def roofline_summary(cfg, classes, rows: int, ctx: int, hbm: float, tfl: float, peak_kind: str):
    """Roofline of every kernel class of an eager decode step at `rows` rows, context `ctx`.

    achieved = the class's ALGORITHMIC work per step (step_work) / its CUDA-event time per
    step (events on the LM stream around each launch, eager timing mode) -- i.e. work per
    launch / mean launch duration.  The bound is the larger of work/peak over the tensor
    and HBM roofs (arithmetic intensity vs the ridge peak_tflops / peak_hbm).  The
    dominant class (largest time) is the headline.  traffic = ncu dram bytes per launch
    of that class (profiles/traffic_r02.json), or null."""
    work = step_work(cfg, rows, float(rows) * ctx, head_slots=1)  # the eager rows share one position
    out = {}
    for name, c in classes.items():
        if c["launches"] <= 0 or c["ms"] <= 0 or name not in work:
            continue
        flops, by = work[name]
        sec = c["ms"] / 1e3
        t_tc, t_hbm = flops / (tfl * 1e12), by / (hbm * 1e9)
        e = {"ms_per_step": round(c["ms"], 4), "launches_per_step": c["launches"],
             "flops_per_step": flops, "bytes_per_step": by,
             "intensity_flop_per_byte": round(flops / by, 1) if by else None}
        if t_tc > t_hbm:
            e.update(bound="tensor", achieved=round(flops / sec / 1e12, 1), peak=tfl, unit="TFLOP/s")
        else:
            e.update(bound="hbm", achieved=round(by / sec / 1e9, 1), peak=hbm, unit="GB/s")
        e["frac"] = round(e["achieved"] / e["peak"], 4)
        out[name] = e
    top = max(out, key=lambda k: out[k]["ms_per_step"])
    t = out[top]
    traffic = None
    prof_path = ROOT / "profiles" / "traffic_r02.json"
    if prof_path.exists():
        traffic = json.loads(prof_path.read_text()).get(top)
    return {"bound": t["bound"], "kernel": top, "achieved": t["achieved"], "peak": t["peak"], "unit": t["unit"],
            "frac": t["frac"], "traffic": traffic, "peak_kind": peak_kind,
            "work": "algorithmic per step / CUDA-event time per step (= per launch / mean launch duration); "
                    "gemm flops = 2 x rows x projection weights, bytes exclude split-K partial planes",
            "classes": out, "ctx": ctx, "rows": rows}


def detok_mac_per_latent_frame(cfg) -> int:
    """Multiply-accumulates of the causal SNAC-style decoder per latent frame (hop = 512
    output samples): input dw k7 + 1x1 latent->D0; per block b the ConvT(k=2s, stride s)
    as the GEMM [x_t | x_{t-1}] . W[(s Co), 2 Ci] at the block's input rate, then 3
    residual units (dw k7 + 1x1 Co->Co) at its output rate; output k7 conv to 1 channel."""
    L, D0 = cfg.latent_dim, cfg.decoder_dim
    ch = [D0]
    for _ in range(4):
        ch.append(ch[-1] // 2)
    mac, pos = 7 * L + L * D0, 1
    for b in range(4):
        Ci, Co, st = ch[b], ch[b + 1], cfg.rates[b]
        mac += pos * 2 * Ci * st * Co
        pos *= st
        mac += 3 * pos * (Co * Co + 7 * Co)
    return mac + pos * 7 * ch[4]


def detok_roofline(dev, tfl: float, hbm: float, n_win: int = 32, calls: int = 12):
    """K4 alone: steady-state detok calls of n_win 7-token windows (one frame = 4 latent
    frames = 2048 samples each, cached left context), as one serving iteration at 256
    streams issues.  CUDA events on the detok stream around each call (graph-captured).
    Work = 2 x MAC per latent frame (detok_mac_per_latent_frame) x latent frames."""
    import torch

    from paper_2602_00269_b200.device import Sampling

    cfg = dev.cfg
    rng = np.random.default_rng(5)
    slots = []
    for i in range(n_win):
        sl = dev.admit(777000 + i, 50, 688, Sampling(temperature=0.0))
        ids = [cfg.audio_base + (k % 7) * cfg.codebook_size + int(rng.integers(cfg.codebook_size))
               for k in range(28 + 7 * calls)]
        dev.write_tokens(sl, 50, ids)
        slots.append(sl)
    dev.detok(np.array([[sl, 1, 0, 28, 28, 0] for sl in slots], np.int32), sync=True)  # first windows
    _, dt_s = dev.streams()
    st = torch.cuda.ExternalStream(dt_s)
    times = []
    for c in range(calls):
        w = np.array([[sl, 2 + c, 7 * (c + 1), 28, 7, 0] for sl in slots], np.int32)
        ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ea.record(st)
        dev.detok(w, sync=False)
        eb.record(st)
        torch.cuda.synchronize()
        times.append(ea.elapsed_time(eb))
    for sl in slots:
        dev.release(sl)
    ms = float(np.median(times[2:]))  # the first calls capture the bucket's graph
    mac = detok_mac_per_latent_frame(cfg)
    flops = 2.0 * mac * 4 * n_win
    # the detok stream runs on its own SM partition (green context) when the context
    # split the GPU: its roofline is that partition's share of the tensor peak
    lm_sms, dt_sms = dev.sm_partition()
    sms = dt_sms if dt_sms > 0 else lm_sms
    peak = tfl * sms / 148.0
    return {"bound": "tensor", "windows_per_call": n_win, "latent_frames_per_call": 4 * n_win,
            "mac_per_latent_frame": mac, "gflop_per_call": round(flops / 1e9, 3), "ms_per_call": round(ms, 4),
            "sms": sms, "achieved": round(flops / (ms / 1e3) / 1e12, 2), "peak": round(peak, 1),
            "peak_full_gpu": tfl, "unit": "TFLOP/s", "frac": round(flops / (ms / 1e3) / 1e12 / peak, 4),
            "audio_s_per_s": round(n_win * 2048 / 24000 / (ms / 1e3), 1)}


DRAIN_S = 20.0  # seconds after the last arrival for a load-test run to finish every request


def slo_run(dev, rate: float, seconds: float, seed: int, prompt: int, ws: int, rank: int, max_batch: int,
            startup_limit: int):
    """One Poisson load test (config 5) at the WHOLE-JOB offered rate: reference workload
    (workload.py:116-156, 688-token outputs), requests routed to the ws replicas with the
    reference router, metrics pooled over ranks (core.py:300-333 definitions)."""
    from paper_2602_00269_b200 import dp
    from paper_2602_00269_b200._ref import scheduler, workload
    from paper_2602_00269_b200.engine import StreamingEngine, orpheus_profile

    prof = orpheus_profile(max_batch=max_batch)
    spec = workload.WorkloadSpec(rate=rate, duration_s=seconds, prompt_dist=workload.fixed(prompt),
                                 output_dist=workload.fixed(688), seed=seed)
    arr = list(enumerate(workload.build_workload(spec)))
    mine = dp.route(arr, ws, seed)[rank]
    policy = scheduler.PolicyConfig(max_lm_batch=max_batch, max_detok_batch=max_batch,
                                    startup_concurrency_limit=startup_limit)
    t_run = time.perf_counter()
    eng = StreamingEngine(dev, prof, policy, seed)
    # A run whose backlog has not drained DRAIN_S after the last arrival is over
    # capacity: it stops there and fails (an overloaded 60 s run otherwise spends
    # minutes draining its queue -- the bench's wall time, not its result).
    tr = eng.run(mine, max_wall_s=seconds + DRAIN_S)
    eng.shutdown()  # releases the slots of requests cut off by the wall limit
    t_served = time.perf_counter()
    rep = dp.gather_pool(dp.local_summary(tr), ws)
    drained = rep["completed"] >= len(arr)
    ok = drained and rep["viability"] >= 0.99 and rep["ttfa_p90"] <= 0.5
    t_end = time.perf_counter()
    return ok, dict(rate=rate, seconds=seconds, requests=len(arr), drained=drained,
                    wall_s=round(t_end - t_run, 1), report_s=round(t_end - t_served, 1), ttfa_p50=rep["ttfa_p50"],
                    ttfa_p90=rep["ttfa_p90"], ttfa_p99=rep["ttfa_p99"], viability=rep["viability"],
                    inverse_rtf=rep["inverse_rtf"], audio_s=rep["audio_s"], completed=rep["completed"], ok=ok)


def run_slo(dev, start: float, seconds: float, probe_seconds: float, seed: int, prompt: int, ws: int = 1,
            rank: int = 0, max_batch: int = 256, startup_limit: int = 16, coarse: float = 8.0,
            fine: float = 2.0, max_full: int = 5):
    """Paper protocol (Poisson arrivals, 60 s runs, p90 TTFA, pooled
    viability): the highest offered rate, on a `fine`-req/s grid, whose full-length run
    keeps viability >= 0.99 and p90 TTFA <= 0.5 s.  Short probes (probe_seconds, `coarse`
    steps) bracket it first; only full-length runs decide the result."""
    sweep = []
    tested = {}  # full-length results by rate (a rate is run at most once)

    def full(rate):
        if rate not in tested:
            ok_, row_ = slo_run(dev, rate, seconds, seed, prompt, ws, rank, max_batch, startup_limit)
            sweep.append(row_)
            tested[rate] = ok_
        return tested[rate]

    r, last_ok = start, None
    while True:  # coarse bracket (short probes)
        ok, row = slo_run(dev, r, probe_seconds, seed, prompt, ws, rank, max_batch, startup_limit)
        sweep.append(row)
        if not ok:
            break
        last_ok, r = r, r + coarse
    n = 0

    def try_full(rate):  # None once the full-length budget is spent
        nonlocal n
        if rate in tested:
            return tested[rate]
        if n >= max_full:
            return None
        n += 1
        return full(rate)

    # Full-length runs decide, each rate at most once and at most max_full of them
    # (bounds the bench's wall time): find a passing and a failing full-length rate
    # (up on the fine grid from the last passing probe, or down from it in coarse
    # steps), then bisect between them on the fine grid.
    lo_pass, hi_fail = None, None
    r = last_ok if last_ok is not None else start - coarse
    while r > 0:
        ok = try_full(r)
        if ok is None:
            break
        if ok:
            lo_pass = r
            break
        hi_fail = r
        r -= coarse
    if lo_pass is not None and hi_fail is None:  # the probe rate passed: go up
        top = (last_ok if last_ok is not None else start) + coarse  # the failing probe
        r = lo_pass + fine
        while r < top:
            ok = try_full(r)
            if ok is None:
                break
            if not ok:
                hi_fail = r
                break
            lo_pass, r = r, r + fine
    while lo_pass is not None and hi_fail is not None and hi_fail - lo_pass > fine:
        mid = lo_pass + fine * max(1, round((hi_fail - lo_pass) / (2 * fine)))
        ok = try_full(mid)
        if ok is None:
            break
        if ok:
            lo_pass = mid
        else:
            hi_fail = mid
    best = lo_pass
    return (best or 0.0), sweep


def cosy_lm_steps(batch: int, ctx: int, steps: int, seed: int, hbm: float, device: int):
    """BASELINE config 4's LM (CosyVoice2-style Qwen2.5-0.5B backbone) alone: graph-captured
    decode steps with sampling (cosy_like params: T .8, top-k 50, top-p .95, rp 1.1) over
    `batch` streams at context `ctx`; speech tokens/s, ms/step, HBM roofline of the step
    (weights + KV read), and the LM floor of time-to-first-chunk per chunk size
    (prefill + chunk decode steps; the token-to-mel/vocoder detokenizer is not built)."""
    import torch

    from paper_2602_00269_b200.config import cosyvoice2
    from paper_2602_00269_b200.device import Sampling, VoxDevice

    cfg = cosyvoice2(max_slots=batch + 8, max_ctx=ctx + steps + 64)
    dev = VoxDevice(cfg, weight_seed=seed, device=device)
    prm = Sampling(temperature=0.8, top_p=0.95, top_k=50, repetition_penalty=1.1)
    slots = [dev.admit(seed * 7919 + i, 50, ctx + steps, prm) for i in range(batch)]
    # KV fill: prompt prefill, then (ctx - 50) sampled decode steps so contexts are real
    for a in range(0, batch, 16):  # <= max_rows per forward
        dev.forward(np.array([[s, p, -1, 0] for s in slots[a:a + 16] for p in range(49)], np.int32),
                    sample=False)
    t0 = time.perf_counter()
    dev.forward(np.array([[slots[0], 0, -1, 0]], np.int32), sample=False, sync=True)
    for k in range(ctx - 50):
        dev.forward(np.array([[s, 49 + k, -1, 1] for s in slots], np.int32))
    dev.synchronize()
    lm_s, _ = dev.streams()
    st = torch.cuda.ExternalStream(lm_s)
    ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    pos0 = ctx - 1
    for k in range(3):  # warm
        dev.forward(np.array([[s, pos0 + k, -1, 1] for s in slots], np.int32))
    dev.synchronize()
    ea.record(st)
    for k in range(steps):
        dev.forward(np.array([[s, pos0 + 3 + k, -1, 1] for s in slots], np.int32))
    eb.record(st)
    torch.cuda.synchronize()
    ms = ea.elapsed_time(eb) / steps
    mean_ctx = pos0 + 3 + steps / 2
    by = cfg.weight_bytes - 2 * cfg.vocab * cfg.d_model + 2 * cfg.codebook_size * cfg.d_model  # serving head
    by += batch * mean_ctx * cfg.kv_bytes_per_token
    # prefill time of one 50-token prompt (graph-less, as the engine runs prefill)
    s_new = dev.admit(seed + 99991, 50, 16, prm)
    t1 = time.perf_counter()
    dev.forward(np.array([[s_new, p, -1, 0] for p in range(49)], np.int32), sample=False, sync=True)
    pre_ms = (time.perf_counter() - t1) * 1e3
    dev.close()
    return {"model": "cosyvoice2-style LM (Qwen2.5-0.5B geometry, q|k|v bias, GQA 14:2, hd 64) random-init",
            "batch": batch, "ctx": ctx, "ms_per_step": round(ms, 4),
            "speech_tokens_per_s": round(batch / (ms / 1e3), 1),
            "audio_s_per_s_lm_only": round(batch / (ms / 1e3) / 25.0, 1),
            "roofline": {"bound": "hbm", "achieved": round(by / (ms / 1e3) / 1e9, 1), "peak": hbm, "unit": "GB/s",
                         "frac": round(by / (ms / 1e3) / 1e9 / hbm, 4), "bytes_per_step": int(by)},
            "lm_first_chunk_floor_ms": {str(c): round(pre_ms + c * ms, 2) for c in (5, 10, 15, 25, 50)},
            "prefill_ms_50_tokens": round(pre_ms, 3), "kv_fill_s": round(time.perf_counter() - t0, 2),
            "detokenizer": cosy_detok_sweep(batch, seed, device, pre_ms, ms)}


def cosy_detok_sweep(batch: int, seed: int, device: int, lm_prefill_ms: float, lm_step_ms: float,
                     chunks=(5, 10, 15, 25, 50), calls: int = 3):
    """K8 CosyVoice2-style detokenizer (flow matching + HiFT-style vocoder) at config-4 dims:
    chunk-size sweep for TTFA vs throughput (cosy_like chunk 15,
    profiles.py:163-179).  Per chunk size: device ms of one call over `batch` streams (steady
    state, every stream with vocoder history) -> detok audio-s/s and tensor roofline on the
    algorithmic FLOPs; device ms of a single request's FIRST call -> the TTFA floor = LM
    prefill + chunk x LM step (measured by cosy_lm_steps at `batch` streams) + that call."""
    from paper_2602_00269_b200.config import CosyDetokConfig
    from paper_2602_00269_b200.cosy_detok import CosyDetokenizer

    _, tflops, _ = _peaks()
    cfg = CosyDetokConfig(max_slots=batch + 1, max_tokens=batch * max(chunks), max_chunk=max(chunks))
    dec = CosyDetokenizer(cfg, seed, device)
    rng = np.random.default_rng(seed)
    out = {"kernel": "K8 csrc/cosy_detok.cu: flow (6-layer encoder, 10 CFG Euler steps x 8-layer estimator) + "
                     "HiFT-style vocoder, every call re-consumes 50 reference tokens",
           "streams": batch, "sweep": []}
    for c in chunks:
        slots = [dec.open(seed * 31 + i) for i in range(batch)]
        ms = []
        for k in range(calls + 1):
            dec.decode(slots, [rng.integers(0, cfg.vocab, c) for _ in slots])
            if k >= 1:
                ms.append(dec.last_ms())
        for s_ in slots:
            dec.release(s_)
        # a single request's first call; the call shape's CUDA graph is captured by an
        # earlier request of the same shape (as in serving), so time the second one
        for k in range(2):
            one = dec.open(seed + c + 1000 * k)
            dec.decode([one], [rng.integers(0, cfg.vocab, c)])
            first_ms = dec.last_ms()
            dec.release(one)
        m = float(np.median(ms))
        fl = dec.flops_per_call(c) * batch
        audio = batch * c / 25.0
        out["sweep"].append({
            "chunk": c, "ms_per_call": round(m, 3), "audio_s_per_s": round(audio / (m / 1e3), 1),
            "first_call_ms_b1": round(first_ms, 3),
            "ttfa_floor_ms": round(lm_prefill_ms + c * lm_step_ms + first_ms, 2),
            "roofline": {"bound": "tensor", "achieved": round(fl / (m / 1e3) / 1e12, 2), "peak": tflops,
                         "unit": "TFLOP/s", "frac": round(fl / (m / 1e3) / 1e12 / tflops, 4),
                         "gflop_per_call": round(fl / 1e9, 1)}})
    out["launches_per_call"] = dec.launch_count() // (len(chunks) * (calls + 2))
    dec.close()
    return out


def csm_frames(batch: int, frames: int, seed: int, hbm: float, device: int, with_detok: bool = True):
    """BASELINE config 3 (CSM-1B-style): frames/s of the multi-codebook path -- one backbone
    forward (codebook 0) + 31 depth-decoder forwards (codebooks 1..31) per frame for
    `batch` streams (greedy), hand-overs on the device.  Roofline bytes per frame =
    backbone weights + 31 x depth weights (one codebook head slice each) + KV reads."""
    import torch

    from paper_2602_00269_b200.config import csm_backbone, csm_depth
    from paper_2602_00269_b200.csm import CsmFrames
    from paper_2602_00269_b200.device import Sampling, VoxDevice

    bcfg = csm_backbone(max_slots=batch + 4, max_ctx=128, max_rows=max(512, batch * 2))
    dcfg = csm_depth(max_slots=batch + 4, max_rows=max(512, batch * 2))
    bb, dp = VoxDevice(bcfg, seed, device), VoxDevice(dcfg, seed + 1, device)
    pipe = CsmFrames(bb, dp)
    g = Sampling(temperature=0.0, repetition_penalty=1.0)
    P = 50
    streams = [pipe.admit(seed * 131 + i, P, frames + 8, g, g) for i in range(batch)]
    for a in range(0, batch, 8):
        pipe.prefill(streams[a:a + 8])
    for _ in range(2):  # warm: graphs for every depth position
        pipe.step(streams)
    torch.cuda.synchronize()
    # device time: events on the backbone's LM stream -- every frame ends there (the
    # depth decoder's codes are linked back into the backbone's frame store)
    bb_lm, _ = bb.streams()
    st_bb = torch.cuda.ExternalStream(bb_lm)
    ea, eb = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    ea.record(st_bb)
    for _ in range(frames):
        pipe.step(streams)
    eb.record(st_bb)
    bb.synchronize()
    dp.synchronize()
    wall = (time.perf_counter() - t0) / frames
    torch.cuda.synchronize()
    dt = ea.elapsed_time(eb) / 1e3 / frames
    dcodes = (bcfg.n_codebooks - 1)

    def layer_bytes(c):
        return 2 * ((c.n_heads + 2 * c.n_kv_heads) * c.head_dim * c.d_model + c.d_model * c.n_heads * c.head_dim
                    + 3 * c.d_model * c.d_ff) * c.n_layers
    ctx = P + 2 + frames / 2
    by = (layer_bytes(bcfg) + 2 * bcfg.codebook_size * bcfg.d_model + batch * ctx * bcfg.kv_bytes_per_token
          + dcodes * (layer_bytes(dcfg) + 2 * dcfg.codebook_size * dcfg.d_model)
          + batch * sum(range(2, 33)) * dcfg.kv_bytes_per_token)
    out = {"model": "csm-1b-style random-init: Llama-1B backbone (16 x 2048, 32q/8kv hd 64) + depth decoder "
                    "(4 x 1024, 8q/2kv hd 128) over 32 codebooks x 2048 codes",
           "batch": batch, "frames_timed": frames, "ms_per_frame": round(dt * 1e3, 3),
           "frames_per_s": round(batch / dt, 1), "audio_s_per_s_lm_only": round(batch / dt * 0.08, 1),
           "forwards_per_frame": 1 + dcodes,
           "roofline": {"bound": "hbm", "achieved": round(by / dt / 1e9, 1), "peak": hbm, "unit": "GB/s",
                        "frac": round(by / dt / 1e9 / hbm, 4), "bytes_per_frame": int(by)},
           "wall_ms_per_frame": round(wall * 1e3, 3),
           "timing": "CUDA events on the backbone stream around the frames (device time; every frame ends "
                     "with the depth codes linked back on that stream)"}
    for s_ in streams:
        pipe.release(s_)
    bb.close()
    dp.close()
    if not with_detok:
        return out
    out["detokenizer"] = mimi_chunks(batch, 10, seed, device)
    out["audio_s_per_s_lm_plus_detok"] = round(1.0 / (1.0 / out["audio_s_per_s_lm_only"] +
                                                       1.0 / out["detokenizer"]["audio_s_per_s"]), 1)
    return out


def mimi_chunks(batch: int, chunk: int, seed: int, device: int, calls: int = 6):
    """K7 Mimi-style detokenizer at config-3 dims: `batch` streams each decoding one
    `chunk`-frame window per call (depth_like profile: chunk_size 10, profiles.py:214-231),
    steady state (streams already hold history).  Device time by CUDA events around the
    kernels; tensor roofline on the algorithmic FLOPs of the decode (MimiDecoder.flops_per_frame)."""
    from paper_2602_00269_b200.config import MimiConfig
    from paper_2602_00269_b200.mimi import MimiDecoder

    _, tflops, _ = _peaks()
    cfg = MimiConfig(max_slots=batch, max_frames=batch * chunk)
    dec = MimiDecoder(cfg, seed, device)
    rng = np.random.default_rng(seed)
    slots = [dec.open() for _ in range(batch)]
    ms = []
    t0 = time.perf_counter()
    for i in range(calls + 2):
        codes = [rng.integers(0, cfg.cb_size, size=(chunk, cfg.n_q)) for _ in range(batch)]
        dec.decode(slots, codes)
        if i >= 2:
            ms.append(dec.last_ms())
    wall = (time.perf_counter() - t0) / (calls + 2)
    m = float(np.median(ms))
    fl = dec.flops_per_frame() * batch * chunk
    audio = batch * chunk / 12.5
    out = {"kernel": "K7 csrc/mimi.cu (sliding-window transformer + SEANet convs as tcgen05 im2col GEMMs)",
           "streams": batch, "frames_per_call": chunk, "ms_per_call": round(m, 3),
           "wall_ms_per_call_incl_copies": round(wall * 1e3, 3), "audio_s_per_s": round(audio / (m / 1e3), 1),
           "launches_per_call": dec.launch_count() // (calls + 2),
           "roofline": {"bound": "tensor", "achieved": round(fl / (m / 1e3) / 1e12, 2), "peak": tflops,
                        "unit": "TFLOP/s", "frac": round(fl / (m / 1e3) / 1e12 / tflops, 4),
                        "gflop_per_call": round(fl / 1e9, 2)}}
    dec.close()
    return out


def reference_host_path(n_rows: int = 60):
    """The reference's OWN host path at the Orpheus vocabulary,
    unmodified speechserve from baseline/_ref: per-row sample() (model_api.py:355-381)
    at V = 156,940 with the Orpheus parameters (profiles.py:192-194) on masked hash
    logits -- the like-for-like baseline of K1 -- and run_scenario (engine.py:460-505) of
    config 1's workload (4 requests x 64 tokens at t=0, orpheus_like, async) whose hot
    path is its hash-logit forward + that sampler.  Single-threaded Python/numpy."""
    from dataclasses import replace

    from speechserve import engine as r_engine
    from speechserve import model_api, profiles, scheduler, workload

    V = 156940
    prof = replace(profiles.builtin_profile("orpheus_like"), vocab_size=V)
    params = prof.sampling_defaults
    state = model_api.SamplingState(seed=1, rng=np.random.default_rng(1),
                                    windows=[model_api._RingWindow(params.penalty_window, V)])
    rows = []
    for i in range(n_rows):
        x = model_api.synthetic_logits(model_api.request_seed(0, i), i, 0, V)
        lo = 128266 + (i % 7) * 4096
        m = np.full(V, -np.inf)
        m[lo:lo + 4096] = x[lo:lo + 4096]
        rows.append(m)
    t0 = time.perf_counter()
    for m in rows:
        model_api.sample(m, params, state)
    sample_ms = (time.perf_counter() - t0) / n_rows * 1e3
    greedy = replace(params, temperature=0.0)
    t0 = time.perf_counter()
    for m in rows:
        model_api.sample(m, greedy, state)
    greedy_ms = (time.perf_counter() - t0) / n_rows * 1e3
    arr = workload.build_workload(workload.WorkloadSpec(rate=0.0, offline_count=4, prompt_dist=workload.fixed(50),
                                                        output_dist=workload.fixed(64), seed=0))
    t0 = time.perf_counter()
    tr = r_engine.run_scenario(arr, prof, scheduler.PolicyConfig(), r_engine.Topology(),
                               r_engine.PipelineMode.ASYNCHRONOUS, seed=0)
    wall = time.perf_counter() - t0
    toks = sum(r.tokens_generated for r in tr.requests)
    return {"sample_ms_per_row": round(sample_ms, 3), "sample_greedy_ms_per_row": round(greedy_ms, 3),
            "sampling": f"T {params.temperature}, top-p {params.top_p}, rp {params.repetition_penalty}, V {V}",
            "run_scenario_wall_s": round(wall, 3), "run_scenario_tokens": toks,
            "run_scenario_tok_per_s": round(toks / wall, 1), "cores": 1,
            "what": "unmodified reference (baseline/_ref): per-row sample() on masked hash logits; run_scenario "
                    "of config 1 (4 x 64 tokens, orpheus_like at V=156,940, async) -- hash-stub LM, no audio"}


def reference_protocol(device: int):
    """The drop-in boundary measured: BASELINE config 1's workload (4 requests x 64 tokens
    at t=0, orpheus_like at V = 156,940, async pipeline) through the UNMODIFIED reference
    SimEngine (engine.py:146 run) with ``engine.executor = B200Executor(...)`` on the
    config-1 model (2-layer Llama, SNAC-style decoder; the host's reference sample()
    still picks every token from the returned logits), next to the same engine with the
    reference's own SyntheticExecutor (hash-stub LM, no audio)."""
    from dataclasses import replace

    from paper_2602_00269_b200._ref import core, profiles, ref_engine, scheduler, workload
    from paper_2602_00269_b200.config import tiny
    from paper_2602_00269_b200.executor import B200Executor

    V = 156940
    prof = replace(profiles.builtin_profile("orpheus_like"), vocab_size=V)
    arr = list(enumerate(workload.build_workload(workload.WorkloadSpec(
        rate=0.0, offline_count=4, prompt_dist=workload.fixed(50), output_dist=workload.fixed(64), seed=0))))
    out = {}
    for name in ("reference_synthetic", "b200_executor"):
        eng = ref_engine.SimEngine(prof, scheduler.PolicyConfig(), ref_engine.PipelineMode.ASYNCHRONOUS, seed=0)
        ex = None
        if name == "b200_executor":
            ex = B200Executor(prof, tiny(max_slots=8, max_ctx=1024, max_rows=256, max_detok_frames=256), 0, device)
            eng.executor = ex
        t0 = time.perf_counter()
        tr = eng.run(arr)
        wall = time.perf_counter() - t0
        rep = core.build_report(tr)
        toks = sum(r.tokens_generated for r in tr.requests)
        out[name] = {"wall_s": round(wall, 3), "tokens": toks, "tok_per_s": round(toks / wall, 1),
                     "requests_completed": rep.requests_completed}
        if ex is not None:
            ex.dev.close()
    out["what"] = ("config 1 (4 x 64 tokens) through the unmodified reference SimEngine: its own SyntheticExecutor "
                   "vs engine.executor = B200Executor (real 2-layer LM + SNAC-style audio on the B200; the "
                   "reference's host sample() at V = 156,940 still picks every token)")
    return out


def cpu_port_sample(seconds_budget: float = 20.0):
    """Oracle port of the same step on host cores (bounded sample); returns audio-s/s."""
    from oracle.cpu_step import time_cpu_step

    return time_cpu_step(budget_s=seconds_budget)


def our_config(args, ws: int) -> dict:
    """The workload both arms report on (the reference arm times a bounded sample of it)."""
    return {"workload": "orpheus-3b-style steady-state serving iteration (config 2)",
            "model": "orpheus-3b-style random-init", "concurrent_streams_per_gpu": args.batch,
            "prompt": args.prompt, "output_tokens": 688, "parallelism": f"dp{ws} (request-sharded replicas)",
            "l2": "inputs larger than L2 (6.6 GB weights + KV per step)"}


def spawn_ranks(n: int) -> int:
    """`bench.py --gpus N` outside torchrun: re-launch this command as N ranks (one
    process per GPU) under torch.distributed.run on 127.0.0.1, NCCL_DEBUG=INFO so the
    rank/device map is in the log; rank 0 prints the JSON line."""
    import socket

    with socket.socket() as s_:
        s_.bind(("127.0.0.1", 0))
        port = s_.getsockname()[1]
    env = dict(os.environ, NCCL_DEBUG=os.environ.get("NCCL_DEBUG", "INFO"), VOX_BENCH_SPAWNED="1")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", str(Path(__file__).resolve()), *sys.argv[1:]]
    return subprocess.run(cmd, env=env).returncode


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=64)
    ap.add_argument("--warmup", type=int, default=8)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--batch", type=int, default=256)
    ap.add_argument("--prompt", type=int, default=50)
    ap.add_argument("--seed", type=int, default=0)
    ap.add_argument("--slo-seconds", type=float, default=60.0, help="full-length run (PAPER.md:257)")
    ap.add_argument("--slo-probe-seconds", type=float, default=30.0, help="bracketing probes")
    ap.add_argument("--slo-start", type=float, default=72.0, help="first offered rate per GPU (req/s)")
    ap.add_argument("--no-slo", action="store_true")
    ap.add_argument("--slo-max-batch", type=int, default=256, help="LM batch cap of the load test")
    ap.add_argument("--slo-startup-limit", type=int, default=16, help="scheduler startup concurrency")
    ap.add_argument("--no-roofline", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-cosy", action="store_true", help="skip the config-4 (CosyVoice2-style LM) line")
    ap.add_argument("--no-csm", action="store_true", help="skip the config-3 (CSM-1B-style frames) line")
    ap.add_argument("--ranks-probe", action="store_true", help="print each rank's (rank, world) and exit")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(spawn_ranks(args.gpus))
    if args.ranks_probe:
        ws, rank, _ = dist_setup("gloo")
        print(json.dumps({"rank": rank, "world": ws}), flush=True)
        if ws > 1:
            import torch.distributed as dist

            dist.barrier()
            dist.destroy_process_group()
        return

    if args.impl == "reference":
        ws, rank, _ = dist_setup("gloo")
        if rank != 0:
            return
        from oracle.cpu_step import time_cpu_step

        r = time_cpu_step(budget_s=60.0, steps=args.steps, warmup=1)
        try:
            host = reference_host_path()
        except Exception as e:  # report, never mask the arm
            host = {"error": repr(e)[:200]}
        line = {"metric": METRIC, "value": round(r["audio_s_per_s"], 5), "unit": UNIT, "impl": "reference",
                "n_gpus": args.gpus, "steps": r["steps"], "warmup": 1, "ms_per_step": round(r["ms_per_step"], 2),
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
                "data": "synthetic", "config": our_config(args, ws),
                "cpu_baseline": {"value": round(r["audio_s_per_s"], 5), "unit": UNIT, "cores": r["cores"],
                                 "kind": "port", "sample": r["sample"]},
                "reference_host_path": host,
                "e2e": {"value": round(r["audio_s_per_s"], 5), "unit": UNIT, "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
        print(json.dumps(line))
        return

    ws, rank, local = dist_setup("nccl")
    import torch

    from paper_2602_00269_b200.build import build
    from paper_2602_00269_b200.config import orpheus3b
    from paper_2602_00269_b200.device import VoxDevice

    if rank == 0:
        build()
    if ws > 1:
        import torch.distributed as dist

        dist.barrier()
    torch.cuda.set_device(local)
    cfg = orpheus3b()
    dev = VoxDevice(cfg, weight_seed=args.seed, device=local)
    hbm, tfl, peak_kind = _peaks()

    res = steady_state_steps(dev, args.batch, 3, args.warmup, args.prompt, args.seed + 1000 * rank)  # graphs warm
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clk:
        res = steady_state_steps(dev, args.batch, args.steps, args.warmup, args.prompt, args.seed + 1000 * rank)
    dev_ms = reduce_max(res["dev_ms"], ws, (torch.device("cuda", local) if _DIST_DEVICE else None))
    wall_s = reduce_max(res["wall_s"], ws, (torch.device("cuda", local) if _DIST_DEVICE else None))
    decoded, chunks, pcm = reduce_sum([res["decoded"], res["chunks"], res["pcm_samples"]], ws,
                                      (torch.device("cuda", local) if _DIST_DEVICE else None))
    audio_s = decoded / res["token_rate"]
    value = audio_s / (dev_ms / 1000.0)
    e2e = audio_s / wall_s

    t_phase = [time.time()]

    def phase(name):  # wall time per bench phase, to stderr (the JSON line stays alone on stdout)
        now = time.time()
        print(f"[bench] {name}: {now - t_phase[0]:.1f} s", file=sys.stderr, flush=True)
        t_phase[0] = now

    phase("headline steps")
    roof = None
    if not args.no_roofline and rank == 0:
        classes, step_ms, ctx, sweep, in_graph, nrows = kernel_roofline(dev, args.batch, args.prompt,
                                                                        args.seed + 77, hbm, tfl)
        roof = roofline_summary(cfg, classes, nrows, ctx, hbm, tfl, peak_kind)
        roof["eager_step_ms"] = round(step_ms, 3)
        roof["graph_critical_path"] = in_graph
        roof["batch_sweep"] = {"ctx": ctx, "points": sweep}
        try:
            roof["detok"] = detok_roofline(dev, tfl, hbm)
        except Exception as e:  # report, never mask the headline
            roof["detok"] = {"error": repr(e)[:200]}

    phase("roofline")
    slo = None
    if not args.no_slo:
        best, sweep = run_slo(dev, args.slo_start * ws, args.slo_seconds, args.slo_probe_seconds, args.seed,
                              args.prompt, ws, rank, args.slo_max_batch, args.slo_startup_limit,
                              coarse=8.0 * ws, fine=2.0 * ws)
        slo = {"max_req_s_at_slo": best, "per_gpu": best / ws, "max_lm_batch": args.slo_max_batch,
               "startup_concurrency_limit": args.slo_startup_limit, "criterion": "viability>=0.99 and p90 TTFA<=0.5s",
               "duration_s": args.slo_seconds, "grid_req_s": 2.0 * ws,
               "protocol": f"{args.slo_probe_seconds:.0f} s probes in {8 * ws} req/s steps bracket the rate; "
                           f"the result is the highest {2 * ws} req/s-grid rate passing a {args.slo_seconds:.0f} s run "
                           f"(at most 5 full-length runs: a passing and a failing rate, then bisection; "
                           f"a run whose backlog is not drained {DRAIN_S:.0f} s after its last arrival fails)",
               "routing": "reference route_dp (seeded uniform), replicas", "sweep": sweep}

    phase("slo")
    cosy = None
    if not args.no_cosy and rank == 0:
        try:
            cosy = cosy_lm_steps(128, 512, 32, args.seed + 5, hbm, local)
        except Exception as e:  # report, never mask the headline
            cosy = {"error": repr(e)[:200]}

    phase("config-4 cosy")
    csm = None
    if not args.no_csm and rank == 0:
        try:
            # 256 streams (the LM frame is latency-bound, so throughput grows with the
            # batch); the 64-stream LM point is kept for comparison
            csm = csm_frames(256, 8, args.seed + 9, hbm, local)
            small = csm_frames(64, 8, args.seed + 9, hbm, local, with_detok=False)
            csm["batch_64_lm"] = {k: small[k] for k in ("ms_per_frame", "audio_s_per_s_lm_only", "roofline")}
        except Exception as e:  # report, never mask the headline
            csm = {"error": repr(e)[:200]}

    phase("config-3 csm")
    proto = None
    if not args.no_cpu and rank == 0:
        try:
            proto = reference_protocol(local)
        except Exception as e:  # report, never mask the headline
            proto = {"error": repr(e)[:200]}

    phase("reference protocol")
    cpu = None
    if not args.no_cpu and rank == 0:
        from oracle.cpu_step import time_cpu_step

        r = time_cpu_step(budget_s=20.0, steps=8, warmup=1)
        cpu = {"value": round(r["audio_s_per_s"], 5), "unit": UNIT, "cores": r["cores"], "kind": "port",
               "sample": r["sample"]}

    phase("cpu baseline")
    if rank == 0:
        steps = args.steps
        h2d = (res["rows"] / steps) * 40 + 64  # RowDev (32 B) + out_index + sample_rows per row
        d2h = (res["decoded"] / steps) * 4 + (res["pcm_samples"] / steps) * 4 + 4
        line = {
            "metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": ws, "steps": steps,
            "warmup": args.warmup, "ms_per_step": round(dev_ms / steps, 4), "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": our_config(args, ws),
            "e2e": {"value": round(e2e, 2), "unit": UNIT, "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h)},
            "gpu_launches": int(res["launches"]),
            "clocks": clk.summary(),
            "roofline": roof,
            "cpu_baseline": cpu,
            "slo": slo,
            "config3_csm_frames": csm,
            "reference_protocol": proto,
            "config4_cosyvoice2_lm": cosy,
            "detail": {"tokens_decoded": decoded, "chunks": chunks, "pcm_samples": pcm,
                       "mean_decode_ctx": round(res["mean_ctx"], 1), "prefill_rows": res["prefill_rows"],
                       "timed": "closed loop: B streams kept live, ages uniform over the 688-token lifetime",
                       "device_ms": round(dev_ms, 3), "wall_s": round(wall_s, 4),
                       "host_blocked_ms_per_step": round(res["wait_s"] * 1000 / steps, 3),
                       "lm_graph_step_ms": round(res["lm_graph_step_ms"], 4),
                       "lm_graph_rows": res["lm_graph_rows"],
                       "req_s_equiv": round(decoded / res["token_rate"] / (688 / res["token_rate"]) / (dev_ms / 1000), 2)},
        }
        print(json.dumps(line))
    dev.close()
    if ws > 1:
        import torch.distributed as dist

        dist.destroy_process_group()


if __name__ == "__main__":
    main()
