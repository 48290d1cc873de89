"""Thin Python handle over one C-ABI context (one GPU, one engine loop)."""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from typing import Optional, Sequence

import numpy as np

from . import _lib
from .config import ModelConfig


@dataclass(frozen=True)
class Sampling:
    """Mirror of the reference SamplingParams (model_api.py:105-121)."""

    temperature: float = 1.0
    top_k: Optional[int] = None
    top_p: float = 1.0
    repetition_penalty: float = 1.0
    penalty_window: int = 64

    MAX_WINDOW = 256  # device ring-window capacity (VoxSampling.penalty_window)

    @classmethod
    def from_ref(cls, p) -> "Sampling":
        if p.penalty_window > cls.MAX_WINDOW:
            # the reference accepts any window (model_api.py:105-121); the device keeps
            # the last <= 256 ids: refuse instead of silently penalising fewer tokens
            raise ValueError(f"penalty_window {p.penalty_window} exceeds the device ring capacity "
                             f"{cls.MAX_WINDOW}")
        return cls(p.temperature, p.top_k, p.top_p, p.repetition_penalty, p.penalty_window)

    def to_c(self) -> _lib.VoxSampling:
        return _lib.VoxSampling(
            float(self.temperature), float(self.top_p), float(self.repetition_penalty),
            int(self.top_k or 0), int(self.penalty_window),
        )


def _ptr(a: np.ndarray, ctype):
    return a.ctypes.data_as(C.POINTER(ctype))


class VoxDevice:
    """Owns a VoxCtx: weights, paged KV pool, token store, detok state."""

    def __init__(self, cfg: ModelConfig, weight_seed: int = 0, device: int = 0):
        self.lib = _lib.load()
        self.cfg = cfg
        c = _lib.VoxModelCfg()
        c.n_layers, c.d_model, c.n_heads = cfg.n_layers, cfg.d_model, cfg.n_heads
        c.n_kv_heads, c.head_dim, c.d_ff, c.vocab = cfg.n_kv_heads, cfg.head_dim, cfg.d_ff, cfg.vocab
        c.rope_theta, c.rms_eps = cfg.rope_theta, cfg.rms_eps
        c.embed_scale = cfg.embed_half_width
        c.text_vocab = cfg.text_vocab
        c.audio_base, c.codebook_size, c.frame_tokens = cfg.audio_base, cfg.codebook_size, cfg.frame_tokens
        c.page_size, c.n_pages, c.max_slots = cfg.page_size, cfg.pages, cfg.max_slots
        c.max_ctx, c.max_rows = cfg.max_ctx, cfg.max_rows
        c.detok_enabled = int(cfg.detok_enabled)
        c.latent_dim, c.decoder_dim, c.n_rates = cfg.latent_dim, cfg.decoder_dim, len(cfg.rates)
        for i, r in enumerate(cfg.rates):
            c.rates[i] = r
        c.max_detok_frames = cfg.max_detok_frames
        c.qkv_bias = int(cfg.qkv_bias)
        c.n_codebooks = int(cfg.n_codebooks)
        c.ext_dim = int(cfg.ext_dim)
        self._c = c
        h = C.c_void_p()
        _lib.check(self.lib.vox_create(device, C.byref(c), C.c_uint64(weight_seed & (2**64 - 1)), C.byref(h)))
        self.ctx = h

    # ------------------------------------------------------------------ lifecycle
    def close(self) -> None:
        if self.ctx:
            self.lib.vox_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _check(self, rc: int) -> None:
        _lib.check(rc, self.ctx)

    # ------------------------------------------------------------------ requests
    def admit(self, req_seed: int, prompt_len: int, target_len: int, sampling: Sampling) -> int:
        slot = C.c_int32()
        p = sampling.to_c()
        self._check(self.lib.vox_admit(self.ctx, C.c_uint64(req_seed & (2**64 - 1)), prompt_len,
                                       target_len, C.byref(p), C.byref(slot)))
        return slot.value

    def release(self, slot: int) -> None:
        self._check(self.lib.vox_release(self.ctx, slot))

    def page_table(self, slot: int) -> np.ndarray:
        cap = (self.cfg.max_ctx + self.cfg.page_size - 1) // self.cfg.page_size
        out = np.zeros(cap, dtype=np.int32)
        n = C.c_int32()
        self._check(self.lib.vox_page_table(self.ctx, slot, _ptr(out, C.c_int32), cap, C.byref(n)))
        return out[: n.value].copy()

    def read_tokens(self, slot: int, pos: int, n: int) -> np.ndarray:
        out = np.zeros(n, dtype=np.int32)
        self._check(self.lib.vox_read_tokens(self.ctx, slot, pos, n, _ptr(out, C.c_int32)))
        return out

    def write_tokens(self, slot: int, pos: int, ids: Sequence[int]) -> None:
        a = np.ascontiguousarray(ids, dtype=np.int32)
        self._check(self.lib.vox_write_tokens(self.ctx, slot, pos, len(a), _ptr(a, C.c_int32)))

    # ------------------------------------------------------------------ LM step
    def forward(self, rows: np.ndarray, sample: bool = True, full_logits: bool = False,
                want_tokens: bool = False, sync: bool = False, graph: bool = True):
        """rows: int32 [n, 4] = (slot, pos, token, sample).  Returns (tokens, logits)."""
        rows = np.ascontiguousarray(rows, dtype=np.int32)
        n = rows.shape[0]
        nsamp = int(rows[:, 3].astype(bool).sum()) if n else 0
        flags = 0
        if sample:
            flags |= _lib.VOX_FWD_SAMPLE
        if full_logits:
            flags |= _lib.VOX_FWD_FULL_LOGITS
        if sync:
            flags |= _lib.VOX_FWD_SYNC
        if not graph:
            flags |= _lib.VOX_FWD_NO_GRAPH
        logits = None
        toks = None
        lp = None
        tp = None
        if full_logits:
            logits = np.empty((nsamp, self.cfg.vocab), dtype=np.float32)
            lp = _ptr(logits, C.c_float)
        if want_tokens:
            toks = np.empty(nsamp, dtype=np.int32)
            tp = _ptr(toks, C.c_int32)
        rp = rows.ctypes.data_as(C.POINTER(_lib.VoxRow))
        self._check(self.lib.vox_forward(self.ctx, rp, n, flags, lp, tp))
        return toks, logits

    def forward_steps(self, rows: np.ndarray, steps: int) -> None:
        """`steps` sampled decode steps over the same rows, pos advancing by one per step,
        issued in one call (no host round trip between steps)."""
        rows = np.ascontiguousarray(rows, dtype=np.int32)
        rp = rows.ctypes.data_as(C.POINTER(_lib.VoxRow))
        self._check(self.lib.vox_forward_steps(self.ctx, rp, rows.shape[0], steps, _lib.VOX_FWD_SAMPLE))

    def read_logits(self):
        """The last forward's head logits as K1 saw them: ([n_rows, ld] fp32, col_base),
        column j = vocabulary id col_base + j (synchronises the LM stream)."""
        n, ld, base = C.c_int32(), C.c_int32(), C.c_int32()
        self._check(self.lib.vox_read_logits(self.ctx, None, 0, 0, C.byref(n), C.byref(ld), C.byref(base)))
        out = np.empty((n.value, ld.value), np.float32)
        self._check(self.lib.vox_read_logits(self.ctx, _ptr(out, C.c_float), n.value, ld.value, None, None, None))
        return out, base.value

    def forward_seq(self) -> int:
        s = C.c_int64()
        self._check(self.lib.vox_forward_seq(self.ctx, C.byref(s)))
        return s.value

    def forward_wait(self, seq: int) -> None:
        self._check(self.lib.vox_forward_wait(self.ctx, seq))

    def sample_logits(self, logits: np.ndarray, params: Sequence[Sampling], windows: Sequence[Sequence[int]],
                      seeds: Sequence[int], steps: Sequence[int], lo=None, hi=None) -> np.ndarray:
        logits = np.ascontiguousarray(logits, dtype=np.float32)
        n, vocab = logits.shape
        wcap = max([len(w) for w in windows] + [1])
        wids = np.zeros((n, wcap), dtype=np.int32)
        wlen = np.zeros(n, dtype=np.int32)
        for i, w in enumerate(windows):
            wids[i, : len(w)] = w
            wlen[i] = len(w)
        parr = (_lib.VoxSampling * n)(*[p.to_c() for p in params])
        s = np.asarray([x & (2**64 - 1) for x in seeds], dtype=np.uint64)
        st = np.asarray(steps, dtype=np.uint64)
        lo_a = np.asarray(lo if lo is not None else [0] * n, dtype=np.int32)
        hi_a = np.asarray(hi if hi is not None else [vocab] * n, dtype=np.int32)
        out = np.empty(n, dtype=np.int32)
        self._check(self.lib.vox_sample_logits(
            self.ctx, _ptr(logits, C.c_float), n, vocab, parr, _ptr(wids, C.c_int32), wcap,
            _ptr(wlen, C.c_int32), _ptr(s, C.c_uint64), _ptr(st, C.c_uint64),
            _ptr(lo_a, C.c_int32), _ptr(hi_a, C.c_int32), _ptr(out, C.c_int32)))
        return out

    # ------------------------------------------------------------------ detokenizer
    def detok(self, windows: np.ndarray, sync: bool = True):
        """windows: int32 [n, 6] = (slot, index, start, length, new_tokens, final).

        sync=True -> (list of per-request PCM arrays, ticket); else (n_samples, ticket).
        """
        w = np.ascontiguousarray(windows, dtype=np.int32)
        n = w.shape[0]
        ns = np.zeros(n, dtype=np.int32)
        ticket = C.c_int64()
        wp = w.ctypes.data_as(C.POINTER(_lib.VoxWindow))
        if sync:
            total_cap = int(self.cfg.max_detok_frames * self.cfg.hop)
            buf = np.empty(total_cap, dtype=np.float32)
            self._check(self.lib.vox_detok(self.ctx, wp, n, _ptr(buf, C.c_float), _ptr(ns, C.c_int32),
                                           C.byref(ticket)))
            out, off = [], 0
            for k in ns:
                out.append(buf[off: off + k].copy())
                off += k
            return out, ticket.value
        self._check(self.lib.vox_detok(self.ctx, wp, n, None, _ptr(ns, C.c_int32), C.byref(ticket)))
        return ns, ticket.value

    def ticket_done(self, ticket: int):
        done = C.c_int32()
        t = C.c_double()
        self._check(self.lib.vox_ticket_query(self.ctx, ticket, C.byref(done), C.byref(t)))
        return bool(done.value), t.value

    def ticket_pcm(self, ticket: int) -> np.ndarray:
        p = C.POINTER(C.c_float)()
        total = C.c_int32()
        self._check(self.lib.vox_ticket_pcm(self.ctx, ticket, C.byref(p), C.byref(total)))
        return np.ctypeslib.as_array(p, shape=(total.value,)).copy() if total.value else np.zeros(0, np.float32)

    def clock_reset(self) -> None:
        self._check(self.lib.vox_clock_reset(self.ctx))

    def synchronize(self) -> None:
        self._check(self.lib.vox_synchronize(self.ctx))

    def streams(self):
        a, b = C.c_void_p(), C.c_void_p()
        self._check(self.lib.vox_streams(self.ctx, C.byref(a), C.byref(b)))
        return a.value, b.value

    # ------------------------------------------------------------------ timing
    def timing(self, on: bool) -> None:
        self._check(self.lib.vox_timing_enable(self.ctx, int(on)))

    def timing_read(self, cls: str):
        ms, n, by = C.c_double(), C.c_int64(), C.c_double()
        self._check(self.lib.vox_timing_read(self.ctx, cls.encode(), C.byref(ms), C.byref(n), C.byref(by)))
        return ms.value, n.value, by.value

    # ------------------------------------------------------------------ CSM-style frames
    def write_frame(self, slot: int, pos: int, ids: np.ndarray) -> None:
        """ids [n_pos, n_codebooks - 1] of codebooks 1.. at positions pos.. (-1 = none)."""
        a = np.ascontiguousarray(ids, dtype=np.int32)
        self._check(self.lib.vox_write_frame(self.ctx, slot, pos, a.shape[0], _ptr(a, C.c_int32)))

    def read_frame(self, slot: int, pos: int, n_pos: int) -> np.ndarray:
        out = np.empty((n_pos, self.cfg.n_codebooks - 1), np.int32)
        self._check(self.lib.vox_read_frame(self.ctx, slot, pos, n_pos, _ptr(out, C.c_int32)))
        return out

    def project_ext(self, src: "VoxDevice", n: int) -> None:
        """ext rows 0..n-1 = src's last sampled final-hidden rows x this ctx's input projector."""
        self._check(self.lib.vox_project_ext(self.ctx, src.ctx, n))

    def link_tokens(self, src: "VoxDevice", links: np.ndarray, offset: int, mode: int) -> None:
        """Device-side token hand-over; links [n, 4] = (dst_slot, dst_pos, src_slot, src_pos)."""
        a = np.ascontiguousarray(links, dtype=np.int32)
        self._check(self.lib.vox_link_tokens(self.ctx, src.ctx, _ptr(a, C.c_int32), a.shape[0], offset, mode))

    def copy_tokens(self, src: "VoxDevice", spans: np.ndarray) -> None:
        """Token-store spans [n, 5] = (dst_slot, dst_pos, src_slot, src_pos, len) from the
        LM context `src` into this (detokenizer) context -- disaggregated LM -> detok."""
        arr = np.ascontiguousarray(spans, np.int32).reshape(-1, 5)
        self._check(self.lib.vox_copy_tokens(self.ctx, src.ctx, arr.ctypes.data_as(_lib._i32p), arr.shape[0]))

    def trace_arm(self, capacity: int = 1 << 20) -> None:
        """Arm the in-graph kernel tracer (one record per CTA of every instrumented kernel)."""
        self._check(self.lib.vox_trace_arm(self.ctx, capacity))

    def trace_read(self, max_records: int = 1 << 20) -> np.ndarray:
        """Records {tag (kernel | grid CTAs << 8), smid, t0_ns, t1_ns}; disarms the tracer."""
        dt = np.dtype([("tag", np.uint32), ("smid", np.uint32), ("t0", np.uint64), ("t1", np.uint64)])
        out = np.zeros(max_records, dt)
        n = C.c_int64()
        self._check(self.lib.vox_trace_read(self.ctx, out.ctypes.data_as(C.c_void_p), max_records, C.byref(n)))
        return out[: n.value]

    def launch_count(self) -> int:
        n = C.c_int64()
        self._check(self.lib.vox_launch_count(self.ctx, C.byref(n)))
        return n.value

    def sm_partition(self) -> tuple[int, int]:
        """(LM-stream SMs, detok-stream SMs); detok 0 = both streams share every SM."""
        lm, dt = C.c_int32(), C.c_int32()
        self._check(self.lib.vox_sm_partition(self.ctx, C.byref(lm), C.byref(dt)))
        return lm.value, dt.value

    def gemm_test(self, w_bits: np.ndarray, x_bits: np.ndarray, bias=None, splits: int = 1, iters: int = 1):
        """K3 alone: w_bits [M,K], x_bits [N,K] uint16 bf16 bits -> (out [N,M] fp32, mean ms)."""
        w = np.ascontiguousarray(w_bits, dtype=np.uint16)
        x = np.ascontiguousarray(x_bits, dtype=np.uint16)
        M, K = w.shape
        N = x.shape[0]
        out = np.empty((N, M), np.float32)
        ms = C.c_double()
        b = None if bias is None else np.ascontiguousarray(bias, dtype=np.float32)
        self._check(self.lib.vox_gemm_test(
            self.ctx, w.ctypes.data_as(C.POINTER(C.c_uint16)), x.ctypes.data_as(C.POINTER(C.c_uint16)),
            None if b is None else _ptr(b, C.c_float), M, N, K, splits, iters, _ptr(out, C.c_float), C.byref(ms)))
        return out, ms.value

    def read_weight(self, name: str, layer: int, shape, dtype) -> np.ndarray:
        out = np.empty(shape, dtype=dtype)
        self._check(self.lib.vox_read_weight(self.ctx, name.encode(), layer, out.ctypes.data_as(C.c_void_p),
                                             out.nbytes))
        return out

    def read_kv(self, layer: int, slot: int, pos: int):
        n = self.cfg.n_kv_heads * self.cfg.head_dim
        k = np.empty(n, dtype=np.float32)
        v = np.empty(n, dtype=np.float32)
        self._check(self.lib.vox_read_kv(self.ctx, layer, slot, pos, _ptr(k, C.c_float), _ptr(v, C.c_float)))
        return k.reshape(self.cfg.n_kv_heads, -1), v.reshape(self.cfg.n_kv_heads, -1)
