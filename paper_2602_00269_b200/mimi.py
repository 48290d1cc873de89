"""MimiDecoder: the K7 streaming detokenizer of BASELINE config 3 (CSM-1B-style).

Host side of ``vox_mimi_*`` (include/voxb200.h, csrc/mimi.cu): one device context
holding the Mimi-style decoder's weights, per-stream conv padding caches and
sliding-window K/V rings.  A stream is opened per request; each ``decode`` call
turns that request's new 12.5 Hz frames (n_q codes each) into 1920 PCM samples per
frame, continuing the stream's history, so the chunks of a stream concatenate to
the full-sequence decode ([3P] transformers ``MimiModel.decode``,
modeling_mimi.py:1613-1680; restated and pinned in oracle/mimi.py).

It serves ``Executor.detokenize_windows`` (model_api.py:213-220) for depth-stage
profiles (profiles.py:214-231), replacing the reference's stub
(profiles.py:333-356): see ``executor.CsmExecutor``.
"""

from __future__ import annotations

import ctypes as C
from typing import Sequence

import numpy as np

from . import _lib
from .config import MimiConfig


def _cfg_struct(cfg: MimiConfig) -> _lib.VoxMimiCfg:
    s = _lib.VoxMimiCfg()
    for f in ("n_q", "n_semantic", "cb_size", "cb_dim", "hidden", "n_layers", "n_heads", "ffn", "window",
              "filters", "kernel", "last_kernel", "res_kernel", "compress", "max_slots", "max_frames"):
        setattr(s, f, int(getattr(cfg, f)))
    s.rope_theta = float(cfg.rope_theta)
    s.eps = float(cfg.eps)
    s.n_ratios = len(cfg.ratios)
    for i, r in enumerate(cfg.ratios):
        s.ratios[i] = int(r)
    return s


class MimiDecoder:
    def __init__(self, cfg: MimiConfig, weight_seed: int = 0, device: int = 0):
        self.lib = _lib.load()
        self.cfg = cfg
        h = C.c_void_p()
        rc = self.lib.vox_mimi_create(device, C.byref(_cfg_struct(cfg)), C.c_uint64(weight_seed), C.byref(h))
        if rc != 0:
            msg = self.lib.vox_mimi_last_error(None)
            raise _lib._STATUS_TO_EXC.get(rc, RuntimeError)(msg.decode() if msg else f"status {rc}")
        self.h = h

    def _check(self, rc: int) -> None:
        _lib.check(rc, mimi=self.h)

    def close(self) -> None:
        if self.h:
            self.lib.vox_mimi_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def open(self) -> int:
        s = C.c_int32()
        self._check(self.lib.vox_mimi_open(self.h, C.byref(s)))
        return s.value

    def release(self, slot: int) -> None:
        self._check(self.lib.vox_mimi_close(self.h, slot))

    def decode(self, slots: Sequence[int], codes: Sequence[np.ndarray]) -> list[np.ndarray]:
        """codes[i]: [n_frames_i, n_q] ints of stream slots[i]'s next frames -> PCM per stream."""
        n = len(slots)
        reqs = (_lib.VoxMimiReq * max(n, 1))()
        mats = []
        for i, (s, c) in enumerate(zip(slots, codes)):
            c = np.asarray(c, np.int32).reshape(-1, self.cfg.n_q)
            reqs[i].slot, reqs[i].n_frames = int(s), c.shape[0]
            mats.append(c)
        allc = np.ascontiguousarray(np.concatenate(mats, axis=0) if mats else np.zeros((0, self.cfg.n_q), np.int32))
        total = allc.shape[0] * self.cfg.frame_samples
        pcm = np.empty(max(total, 1), np.float32)
        ns = C.c_int64()
        self._check(self.lib.vox_mimi_decode(self.h, reqs, n, allc.ctypes.data_as(_lib._i32p),
                                             pcm.ctypes.data_as(_lib._f32p), C.byref(ns)))
        assert ns.value == total
        out, a = [], 0
        for c in mats:
            b = a + c.shape[0] * self.cfg.frame_samples
            out.append(pcm[a:b].copy())
            a = b
        return out

    def last_ms(self) -> float:
        """CUDA-event time of the last decode's kernels."""
        v = C.c_double()
        self._check(self.lib.vox_mimi_last_ms(self.h, C.byref(v)))
        return v.value

    def flops_per_frame(self, ctx: int | None = None) -> float:
        """Algorithmic FLOPs per 12.5 Hz frame (2 per MAC): transformer projections +
        attention over a window of `ctx` keys (default: full window), SEANet convs."""
        c = self.cfg
        D, F, L = c.hidden, c.ffn, c.n_layers
        ctx = c.window if ctx is None else ctx
        pos = 2
        fl = pos * L * 2 * (4 * D * D + 2 * D * F + 2 * ctx * D)
        ch = c.channels
        fl += pos * 2 * c.kernel * D * ch[0]
        rows = pos
        for b, s in enumerate(c.ratios):
            Ci, Co = ch[b], ch[b + 1]
            hh = Co // c.compress
            fl += rows * 2 * (2 * Ci) * (s * Co)
            rows *= s
            fl += rows * 2 * (c.res_kernel * Co * hh + hh * Co)
        fl += rows * 2 * c.last_kernel * ch[-1]
        return float(fl)

    def launch_count(self) -> int:
        v = C.c_int64()
        self._check(self.lib.vox_mimi_launch_count(self.h, C.byref(v)))
        return v.value
