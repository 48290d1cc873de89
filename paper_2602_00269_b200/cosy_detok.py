"""CosyDetokenizer: the K8 detokenizer of BASELINE config 4 (CosyVoice2-style).

Host side of ``vox_cosy_*`` (include/voxb200.h, csrc/cosy_detok.cu): chunked
token-to-mel flow matching (every call re-consumes the request's reference tokens,
profiles.py:135 ``ref_window_tokens``) followed by a causal HiFT-style
vocoder that keeps each request's conv histories and iSTFT tail on the device, so a
request's chunks concatenate to one continuous 24 kHz stream (960 samples per token).
Serves ``Executor.detokenize_windows`` (model_api.py:213-220) for cosy_like
(profiles.py:163-179), replacing the stub at profiles.py:333-356.
"""

from __future__ import annotations

import ctypes as C
from typing import Sequence

import numpy as np

from . import _lib
from .config import CosyDetokConfig


def _cfg_struct(cfg: CosyDetokConfig) -> _lib.VoxCosyCfg:
    s = _lib.VoxCosyCfg()
    for f in ("vocab", "ref_tokens", "d_enc", "enc_layers", "enc_heads", "enc_ffn", "mel", "d_est", "est_layers",
              "est_heads", "est_ffn", "n_steps", "voc_ch", "voc_kernel", "res_kernel", "post_kernel", "n_fft", "hop",
              "max_slots", "max_tokens", "max_chunk"):
        setattr(s, f, int(getattr(cfg, f)))
    for f in ("cfg_rate", "rope_theta", "eps", "slope"):
        setattr(s, f, float(getattr(cfg, f)))
    s.n_ratios = len(cfg.ratios)
    for i, r in enumerate(cfg.ratios):
        s.ratios[i] = int(r)
    return s


class CosyDetokenizer:
    def __init__(self, cfg: CosyDetokConfig, weight_seed: int = 0, device: int = 0):
        self.lib = _lib.load()
        self.cfg = cfg
        h = C.c_void_p()
        rc = self.lib.vox_cosy_create(device, C.byref(_cfg_struct(cfg)), C.c_uint64(weight_seed), C.byref(h))
        if rc != 0:
            msg = self.lib.vox_cosy_last_error(None)
            raise _lib._STATUS_TO_EXC.get(rc, RuntimeError)(msg.decode() if msg else f"status {rc}")
        self.h = h

    def _check(self, rc: int) -> None:
        _lib.check(rc, cosy=self.h)

    def close(self) -> None:
        if self.h:
            self.lib.vox_cosy_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def open(self, req_seed: int) -> int:
        s = C.c_int32()
        self._check(self.lib.vox_cosy_open(self.h, C.c_uint64(req_seed & ((1 << 64) - 1)), C.byref(s)))
        return s.value

    def release(self, slot: int) -> None:
        self._check(self.lib.vox_cosy_close(self.h, slot))

    def decode(self, slots: Sequence[int], tokens: Sequence[np.ndarray]) -> list[np.ndarray]:
        """tokens[i]: new speech tokens of stream slots[i] -> its next PCM chunk."""
        n = len(slots)
        reqs = (_lib.VoxCosyReq * max(n, 1))()
        mats = []
        for i, (s, t) in enumerate(zip(slots, tokens)):
            t = np.asarray(t, np.int32).reshape(-1)
            reqs[i].slot, reqs[i].n_tokens = int(s), t.size
            mats.append(t)
        allt = np.ascontiguousarray(np.concatenate(mats) if mats else np.zeros(0, np.int32))
        total = allt.size * self.cfg.samples_per_token
        pcm = np.empty(max(total, 1), np.float32)
        ns = C.c_int64()
        self._check(self.lib.vox_cosy_decode(self.h, reqs, n, allt.ctypes.data_as(_lib._i32p),
                                             pcm.ctypes.data_as(_lib._f32p), C.byref(ns)))
        assert ns.value == total
        out, a = [], 0
        for t in mats:
            b = a + t.size * self.cfg.samples_per_token
            out.append(pcm[a:b].copy())
            a = b
        return out

    def last_ms(self) -> float:
        v = C.c_double()
        self._check(self.lib.vox_cosy_last_ms(self.h, C.byref(v)))
        return v.value

    def launch_count(self) -> int:
        v = C.c_int64()
        self._check(self.lib.vox_cosy_launch_count(self.h, C.byref(v)))
        return v.value

    def flops_per_call(self, chunk: int) -> float:
        """Algorithmic FLOPs of one request's call with `chunk` new tokens (2 per MAC)."""
        c = self.cfg
        T = c.ref_tokens + chunk
        R = 2 * T

        def xf(rows, d, ffn):
            return rows * 2 * (4 * d * d + 2 * d * ffn) + 4 * rows * rows * d

        fl = c.enc_layers * xf(T, c.d_enc, c.enc_ffn) + T * 2 * c.d_enc * c.mel
        fl += c.n_steps * 2 * (R * 2 * 4 * c.mel * c.d_est + c.est_layers * xf(R, c.d_est, c.est_ffn)
                               + R * 2 * c.d_est * c.mel)
        ch, rows = c.voc_channels, 2 * chunk
        fl += rows * 2 * c.voc_kernel * c.mel * ch[0]
        for b, s in enumerate(c.ratios):
            Ci, Co = ch[b], ch[b + 1]
            fl += rows * 2 * 2 * Ci * s * Co
            rows *= s
            fl += 2 * rows * 2 * c.res_kernel * Co * Co
        fl += rows * 2 * c.post_kernel * ch[-1] * (c.n_fft + 2)
        return float(fl)
