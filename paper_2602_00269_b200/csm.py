"""CSM-style multi-codebook frame generation (BASELINE config 3).

The reference's depth stage (model_api.py:438-458 depth_forward, engine.py:277-301)
fills codebooks 1..n-1 of every position after the backbone produced codebook 0.
Here both transformers are device contexts running the same kernels as the Orpheus
path (tcgen05 GEMMs, paged attention, fused sampler):

  backbone  (csm_backbone): input = sum of the frame's codebook embeddings; head =
            codebook-0 rows -> samples c0 of the next frame into its token store.
  depth     (csm_depth):    position 0 = projected backbone final hidden
            (vox_project_ext), position 1 = c0, position k samples codebook k.

Hand-overs stay on the device (vox_link_tokens): c0 -> depth position 1, and the
depth's codebook 1..n-1 codes -> the backbone's frame store at the next position, so
one frame is 1 backbone forward + (n-1) depth forwards with no host round trip.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from .device import Sampling, VoxDevice


@dataclass
class CsmStream:
    bslot: int
    dslot: int
    pos: int  # backbone position whose input is fed next (last prompt position, then frames)


class CsmFrames:
    def __init__(self, backbone: VoxDevice, depth: VoxDevice):
        self.bb, self.dp = backbone, depth
        self.C = backbone.cfg.n_codebooks
        self.base = backbone.cfg.audio_base  # backbone id of codebook-0 code 0
        if depth.cfg.frame_tokens != self.C - 1 or depth.cfg.ext_dim != backbone.cfg.d_model:
            raise ValueError("backbone / depth decoder geometry mismatch")

    def admit(self, seed: int, prompt_len: int, n_frames: int, sampling: Sampling,
              depth_sampling: Sampling) -> CsmStream:
        bslot = self.bb.admit(seed, prompt_len, n_frames, sampling)
        dslot = self.dp.admit(seed ^ 0x5EED5EED, 2, self.C - 1, depth_sampling)
        return CsmStream(bslot, dslot, prompt_len - 1)

    def prefill(self, streams: list[CsmStream]) -> None:
        rows = [[s.bslot, p, -1, 0] for s in streams for p in range(s.pos)]
        if rows:
            self.bb.forward(np.array(rows, np.int32), sample=False)

    def step(self, streams: list[CsmStream]) -> None:
        """One frame for every stream: c0 (backbone) then codebooks 1..C-1 (depth)."""
        n = len(streams)
        self.bb.forward(np.array([[s.bslot, s.pos, -1, 1] for s in streams], np.int32))
        self.dp.project_ext(self.bb, n)
        self.dp.link_tokens(self.bb, np.array([[s.dslot, 1, s.bslot, s.pos + 1] for s in streams], np.int32),
                            -self.base, 0)
        rows = [[s.dslot, 0, -2, 0] for s in streams] + [[s.dslot, 1, -1, 1] for s in streams]
        self.dp.forward(np.array(rows, np.int32))
        if self.C > 2:  # positions 2 .. C-1 in one call
            self.dp.forward_steps(np.array([[s.dslot, 2, -1, 1] for s in streams], np.int32), self.C - 2)
        self.bb.link_tokens(self.dp, np.array([[s.bslot, s.pos + 1, s.dslot, 2] for s in streams], np.int32),
                            self.base, 1)
        for s in streams:
            s.pos += 1

    def frame(self, s: CsmStream, pos: int) -> np.ndarray:
        """Codes (per-codebook indices 0..2047) of the frame at backbone position pos."""
        c0 = int(self.bb.read_tokens(s.bslot, pos, 1)[0])
        rest = self.bb.read_frame(s.bslot, pos, 1)[0]
        cs = self.bb.cfg.codebook_size
        return np.array([c0 - self.base] + [int(r) - self.base - (k + 1) * cs for k, r in enumerate(rest)])

    def release(self, s: CsmStream) -> None:
        self.bb.release(s.bslot)
        self.dp.release(s.dslot)
