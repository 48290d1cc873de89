"""Synthetic request inputs (TEST INFRASTRUCTURE ONLY).

request_seed follows model_api.py:54-55; prompt ids mirror csrc/vox_api.cu
(prompt_id): mix64(req_seed + 0x632BE59BD9B4E019*(i+1)) mod text_vocab.
"""

from __future__ import annotations

from .weights import MASK64, mix64


def request_seed(run_seed: int, request_id: int) -> int:
    """model_api.py:54-55."""
    return mix64(mix64(run_seed & MASK64) ^ (request_id & MASK64))


def prompt_ids(req_seed: int, n: int, text_vocab: int) -> list[int]:
    return [mix64((req_seed + 0x632BE59BD9B4E019 * (i + 1)) & MASK64) % text_vocab for i in range(n)]
