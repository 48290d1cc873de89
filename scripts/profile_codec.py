"""Profiling driver for the codec detokenizers (K7 Mimi, K8 CosyVoice2-style): one warm
steady-state decode call inside cudaProfilerStart/Stop, for

  ncu --profile-from-start off --metrics gpu__time_duration.sum --csv ... \\
      python scripts/profile_codec.py --model cosy --batch 128 --chunk 15
"""

import argparse
import ctypes
import sys
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(ROOT / "baseline" / "_ref"))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", choices=["cosy", "mimi"], default="cosy")
    ap.add_argument("--batch", type=int, default=128)
    ap.add_argument("--chunk", type=int, default=15)
    a = ap.parse_args()
    rt = ctypes.CDLL("libcudart.so.12") if Path("/usr/local/cuda/lib64/libcudart.so.12").exists() else None
    rng = np.random.default_rng(0)
    if a.model == "cosy":
        from paper_2602_00269_b200.config import CosyDetokConfig
        from paper_2602_00269_b200.cosy_detok import CosyDetokenizer

        cfg = CosyDetokConfig(max_slots=a.batch, max_tokens=a.batch * a.chunk, max_chunk=max(a.chunk, 15))
        dec = CosyDetokenizer(cfg, 1)
        slots = [dec.open(i) for i in range(a.batch)]
        mk = lambda: [rng.integers(0, cfg.vocab, a.chunk) for _ in slots]  # noqa: E731
    else:
        from paper_2602_00269_b200.config import MimiConfig
        from paper_2602_00269_b200.mimi import MimiDecoder

        cfg = MimiConfig(max_slots=a.batch, max_frames=a.batch * a.chunk)
        dec = MimiDecoder(cfg, 1)
        slots = [dec.open() for _ in range(a.batch)]
        mk = lambda: [rng.integers(0, cfg.cb_size, size=(a.chunk, cfg.n_q)) for _ in slots]  # noqa: E731
    dec.decode(slots, mk())
    dec.decode(slots, mk())
    print("warm call ms", dec.last_ms(), flush=True)
    if rt:
        rt.cudaProfilerStart()
    dec.decode(slots, mk())
    if rt:
        rt.cudaProfilerStop()
    print("profiled call ms", dec.last_ms())
    dec.close()


if __name__ == "__main__":
    main()
