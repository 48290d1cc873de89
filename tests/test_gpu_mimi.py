"""K7 Mimi-style streaming detokenizer (csrc/mimi.cu) vs oracle/mimi.py.

The oracle is pinned to transformers' MimiModel.decode (tests/test_mimi_oracle.py).
Bar (BASELINE north_star): audio within max-abs 2e-2 and SNR >= 35 dB of the
full-sequence decode; chunked streaming decode with cached state must equal the
device's own one-shot decode of the same frames.
"""

import numpy as np
import pytest

from oracle.mimi import MimiOracle
from paper_2602_00269_b200.config import MimiConfig, tiny_mimi

pytestmark = pytest.mark.gpu

_ERRS = [ValueError]


def _snr(ref, got):
    return 10 * np.log10((ref.astype(np.float64) ** 2).sum() / max(((got - ref).astype(np.float64) ** 2).sum(), 1e-30))


def _codes(cfg, F, seed):
    return np.random.default_rng(seed).integers(0, cfg.cb_size, size=(F, cfg.n_q)).astype(np.int32)


@pytest.mark.parametrize("window", [250, 16])
def test_one_shot_decode_vs_oracle(window):
    from paper_2602_00269_b200.mimi import MimiDecoder

    cfg = tiny_mimi(window=window)
    dec = MimiDecoder(cfg, weight_seed=11)
    orc = MimiOracle(cfg, 11)
    codes = _codes(cfg, 8, 3)
    s = dec.open()
    pcm = dec.decode([s], [codes])[0]
    ref_dev = orc.decode(codes, exact=False)
    ref = orc.decode(codes, exact=True)
    assert pcm.shape == ref.shape == (8 * cfg.frame_samples,)
    e_dev, e_ref = np.abs(pcm - ref_dev).max(), np.abs(pcm - ref).max()
    print(f"mimi one-shot window {window}: |dev-oracle(device rounding)| {e_dev:.2e}, |dev-oracle(exact)| {e_ref:.2e}, "
          f"SNR {_snr(ref, pcm):.1f} dB")
    assert e_ref < 2e-2 and _snr(ref, pcm) >= 35
    dec.release(s)
    dec.close()


def test_streaming_chunks_equal_full_decode():
    """3 streams, frame chunks of different sizes interleaved across calls (window 16
    so the K/V rings wrap); each stream's concatenated chunks == one-shot decode."""
    from paper_2602_00269_b200.mimi import MimiDecoder

    cfg = tiny_mimi(window=16)
    dec = MimiDecoder(cfg, weight_seed=5)
    orc = MimiOracle(cfg, 5)
    plans = [[3, 5, 1, 4, 7], [1, 1, 8, 2, 8], [6, 6, 4, 4, 0]]
    codes = [_codes(cfg, sum(p), 100 + i) for i, p in enumerate(plans)]
    slots = [dec.open() for _ in plans]
    out = [[] for _ in plans]
    pos = [0, 0, 0]
    for step in range(5):
        ids, cs = [], []
        for i, p in enumerate(plans):
            if p[step]:
                ids.append(i)
                cs.append(codes[i][pos[i]:pos[i] + p[step]])
                pos[i] += p[step]
        pcms = dec.decode([slots[i] for i in ids], cs)
        for i, pcm in zip(ids, pcms):
            out[i].append(pcm)
    one = MimiDecoder(cfg, weight_seed=5)
    for i in range(3):
        got = np.concatenate(out[i])
        s1 = one.open()
        full = one.decode([s1], [codes[i]])[0]
        ref = orc.decode(codes[i], exact=True)
        assert got.shape == full.shape == ref.shape
        d = np.abs(got - full).max()
        print(f"stream {i}: |chunked - one-shot| {d:.2e}, SNR vs oracle {_snr(ref, got):.1f} dB")
        assert d < 1e-4, d
        assert np.abs(got - ref).max() < 2e-2 and _snr(ref, got) >= 35
    for s in slots:
        dec.release(s)
    dec.close()
    one.close()


def test_config3_dims():
    """Production Mimi dims (32 codebooks, 8 transformer layers, window 250), 2 streams
    in one call then a second chunk each."""
    from paper_2602_00269_b200.mimi import MimiDecoder

    cfg = MimiConfig(max_slots=4, max_frames=32)
    dec = MimiDecoder(cfg, weight_seed=21)
    orc = MimiOracle(cfg, 21)
    codes = [_codes(cfg, 7, 1), _codes(cfg, 5, 2)]
    a, b = dec.open(), dec.open()
    p1 = dec.decode([a, b], [codes[0][:4], codes[1][:3]])
    p2 = dec.decode([b, a], [codes[1][3:], codes[0][4:]])
    got = [np.concatenate([p1[0], p2[1]]), np.concatenate([p1[1], p2[0]])]
    for i in range(2):
        ref = orc.decode(codes[i], exact=True)
        snr = _snr(ref, got[i])
        print(f"config-3 Mimi stream {i}: max-abs {np.abs(got[i] - ref).max():.2e}, SNR {snr:.1f} dB, "
              f"rms {np.sqrt((ref ** 2).mean()):.3f}")
        assert np.abs(got[i] - ref).max() < 2e-2 and snr >= 35
    assert dec.launch_count() > 0
    dec.close()


def test_errors():
    from paper_2602_00269_b200._ref import errors
    from paper_2602_00269_b200.mimi import MimiDecoder

    cfg = tiny_mimi(max_frames=8, max_slots=2)
    dec = MimiDecoder(cfg, weight_seed=1)
    with pytest.raises(errors.CacheMissing):
        dec.decode([0], [_codes(cfg, 1, 0)])
    s = dec.open()
    bad = _codes(cfg, 1, 0)
    bad[0, 0] = cfg.cb_size
    with pytest.raises(ValueError):
        dec.decode([s], [bad])
    with pytest.raises(errors.BatchTooLarge):
        dec.decode([s], [_codes(cfg, 9, 0)])
    dec.open()
    with pytest.raises(MemoryError):
        dec.open()
    dec.close()
