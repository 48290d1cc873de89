"""Pin oracle/mimi.py to transformers' MimiModel.decode (the published algorithm of
BASELINE config 3's detokenizer; [3P] transformers 5.5.0 modeling_mimi.py:1613-1680)."""

import numpy as np
import pytest

from oracle.mimi import MimiOracle
from paper_2602_00269_b200.config import tiny_mimi

torch = pytest.importorskip("torch")
transformers = pytest.importorskip("transformers")


def _hf_model(cfg, orc):
    from transformers import MimiConfig, MimiModel

    hc = MimiConfig(num_quantizers=cfg.n_q, num_semantic_quantizers=cfg.n_semantic, codebook_size=cfg.cb_size,
                    codebook_dim=cfg.cb_dim, hidden_size=cfg.hidden, num_hidden_layers=cfg.n_layers,
                    num_attention_heads=cfg.n_heads, num_key_value_heads=cfg.n_heads, intermediate_size=cfg.ffn,
                    sliding_window=cfg.window, num_filters=cfg.filters, upsampling_ratios=list(cfg.ratios),
                    kernel_size=cfg.kernel, last_kernel_size=cfg.last_kernel, residual_kernel_size=cfg.res_kernel,
                    compress=cfg.compress, norm_eps=cfg.eps, rope_parameters={"rope_type": "default",
                                                                              "rope_theta": cfg.rope_theta},
                    vector_quantization_hidden_dimension=cfg.cb_dim, use_causal_conv=True)
    hc._attn_implementation = "eager"
    torch.manual_seed(0)
    m = MimiModel(hc).eval()
    sd = {k: torch.from_numpy(np.ascontiguousarray(v)) for k, v in orc.w.torch_layout().items()}
    missing = set(sd) - set(m.state_dict())
    assert not missing, sorted(missing)[:5]
    m.load_state_dict(sd, strict=False)
    return m


@pytest.mark.parametrize("F,window", [(6, 250), (20, 16)])
def test_oracle_equals_transformers_mimi_decode(F, window):
    cfg = tiny_mimi(window=window)
    orc = MimiOracle(cfg, 77)
    rng = np.random.default_rng(F)
    codes = rng.integers(0, cfg.cb_size, size=(F, cfg.n_q))
    m = _hf_model(cfg, orc)
    with torch.no_grad():
        ref = m.decode(torch.from_numpy(codes.T[None].copy())).audio_values[0, 0].numpy()
    got = orc.decode(codes, exact=True)
    assert got.shape == ref.shape == (F * cfg.frame_samples,)
    err = np.abs(got - ref).max()
    assert err < 2e-4 * max(1.0, np.abs(ref).max()), err
    # the device's rounding points stay inside the audio tolerance of the exact decode
    dev = orc.decode(codes, exact=False)
    snr = 10 * np.log10((ref ** 2).sum() / ((dev - ref) ** 2).sum())
    assert np.abs(dev - ref).max() < 2e-2 and snr > 35, (np.abs(dev - ref).max(), snr)
    print(f"mimi oracle F={F} window={window}: |oracle-hf| {err:.2e}, device-rounding SNR {snr:.1f} dB, "
          f"rms {np.sqrt((ref ** 2).mean()):.3f}")


def test_oracle_is_causal():
    """The decode of a prefix equals the prefix of the decode (so a stateful chunked
    decode must reproduce the full-sequence decode exactly)."""
    cfg = tiny_mimi(window=16)
    orc = MimiOracle(cfg, 5)
    codes = np.random.default_rng(1).integers(0, cfg.cb_size, size=(12, cfg.n_q))
    full = orc.decode(codes, exact=False)
    part = orc.decode(codes[:7], exact=False)
    assert np.allclose(full[: part.size], part, atol=1e-5)
