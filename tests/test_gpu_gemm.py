"""K3 tcgen05 GEMM vs a float64 numpy reference over every tile width and split-K."""

import numpy as np
import pytest

from oracle.weights import bf16_round

pytestmark = pytest.mark.gpu


def _bits(a):
    return (bf16_round(a).view(np.uint32) >> 16).astype(np.uint16)


@pytest.mark.parametrize("M,N,K,splits", [
    (128, 1, 64, 1), (128, 16, 128, 1), (256, 5, 256, 2), (384, 31, 512, 4),
    (512, 64, 768, 3), (200, 100, 1024, 1), (1024, 128, 2048, 8), (64, 300, 64, 1),
    (4096, 257, 2048, 1), (128, 1024, 256, 1), (156940 // 10, 7, 256, 1),
])
@pytest.mark.parametrize("packed", [0, 1])
def test_gemm_matches_numpy(tiny_dev, monkeypatch, M, N, K, splits, packed):
    # packed=1 streams W from the packed 16 KB tile layout (init.cu), the decode path
    monkeypatch.setenv("VOX_GEMM_PACKED_TEST", str(packed))
    rng = np.random.default_rng(M * 7 + N)
    w = bf16_round(rng.uniform(-1, 1, size=(M, K)).astype(np.float32))
    x = bf16_round(rng.uniform(-1, 1, size=(N, K)).astype(np.float32))
    bias = rng.uniform(-1, 1, size=M).astype(np.float32) if splits == 1 else None
    out, _ = tiny_dev.gemm_test(_bits(w), _bits(x), bias, splits)
    ref = x.astype(np.float64) @ w.astype(np.float64).T
    if bias is not None:
        ref += bias
    err = np.abs(out - ref).max()
    assert err < 1e-3 * np.sqrt(K), (err, np.unravel_index(np.argmax(np.abs(out - ref)), out.shape))


@pytest.mark.parametrize("M,N,K", [(3072, 224, 3072), (1024, 256, 2048), (5120, 64, 1024), (640, 100, 512)])
@pytest.mark.parametrize("splits", [2, 3, 5, 8])
def test_gemm_decode_split_k(tiny_dev, monkeypatch, M, N, K, splits):
    """Decode GEMM (one n-tile of all rows) with forced split-K fp32 planes."""
    monkeypatch.setenv("VOX_GEMM_PACKED_TEST", "1")
    monkeypatch.setenv("VOX_GEMM_SPLITS_TEST", str(splits))
    rng = np.random.default_rng(M + N + splits)
    w = bf16_round(rng.uniform(-1, 1, size=(M, K)).astype(np.float32))
    x = bf16_round(rng.uniform(-1, 1, size=(N, K)).astype(np.float32))
    out, _ = tiny_dev.gemm_test(_bits(w), _bits(x), None, splits)
    ref = x.astype(np.float64) @ w.astype(np.float64).T
    err = np.abs(out - ref).max()
    assert err < 1e-3 * np.sqrt(K), err


@pytest.mark.parametrize("M,N,K", [(1024, 300, 512), (2048, 512, 1024), (640, 448, 768), (3072, 273, 3072),
                                   (1024, 384, 1024), (16384, 288, 3072), (640, 257, 512)])
def test_gemm_two_row_tiles(tiny_dev, monkeypatch, M, N, K):
    """257..384 rows: one n-tile, two MMAs per k-step (N = 256 + rest);
    385..512 rows: the decode GEMM splits the rows over two n-tiles."""
    monkeypatch.setenv("VOX_GEMM_PACKED_TEST", "1")
    rng = np.random.default_rng(M + N)
    w = bf16_round(rng.uniform(-1, 1, size=(M, K)).astype(np.float32))
    x = bf16_round(rng.uniform(-1, 1, size=(N, K)).astype(np.float32))
    out, _ = tiny_dev.gemm_test(_bits(w), _bits(x), None, 1)
    ref = x.astype(np.float64) @ w.astype(np.float64).T
    assert np.abs(out - ref).max() < 1e-3 * np.sqrt(K)


@pytest.mark.parametrize("M,N,K", [(256, 4096, 256), (768, 5000, 256), (1024, 3000, 1024), (80, 2500, 512),
                                   (384, 4100, 768)])
@pytest.mark.parametrize("mt", [1, 2])
def test_gemm_persistent(tiny_dev, monkeypatch, M, N, K, mt):
    """The codec detokenizers' persistent many-tile GEMM (gemm_persist_kernel): TMA ring
    across tiles, double-buffered TMEM, direct epilogue with bias; ragged M and N tails."""
    monkeypatch.setenv("VOX_GEMM_PERSIST_TEST", str(mt))
    rng = np.random.default_rng(M + N + K + mt)
    w = bf16_round(rng.uniform(-1, 1, size=(M, K)).astype(np.float32))
    x = bf16_round(rng.uniform(-1, 1, size=(N, K)).astype(np.float32))
    bias = rng.uniform(-1, 1, size=M).astype(np.float32)
    out, _ = tiny_dev.gemm_test(_bits(w), _bits(x), bias, 1)
    ref = x.astype(np.float64) @ w.astype(np.float64).T + bias
    assert np.abs(out - ref).max() < 1e-3 * np.sqrt(K)
