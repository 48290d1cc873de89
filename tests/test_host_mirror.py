"""CPU: the numpy oracle reproduces the device init/prompt arithmetic bit-for-bit.

A host-only probe is compiled with nvcc from the SAME header the kernels use
(csrc/common.cuh: mix64, tensor_key, unit_pm1) and its output is compared with
oracle/weights.py — no GPU needed.
"""

import shutil
import subprocess
from pathlib import Path

import numpy as np
import pytest

from oracle import weights as ow
from oracle.workload import prompt_ids, request_seed

ROOT = Path(__file__).resolve().parent.parent
PROBE = r"""
#include <cstdio>
#include <cmath>
#include <cuda_bf16.h>
#include "common.cuh"
using namespace vox;
int main() {
  const uint64_t keys[3] = {tensor_key(1234, 1, 0), tensor_key(1234, 5, 1), tensor_key(7, 130, 11)};
  for (int t = 0; t < 3; ++t) {
    printf("%llu\n", (unsigned long long)keys[t]);
    for (int i = 0; i < 8; ++i) {
      float u = unit_pm1(mix64(keys[t] + (uint64_t)i));
      float v = u * std::sqrt(3.0f / 256);
      __nv_bfloat16 b = __float2bfloat16_rn(v);
      printf("%.9g %.9g\n", u, __bfloat162float(b));
    }
  }
  // prompt ids (csrc/vox_api.cu:prompt_id)
  uint64_t rs = 0x1234567890abcdefull;
  for (int i = 0; i < 4; ++i)
    printf("%llu\n", (unsigned long long)(mix64(rs + 0x632BE59BD9B4E019ull * (uint64_t)(i + 1)) % 128000ull));
  return 0;
}
"""


@pytest.fixture(scope="module")
def probe_out(tmp_path_factory):
    nvcc = shutil.which("nvcc") or "/usr/local/cuda/bin/nvcc"
    if not Path(nvcc).exists():
        pytest.skip("nvcc not available")
    d = tmp_path_factory.mktemp("probe")
    src = d / "probe.cu"
    src.write_text(PROBE)
    exe = d / "probe"
    subprocess.run([nvcc, "-std=c++17", "-I", str(ROOT / "paper_2602_00269_b200" / "csrc"), "-o", str(exe), str(src)],
                   check=True, capture_output=True)
    return subprocess.run([str(exe)], check=True, capture_output=True, text=True).stdout.split()


def test_init_mirror_bit_exact(probe_out):
    it = iter(probe_out)
    for seed, tid, layer in [(1234, 1, 0), (1234, 5, 1), (7, 130, 11)]:
        key = ow.tensor_key(seed, tid, layer)
        assert int(next(it)) == key
        u = ow.unit_pm1(8, key)
        b = ow.init_bf16(8, key, np.sqrt(np.float32(3.0) / np.float32(256)))
        for i in range(8):
            assert np.float32(float(next(it))) == u[i]
            assert np.float32(float(next(it))) == b[i]


def test_prompt_ids_mirror(probe_out):
    tail = [int(x) for x in probe_out[-4:]]
    assert tail == prompt_ids(0x1234567890ABCDEF, 4, 128000)


def test_request_seed_matches_reference():
    from paper_2602_00269_b200._ref import model_api

    for rid in range(20):
        assert request_seed(3, rid) == model_api.request_seed(3, rid)


def test_bf16_round_matches_torch():
    torch = pytest.importorskip("torch")
    x = np.random.default_rng(0).normal(size=4096).astype(np.float32) * 3
    ref = torch.from_numpy(x).to(torch.bfloat16).to(torch.float32).numpy()
    assert np.array_equal(ow.bf16_round(x), ref)
