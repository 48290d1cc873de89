// init.cu — seeded, counter-based random-init weights.
//
// w[i] = bf16_rn(unit_pm1(mix64(key + i)) * scale): one IEEE fp32 multiply
// and one RNE rounding, so oracle/weights.py reproduces every element
// bit-for-bit on the CPU (no Box-Muller, no FMA contraction).
#include "common.cuh"
#include "kernels.h"

namespace vox {

__global__ void init_bf16_kernel(bf16* __restrict__ w, int64_t n, uint64_t key, float scale) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += stride) {
    const float u = unit_pm1(mix64(key + static_cast<uint64_t>(i)));
    w[i] = __float2bfloat16_rn(__fmul_rn(u, scale));
  }
}

__global__ void init_f32_kernel(float* __restrict__ w, int64_t n, uint64_t key, float scale,
                                float offset) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += stride) {
    const float u = unit_pm1(mix64(key + static_cast<uint64_t>(i)));
    const float v = __fadd_rn(__fmul_rn(u, scale), offset);
    w[i] = __bfloat162float(__float2bfloat16_rn(v));
  }
}

void launch_init_bf16(bf16* w, int64_t n, uint64_t key, float scale, cudaStream_t st) {
  const int64_t blocks = (n + 255) / 256;
  init_bf16_kernel<<<static_cast<int>(blocks < 148 * 64 ? blocks : 148 * 64), 256, 0, st>>>(
      w, n, key, scale);
}

void launch_init_f32(float* w, int64_t n, uint64_t key, float scale, float offset,
                     cudaStream_t st) {
  const int64_t blocks = (n + 255) / 256;
  init_f32_kernel<<<static_cast<int>(blocks < 148 * 64 ? blocks : 148 * 64), 256, 0, st>>>(
      w, n, key, scale, offset);
}

}  // namespace vox
