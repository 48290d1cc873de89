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

// Same values as init_bf16_kernel for the logical matrix W[row0 + m][k] (row
// stride K), written in the UMMA-ready PACKED layout the GEMM streams:
//   [M/128 tiles][K/64 k-blocks][128 rows][64 cols], each 16 KB tile already in
//   the 128B-swizzled K-major shared-memory layout (16-byte chunk c of row r is
//   stored at chunk c ^ (r & 7)).  Rows beyond M (tile padding) are zero.
// One k-block of one 128-row tile is then a single contiguous 16 KB bulk copy
// (sequential DRAM bursts) instead of 128 strided 128-byte rows.
// half > 0: gate|up interleave -- packed row r of tile t holds logical row
// (r < 64 ? 64 t + r : half + 64 t + r - 64), so each 128-row tile carries the
// gate and up rows of the same 64 features (fused SiLU(gate) * up epilogue).
__device__ __forceinline__ int64_t packed_logical_row(int64_t m, int64_t half) {
  if (half <= 0) return m;
  const int64_t t = m >> 7, r = m & 127;
  return r < 64 ? 64 * t + r : half + 64 * t + (r - 64);
}

__global__ void init_bf16_packed_kernel(bf16* __restrict__ w, int64_t M, int64_t K,
                                        int64_t row0, uint64_t key, float scale, int64_t half) {
  const int64_t n_kb = K / 64;
  const int64_t total = (M + 255) / 256 * 256 * K;  // = packed_elems(M, K)
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; j < total;
       j += stride) {
    const int64_t t = j >> 13, within = j & 8191;
    const int r = static_cast<int>(within >> 6);
    const int c = static_cast<int>((within >> 3) & 7) ^ (r & 7);
    const int e = static_cast<int>(within & 7);
    const int64_t m = (t / n_kb) * 128 + r;
    const int64_t k = (t % n_kb) * 64 + c * 8 + e;
    float v = 0.f;
    if (m < M) {
      const int64_t ml = packed_logical_row(m, half);
      v = __fmul_rn(unit_pm1(mix64(key + static_cast<uint64_t>((row0 + ml) * K + k))), scale);
    }
    w[j] = __float2bfloat16_rn(v);
  }
}

void launch_init_bf16_packed(bf16* w, int64_t M, int64_t K, int64_t row0, uint64_t key,
                             float scale, cudaStream_t st, int64_t interleave_half) {
  init_bf16_packed_kernel<<<148 * 64, 256, 0, st>>>(w, M, K, row0, key, scale, interleave_half);
}

// logical [M][K] -> packed tiles (same layout as init_bf16_packed_kernel)
__global__ void pack_bf16_kernel(const bf16* __restrict__ src, bf16* __restrict__ dst, int64_t M,
                                 int64_t K) {
  const int64_t n_kb = K / 64;
  const int64_t total = (M + 255) / 256 * 256 * K;  // = packed_elems(M, K)
  for (int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; j < total;
       j += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t t = j >> 13, within = j & 8191;
    const int r = static_cast<int>(within >> 6);
    const int c = static_cast<int>((within >> 3) & 7) ^ (r & 7);
    const int64_t m = (t / n_kb) * 128 + r;
    const int64_t k = (t % n_kb) * 64 + c * 8 + (within & 7);
    dst[j] = m < M ? src[m * K + k] : __float2bfloat16_rn(0.f);
  }
}

void launch_pack_bf16(const bf16* src, bf16* dst, int64_t M, int64_t K, cudaStream_t st) {
  pack_bf16_kernel<<<148 * 16, 256, 0, st>>>(src, dst, M, K);
}

// Reads `bytes` (multiple of 16) and writes one word per block: leaves L2
// holding clean lines of an unrelated buffer (microbenchmark L2 flush).
__global__ void l2_flush_kernel(const uint4* __restrict__ p, int64_t n, uint32_t* sink) {
  uint32_t acc = 0;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const uint4 v = p[i];
    acc ^= v.x ^ v.y ^ v.z ^ v.w;
  }
  if (acc == 0x9E3779B9u) sink[blockIdx.x] = acc;  // practically never: keeps the loads live
}

void launch_l2_flush(const void* buf, size_t bytes, uint32_t* sink, cudaStream_t st) {
  l2_flush_kernel<<<148 * 8, 512, 0, st>>>(static_cast<const uint4*>(buf),
                                           static_cast<int64_t>(bytes / 16), sink);
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
