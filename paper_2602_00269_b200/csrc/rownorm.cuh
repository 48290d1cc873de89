// rownorm.cuh -- split-K reduce + residual add + RMSNorm of one activation row,
// shared by resid_norm_kernel (lm_kernels.cu) and the decode GEMM's fused norm
// prologue (gemm_tc.cu), so both produce bit-identical rows.
#pragma once
#include "common.cuh"

namespace vox {

VOX_DEV float block_sum256(float v, float* red) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) red[w] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    float t = (l < 8) ? red[l] : 0.f;
    t = warp_sum(t);
    if (l == 0) red[8] = t;
  }
  __syncthreads();
  return red[8];
}

// block-wide sum for blockDim.x <= 1024 (multiple of 32); red holds >= 33 floats
VOX_DEV float block_sum_any(float v, float* red) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31, nw = blockDim.x >> 5;
  if (l == 0) red[w] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    float t = (l < nw) ? red[l] : 0.f;
    t = warp_sum(t);
    if (l == 0) red[32] = t;
  }
  __syncthreads();
  return red[32];
}

VOX_DEV float4 add4(float4 a, float4 b) { return make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w); }

// sum of the split-K partial planes at float4 index i (fixed split order).  The
// plane loads are issued G at a time before the first add so their L2 latencies
// overlap (a plain running sum serialises one L2 round trip per plane); the
// additions still run plane 0, 1, 2, ... so the result is bit-identical.
template <int G = 4>
VOX_DEV float4 sum_splits4(const float4* __restrict__ w, int splits, int64_t split_stride4,
                           int64_t i) {
  float4 a = w[i];
  for (int s0 = 1; s0 < splits; s0 += G) {
    float4 t[G];
#pragma unroll
    for (int u = 0; u < G; ++u)
      if (s0 + u < splits) t[u] = w[(s0 + u) * split_stride4 + i];
#pragma unroll
    for (int u = 0; u < G; ++u)
      if (s0 + u < splits) a = add4(a, t[u]);
  }
  return a;
}

VOX_DEV void store_bf16x4(bf16* dst, float a, float b, float c, float d) {
  __nv_bfloat162 lo = __floats2bfloat162_rn(a, b);
  __nv_bfloat162 hi = __floats2bfloat162_rn(c, d);
  uint2 u;
  u.x = *reinterpret_cast<uint32_t*>(&lo);
  u.y = *reinterpret_cast<uint32_t*>(&hi);
  *reinterpret_cast<uint2*>(dst) = u;
}

// x = bf16(h * inv * w) in the oracle's rounding order (two fp32 products)
VOX_DEV void norm_store4(bf16* x, float4 h, float inv, float4 w) {
  store_bf16x4(x, __fmul_rn(__fmul_rn(h.x, inv), w.x), __fmul_rn(__fmul_rn(h.y, inv), w.y),
               __fmul_rn(__fmul_rn(h.z, inv), w.z), __fmul_rn(__fmul_rn(h.w, inv), w.w));
}

// h[r] += sum of the split planes at row r; x_out[orow] = bf16(h * rsqrt(mean(h^2) + eps) * nw)
// (orow < 0: h only).  Any blockDim.x that is a multiple of 32, <= 1024; red >= 33 floats.
VOX_DEV void resid_norm_row(int r, const float* __restrict__ ws, int splits, int64_t split_stride,
                            int d, float eps, float* __restrict__ h, const float* __restrict__ nw,
                            bf16* __restrict__ x_out, int orow, float* red) {
  float4* h4 = reinterpret_cast<float4*>(h + static_cast<int64_t>(r) * d);
  const float4* w4 = reinterpret_cast<const float4*>(ws + static_cast<int64_t>(r) * d);
  const int64_t ss4 = split_stride / 4;
  const int d4 = d / 4;
  const int nt = blockDim.x;
  float ss = 0.f;
#pragma unroll 4
  for (int i = threadIdx.x; i < d4; i += nt) {
    const float4 v = add4(h4[i], sum_splits4(w4, splits, ss4, i));
    h4[i] = v;
    ss = fmaf(v.x, v.x, ss);
    ss = fmaf(v.y, v.y, ss);
    ss = fmaf(v.z, v.z, ss);
    ss = fmaf(v.w, v.w, ss);
  }
  ss = block_sum_any(ss, red);
  if (orow < 0) return;
  const float inv = 1.0f / sqrtf(ss / static_cast<float>(d) + eps);
  const float4* n4 = reinterpret_cast<const float4*>(nw);
  bf16* xr = x_out + static_cast<int64_t>(orow) * d;
  for (int i = threadIdx.x; i < d4; i += nt) norm_store4(xr + 4 * i, h4[i], inv, n4[i]);
}

}  // namespace vox
