// codec_common.cuh — kernels shared by the streaming codec decoders (K7 mimi.cu,
// K8 cosy_detok.cu): per-stream row segments, parity-double-buffered state, LayerNorm,
// GELU, causal-conv im2col with cached history, history update, and the tcgen05 GEMM
// call (gemm_tc.cu) on plain row-major bf16 weights.
#pragma once
#include <cstdlib>
#include <cuda.h>

#include <string>

#include "common.cuh"
#include "kernels.h"

namespace vox {
namespace {

// one stream's rows in a call: at a level with u rows per unit (frame / mel frame),
// stream rows are [f_off * u, (f_off + nf) * u); pos0 = its first unit's position
struct SegDev {
  int32_t slot, f_off, nf, parity, pos0, aux, pad_[2];
};

enum : int { kActNone = 0, kActElu = 1, kActLeaky = 2 };

struct StateView {  // one slot's state, parity half `p` read, `1 - p` written
  float* base;
  int64_t slot_floats, half;
  VOX_DEV const float* in(const SegDev& q, int64_t off) const {
    return base + q.slot * slot_floats + q.parity * half + off;
  }
  VOX_DEV float* out(const SegDev& q, int64_t off) const {
    return base + q.slot * slot_floats + (1 - q.parity) * half + off;
  }
};

VOX_DEV float elu(float x) { return x > 0.f ? x : expm1f(x); }

template <int NT>
VOX_DEV float block_sum(float v, float* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < NT / 32; ++i) s += red[i];
  return s;
}

VOX_DEV float act_fn(float x, int act, float slope) {
  return act == kActElu ? elu(x) : act == kActLeaky ? (x > 0.f ? x : slope * x) : x;
}

// h (+= ls * tmp) ; x = bf16(LayerNorm(h) * w + b).  One warp per row, NV = D / 32 values
// per lane held in registers (D in {256, 512, 1024}).
template <int NV>
__global__ void __launch_bounds__(128) codec_ln_kernel(float* __restrict__ h, const float* __restrict__ tmp,
                                                      const float* __restrict__ ls, const float* __restrict__ w,
                                                      const float* __restrict__ b, bf16* __restrict__ x, float eps,
                                                      int64_t rows) {
  constexpr int D = NV * 32;
  const int64_t r = static_cast<int64_t>(blockIdx.x) * 4 + (threadIdx.x >> 5);
  if (r >= rows) return;
  const int lane = threadIdx.x & 31;
  float v[NV];
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int c = lane + 32 * i;
    float a = h[r * D + c];
    if (tmp != nullptr) {
      a = a + ls[c] * tmp[r * D + c];
      h[r * D + c] = a;
    }
    v[i] = a;
    s += a;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  const float mean = s / static_cast<float>(D);
  float ss = 0.f;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    v[i] -= mean;
    ss += v[i] * v[i];
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  const float sd = sqrtf(ss / static_cast<float>(D) + eps);
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int c = lane + 32 * i;
    x[r * D + c] = f32_to_bf16(v[i] / sd * w[c] + b[c]);
  }
}

inline void launch_codec_ln(float* h, const float* tmp, const float* ls, const float* w, const float* b, bf16* x,
                            int D, float eps, int64_t rows, cudaStream_t st) {
  const unsigned grid = static_cast<unsigned>((rows + 3) / 4);
  switch (D) {
    case 256: codec_ln_kernel<8><<<grid, 128, 0, st>>>(h, tmp, ls, w, b, x, eps, rows); break;
    case 512: codec_ln_kernel<16><<<grid, 128, 0, st>>>(h, tmp, ls, w, b, x, eps, rows); break;
    case 768: codec_ln_kernel<24><<<grid, 128, 0, st>>>(h, tmp, ls, w, b, x, eps, rows); break;
    default: codec_ln_kernel<32><<<grid, 128, 0, st>>>(h, tmp, ls, w, b, x, eps, rows); break;
  }
}

__global__ void codec_gelu_kernel(const float* __restrict__ x, bf16* __restrict__ y, int64_t n) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) {
    const float v = x[i];
    y[i] = f32_to_bf16(0.5f * v * (1.f + erff(v * 0.70710678118654752f)));
  }
}

// Causal-conv operand: out[r][j*C + c] = act(x[t - (k-1) + j][c]) (history rows of
// the previous chunk for negative indices), zero for cols >= k*C (K padding).
__global__ void codec_im2col_kernel(const float* __restrict__ x, int C, int k, int act, float slope, int Kp, int u,
                                   const int32_t* __restrict__ frame_req, const SegDev* __restrict__ reqs,
                                   StateView sv, int64_t off, int64_t rows, bf16* __restrict__ out) {
  const int chunks = Kp / 8;
  const int64_t idx = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (idx >= rows * chunks) return;
  const int64_t r = idx / chunks;
  const int col0 = static_cast<int>(idx % chunks) * 8;
  uint4 pk = make_uint4(0, 0, 0, 0);
  if (col0 < k * C) {
    const SegDev q = reqs[frame_req[r / u]];
    const int64_t t = r - static_cast<int64_t>(q.f_off) * u;
    const int j = col0 / C, c0 = col0 % C;
    const int64_t src = t - (k - 1) + j;
    const float* p = src >= 0 ? x + (r - t + src) * C + c0 : sv.in(q, off) + ((k - 1) + src) * C + c0;
    const float4 a = *reinterpret_cast<const float4*>(p);
    const float4 b = *reinterpret_cast<const float4*>(p + 4);
    float v[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
    __nv_bfloat162 h2[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float v0 = act_fn(v[2 * i], act, slope);
      const float v1 = act_fn(v[2 * i + 1], act, slope);
      h2[i] = __floats2bfloat162_rn(v0, v1);
    }
    pk = *reinterpret_cast<uint4*>(h2);
  }
  *reinterpret_cast<uint4*>(out + r * Kp + col0) = pk;
}

// next chunk's history: the last k-1 rows of (old history ++ this chunk's rows)
__global__ void codec_hist_kernel(const float* __restrict__ x, int C, int k, int u,
                                 const SegDev* __restrict__ reqs, StateView sv, int64_t off) {
  const SegDev q = reqs[blockIdx.x];
  const int64_t n = static_cast<int64_t>(q.nf) * u, ro = static_cast<int64_t>(q.f_off) * u;
  for (int e = threadIdx.x; e < (k - 1) * C; e += blockDim.x) {
    const int m = e / C, c = e % C;
    const int64_t src = n - (k - 1) + m;
    sv.out(q, off)[e] = src >= 0 ? x[(ro + src) * C + c] : sv.in(q, off)[((k - 1) + src) * C + c];
  }
}


// out[rows, M] (+bias, +resid) = x[rows, K] . W[M, K]^T on the 1-CTA tcgen05 kernel, one split
// gelu_out != null: the epilogue writes bf16(GELU(acc + bias)) there ([rows][M]) instead of fp32 out
inline cudaError_t codec_gemm(const CUtensorMap& tw, int M, const bf16* x, int K, int64_t rows, float* out,
                              int64_t ldo, const float* bias, const float* resid, int64_t ldr, cudaStream_t st,
                              int64_t* launches, bf16* gelu_out = nullptr) {
  if (rows <= 0) return cudaSuccess;
  // many-row GEMMs: 128-row activation tiles (3-stage, 96 KB ring, 128 TMEM
  // columns) so two CTAs share an SM and one's epilogue overlaps the other's
  // loads and MMAs (the 256-row tile ran one CTA per SM, load -> MMA -> epilogue
  // serialised per wave)
  const int bn = gemm_bn_for_rows(static_cast<int>(rows < 128 ? rows : 128));
  CUtensorMap tx;
  if (!make_tmap_bf16(&tx, x, K, rows, static_cast<uint64_t>(K) * 2, bn)) return cudaErrorInvalidValue;
  GemmArgs a{};
  a.M = M;
  a.N = static_cast<int>(rows);
  a.K = K;
  a.out = out;
  a.ldo = ldo;
  a.split_stride = rows * ldo;
  a.bias = bias;
  a.resid = resid;
  a.ldr = ldr;
  a.m_valid = M;
  if (gelu_out != nullptr) {
    a.epi = 2;
    a.act = gelu_out;
    a.ld_act = M;
  }
  ++*launches;
  // many tiles: the persistent kernel (epilogue of tile t overlaps tile t+1)
  // (M >= 256: 256-row weight tiles, so each activation stage feeds two MMAs)
  static const int persist = getenv("VOX_CODEC_PERSIST") ? atoi(getenv("VOX_CODEC_PERSIST")) : 2;
  const int64_t tiles = (rows + bn - 1) / bn * ((M + 127) / 128);
  if (persist > 0 && bn == 128 && tiles >= 2 * kNumSMs)
    return gemm_launch_persist(tw, tx, a, bn, (persist == 2 && M >= 256) ? 2 : 1, st);
  return gemm_launch(tw, tx, a, 1, bn, 1, st);
}

inline bool codec_wmap(CUtensorMap* t, const bf16* w, int M, int K) {
  return make_tmap_bf16(t, w, K, M, static_cast<uint64_t>(K) * 2, 128);
}

}  // namespace
}  // namespace vox
