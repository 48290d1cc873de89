// cosy_detok.cu — K8: CosyVoice2-style chunked detokenizer (BASELINE config 4): token-to-mel
// flow matching + HiFT-style vocoder, restated in oracle/cosy_detok.py (public CosyVoice2
// architecture; "a flow-matching module built on Transformer layers and a
// HiFi-GAN vocoder") at the chunking VoxServe uses (every call consumes the
// request's reference tokens plus the chunk's new tokens; profiles.py:135
// ref_window_tokens = 50).  Replaces the reference's stub detokenizer
// (profiles.py:333-356) for the cosy_like profile (profiles.py:163-179).
//
// One decode call over n requests with C_i new tokens each:
//   flow (rows per request: T_i = ref + C_i tokens, 2 T_i mel frames, x2 for CFG)
//     cd_embed -> enc_layers x {LN, QKV GEMM, cd_rope, cd_attn (full, per request),
//     O GEMM (+h), LN, fc1 GEMM, GELU, fc2 GEMM (+h)} -> LN -> mu GEMM
//     cd_noise (x0, keyed by request seed + call index)
//     n_steps x {cd_est_in (cond | uncond operand) -> in GEMM (+ b_in + temb(t_i)) ->
//                est_layers x {...} -> LN -> out GEMM -> cd_euler (CFG combine, x += dt v)}
//   vocoder (stateful per request: conv histories + iSTFT overlap tail, chunk parity):
//     cd_gather_mel -> k7 conv -> per ratio {LReLU ConvT GEMM, residual block} ->
//     k7 conv_post GEMM -> cd_istft_frames -> cd_ola (+ history)
// Every GEMM is the tcgen05/TMEM/TMA kernel of gemm_tc.cu; every conv is an im2col
// operand (codec_common.cuh) + that GEMM.
#include <cuda.h>

#include <algorithm>
#include <map>
#include <tuple>
#include <cmath>
#include <mutex>
#include <string>
#include <vector>

#include "codec_common.cuh"

namespace vox {
namespace {

enum : uint64_t {
  T_CD_EMB = 400, T_CD_ENC = 401, T_CD_ELNFW = 409, T_CD_ELNFB = 410, T_CD_MU = 411, T_CD_MUB = 412,
  T_CD_SPK = 413, T_CD_REFTOK = 414, T_CD_REFMEL = 415, T_CD_NOISE = 416,
  T_CD_IN = 420, T_CD_INB = 421, T_CD_T1 = 422, T_CD_T1B = 423, T_CD_T2 = 424, T_CD_T2B = 425,
  T_CD_EST = 430, T_CD_OLNW = 438, T_CD_OLNB = 439, T_CD_OUT = 440, T_CD_OUTB = 441,
  T_CD_VPRE = 450, T_CD_VPREB = 451, T_CD_UPW = 452, T_CD_UPB = 453,
  T_CD_R1W = 454, T_CD_R1B = 455, T_CD_R2W = 456, T_CD_R2B = 457, T_CD_VPOST = 458, T_CD_VPOSTB = 459,
};

constexpr int kCdMaxGraphs = 64;  // call shapes kept as CUDA graphs
constexpr int kCdMaxRows = 256;  // rows of one attention group (2 * (ref + max_chunk))

VOX_DEV uint64_t seg_key(const SegDev& q) {
  return static_cast<uint64_t>(static_cast<uint32_t>(q.pad_[0])) |
         (static_cast<uint64_t>(static_cast<uint32_t>(q.pad_[1])) << 32);
}

// token rows: [ref tokens of the slot | the call's new tokens]; aux = offset of the
// request's new tokens in the staged token array
__global__ void __launch_bounds__(128) cd_embed_kernel(const int32_t* __restrict__ row_seg,
                                                       const SegDev* __restrict__ seg, const int32_t* __restrict__ reftok,
                                                       int ref, const int32_t* __restrict__ newtok,
                                                       const float* __restrict__ emb, int D, float* __restrict__ h) {
  const int64_t r = blockIdx.x;
  const SegDev q = seg[row_seg[r]];
  const int t = static_cast<int>(r - q.f_off);
  const int tok = t < ref ? reftok[q.slot * ref + t] : newtok[q.aux + t - ref];
  for (int c = threadIdx.x; c < D; c += blockDim.x) h[r * D + c] = emb[static_cast<int64_t>(tok) * D + c];
}

// Full (bidirectional) attention inside each segment with RoPE (rotate-half, position =
// row index in the segment) applied while staging: one CTA (8 warps) per (segment, head);
// the head's K (row stride hd + 1: conflict-free column reads) and V live in shared
// memory, each warp takes 4 queries at a time (every K/V element read from smem feeds 4
// query FMAs).  hd <= 64, segment rows <= kCdMaxRows.
constexpr int kAttnQ = 4;
__global__ void __launch_bounds__(256) cd_attn_kernel(const float* __restrict__ qkv, const SegDev* __restrict__ seg,
                                                      int D, int hd, const float* __restrict__ inv_freq,
                                                      bf16* __restrict__ out) {
  extern __shared__ float sm[];
  const SegDev q = seg[blockIdx.x];
  const int hh = blockIdx.y;
  const int n = q.nf, half = hd / 2, ks = hd + 1;
  float* Ks = sm;                       // [n][hd + 1]
  float* Vs = Ks + n * ks;              // [n][hd]
  float* Ps = Vs + n * hd;              // [8][kAttnQ][n]
  float* Qs = Ps + 8 * kAttnQ * n;      // [8][kAttnQ][hd]
  const float* base = qkv + static_cast<int64_t>(q.f_off) * 3 * D + hh * hd;
  for (int e = threadIdx.x; e < n * half; e += blockDim.x) {
    const int j = e / half, i = e % half;
    float sn, cs;
    sincosf(static_cast<float>(j) * inv_freq[i], &sn, &cs);
    const float* kr = base + static_cast<int64_t>(j) * 3 * D + D;
    const float k0 = kr[i], k1 = kr[i + half];
    Ks[j * ks + i] = k0 * cs - k1 * sn;
    Ks[j * ks + i + half] = k1 * cs + k0 * sn;
  }
  for (int e = threadIdx.x; e < n * hd; e += blockDim.x) {
    const int j = e / hd, d = e % hd;
    Vs[e] = base[static_cast<int64_t>(j) * 3 * D + 2 * D + d];
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const float scale = rsqrtf(static_cast<float>(hd));
  float* P = Ps + warp * kAttnQ * n;
  float* Q = Qs + warp * kAttnQ * hd;
  for (int t0 = warp * kAttnQ; t0 < n; t0 += 8 * kAttnQ) {
    for (int e = lane; e < kAttnQ * half; e += 32) {
      const int qi = e / half, i = e % half, t = t0 + qi;
      float q0 = 0.f, q1 = 0.f, sn = 0.f, cs = 1.f;
      if (t < n) {
        const float* qr = base + static_cast<int64_t>(t) * 3 * D;
        q0 = qr[i];
        q1 = qr[i + half];
        sincosf(static_cast<float>(t) * inv_freq[i], &sn, &cs);
      }
      Q[qi * hd + i] = q0 * cs - q1 * sn;
      Q[qi * hd + i + half] = q1 * cs + q0 * sn;
    }
    __syncwarp();
    float mx[kAttnQ];
#pragma unroll
    for (int qi = 0; qi < kAttnQ; ++qi) mx[qi] = -INFINITY;
    for (int j = lane; j < n; j += 32) {
      float s[kAttnQ] = {};
      const float* kr = Ks + j * ks;
      for (int d = 0; d < hd; ++d) {
        const float kv = kr[d];
#pragma unroll
        for (int qi = 0; qi < kAttnQ; ++qi) s[qi] += Q[qi * hd + d] * kv;
      }
#pragma unroll
      for (int qi = 0; qi < kAttnQ; ++qi) {
        P[qi * n + j] = s[qi] * scale;
        mx[qi] = fmaxf(mx[qi], s[qi] * scale);
      }
    }
    float sum[kAttnQ];
#pragma unroll
    for (int qi = 0; qi < kAttnQ; ++qi) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) mx[qi] = fmaxf(mx[qi], __shfl_xor_sync(0xffffffffu, mx[qi], o));
      sum[qi] = 0.f;
    }
    for (int j = lane; j < n; j += 32)
#pragma unroll
      for (int qi = 0; qi < kAttnQ; ++qi) {
        const float e = __expf(P[qi * n + j] - mx[qi]);
        P[qi * n + j] = e;
        sum[qi] += e;
      }
#pragma unroll
    for (int qi = 0; qi < kAttnQ; ++qi)
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) sum[qi] += __shfl_xor_sync(0xffffffffu, sum[qi], o);
    __syncwarp();
    for (int d = lane; d < hd; d += 32) {
      float o[kAttnQ] = {};
      for (int j = 0; j < n; ++j) {
        const float vv = Vs[j * hd + d];
#pragma unroll
        for (int qi = 0; qi < kAttnQ; ++qi) o[qi] += P[qi * n + j] * vv;
      }
#pragma unroll
      for (int qi = 0; qi < kAttnQ; ++qi)
        if (t0 + qi < n) out[(static_cast<int64_t>(q.f_off) + t0 + qi) * D + hh * hd + d] = f32_to_bf16(o[qi] / sum[qi]);
    }
    __syncwarp();
  }
}

inline size_t cd_attn_smem(int n, int hd) {
  return sizeof(float) * (static_cast<size_t>(n) * (hd + 1) + static_cast<size_t>(n) * hd + 8 * kAttnQ * n +
                          8 * kAttnQ * hd);
}

// ---------------------------------------------------------------------------
// Tensor-core variant (hd = 64): mma.sync m16n8k16 bf16 -> fp32, flash-style online
// softmax over 64-key blocks.  One CTA (8 warps) per (segment, head): RoPE'd K staged as
// bf16 [key][72] (B operand of S = Q K^T: 32-bit fragment loads, conflict-free), V staged
// transposed as bf16 [dim][npad + 8] (B operand of O = P V); each warp takes 16 query rows
// at a time, P goes from the S accumulators straight into A fragments (no smem).
// Rounding: Q, K, V and P in bf16, scores / softmax / O in fp32 (the estimator's GEMM
// operands are bf16 too).
// ---------------------------------------------------------------------------
VOX_DEV void mma16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};\n"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
VOX_DEV uint32_t pack2(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

constexpr int kTcHd = 64, kTcKs = 72;
inline int cd_tc_npad(int n) { return (n + 63) / 64 * 64; }
// one warp per 16 query rows of the longest segment (<= 16 warps)
inline int cd_attn_tc_warps(int n) { const int w = (n + 15) / 16; return w < 1 ? 1 : (w > 16 ? 16 : w); }
inline size_t cd_attn_tc_smem(int n) {
  const int np = cd_tc_npad(n);
  return 2 * (static_cast<size_t>(np) * kTcKs + static_cast<size_t>(kTcHd) * (np + 8) +
              static_cast<size_t>(cd_attn_tc_warps(n)) * 16 * kTcKs);
}
// RoPE (cos, sin) table [kCdMaxRows][hd / 2], filled once with the same sincosf
// expression the attention kernels used per element (bit-identical values)
__global__ void cd_rope_table_kernel(const float* __restrict__ inv_freq, int half, float2* __restrict__ tab) {
  const int j = blockIdx.x, i = threadIdx.x;
  if (i < half) {
    float sn, cs;
    sincosf(static_cast<float>(j) * inv_freq[i], &sn, &cs);
    tab[j * half + i] = make_float2(cs, sn);
  }
}

__global__ void __launch_bounds__(512) cd_attn_tc_kernel(const float* __restrict__ qkv, const SegDev* __restrict__ seg,
                                                         int D, const float2* __restrict__ rope,
                                                         bf16* __restrict__ out) {
  extern __shared__ __align__(16) uint8_t smraw[];
  const SegDev q = seg[blockIdx.x];
  const int hh = blockIdx.y;
  const int n = q.nf, np = (n + 63) / 64 * 64, VS = np + 8;
  constexpr int half = kTcHd / 2;
  bf16* Ks = reinterpret_cast<bf16*>(smraw);          // [np][72]
  bf16* Vt = Ks + np * kTcKs;                          // [64][np + 8]
  bf16* Qs = Vt + kTcHd * VS;                          // [8 warps][16][72]
  const float* base = qkv + static_cast<int64_t>(q.f_off) * 3 * D + hh * kTcHd;
  // staging: 4 consecutive dims per thread (float4 loads), loops unrolled so
  // several rows' loads are in flight (the staging is latency-bound otherwise)
#pragma unroll 4
  for (int e = threadIdx.x; e < np * (half / 4); e += blockDim.x) {
    const int j = e / (half / 4), i = (e % (half / 4)) * 4;
    float4 k0 = make_float4(0.f, 0.f, 0.f, 0.f), k1 = k0;
    float2 r[4] = {make_float2(1.f, 0.f), make_float2(1.f, 0.f), make_float2(1.f, 0.f), make_float2(1.f, 0.f)};
    if (j < n) {
      const float* kr = base + static_cast<int64_t>(j) * 3 * D + D;
      k0 = *reinterpret_cast<const float4*>(kr + i);
      k1 = *reinterpret_cast<const float4*>(kr + i + half);
#pragma unroll
      for (int u = 0; u < 4; ++u) r[u] = rope[j * half + i + u];
    }
    const float a0[4] = {k0.x, k0.y, k0.z, k0.w}, a1[4] = {k1.x, k1.y, k1.z, k1.w};
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      Ks[j * kTcKs + i + u] = f32_to_bf16(a0[u] * r[u].x - a1[u] * r[u].y);
      Ks[j * kTcKs + i + u + half] = f32_to_bf16(a1[u] * r[u].x + a0[u] * r[u].y);
    }
  }
#pragma unroll 4
  for (int e = threadIdx.x; e < np * (kTcHd / 4); e += blockDim.x) {
    const int j = e / (kTcHd / 4), d = (e % (kTcHd / 4)) * 4;
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
    if (j < n) v = *reinterpret_cast<const float4*>(base + static_cast<int64_t>(j) * 3 * D + 2 * D + d);
    Vt[d * VS + j] = f32_to_bf16(v.x);
    Vt[(d + 1) * VS + j] = f32_to_bf16(v.y);
    Vt[(d + 2) * VS + j] = f32_to_bf16(v.z);
    Vt[(d + 3) * VS + j] = f32_to_bf16(v.w);
  }
  __syncthreads();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t = lane & 3;
  const int nw = blockDim.x >> 5;
  const float sl2 = rsqrtf(static_cast<float>(kTcHd)) * 1.4426950408889634f;  // scale * log2(e)
  bf16* Q = Qs + warp * 16 * kTcKs;
  for (int t0 = warp * 16; t0 < n; t0 += nw * 16) {
#pragma unroll
    for (int e = lane; e < 16 * (half / 4); e += 32) {
      const int rr = e / (half / 4), i = (e % (half / 4)) * 4, row = t0 + rr;
      float4 q0 = make_float4(0.f, 0.f, 0.f, 0.f), q1 = q0;
      float2 cs[4] = {make_float2(1.f, 0.f), make_float2(1.f, 0.f), make_float2(1.f, 0.f), make_float2(1.f, 0.f)};
      if (row < n) {
        const float* qr = base + static_cast<int64_t>(row) * 3 * D;
        q0 = *reinterpret_cast<const float4*>(qr + i);
        q1 = *reinterpret_cast<const float4*>(qr + i + half);
#pragma unroll
        for (int u = 0; u < 4; ++u) cs[u] = rope[row * half + i + u];
      }
      const float a0[4] = {q0.x, q0.y, q0.z, q0.w}, a1[4] = {q1.x, q1.y, q1.z, q1.w};
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        Q[rr * kTcKs + i + u] = f32_to_bf16(a0[u] * cs[u].x - a1[u] * cs[u].y);
        Q[rr * kTcKs + i + u + half] = f32_to_bf16(a1[u] * cs[u].x + a0[u] * cs[u].y);
      }
    }
    __syncwarp();
    uint32_t qa[4][4];
#pragma unroll
    for (int ks = 0; ks < 4; ++ks) {
      qa[ks][0] = *reinterpret_cast<const uint32_t*>(&Q[g * kTcKs + ks * 16 + 2 * t]);
      qa[ks][1] = *reinterpret_cast<const uint32_t*>(&Q[(g + 8) * kTcKs + ks * 16 + 2 * t]);
      qa[ks][2] = *reinterpret_cast<const uint32_t*>(&Q[g * kTcKs + ks * 16 + 2 * t + 8]);
      qa[ks][3] = *reinterpret_cast<const uint32_t*>(&Q[(g + 8) * kTcKs + ks * 16 + 2 * t + 8]);
    }
    float o[8][4] = {};
    float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;
    for (int kb = 0; kb < np; kb += 64) {
      float sc[8][4] = {};
#pragma unroll
      for (int nt = 0; nt < 8; ++nt) {
        const bf16* kr = Ks + (kb + nt * 8 + g) * kTcKs + 2 * t;
#pragma unroll
        for (int ks = 0; ks < 4; ++ks)
          mma16816(sc[nt], qa[ks], *reinterpret_cast<const uint32_t*>(kr + ks * 16),
                   *reinterpret_cast<const uint32_t*>(kr + ks * 16 + 8));
      }
      float x0 = -INFINITY, x1 = -INFINITY;
#pragma unroll
      for (int nt = 0; nt < 8; ++nt)
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int key = kb + nt * 8 + 2 * t + (e & 1);
          const float v = key < n ? sc[nt][e] * sl2 : -INFINITY;
          sc[nt][e] = v;
          if (e < 2) x0 = fmaxf(x0, v); else x1 = fmaxf(x1, v);
        }
#pragma unroll
      for (int off = 1; off < 4; off <<= 1) {
        x0 = fmaxf(x0, __shfl_xor_sync(0xffffffffu, x0, off));
        x1 = fmaxf(x1, __shfl_xor_sync(0xffffffffu, x1, off));
      }
      const float n0 = fmaxf(m0, x0), n1 = fmaxf(m1, x1);
      const float al0 = exp2f(m0 - n0), al1 = exp2f(m1 - n1);
      m0 = n0;
      m1 = n1;
      l0 *= al0;
      l1 *= al1;
#pragma unroll
      for (int dt = 0; dt < 8; ++dt) {
        o[dt][0] *= al0; o[dt][1] *= al0; o[dt][2] *= al1; o[dt][3] *= al1;
      }
#pragma unroll
      for (int nt = 0; nt < 8; ++nt) {
        sc[nt][0] = exp2f(sc[nt][0] - m0);
        sc[nt][1] = exp2f(sc[nt][1] - m0);
        sc[nt][2] = exp2f(sc[nt][2] - m1);
        sc[nt][3] = exp2f(sc[nt][3] - m1);
        l0 += sc[nt][0] + sc[nt][1];
        l1 += sc[nt][2] + sc[nt][3];
      }
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        const uint32_t pa[4] = {pack2(sc[2 * kk][0], sc[2 * kk][1]), pack2(sc[2 * kk][2], sc[2 * kk][3]),
                                pack2(sc[2 * kk + 1][0], sc[2 * kk + 1][1]),
                                pack2(sc[2 * kk + 1][2], sc[2 * kk + 1][3])};
#pragma unroll
        for (int dt = 0; dt < 8; ++dt) {
          const bf16* vr = Vt + (dt * 8 + g) * VS + kb + kk * 16 + 2 * t;
          mma16816(o[dt], pa, *reinterpret_cast<const uint32_t*>(vr), *reinterpret_cast<const uint32_t*>(vr + 8));
        }
      }
    }
#pragma unroll
    for (int off = 1; off < 4; off <<= 1) {
      l0 += __shfl_xor_sync(0xffffffffu, l0, off);
      l1 += __shfl_xor_sync(0xffffffffu, l1, off);
    }
    const int r0 = t0 + g, r1 = t0 + g + 8;
#pragma unroll
    for (int dt = 0; dt < 8; ++dt) {
      const int d = hh * kTcHd + dt * 8 + 2 * t;
      if (r0 < n)
        *reinterpret_cast<__nv_bfloat162*>(out + (static_cast<int64_t>(q.f_off) + r0) * D + d) =
            __floats2bfloat162_rn(o[dt][0] / l0, o[dt][1] / l0);
      if (r1 < n)
        *reinterpret_cast<__nv_bfloat162*>(out + (static_cast<int64_t>(q.f_off) + r1) * D + d) =
            __floats2bfloat162_rn(o[dt][2] / l1, o[dt][3] / l1);
    }
    __syncwarp();
  }
}

// x0: unit-variance uniform noise, bit-identical to oracle/weights.py:cosy_noise
__global__ void cd_noise_kernel(const int32_t* __restrict__ row_seg, const SegDev* __restrict__ seg, int M,
                                int64_t rows, float* __restrict__ x) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= rows * M) return;
  const int64_t r = i / M;
  const int c = static_cast<int>(i % M);
  const SegDev q = seg[row_seg[r >> 1]];
  const int64_t t = r - 2LL * q.f_off;
  const float u = unit_pm1(mix64(seg_key(q) + static_cast<uint64_t>(t * M + c)));
  x[i] = __bfloat162float(__float2bfloat16_rn(__fadd_rn(__fmul_rn(u, sqrtf(3.0f)), 0.f)));
}

// estimator operand [2 R][4 M] bf16: cond branch rows [x | mu[t/2] | spk | refmel or 0],
// uncond branch rows (R + r) [x | 0 | 0 | 0]
__global__ void cd_est_in_kernel(const float* __restrict__ x, const float* __restrict__ mu,
                                 const int32_t* __restrict__ row_seg, const SegDev* __restrict__ seg,
                                 const float* __restrict__ spk, const float* __restrict__ refmel, int ref, int M,
                                 int64_t R, bf16* __restrict__ out) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= 2 * R * 4 * M) return;
  const int64_t row = i / (4 * M);
  const int col = static_cast<int>(i % (4 * M));
  const bool unc = row >= R;
  const int64_t r = unc ? row - R : row;
  const int part = col / M, c = col % M;
  float v = 0.f;
  if (part == 0) {
    v = x[r * M + c];
  } else if (!unc) {
    const SegDev q = seg[row_seg[r >> 1]];
    const int64_t t = r - 2LL * q.f_off;
    if (part == 1) v = mu[(r >> 1) * M + c];
    else if (part == 2) v = spk[static_cast<int64_t>(q.slot) * M + c];
    else if (t < 2 * ref) v = refmel[(static_cast<int64_t>(q.slot) * 2 * ref + t) * M + c];
  }
  out[i] = f32_to_bf16(v);
}

__global__ void cd_euler_kernel(float* __restrict__ x, const float* __restrict__ v, int64_t n, float dt, float lam) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i < n) x[i] = x[i] + dt * ((1.f + lam) * v[i] - lam * v[n + i]);
}

// vocoder input: the new mel frames of each request (flow rows 2 ref .. 2 T - 1)
__global__ void cd_gather_mel_kernel(const float* __restrict__ x, const int32_t* __restrict__ vrow_seg,
                                     const SegDev* __restrict__ vseg, const SegDev* __restrict__ fseg, int ref,
                                     int M, int64_t rows, float* __restrict__ mel) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= rows * M) return;
  const int64_t r = i / M;
  const int c = static_cast<int>(i % M);
  const int g = vrow_seg[r];
  const int64_t t = r - vseg[g].f_off;
  mel[i] = x[(2LL * fseg[g].f_off + 2 * ref + t) * M + c];
}

// windowed frames of the causal iSTFT: spec rows [J][2 nb] -> wf [J][n_fft]
__global__ void cd_istft_frames_kernel(const float* __restrict__ spec, int nfft, int64_t J, float* __restrict__ wf) {
  const int64_t j = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (j >= J) return;
  const int nb = nfft / 2 + 1;
  float re[16], im[16];
  for (int k = 0; k < nb; ++k) {
    const float mag = fminf(expf(spec[j * 2 * nb + k]), 100.f);
    const float ph = sinf(spec[j * 2 * nb + nb + k]);
    float s, c;
    sincosf(ph, &s, &c);
    re[k] = mag * c;
    im[k] = mag * s;
  }
  const float two_pi_n = 6.283185307179586f / static_cast<float>(nfft);
  for (int t = 0; t < nfft; ++t) {
    float acc = re[0] + ((t & 1) ? -re[nb - 1] : re[nb - 1]);
    for (int k = 1; k < nb - 1; ++k) {
      float s, c;
      sincosf(two_pi_n * static_cast<float>((k * t) % nfft), &s, &c);
      acc += 2.f * (re[k] * c - im[k] * s);
    }
    const float w = 0.5f - 0.5f * cospif(2.f * static_cast<float>(t) / static_cast<float>(nfft));
    wf[j * nfft + t] = w * acc / static_cast<float>(nfft);
  }
}

// overlap-add: sample hop*j + a = sum_q wf[j - q][a + hop q] / env (frames of earlier
// calls from the state, zero before the stream start); one thread per output sample
__global__ void cd_ola_kernel(const float* __restrict__ wf, int nfft, int hop, int u,
                              const int32_t* __restrict__ vrow_seg, const SegDev* __restrict__ vseg, StateView sv,
                              int64_t off, int64_t frames, float* __restrict__ pcm) {
  const int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (i >= frames * hop) return;
  const int64_t j = i / hop;
  const int a = static_cast<int>(i % hop);
  const SegDev q = vseg[vrow_seg[j / u]];
  const int64_t t = j - static_cast<int64_t>(q.f_off) * u;
  const int nq = nfft / hop;
  float acc = 0.f, env = 0.f;
  for (int k = 0; k < nq; ++k) {
    const int idx = a + hop * k;
    const float w = 0.5f - 0.5f * cospif(2.f * static_cast<float>(idx) / static_cast<float>(nfft));
    env += w * w;
    const int64_t src = t - k;
    const float* row = src >= 0 ? wf + (j - k) * nfft : sv.in(q, off) + ((nq - 1) + src) * nfft;
    acc += row[idx];
  }
  pcm[i] = acc / env;
}

// temb(t) + b_in for one ODE step: sinusoid(1000 t) -> t1 -> SiLU -> t2 (one CTA, ds threads)
__global__ void cd_temb_kernel(const float* __restrict__ t1, const float* __restrict__ t1b,
                               const float* __restrict__ t2, const float* __restrict__ t2b,
                               const float* __restrict__ b_in, int ds, float t, float* __restrict__ out) {
  extern __shared__ float sh[];
  float* e = sh;
  float* a = sh + ds;
  const int half = ds / 2;
  for (int i = threadIdx.x; i < half; i += blockDim.x) {
    const float fr = expf(-9.210340371976184f * static_cast<float>(i) / static_cast<float>(half));
    const float arg = 1000.f * t * fr;
    e[i] = sinf(arg);
    e[half + i] = cosf(arg);
  }
  __syncthreads();
  for (int o = threadIdx.x; o < ds; o += blockDim.x) {
    float s = t1b[o];
    for (int k = 0; k < ds; ++k) s += t1[static_cast<int64_t>(o) * ds + k] * e[k];
    a[o] = s / (1.f + expf(-s));
  }
  __syncthreads();
  for (int o = threadIdx.x; o < ds; o += blockDim.x) {
    float s = t2b[o];
    for (int k = 0; k < ds; ++k) s += t2[static_cast<int64_t>(o) * ds + k] * a[k];
    out[o] = s + b_in[o];
  }
}

__global__ void cd_reftok_kernel(int32_t* __restrict__ out, int n, uint64_t key, int vocab) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = static_cast<int32_t>(mix64(key + static_cast<uint64_t>(i)) % static_cast<uint64_t>(vocab));
}

}  // namespace
}  // namespace vox

using namespace vox;

struct CdXf {
  float *ln1w, *ln1b, *ln2w, *ln2b;
  bf16 *qkv, *o, *fc1, *fc2;
  CUtensorMap tm_qkv, tm_o, tm_fc1, tm_fc2;
};
struct CdBlock {
  bf16 *upw, *r1w, *r2w;
  float *upb, *r1b, *r2b;
  CUtensorMap tm_up, tm_r1, tm_r2;
};

struct VoxCosy {
  int device = 0;
  VoxCosyCfg cfg{};
  std::string err;
  cudaStream_t st = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;
  double last_ms = 0.0;
  int64_t launches = 0;
  // one CUDA graph per call shape (requests, token rows, vocoder rows, longest
  // segment): a call is ~700 launches, host-bound at small batches without it
  std::map<std::tuple<int, int64_t, int64_t, int>, cudaGraphExec_t> graphs;
  std::map<std::tuple<int, int64_t, int64_t, int>, int64_t> graph_launches;
  bool no_graphs = getenv("VOX_NO_GRAPH") != nullptr;
  // weights
  float* emb = nullptr;
  std::vector<CdXf> enc, est;
  float *elnfw = nullptr, *elnfb = nullptr, *mub = nullptr, *olnw = nullptr, *olnb = nullptr, *outb = nullptr;
  bf16 *mu = nullptr, *w_in = nullptr, *w_out = nullptr;
  CUtensorMap tm_mu, tm_in, tm_out;
  float* step_bias = nullptr;  // [n_steps][d_est] = b_in + temb(t_i)
  std::vector<float> ts;
  float *inv_enc = nullptr, *inv_est = nullptr;
  float2 *rope_enc = nullptr, *rope_est = nullptr;  // [kCdMaxRows][hd / 2] (cos, sin)
  bf16 *vpre = nullptr, *vpost = nullptr;
  float *vpreb = nullptr, *vpostb = nullptr;
  CUtensorMap tm_vpre, tm_vpost;
  int kp_pre = 0, kp_post = 0;
  std::vector<CdBlock> blocks;
  std::vector<int> ch;
  // per-slot request tensors + vocoder state
  int32_t* reftok = nullptr;
  float *spk = nullptr, *refmel = nullptr, *state = nullptr;
  int64_t half = 0, off_pre = 0, off_ct[4] = {}, off_r1[4] = {}, off_r2[4] = {}, off_post = 0, off_ola = 0;
  std::vector<int> used, parity, calls;
  std::vector<uint64_t> seeds;
  // workspaces
  int64_t max_erows = 0, max_vrows = 0;
  int max_seg = 0;  // token rows of the longest request in the current call
  bool attn_fp32 = getenv("VOX_COSY_ATTN_FP32") != nullptr;  // A/B: CUDA-core fp32 attention
  float *h = nullptr, *qkv = nullptr, *tmp = nullptr, *mu_t = nullptr, *x = nullptr, *v = nullptr, *z = nullptr;
  float *mel = nullptr, *va = nullptr, *vb = nullptr, *vt = nullptr, *spec = nullptr, *wf = nullptr, *pcm = nullptr;
  bf16 *xbf = nullptr, *col = nullptr;
  int32_t *d_stage = nullptr, *h_stage = nullptr;
  size_t stage_ints = 0;
  float* h_pcm = nullptr;
};

namespace {
std::mutex g_cd_mu;
std::string g_cd_err;

int cfail(VoxCosy* m, int code, const std::string& msg) {
  if (m) m->err = msg;
  std::lock_guard<std::mutex> g(g_cd_mu);
  g_cd_err = msg;
  return code;
}

#define CCK(x)                                                                                          \
  do {                                                                                                  \
    cudaError_t e_ = (x);                                                                               \
    if (e_ != cudaSuccess) return cfail(m, VOX_ERR_CUDA, std::string(#x ": ") + cudaGetErrorString(e_)); \
  } while (0)
#define CRET(x)                  \
  do {                           \
    int r_ = (x);                \
    if (r_ != VOX_OK) return r_; \
  } while (0)
#define CLK(...)              \
  do {                        \
    __VA_ARGS__;              \
    m->launches++;            \
    CCK(cudaGetLastError());  \
  } while (0)

template <typename T>
cudaError_t cal(T** p, size_t n) {
  return cudaMalloc(reinterpret_cast<void**>(p), sizeof(T) * (n > 0 ? n : 1));
}

int gemm(VoxCosy* m, const CUtensorMap& tw, int M, const bf16* x, int K, int64_t rows, float* out, int64_t ldo,
         const float* bias, const float* resid, int64_t ldr, bf16* gelu_out = nullptr) {
  const cudaError_t e = codec_gemm(tw, M, x, K, rows, out, ldo, bias, resid, ldr, m->st, &m->launches, gelu_out);
  if (e != cudaSuccess) return cfail(m, VOX_ERR_CUDA, std::string("cosy gemm: ") + cudaGetErrorString(e));
  return VOX_OK;
}

int wmap(VoxCosy* m, CUtensorMap* t, const bf16* w, int M, int K) {
  return codec_wmap(t, w, M, K) ? VOX_OK : cfail(m, VOX_ERR_CUDA, "cosy: weight map");
}

struct Stage {  // host/device staging layout (int32 units)
  size_t fseg, vseg, gseg, row_seg, mrow_seg, vrow_seg, toks, total;
};
Stage stage_layout(const VoxCosyCfg& g, int64_t E, int64_t V) {
  Stage s{};
  s.fseg = 0;
  s.vseg = 8 * static_cast<size_t>(g.max_slots);
  s.gseg = s.vseg + 8 * static_cast<size_t>(g.max_slots);
  s.row_seg = s.gseg + 16 * static_cast<size_t>(g.max_slots);
  s.mrow_seg = s.row_seg + E;
  s.vrow_seg = s.mrow_seg + 4 * E;
  s.toks = s.vrow_seg + V;
  s.total = s.toks + g.max_tokens;
  return s;
}

int create(VoxCosy* m, uint64_t seed) {
  const VoxCosyCfg& g = m->cfg;
  cudaStream_t st = m->st;
  const int de = g.d_enc, ds = g.d_est, M = g.mel;
  auto key = [&](uint64_t tid, uint64_t l) { return tensor_key(seed, tid, l); };
  auto bf = [&](bf16** p, int64_t n, uint64_t tid, uint64_t l, float scale) -> int {
    CCK(cal(p, n));
    launch_init_bf16(*p, n, key(tid, l), scale, st);
    CCK(cudaGetLastError());
    return VOX_OK;
  };
  auto fl = [&](float** p, int64_t n, uint64_t tid, uint64_t l, float scale, float off) -> int {
    CCK(cal(p, n));
    launch_init_f32(*p, n, key(tid, l), scale, off, st);
    CCK(cudaGetLastError());
    return VOX_OK;
  };
  // [Mr, K] generated then zero-padded to [Mr, Kp] (K not a multiple of 64)
  auto bf_pad = [&](bf16** p, int Mr, int K, int Kp, uint64_t tid, float scale) -> int {
    bf16* raw;
    CRET(bf(&raw, static_cast<int64_t>(Mr) * K, tid, 0, scale));
    CCK(cal(p, static_cast<size_t>(Mr) * Kp));
    CCK(cudaMemsetAsync(*p, 0, static_cast<size_t>(Mr) * Kp * 2, st));
    CCK(cudaMemcpy2DAsync(*p, Kp * 2, raw, K * 2, K * 2, Mr, cudaMemcpyDeviceToDevice, st));
    CCK(cudaStreamSynchronize(st));
    cudaFree(raw);
    return VOX_OK;
  };
  auto xf = [&](std::vector<CdXf>& v, int nl, uint64_t base, int d, int ffn) -> int {
    v.resize(nl);
    for (int l = 0; l < nl; ++l) {
      CdXf& w = v[l];
      CRET(fl(&w.ln1w, d, base + 0, l, 0.25f, 1.f));
      CRET(fl(&w.ln1b, d, base + 1, l, 0.05f, 0.f));
      CRET(fl(&w.ln2w, d, base + 2, l, 0.25f, 1.f));
      CRET(fl(&w.ln2b, d, base + 3, l, 0.05f, 0.f));
      CRET(bf(&w.qkv, 3LL * d * d, base + 4, l, std::sqrt(3.0f / d)));
      CRET(bf(&w.o, static_cast<int64_t>(d) * d, base + 5, l, 0.5f * std::sqrt(3.0f / d)));
      CRET(bf(&w.fc1, static_cast<int64_t>(ffn) * d, base + 6, l, std::sqrt(3.0f / d)));
      CRET(bf(&w.fc2, static_cast<int64_t>(d) * ffn, base + 7, l, 0.5f * std::sqrt(3.0f / ffn)));
      CRET(wmap(m, &w.tm_qkv, w.qkv, 3 * d, d));
      CRET(wmap(m, &w.tm_o, w.o, d, d));
      CRET(wmap(m, &w.tm_fc1, w.fc1, ffn, d));
      CRET(wmap(m, &w.tm_fc2, w.fc2, d, ffn));
    }
    return VOX_OK;
  };
  CRET(fl(&m->emb, static_cast<int64_t>(g.vocab) * de, T_CD_EMB, 0, 1.f, 0.f));
  CRET(xf(m->enc, g.enc_layers, T_CD_ENC, de, g.enc_ffn));
  CRET(fl(&m->elnfw, de, T_CD_ELNFW, 0, 0.25f, 1.f));
  CRET(fl(&m->elnfb, de, T_CD_ELNFB, 0, 0.05f, 0.f));
  CRET(bf(&m->mu, static_cast<int64_t>(M) * de, T_CD_MU, 0, std::sqrt(3.0f / de)));
  CRET(fl(&m->mub, M, T_CD_MUB, 0, 0.05f, 0.f));
  CRET(wmap(m, &m->tm_mu, m->mu, M, de));
  CRET(bf(&m->w_in, static_cast<int64_t>(ds) * 4 * M, T_CD_IN, 0, std::sqrt(3.0f / (4 * M))));
  CRET(wmap(m, &m->tm_in, m->w_in, ds, 4 * M));
  {
    float *b_in, *t1, *t1b, *t2, *t2b;
    CRET(fl(&b_in, ds, T_CD_INB, 0, 0.05f, 0.f));
    CRET(fl(&t1, static_cast<int64_t>(ds) * ds, T_CD_T1, 0, std::sqrt(3.0f / ds), 0.f));
    CRET(fl(&t1b, ds, T_CD_T1B, 0, 0.05f, 0.f));
    CRET(fl(&t2, static_cast<int64_t>(ds) * ds, T_CD_T2, 0, std::sqrt(3.0f / ds), 0.f));
    CRET(fl(&t2b, ds, T_CD_T2B, 0, 0.05f, 0.f));
    CCK(cal(&m->step_bias, static_cast<size_t>(g.n_steps) * ds));
    m->ts.resize(g.n_steps + 1);
    for (int i = 0; i <= g.n_steps; ++i)
      m->ts[i] = static_cast<float>(1.0 - std::cos(M_PI / 2 * static_cast<double>(i) / g.n_steps));
    for (int i = 0; i < g.n_steps; ++i)
      cd_temb_kernel<<<1, 256, 2 * ds * sizeof(float), st>>>(t1, t1b, t2, t2b, b_in, ds, m->ts[i],
                                                              m->step_bias + static_cast<int64_t>(i) * ds);
    CCK(cudaGetLastError());
    CCK(cudaStreamSynchronize(st));
    for (float* p : {b_in, t1, t1b, t2, t2b}) cudaFree(p);
  }
  CRET(xf(m->est, g.est_layers, T_CD_EST, ds, g.est_ffn));
  CRET(fl(&m->olnw, ds, T_CD_OLNW, 0, 0.25f, 1.f));
  CRET(fl(&m->olnb, ds, T_CD_OLNB, 0, 0.05f, 0.f));
  CRET(bf(&m->w_out, static_cast<int64_t>(M) * ds, T_CD_OUT, 0, std::sqrt(3.0f / ds)));
  CRET(fl(&m->outb, M, T_CD_OUTB, 0, 0.05f, 0.f));
  CRET(wmap(m, &m->tm_out, m->w_out, M, ds));
  auto inv = [&](float** p, int d, int heads) -> int {
    const int hd = d / heads;
    std::vector<float> v(hd / 2);
    for (int i = 0; i < hd / 2; ++i) v[i] = 1.0f / std::pow(g.rope_theta, static_cast<float>(2 * i) / hd);
    CCK(cal(p, v.size()));
    CCK(cudaMemcpy(*p, v.data(), v.size() * 4, cudaMemcpyHostToDevice));
    return VOX_OK;
  };
  CRET(inv(&m->inv_enc, de, g.enc_heads));
  CRET(inv(&m->inv_est, ds, g.est_heads));
  CCK(cal(&m->rope_enc, static_cast<size_t>(kCdMaxRows) * (de / g.enc_heads / 2)));
  CCK(cal(&m->rope_est, static_cast<size_t>(kCdMaxRows) * (ds / g.est_heads / 2)));
  cd_rope_table_kernel<<<kCdMaxRows, 64, 0, st>>>(m->inv_enc, de / g.enc_heads / 2, m->rope_enc);
  cd_rope_table_kernel<<<kCdMaxRows, 64, 0, st>>>(m->inv_est, ds / g.est_heads / 2, m->rope_est);
  CCK(cudaGetLastError());
  // vocoder
  const std::vector<int>& ch = m->ch;
  m->kp_pre = (g.voc_kernel * M + 63) / 64 * 64;
  CRET(bf_pad(&m->vpre, ch[0], g.voc_kernel * M, m->kp_pre, T_CD_VPRE, std::sqrt(3.0f / (g.voc_kernel * M))));
  CRET(fl(&m->vpreb, ch[0], T_CD_VPREB, 0, 0.05f, 0.f));
  CRET(wmap(m, &m->tm_vpre, m->vpre, ch[0], m->kp_pre));
  m->blocks.resize(g.n_ratios);
  for (int b = 0; b < g.n_ratios; ++b) {
    CdBlock& w = m->blocks[b];
    const int Ci = ch[b], Co = ch[b + 1], s = g.ratios[b];
    CRET(bf(&w.upw, static_cast<int64_t>(s) * Co * 2 * Ci, T_CD_UPW, b, std::sqrt(3.0f / (2.0f * Ci))));
    float* small;
    CRET(fl(&small, Co, T_CD_UPB, b, 0.05f, 0.f));
    CCK(cal(&w.upb, static_cast<size_t>(s) * Co));
    for (int j = 0; j < s; ++j)
      CCK(cudaMemcpyAsync(w.upb + static_cast<int64_t>(j) * Co, small, Co * 4, cudaMemcpyDeviceToDevice, st));
    CRET(bf(&w.r1w, static_cast<int64_t>(Co) * g.res_kernel * Co, T_CD_R1W, b, std::sqrt(3.0f / (g.res_kernel * Co))));
    CRET(fl(&w.r1b, Co, T_CD_R1B, b, 0.05f, 0.f));
    CRET(bf(&w.r2w, static_cast<int64_t>(Co) * g.res_kernel * Co, T_CD_R2W, b,
            0.5f * std::sqrt(3.0f / (g.res_kernel * Co))));
    CRET(fl(&w.r2b, Co, T_CD_R2B, b, 0.05f, 0.f));
    CCK(cudaStreamSynchronize(st));
    cudaFree(small);
    CRET(wmap(m, &w.tm_up, w.upw, s * Co, 2 * Ci));
    CRET(wmap(m, &w.tm_r1, w.r1w, Co, g.res_kernel * Co));
    CRET(wmap(m, &w.tm_r2, w.r2w, Co, g.res_kernel * Co));
  }
  const int nb2 = g.n_fft + 2, C4 = ch[g.n_ratios];
  m->kp_post = (g.post_kernel * C4 + 63) / 64 * 64;
  CRET(bf_pad(&m->vpost, nb2, g.post_kernel * C4, m->kp_post, T_CD_VPOST, std::sqrt(3.0f / (g.post_kernel * C4))));
  CRET(fl(&m->vpostb, nb2, T_CD_VPOSTB, 0, 0.05f, 0.f));
  CRET(wmap(m, &m->tm_vpost, m->vpost, nb2, m->kp_post));
  // per-slot tensors + state
  CCK(cal(&m->reftok, static_cast<size_t>(g.max_slots) * g.ref_tokens));
  CCK(cal(&m->spk, static_cast<size_t>(g.max_slots) * M));
  CCK(cal(&m->refmel, static_cast<size_t>(g.max_slots) * 2 * g.ref_tokens * M));
  int64_t off = 0;
  m->off_pre = off;
  off += static_cast<int64_t>(g.voc_kernel - 1) * M;
  for (int b = 0; b < g.n_ratios; ++b) {
    m->off_ct[b] = off;
    off += ch[b];
    m->off_r1[b] = off;
    off += static_cast<int64_t>(g.res_kernel - 1) * ch[b + 1];
    m->off_r2[b] = off;
    off += static_cast<int64_t>(g.res_kernel - 1) * ch[b + 1];
  }
  m->off_post = off;
  off += static_cast<int64_t>(g.post_kernel - 1) * C4;
  m->off_ola = off;
  off += static_cast<int64_t>(g.n_fft / g.hop - 1) * g.n_fft;
  m->half = (off + 63) / 64 * 64;
  CCK(cal(&m->state, static_cast<size_t>(g.max_slots) * 2 * m->half));
  CCK(cudaMemset(m->state, 0, static_cast<size_t>(g.max_slots) * 2 * m->half * 4));
  m->used.assign(g.max_slots, 0);
  m->parity.assign(g.max_slots, 0);
  m->calls.assign(g.max_slots, 0);
  m->seeds.assign(g.max_slots, 0);
  // workspaces
  const int64_t E = static_cast<int64_t>(g.max_tokens) + static_cast<int64_t>(g.max_slots) * g.ref_tokens;
  m->max_erows = E;
  const int64_t Rm = 2 * E, Re2 = 2 * Rm;  // mel rows, estimator rows (both CFG branches)
  const int64_t dmax = std::max(de, ds), fmax = std::max<int64_t>(std::max(g.enc_ffn, g.est_ffn), 4 * M);
  CCK(cal(&m->h, E * de));
  CCK(cal(&m->z, Re2 * ds));
  CCK(cal(&m->qkv, std::max(E * 3 * de, Re2 * 3 * ds)));
  CCK(cal(&m->tmp, std::max(E * g.enc_ffn, Re2 * g.est_ffn)));
  CCK(cal(&m->xbf, std::max(E, Re2) * std::max(dmax, fmax)));
  CCK(cal(&m->mu_t, E * M));
  CCK(cal(&m->x, Rm * M));
  CCK(cal(&m->v, Re2 * M));
  const int64_t V = 2LL * g.max_tokens;  // vocoder mel frames per call
  m->max_vrows = V;
  int64_t u = 1, mx = V * ch[0], mcol = V * m->kp_pre;
  for (int b = 0; b < g.n_ratios; ++b) {
    mcol = std::max<int64_t>(mcol, V * u * 2 * ch[b]);
    u *= g.ratios[b];
    mx = std::max<int64_t>(mx, V * u * ch[b + 1]);
    mcol = std::max<int64_t>(mcol, V * u * g.res_kernel * ch[b + 1]);
  }
  mcol = std::max<int64_t>(mcol, V * u * m->kp_post);
  CCK(cal(&m->mel, V * M));
  CCK(cal(&m->va, mx));
  CCK(cal(&m->vb, mx));
  CCK(cal(&m->vt, mx));
  CCK(cal(&m->col, mcol));
  CCK(cal(&m->spec, V * u * nb2));
  CCK(cal(&m->wf, V * u * g.n_fft));
  CCK(cal(&m->pcm, V * u * g.hop));
  // staging: fseg[max_slots] vseg[max_slots] (8 ints each) | row_seg[E] | vrow_seg[V] | tokens[max_tokens]
  m->stage_ints = stage_layout(g, E, V).total;
  CCK(cal(&m->d_stage, m->stage_ints));
  CCK(cudaHostAlloc(&m->h_stage, m->stage_ints * 4, cudaHostAllocDefault));
  CCK(cudaHostAlloc(&m->h_pcm, V * u * g.hop * 4, cudaHostAllocDefault));
  return VOX_OK;
}

int xf_layers(VoxCosy* m, std::vector<CdXf>& layers, float* h, int64_t rows, int d, int heads, int ffn, int nseg,
              const int32_t* row_seg, const SegDev* seg, const float* inv, const float2* rope, int max_rows) {
  (void)row_seg;
  const VoxCosyCfg& g = m->cfg;
  cudaStream_t st = m->st;
  const int hd = d / heads;
  for (auto& w : layers) {
    CLK(launch_codec_ln(h, nullptr, nullptr, w.ln1w, w.ln1b, m->xbf, d, g.eps, rows, st));
    CRET(gemm(m, w.tm_qkv, 3 * d, m->xbf, d, rows, m->qkv, 3 * d, nullptr, nullptr, 0));
    if (hd == kTcHd && !m->attn_fp32)
      CLK(cd_attn_tc_kernel<<<dim3(nseg, heads), 32 * cd_attn_tc_warps(max_rows), cd_attn_tc_smem(max_rows), st>>>(
          m->qkv, seg, d, rope, m->xbf));
    else
      CLK(cd_attn_kernel<<<dim3(nseg, heads), 256, cd_attn_smem(max_rows, hd), st>>>(m->qkv, seg, d, hd, inv, m->xbf));
    CRET(gemm(m, w.tm_o, d, m->xbf, d, rows, h, d, nullptr, h, d));
    CLK(launch_codec_ln(h, nullptr, nullptr, w.ln2w, w.ln2b, m->xbf, d, g.eps, rows, st));
    // fc1 with GELU + bf16 in its epilogue (the fp32 [rows][ffn] round trip and the
    // GELU launch are gone); the activations land in tmp's storage
    bf16* act = reinterpret_cast<bf16*>(m->tmp);
    CRET(gemm(m, w.tm_fc1, ffn, m->xbf, d, rows, nullptr, ffn, nullptr, nullptr, 0, act));
    CRET(gemm(m, w.tm_fc2, d, act, ffn, rows, h, d, nullptr, h, d));
  }
  return VOX_OK;
}

int enqueue(VoxCosy* m, int n, int64_t E, int64_t V) {
  const VoxCosyCfg& g = m->cfg;
  cudaStream_t st = m->st;
  const int de = g.d_enc, ds = g.d_est, M = g.mel, ref = g.ref_tokens;
  const Stage L = stage_layout(g, m->max_erows, m->max_vrows);
  const SegDev* fseg = reinterpret_cast<const SegDev*>(m->d_stage + L.fseg);
  const SegDev* vseg = reinterpret_cast<const SegDev*>(m->d_stage + L.vseg);
  const SegDev* gseg = reinterpret_cast<const SegDev*>(m->d_stage + L.gseg);
  const int32_t* row_seg = m->d_stage + L.row_seg;
  const int32_t* mrow_seg = m->d_stage + L.mrow_seg;
  const int32_t* vrow_seg = m->d_stage + L.vrow_seg;
  const int32_t* toks = m->d_stage + L.toks;
  StateView sv{m->state, 2 * m->half, m->half};
  // ---------------- flow: encoder over [ref | new] tokens
  CLK(cd_embed_kernel<<<static_cast<unsigned>(E), 128, 0, st>>>(row_seg, fseg, m->reftok, ref, toks, m->emb, de, m->h));
  CRET(xf_layers(m, m->enc, m->h, E, de, g.enc_heads, g.enc_ffn, n, row_seg, fseg, m->inv_enc, m->rope_enc,
                 m->max_seg));
  CLK(launch_codec_ln(m->h, nullptr, nullptr, m->elnfw, m->elnfb, m->xbf, de, g.eps, E, st));
  CRET(gemm(m, m->tm_mu, M, m->xbf, de, E, m->mu_t, M, m->mub, nullptr, 0));
  // ---------------- flow matching ODE (CFG: rows [0, R) cond, [R, 2R) uncond)
  const int64_t R = 2 * E;
  const int64_t nx = R * M;
  CLK(cd_noise_kernel<<<static_cast<unsigned>((nx + 255) / 256), 256, 0, st>>>(row_seg, fseg, M, R, m->x));
  const float lam = g.cfg_rate;
  for (int i = 0; i < g.n_steps; ++i) {
    const int64_t ne = 2 * R * 4 * M;
    CLK(cd_est_in_kernel<<<static_cast<unsigned>((ne + 255) / 256), 256, 0, st>>>(m->x, m->mu_t, row_seg, fseg, m->spk,
                                                                                 m->refmel, ref, M, R, m->xbf));
    CRET(gemm(m, m->tm_in, ds, m->xbf, 4 * M, 2 * R, m->z, ds, m->step_bias + static_cast<int64_t>(i) * ds, nullptr, 0));
    CRET(xf_layers(m, m->est, m->z, 2 * R, ds, g.est_heads, g.est_ffn, 2 * n, mrow_seg, gseg, m->inv_est,
                   m->rope_est, 2 * m->max_seg));
    CLK(launch_codec_ln(m->z, nullptr, nullptr, m->olnw, m->olnb, m->xbf, ds, g.eps, 2 * R, st));
    CRET(gemm(m, m->tm_out, M, m->xbf, ds, 2 * R, m->v, M, m->outb, nullptr, 0));
    CLK(cd_euler_kernel<<<static_cast<unsigned>((nx + 255) / 256), 256, 0, st>>>(m->x, m->v, nx, m->ts[i + 1] - m->ts[i], lam));
  }
  // ---------------- vocoder over the new mel frames (stateful)
  {
    const int64_t ne = V * M;
    CLK(cd_gather_mel_kernel<<<static_cast<unsigned>((ne + 255) / 256), 256, 0, st>>>(m->x, vrow_seg, vseg, fseg, ref, M, V, m->mel));
  }
  auto im2col = [&](const float* x, int C, int k, int act, int Kp, int u, int64_t off, int64_t rows) -> int {
    const int64_t tot = rows * (Kp / 8);
    CLK(codec_im2col_kernel<<<static_cast<unsigned>((tot + 255) / 256), 256, 0, st>>>(x, C, k, act, g.slope, Kp, u, vrow_seg,
                                                                                      vseg, sv, off, rows, m->col));
    if (k > 1) CLK(codec_hist_kernel<<<n, 256, 0, st>>>(x, C, k, u, vseg, sv, off));
    return VOX_OK;
  };
  const std::vector<int>& ch = m->ch;
  CRET(im2col(m->mel, M, g.voc_kernel, kActNone, m->kp_pre, 1, m->off_pre, V));
  CRET(gemm(m, m->tm_vpre, ch[0], m->col, m->kp_pre, V, m->va, ch[0], m->vpreb, nullptr, 0));
  float *x = m->va, *y = m->vb;
  int u = 1;
  for (int b = 0; b < g.n_ratios; ++b) {
    const CdBlock& w = m->blocks[b];
    const int Ci = ch[b], Co = ch[b + 1], s = g.ratios[b];
    const int64_t rows = V * u;
    CRET(im2col(x, Ci, 2, kActLeaky, 2 * Ci, u, m->off_ct[b], rows));
    CRET(gemm(m, w.tm_up, s * Co, m->col, 2 * Ci, rows, y, static_cast<int64_t>(s) * Co, w.upb, nullptr, 0));
    u *= s;
    const int64_t rows2 = V * u;
    CRET(im2col(y, Co, g.res_kernel, kActLeaky, g.res_kernel * Co, u, m->off_r1[b], rows2));
    CRET(gemm(m, w.tm_r1, Co, m->col, g.res_kernel * Co, rows2, m->vt, Co, w.r1b, nullptr, 0));
    CRET(im2col(m->vt, Co, g.res_kernel, kActLeaky, g.res_kernel * Co, u, m->off_r2[b], rows2));
    CRET(gemm(m, w.tm_r2, Co, m->col, g.res_kernel * Co, rows2, y, Co, w.r2b, y, Co));
    std::swap(x, y);
  }
  const int C4 = ch[g.n_ratios], nb2 = g.n_fft + 2;
  const int64_t J = V * u;
  CRET(im2col(x, C4, g.post_kernel, kActLeaky, m->kp_post, u, m->off_post, J));
  CRET(gemm(m, m->tm_vpost, nb2, m->col, m->kp_post, J, m->spec, nb2, m->vpostb, nullptr, 0));
  CLK(cd_istft_frames_kernel<<<static_cast<unsigned>((J + 127) / 128), 128, 0, st>>>(m->spec, g.n_fft, J, m->wf));
  CLK(cd_ola_kernel<<<static_cast<unsigned>((J * g.hop + 255) / 256), 256, 0, st>>>(m->wf, g.n_fft, g.hop, u, vrow_seg,
                                                                                   vseg, sv, m->off_ola, J, m->pcm));
  CLK(codec_hist_kernel<<<n, 256, 0, st>>>(m->wf, g.n_fft, g.n_fft / g.hop, u, vseg, sv, m->off_ola));
  return VOX_OK;
}

}  // namespace

extern "C" {

const char* vox_cosy_last_error(const VoxCosy* m) {
  if (m) return m->err.c_str();
  return g_cd_err.c_str();
}

void vox_cosy_destroy(VoxCosy* m) {
  if (!m) return;
  cudaSetDevice(m->device);
  if (m->st) cudaStreamSynchronize(m->st);
  for (auto& kv : m->graphs) cudaGraphExecDestroy(kv.second);
  for (auto* v : {&m->enc, &m->est})
    for (auto& w : *v)
      for (void* p : {static_cast<void*>(w.ln1w), static_cast<void*>(w.ln1b), static_cast<void*>(w.ln2w),
                      static_cast<void*>(w.ln2b), static_cast<void*>(w.qkv), static_cast<void*>(w.o),
                      static_cast<void*>(w.fc1), static_cast<void*>(w.fc2)})
        cudaFree(p);
  for (auto& w : m->blocks)
    for (void* p : {static_cast<void*>(w.upw), static_cast<void*>(w.r1w), static_cast<void*>(w.r2w),
                    static_cast<void*>(w.upb), static_cast<void*>(w.r1b), static_cast<void*>(w.r2b)})
      cudaFree(p);
  for (void* p : {static_cast<void*>(m->emb), static_cast<void*>(m->elnfw), static_cast<void*>(m->elnfb),
                  static_cast<void*>(m->mub), static_cast<void*>(m->olnw), static_cast<void*>(m->olnb),
                  static_cast<void*>(m->outb), static_cast<void*>(m->mu), static_cast<void*>(m->w_in),
                  static_cast<void*>(m->w_out), static_cast<void*>(m->step_bias), static_cast<void*>(m->inv_enc),
                  static_cast<void*>(m->inv_est), static_cast<void*>(m->rope_enc), static_cast<void*>(m->rope_est),
                  static_cast<void*>(m->vpre), static_cast<void*>(m->vpost),
                  static_cast<void*>(m->vpreb), static_cast<void*>(m->vpostb), static_cast<void*>(m->reftok),
                  static_cast<void*>(m->spk), static_cast<void*>(m->refmel), static_cast<void*>(m->state),
                  static_cast<void*>(m->h), static_cast<void*>(m->qkv), static_cast<void*>(m->tmp),
                  static_cast<void*>(m->mu_t), static_cast<void*>(m->x), static_cast<void*>(m->v),
                  static_cast<void*>(m->z), static_cast<void*>(m->mel), static_cast<void*>(m->va),
                  static_cast<void*>(m->vb), static_cast<void*>(m->vt), static_cast<void*>(m->spec),
                  static_cast<void*>(m->wf), static_cast<void*>(m->pcm), static_cast<void*>(m->xbf),
                  static_cast<void*>(m->col), static_cast<void*>(m->d_stage)})
    cudaFree(p);
  if (m->h_stage) cudaFreeHost(m->h_stage);
  if (m->h_pcm) cudaFreeHost(m->h_pcm);
  if (m->ev0) cudaEventDestroy(m->ev0);
  if (m->ev1) cudaEventDestroy(m->ev1);
  if (m->st) cudaStreamDestroy(m->st);
  delete m;
}

int vox_cosy_create(int device, const VoxCosyCfg* cfg, uint64_t seed, VoxCosy** out) {
  VoxCosy* m = nullptr;
  if (!cfg || !out) return cfail(m, VOX_ERR_INVALID, "null argument");
  *out = nullptr;
  const VoxCosyCfg& g = *cfg;
  auto bad_xf = [](int d, int heads, int ffn) {
    return (d != 256 && d != 512 && d != 768 && d != 1024) || heads < 1 || d % heads || (d / heads) % 2 || d / heads > 64 || ffn % 64;
  };
  if (bad_xf(g.d_enc, g.enc_heads, g.enc_ffn) || bad_xf(g.d_est, g.est_heads, g.est_ffn) || g.mel % 16 ||
      g.enc_layers < 0 || g.est_layers < 0 || g.n_steps < 1 || g.vocab < 1 || g.ref_tokens < 0 ||
      2 * (g.ref_tokens + g.max_chunk) > kCdMaxRows || g.max_chunk < 1 || g.max_tokens < 1 || g.max_slots < 1 ||
      g.n_ratios < 1 || g.n_ratios > 4 || g.n_fft != 16 || g.hop < 1 || g.n_fft % g.hop || g.voc_ch % 64 ||
      (g.voc_ch >> g.n_ratios) % 64 || g.voc_kernel < 1 || g.res_kernel < 1 || g.post_kernel < 1)
    return cfail(m, VOX_ERR_INVALID, "unsupported CosyVoice2-style detokenizer configuration");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev)
    return cfail(m, VOX_ERR_NO_DEVICE, "no CUDA device");
  cudaDeviceProp prop{};
  cudaGetDeviceProperties(&prop, device);
  if (prop.major != 10) return cfail(m, VOX_ERR_NO_DEVICE, "requires an sm_100 (B200) device");
  m = new VoxCosy();
  m->device = device;
  m->cfg = g;
  m->ch.push_back(g.voc_ch);
  for (int b = 0; b < g.n_ratios; ++b) m->ch.push_back(m->ch.back() / 2);
  cudaSetDevice(device);
  int lo = 0, hi = 0;
  cudaDeviceGetStreamPriorityRange(&lo, &hi);
  int rc = cudaStreamCreateWithPriority(&m->st, cudaStreamNonBlocking, lo) == cudaSuccess ? VOX_OK : VOX_ERR_CUDA;
  if (rc == VOX_OK && (cudaEventCreate(&m->ev0) != cudaSuccess || cudaEventCreate(&m->ev1) != cudaSuccess))
    rc = cfail(m, VOX_ERR_CUDA, "event create");
  if (rc == VOX_OK && cudaFuncSetAttribute(cd_attn_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           static_cast<int>(cd_attn_smem(kCdMaxRows, 64))) != cudaSuccess)
    rc = cfail(m, VOX_ERR_CUDA, "attention smem attribute");
  if (rc == VOX_OK && cudaFuncSetAttribute(cd_attn_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                           static_cast<int>(cd_attn_tc_smem(kCdMaxRows))) != cudaSuccess)
    rc = cfail(m, VOX_ERR_CUDA, "attention smem attribute");
  if (rc == VOX_OK) rc = create(m, seed);
  if (rc == VOX_OK && cudaStreamSynchronize(m->st) != cudaSuccess) rc = cfail(m, VOX_ERR_CUDA, "init sync");
  if (rc != VOX_OK) {
    g_cd_err = m->err;
    vox_cosy_destroy(m);
    return rc;
  }
  *out = m;
  return VOX_OK;
}

int vox_cosy_open(VoxCosy* m, uint64_t req_seed, int32_t* slot) {
  if (!m || !slot) return cfail(m, VOX_ERR_INVALID, "null argument");
  const VoxCosyCfg& g = m->cfg;
  cudaSetDevice(m->device);
  for (int s = 0; s < g.max_slots; ++s)
    if (!m->used[s]) {
      cudaStream_t st = m->st;
      CCK(cudaMemsetAsync(m->state + static_cast<int64_t>(s) * 2 * m->half, 0, 2 * m->half * 4, st));
      if (g.ref_tokens > 0) {
        cd_reftok_kernel<<<(g.ref_tokens + 127) / 128, 128, 0, st>>>(m->reftok + static_cast<int64_t>(s) * g.ref_tokens,
                                                                     g.ref_tokens, tensor_key(req_seed, T_CD_REFTOK, 0),
                                                                     g.vocab);
        launch_init_f32(m->refmel + static_cast<int64_t>(s) * 2 * g.ref_tokens * g.mel, 2LL * g.ref_tokens * g.mel,
                        tensor_key(req_seed, T_CD_REFMEL, 0), 1.f, 0.f, st);
      }
      launch_init_f32(m->spk + static_cast<int64_t>(s) * g.mel, g.mel, tensor_key(req_seed, T_CD_SPK, 0), 1.f, 0.f, st);
      CCK(cudaGetLastError());
      m->used[s] = 1;
      m->parity[s] = 0;
      m->calls[s] = 0;
      m->seeds[s] = req_seed;
      *slot = s;
      return VOX_OK;
    }
  return cfail(m, VOX_ERR_OUT_OF_MEMORY, "no free detokenizer slot");
}

int vox_cosy_close(VoxCosy* m, int32_t slot) {
  if (!m || slot < 0 || slot >= m->cfg.max_slots || !m->used[slot])
    return cfail(m, VOX_ERR_CACHE_MISSING, "close of an unknown detokenizer stream");
  m->used[slot] = 0;
  return VOX_OK;
}

int vox_cosy_decode(VoxCosy* m, const VoxCosyReq* reqs, int32_t n, const int32_t* tokens, float* pcm_out,
                    int64_t* n_samples) {
  if (!m || (!reqs && n > 0) || !tokens) return cfail(m, VOX_ERR_INVALID, "null argument");
  if (n <= 0) return cfail(m, VOX_ERR_EMPTY_BATCH, "empty detokenizer batch");
  const VoxCosyCfg& g = m->cfg;
  if (n > g.max_slots) return cfail(m, VOX_ERR_BATCH_TOO_LARGE, "more requests than detokenizer slots");
  cudaSetDevice(m->device);
  const Stage L = stage_layout(g, m->max_erows, m->max_vrows);
  int32_t* hs = m->h_stage;
  m->max_seg = 0;
  SegDev* fseg = reinterpret_cast<SegDev*>(hs + L.fseg);
  SegDev* vseg = reinterpret_cast<SegDev*>(hs + L.vseg);
  SegDev* gseg = reinterpret_cast<SegDev*>(hs + L.gseg);
  int64_t E = 0, V = 0, C = 0;
  std::vector<int> seen;
  for (int i = 0; i < n; ++i) {
    const VoxCosyReq& r = reqs[i];
    if (r.slot < 0 || r.slot >= g.max_slots || !m->used[r.slot])
      return cfail(m, VOX_ERR_CACHE_MISSING, "decode of an unopened detokenizer stream");
    if (std::find(seen.begin(), seen.end(), r.slot) != seen.end())
      return cfail(m, VOX_ERR_INVALID, "a request appears twice in one detokenizer batch");
    seen.push_back(r.slot);
    if (r.n_tokens < 1) return cfail(m, VOX_ERR_INVALID, "detokenizer request without tokens");
    if (r.n_tokens > g.max_chunk) return cfail(m, VOX_ERR_BATCH_TOO_LARGE, "chunk exceeds max_chunk tokens");
    if (C + r.n_tokens > g.max_tokens) return cfail(m, VOX_ERR_BATCH_TOO_LARGE, "batch exceeds max_tokens");
    const int T = g.ref_tokens + r.n_tokens;
    m->max_seg = std::max(m->max_seg, T);
    const uint64_t key = tensor_key(m->seeds[r.slot], T_CD_NOISE, static_cast<uint64_t>(m->calls[r.slot]));
    fseg[i] = SegDev{r.slot, static_cast<int32_t>(E), T, m->parity[r.slot], 0, static_cast<int32_t>(C),
                     {static_cast<int32_t>(key & 0xffffffffu), static_cast<int32_t>(key >> 32)}};
    vseg[i] = SegDev{r.slot, static_cast<int32_t>(V), 2 * r.n_tokens, m->parity[r.slot], 0, 0, {0, 0}};
    for (int t = 0; t < T; ++t) hs[L.row_seg + E + t] = i;
    for (int t = 0; t < 2 * r.n_tokens; ++t) hs[L.vrow_seg + V + t] = i;
    for (int t = 0; t < r.n_tokens; ++t) {
      const int32_t tok = tokens[C + t];
      if (tok < 0 || tok >= g.vocab) return cfail(m, VOX_ERR_INVALID, "speech token outside the vocabulary");
      hs[L.toks + C + t] = tok;
    }
    E += T;
    V += 2 * r.n_tokens;
    C += r.n_tokens;
  }
  // estimator groups: cond (rows 2 f_off ..) then uncond (rows R + 2 f_off ..), mel-row units
  const int64_t R = 2 * E;
  for (int i = 0; i < n; ++i) {
    gseg[i] = SegDev{fseg[i].slot, 2 * fseg[i].f_off, 2 * fseg[i].nf, 0, 0, 0, {0, 0}};
    gseg[n + i] = SegDev{fseg[i].slot, static_cast<int32_t>(R + 2 * fseg[i].f_off), 2 * fseg[i].nf, 0, 0, 0, {0, 0}};
    for (int t = 0; t < 2 * fseg[i].nf; ++t) {
      hs[L.mrow_seg + 2 * fseg[i].f_off + t] = i;
      hs[L.mrow_seg + R + 2 * fseg[i].f_off + t] = n + i;
    }
  }
  CCK(cudaMemcpyAsync(m->d_stage, hs, L.total * 4, cudaMemcpyHostToDevice, m->st));
  CCK(cudaEventRecord(m->ev0, m->st));
  {
    const auto key = std::make_tuple(n, E, V, m->max_seg);
    auto it = m->graphs.find(key);
    if (m->no_graphs || (it == m->graphs.end() && m->graphs.size() >= kCdMaxGraphs)) {
      CRET(enqueue(m, n, E, V));
    } else if (it == m->graphs.end()) {
      // first call of this shape: run it eagerly (sets kernel attributes), then capture
      const int64_t before = m->launches;
      CRET(enqueue(m, n, E, V));
      const int64_t per_call = m->launches - before;
      cudaGraph_t graph;
      CCK(cudaStreamBeginCapture(m->st, cudaStreamCaptureModeThreadLocal));
      const int rc = enqueue(m, n, E, V);
      const cudaError_t ce = cudaStreamEndCapture(m->st, &graph);
      if (rc != VOX_OK) return rc;
      CCK(ce);
      cudaGraphExec_t ex;
      CCK(cudaGraphInstantiate(&ex, graph, 0));
      cudaGraphDestroy(graph);
      m->graphs[key] = ex;
      m->graph_launches[key] = per_call;
      m->launches = before + per_call;
    } else {
      CCK(cudaGraphLaunch(it->second, m->st));
      m->launches += m->graph_launches[key];
    }
  }
  CCK(cudaEventRecord(m->ev1, m->st));
  int64_t spm = g.hop;
  for (int b = 0; b < g.n_ratios; ++b) spm *= g.ratios[b];
  const int64_t total = V * spm;
  CCK(cudaMemcpyAsync(m->h_pcm, m->pcm, total * 4, cudaMemcpyDeviceToHost, m->st));
  CCK(cudaStreamSynchronize(m->st));
  float ms = 0.f;
  CCK(cudaEventElapsedTime(&ms, m->ev0, m->ev1));
  m->last_ms = ms;
  if (pcm_out) std::copy(m->h_pcm, m->h_pcm + total, pcm_out);
  if (n_samples) *n_samples = total;
  for (int i = 0; i < n; ++i) {
    m->parity[reqs[i].slot] ^= 1;
    m->calls[reqs[i].slot] += 1;
  }
  return VOX_OK;
}

int vox_cosy_last_ms(VoxCosy* m, double* ms) {
  if (!m || !ms) return cfail(m, VOX_ERR_INVALID, "null argument");
  *ms = m->last_ms;
  return VOX_OK;
}

int vox_cosy_launch_count(VoxCosy* m, int64_t* launches) {
  if (!m || !launches) return cfail(m, VOX_ERR_INVALID, "null argument");
  *launches = m->launches;
  return VOX_OK;
}

}  // extern "C"
