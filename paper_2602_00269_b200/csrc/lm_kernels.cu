// lm_kernels.cu — the fused elementwise / attention kernels of one decode step.
//
// Layouts (HBM):
//   h        [rows, d]            fp32 residual stream
//   x        [rows, d]            bf16 GEMM input (normalised)
//   ws       [splits, rows, N]    fp32 split-K partials written by gemm_tc.cu
//   q        [rows, H, hd]        bf16 (RoPE applied)
//   K/V pool [layer][page][kv_head][page_size][hd] bf16 (one head's page is
//            page_size*hd contiguous elements -> coalesced 4 KB per head-page)
//   page_table [slot][max_pages_per_slot] int32
// Rows with slot < 0 are padding and are skipped.
#include "common.cuh"
#include "kernels.h"

namespace vox {

template <int NT>
VOX_DEV float block_sum(float v, float* red) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) red[w] = v;
  __syncthreads();
  float t = 0.f;
  if (threadIdx.x < 32) {
    t = (l < NT / 32) ? red[l] : 0.f;
    t = warp_sum(t);
    if (l == 0) red[32] = t;
  }
  __syncthreads();
  t = red[32];
  __syncthreads();
  return t;
}

// ---------------------------------------------------------------------------
// embedding gather + first RMSNorm
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) embed_norm_kernel(const RowDev* __restrict__ rows,
                                                         int* __restrict__ token_store,
                                                         int max_ctx, const bf16* __restrict__ emb,
                                                         const float* __restrict__ nw, int d,
                                                         float eps, float* __restrict__ h,
                                                         bf16* __restrict__ x) {
  __shared__ float red[33];
  const int r = blockIdx.x;
  const RowDev rw = rows[r];
  if (rw.slot < 0) return;
  int* ts = token_store + static_cast<int64_t>(rw.slot) * max_ctx + rw.pos;
  int tok = rw.token;
  if (tok >= 0) {
    if (threadIdx.x == 0) *ts = tok;
  } else {
    tok = *ts;
  }
  const bf16* e = emb + static_cast<int64_t>(tok) * d;
  float* hr = h + static_cast<int64_t>(r) * d;
  float ss = 0.f;
  for (int i = threadIdx.x; i < d; i += 256) {
    const float v = __bfloat162float(e[i]);
    hr[i] = v;
    ss = fmaf(v, v, ss);
  }
  ss = block_sum<256>(ss, red);
  const float inv = 1.0f / sqrtf(ss / static_cast<float>(d) + eps);
  bf16* xr = x + static_cast<int64_t>(r) * d;
  for (int i = threadIdx.x; i < d; i += 256)
    xr[i] = __float2bfloat16_rn(__fmul_rn(__fmul_rn(hr[i], inv), nw[i]));
}

void launch_embed_norm(const RowDev* rows, int n, int* token_store, int max_ctx, const bf16* emb,
                       const float* norm_w, const LmDims& dm, float* h, bf16* x,
                       cudaStream_t st) {
  embed_norm_kernel<<<n, 256, 0, st>>>(rows, token_store, max_ctx, emb, norm_w, dm.d, dm.eps, h,
                                       x);
}

// ---------------------------------------------------------------------------
// split-K reduce of the QKV projection + RoPE + paged KV append
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256)
    qkv_rope_append_kernel(const RowDev* __restrict__ rows, const float* __restrict__ ws,
                           int splits, int64_t split_stride, LmDims dm,
                           const float* __restrict__ inv_freq, const int* __restrict__ page_table,
                           bf16* __restrict__ kc, bf16* __restrict__ vc, bf16* __restrict__ q_out) {
  const int r = blockIdx.x;
  const RowDev rw = rows[r];
  if (rw.slot < 0) return;
  const int hd = dm.hd, half = hd / 2;
  const int nqkv = (dm.n_heads + 2 * dm.n_kv) * hd;
  const float* wr = ws + static_cast<int64_t>(r) * nqkv;
  const int page = page_table[static_cast<int64_t>(rw.slot) * dm.max_pages_per_slot +
                              rw.pos / dm.page_size];
  const int off = rw.pos % dm.page_size;
  const int n_pairs = (dm.n_heads + dm.n_kv) * half;
  for (int p = threadIdx.x; p < n_pairs; p += 256) {
    const int head = p / half, i = p % half;
    const int col = head * hd + i;
    float x1 = 0.f, x2 = 0.f;
    for (int s = 0; s < splits; ++s) {
      x1 += wr[s * split_stride + col];
      x2 += wr[s * split_stride + col + half];
    }
    const float ang = __fmul_rn(static_cast<float>(rw.pos), inv_freq[i]);
    double sn, cs;
    sincos(static_cast<double>(ang), &sn, &cs);
    const float c = static_cast<float>(cs), sv = static_cast<float>(sn);
    const float o1 = __fsub_rn(__fmul_rn(x1, c), __fmul_rn(x2, sv));
    const float o2 = __fadd_rn(__fmul_rn(x2, c), __fmul_rn(x1, sv));
    if (head < dm.n_heads) {
      bf16* q = q_out + (static_cast<int64_t>(r) * dm.n_heads + head) * hd;
      q[i] = __float2bfloat16_rn(o1);
      q[i + half] = __float2bfloat16_rn(o2);
    } else {
      const int kvh = head - dm.n_heads;
      bf16* k = kc + ((static_cast<int64_t>(page) * dm.n_kv + kvh) * dm.page_size + off) * hd;
      k[i] = __float2bfloat16_rn(o1);
      k[i + half] = __float2bfloat16_rn(o2);
    }
  }
  const int vbase = (dm.n_heads + dm.n_kv) * hd;
  for (int e = threadIdx.x; e < dm.n_kv * hd; e += 256) {
    float v = 0.f;
    for (int s = 0; s < splits; ++s) v += wr[s * split_stride + vbase + e];
    const int kvh = e / hd, dd = e % hd;
    vc[((static_cast<int64_t>(page) * dm.n_kv + kvh) * dm.page_size + off) * hd + dd] =
        __float2bfloat16_rn(v);
  }
}

void launch_qkv_rope_append(const RowDev* rows, int n, const float* ws, int splits,
                            int64_t split_stride, const LmDims& dm, const float* inv_freq,
                            const int* page_table, bf16* kc, bf16* vc, bf16* q_out,
                            cudaStream_t st) {
  qkv_rope_append_kernel<<<n, 256, 0, st>>>(rows, ws, splits, split_stride, dm, inv_freq,
                                            page_table, kc, vc, q_out);
}

// ---------------------------------------------------------------------------
// paged GQA decode attention.  One CTA per (row, kv head); the G = H/KV query
// heads sharing the kv head are processed together so every K/V byte is read
// once.  Each warp takes 4 tokens at a time (8 lanes per token, hd/8 dims per
// lane, 16/32-byte vector loads, coalesced within the head-page), online
// softmax in fp32, then a 4-warp merge through shared memory.
// ---------------------------------------------------------------------------
template <int HD, int G>
__global__ void __launch_bounds__(128)
    attn_decode_kernel(const RowDev* __restrict__ rows, const bf16* __restrict__ q,
                       const bf16* __restrict__ kc, const bf16* __restrict__ vc,
                       const int* __restrict__ page_table, LmDims dm, bf16* __restrict__ out) {
  constexpr int DPL = HD / 8;  // dims per lane
  __shared__ float s_m[4][G], s_l[4][G];
  __shared__ float s_acc[4][G][HD];
  const int r = blockIdx.x, kvh = blockIdx.y;
  const RowDev rw = rows[r];
  if (rw.slot < 0) return;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int sub = lane >> 3, dl = (lane & 7) * DPL;
  const int L = rw.pos + 1;
  const float scale = 1.0f / sqrtf(static_cast<float>(HD));

  float qv[G][DPL];
#pragma unroll
  for (int g = 0; g < G; ++g) {
    const bf16* qp = q + (static_cast<int64_t>(r) * dm.n_heads + kvh * G + g) * HD + dl;
#pragma unroll
    for (int j = 0; j < DPL; ++j) qv[g][j] = __bfloat162float(qp[j]);
  }
  float m[G], l[G], acc[G][DPL];
#pragma unroll
  for (int g = 0; g < G; ++g) {
    m[g] = -INFINITY;
    l[g] = 0.f;
#pragma unroll
    for (int j = 0; j < DPL; ++j) acc[g][j] = 0.f;
  }
  const int* pt = page_table + static_cast<int64_t>(rw.slot) * dm.max_pages_per_slot;
  const int n_chunks = (L + 3) / 4;
  for (int c = warp; c < n_chunks; c += 4) {
    const int t = c * 4 + sub;
    const bool valid = t < L;
    float kf[DPL], vf[DPL];
    if (valid) {
      const int page = pt[t / dm.page_size];
      const int64_t base =
          ((static_cast<int64_t>(page) * dm.n_kv + kvh) * dm.page_size + (t % dm.page_size)) *
              HD +
          dl;
      const uint4* kp = reinterpret_cast<const uint4*>(kc + base);
      const uint4* vp = reinterpret_cast<const uint4*>(vc + base);
#pragma unroll
      for (int j = 0; j < DPL / 8; ++j) {
        const uint4 ku = kp[j], vu = vp[j];
        const bf16* kb = reinterpret_cast<const bf16*>(&ku);
        const bf16* vb = reinterpret_cast<const bf16*>(&vu);
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          kf[j * 8 + e] = __bfloat162float(kb[e]);
          vf[j * 8 + e] = __bfloat162float(vb[e]);
        }
      }
    } else {
#pragma unroll
      for (int j = 0; j < DPL; ++j) kf[j] = vf[j] = 0.f;
    }
#pragma unroll
    for (int g = 0; g < G; ++g) {
      float s = 0.f;
#pragma unroll
      for (int j = 0; j < DPL; ++j) s = fmaf(qv[g][j], kf[j], s);
      s += __shfl_xor_sync(0xffffffffu, s, 1);
      s += __shfl_xor_sync(0xffffffffu, s, 2);
      s += __shfl_xor_sync(0xffffffffu, s, 4);
      s = valid ? s * scale : -INFINITY;
      float cm = fmaxf(s, __shfl_xor_sync(0xffffffffu, s, 8));
      cm = fmaxf(cm, __shfl_xor_sync(0xffffffffu, cm, 16));
      const float nm = fmaxf(m[g], cm);
      const float corr = expf(m[g] - nm);  // m = -inf initially -> 0
      const float pr = valid ? expf(s - nm) : 0.f;
      l[g] = l[g] * corr + pr;
#pragma unroll
      for (int j = 0; j < DPL; ++j) acc[g][j] = fmaf(pr, vf[j], acc[g][j] * corr);
      m[g] = nm;
    }
  }
  // merge the 4 token sub-groups inside the warp (same m per warp already)
#pragma unroll
  for (int g = 0; g < G; ++g) {
    l[g] += __shfl_xor_sync(0xffffffffu, l[g], 8);
    l[g] += __shfl_xor_sync(0xffffffffu, l[g], 16);
#pragma unroll
    for (int j = 0; j < DPL; ++j) {
      acc[g][j] += __shfl_xor_sync(0xffffffffu, acc[g][j], 8);
      acc[g][j] += __shfl_xor_sync(0xffffffffu, acc[g][j], 16);
    }
    if (lane == 0) {
      s_m[warp][g] = m[g];
      s_l[warp][g] = l[g];
    }
    if (sub == 0) {
#pragma unroll
      for (int j = 0; j < DPL; ++j) s_acc[warp][g][dl + j] = acc[g][j];
    }
  }
  __syncthreads();
  // merge the 4 warps: thread handles (g, dim) pairs
  for (int idx = threadIdx.x; idx < G * HD; idx += 128) {
    const int g = idx / HD, dd = idx % HD;
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < 4; ++w) M = fmaxf(M, s_m[w][g]);
    float Ls = 0.f, A = 0.f;
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      const float f = (s_m[w][g] == -INFINITY) ? 0.f : expf(s_m[w][g] - M);
      Ls += s_l[w][g] * f;
      A += s_acc[w][g][dd] * f;
    }
    out[(static_cast<int64_t>(r) * dm.n_heads + kvh * G + g) * HD + dd] =
        __float2bfloat16_rn(A / Ls);
  }
}

template <int HD>
static void attn_dispatch_g(const RowDev* rows, int n, const bf16* q, const bf16* kc,
                            const bf16* vc, const int* pt, const LmDims& dm, bf16* out,
                            cudaStream_t st) {
  dim3 grid(n, dm.n_kv);
  switch (dm.n_heads / dm.n_kv) {
    case 1: attn_decode_kernel<HD, 1><<<grid, 128, 0, st>>>(rows, q, kc, vc, pt, dm, out); break;
    case 2: attn_decode_kernel<HD, 2><<<grid, 128, 0, st>>>(rows, q, kc, vc, pt, dm, out); break;
    case 3: attn_decode_kernel<HD, 3><<<grid, 128, 0, st>>>(rows, q, kc, vc, pt, dm, out); break;
    case 4: attn_decode_kernel<HD, 4><<<grid, 128, 0, st>>>(rows, q, kc, vc, pt, dm, out); break;
    default: break;  // rejected at vox_create
  }
}

void launch_attn_decode(const RowDev* rows, int n, const bf16* q, const bf16* kc, const bf16* vc,
                        const int* page_table, const LmDims& dm, bf16* out, cudaStream_t st) {
  if (dm.hd == 64)
    attn_dispatch_g<64>(rows, n, q, kc, vc, page_table, dm, out, st);
  else
    attn_dispatch_g<128>(rows, n, q, kc, vc, page_table, dm, out, st);
}

// ---------------------------------------------------------------------------
// split-K reduce + residual add + RMSNorm (optionally compacting output rows)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256)
    resid_norm_kernel(const RowDev* __restrict__ rows, const float* __restrict__ ws, int splits,
                      int64_t split_stride, int d, float eps, float* __restrict__ h,
                      const float* __restrict__ nw, bf16* __restrict__ x_out,
                      const int* __restrict__ out_index) {
  __shared__ float red[33];
  const int r = blockIdx.x;
  if (rows[r].slot < 0) return;
  float* hr = h + static_cast<int64_t>(r) * d;
  const float* wr = ws + static_cast<int64_t>(r) * d;
  float ss = 0.f;
  for (int i = threadIdx.x; i < d; i += 256) {
    float a = 0.f;
    for (int s = 0; s < splits; ++s) a += wr[s * split_stride + i];
    const float v = hr[i] + a;
    hr[i] = v;
    ss = fmaf(v, v, ss);
  }
  ss = block_sum<256>(ss, red);
  const int orow = out_index ? out_index[r] : r;
  if (orow < 0) return;
  const float inv = 1.0f / sqrtf(ss / static_cast<float>(d) + eps);
  bf16* xr = x_out + static_cast<int64_t>(orow) * d;
  for (int i = threadIdx.x; i < d; i += 256)
    xr[i] = __float2bfloat16_rn(__fmul_rn(__fmul_rn(hr[i], inv), nw[i]));
}

void launch_resid_norm(const RowDev* rows, int n, const float* ws, int splits,
                       int64_t split_stride, const LmDims& dm, float* h, const float* norm_w,
                       bf16* x_out, const int* out_index, cudaStream_t st) {
  resid_norm_kernel<<<n, 256, 0, st>>>(rows, ws, splits, split_stride, dm.d, dm.eps, h, norm_w,
                                       x_out, out_index);
}

// ---------------------------------------------------------------------------
// split-K reduce of gate|up + SiLU(gate) * up
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256)
    silu_mul_kernel(const RowDev* __restrict__ rows, const float* __restrict__ ws, int splits,
                    int64_t split_stride, int dff, bf16* __restrict__ a_out) {
  const int r = blockIdx.x;
  if (rows[r].slot < 0) return;
  const float* wr = ws + static_cast<int64_t>(r) * 2 * dff;
  bf16* ar = a_out + static_cast<int64_t>(r) * dff;
  for (int j = threadIdx.x; j < dff; j += 256) {
    float g = 0.f, u = 0.f;
    for (int s = 0; s < splits; ++s) {
      g += wr[s * split_stride + j];
      u += wr[s * split_stride + dff + j];
    }
    const float sg = __fdiv_rn(g, __fadd_rn(1.0f, expf(-g)));
    ar[j] = __float2bfloat16_rn(__fmul_rn(sg, u));
  }
}

void launch_silu_mul(const RowDev* rows, int n, const float* ws, int splits, int64_t split_stride,
                     const LmDims& dm, bf16* a_out, cudaStream_t st) {
  silu_mul_kernel<<<n, 256, 0, st>>>(rows, ws, splits, split_stride, dm.dff, a_out);
}

}  // namespace vox
