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
