// lm_kernels.cu — fused elementwise kernels of one decode step (K5).
//
// Each follows a tcgen05 GEMM and folds its split-K reduction into the op
// that consumes it, with 16-byte vector loads (one CTA per row, 256 threads):
//   embed_norm        embedding gather + first RMSNorm
//   qkv_rope_append   QKV split-K reduce + RoPE (table) + paged KV append
//   resid_norm        O/down split-K reduce + residual add + RMSNorm
//   silu_mul          gate|up split-K reduce + SiLU(gate) * up
// Layouts (HBM):
//   h        [rows, d]            fp32 residual stream
//   x        [rows, d]            bf16 GEMM input (normalised)
//   ws       [splits, rows, N]    fp32 split-K partials written by gemm_tc.cu
//   q        [rows, H, hd]        bf16 (RoPE applied)
//   K pool   [layer][page][kv_head][page_size][hd] bf16 (one head's page is
//            page_size*hd contiguous elements -> one 4 KB bulk copy per head-page)
//   V pool   [layer][page][kv_head][hd][page_size] bf16 (transposed head-page)
//   page_table [slot][max_pages_per_slot] int32
// Rows with slot < 0 are padding and are skipped.
#include "common.cuh"
#include "kernels.h"
#include "rownorm.cuh"
#include <cstdlib>

namespace vox {
VOX_TRACE_TU(trace_set_lm)


// ---------------------------------------------------------------------------
// embedding gather + first RMSNorm
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) embed_norm_kernel(const RowDev* __restrict__ rows,
                                                         int* __restrict__ token_store,
                                                         const int* __restrict__ frame, int nfc,
                                                         const float* __restrict__ ext,
                                                         int max_ctx, const bf16* __restrict__ emb,
                                                         const float* __restrict__ nw, int d,
                                                         float eps, float* __restrict__ h,
                                                         bf16* __restrict__ x) {
  VOX_TRACE(kTrEmbedNorm);
  griddep_wait();
  griddep_launch();
  __shared__ float red[9];
  const int r = blockIdx.x;
  const RowDev rw = rows[r];
  if (rw.slot < 0) return;
  int* ts = token_store + static_cast<int64_t>(rw.slot) * max_ctx + rw.pos;
  float4* h4 = reinterpret_cast<float4*>(h + static_cast<int64_t>(r) * d);
  const int d4 = d / 4;
  float ss = 0.f;
  if (rw.token == -2) {  // external input row (projected hidden state, vox_project_ext)
    const float4* x4 = reinterpret_cast<const float4*>(ext + static_cast<int64_t>(r) * d);
    for (int i = threadIdx.x; i < d4; i += 256) {
      const float4 v = x4[i];
      h4[i] = v;
      ss = fmaf(v.x, v.x, ss);
      ss = fmaf(v.y, v.y, ss);
      ss = fmaf(v.z, v.z, ss);
      ss = fmaf(v.w, v.w, ss);
    }
  }
  int tok = rw.token;
  if (tok >= 0) {
    if (threadIdx.x == 0) *ts = tok;
  } else {
    tok = *ts;
  }
  // multi-codebook frame: ids of codebooks 1..nfc summed in codebook order
  const int* fr = frame != nullptr ? frame + (static_cast<int64_t>(rw.slot) * max_ctx + rw.pos) * nfc : nullptr;
  const bf16* e = emb + static_cast<int64_t>(tok) * d;
  for (int i = threadIdx.x; i < d4 && rw.token != -2; i += 256) {
    const uint2 u = *reinterpret_cast<const uint2*>(e + 4 * i);
    const bf16* b = reinterpret_cast<const bf16*>(&u);
    float4 v = make_float4(__bfloat162float(b[0]), __bfloat162float(b[1]),
                           __bfloat162float(b[2]), __bfloat162float(b[3]));
    for (int cb = 0; cb < nfc && fr != nullptr; ++cb) {
      const int id = fr[cb];
      if (id < 0) continue;
      const uint2 u2 = *reinterpret_cast<const uint2*>(emb + static_cast<int64_t>(id) * d + 4 * i);
      const bf16* b2 = reinterpret_cast<const bf16*>(&u2);
      v.x = __fadd_rn(v.x, __bfloat162float(b2[0]));
      v.y = __fadd_rn(v.y, __bfloat162float(b2[1]));
      v.z = __fadd_rn(v.z, __bfloat162float(b2[2]));
      v.w = __fadd_rn(v.w, __bfloat162float(b2[3]));
    }
    h4[i] = v;
    ss = fmaf(v.x, v.x, ss);
    ss = fmaf(v.y, v.y, ss);
    ss = fmaf(v.z, v.z, ss);
    ss = fmaf(v.w, v.w, ss);
  }
  ss = block_sum256(ss, red);
  const float inv = 1.0f / sqrtf(ss / static_cast<float>(d) + eps);
  const float4* w4 = reinterpret_cast<const float4*>(nw);
  bf16* xr = x + static_cast<int64_t>(r) * d;
  for (int i = threadIdx.x; i < d4; i += 256) norm_store4(xr + 4 * i, h4[i], inv, w4[i]);
}

void launch_embed_norm(const RowDev* rows, int n, int* token_store, const int* frame, int nfc,
                       const float* ext, int max_ctx, const bf16* emb,
                       const float* norm_w, const LmDims& dm, float* h, bf16* x,
                       cudaStream_t st) {
  launch_k(embed_norm_kernel, dim3(n), dim3(256), 0, st, rows, token_store, frame, nfc, ext, max_ctx,
           emb, norm_w, dm.d, dm.eps, h, x);
}

// multi-step decode (vox_forward_steps): every live row moves to its next position and
// takes its input from the token store (the previous step's sample); one row per
// slot, so the row's position is also the lowest position it appends (fresh)
__global__ void advance_rows_kernel(RowDev* rows, int n) {
  griddep_wait();
  griddep_launch();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n && rows[i].slot >= 0) {
    rows[i].pos += 1;
    rows[i].token = -1;
    rows[i].fresh = rows[i].pos;
  }
}

void launch_advance_rows(RowDev* rows, int n, cudaStream_t st) {
  launch_k(advance_rows_kernel, dim3((n + 127) / 128), dim3(128), 0, st, rows, n);
}

// token hand-over between two contexts (CSM backbone <-> depth decoder)
__global__ void link_tokens_kernel(const int* __restrict__ links, int n, const int* __restrict__ src_ts,
                                   int src_max_ctx, int* __restrict__ dst, int dst_max_ctx, int nfc,
                                   int offset, int mode) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (mode == 0) {
    if (i >= n) return;
    const int* l = links + 4 * i;
    dst[static_cast<int64_t>(l[0]) * dst_max_ctx + l[1]] = src_ts[static_cast<int64_t>(l[2]) * src_max_ctx + l[3]] + offset;
  } else {
    if (i >= n * nfc) return;
    const int j = i / nfc, k = i % nfc;
    const int* l = links + 4 * j;
    dst[(static_cast<int64_t>(l[0]) * dst_max_ctx + l[1]) * nfc + k] =
        src_ts[static_cast<int64_t>(l[2]) * src_max_ctx + l[3] + k] + offset;
  }
}

void launch_link_tokens(const int* links, int n, const int* src_ts, int src_max_ctx, int* dst,
                        int dst_max_ctx, int nfc, int offset, int mode, cudaStream_t st) {
  const int total = mode == 0 ? n : n * nfc;
  link_tokens_kernel<<<(total + 127) / 128, 128, 0, st>>>(links, n, src_ts, src_max_ctx, dst, dst_max_ctx,
                                                          nfc, offset, mode);
}

// ---------------------------------------------------------------------------
// split-K reduce of the QKV projection + RoPE + paged KV append.
// rope[pos][i] = (cos, sin) of float(pos) * inv_freq[i] (fp64 -> fp32 table).
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256)
    qkv_rope_append_kernel(const RowDev* __restrict__ rows, const float* __restrict__ ws,
                           const float* __restrict__ bias, int splits, int64_t split_stride, LmDims dm,
                           const float2* __restrict__ rope, const int* __restrict__ page_table,
                           bf16* __restrict__ kc, bf16* __restrict__ vc, bf16* __restrict__ q_out) {
  VOX_TRACE(kTrQkvRope);
  // row descriptor, page-table entry and the RoPE table of this thread's first
  // item do not depend on the QKV GEMM: load them before waiting for it
  const int r = blockIdx.x;
  const RowDev rw = rows[r];
  const int hd = dm.hd, half = hd / 2;
  const int q4 = half / 4;
  const int n_items = (dm.n_heads + dm.n_kv) * q4;
  const int cta_stride = 256 * gridDim.y;
  const int it0 = threadIdx.x + 256 * blockIdx.y;
  int page = 0;
  float2 cs0[4];
  if (rw.slot >= 0) {
    page = page_table[static_cast<int64_t>(rw.slot) * dm.max_pages_per_slot + rw.pos / dm.page_size];
    if (it0 < n_items) {
      const float2* rp0 = rope + static_cast<int64_t>(rw.pos) * half + (it0 % q4) * 4;
#pragma unroll
      for (int e = 0; e < 4; ++e) cs0[e] = rp0[e];
    }
  }
  griddep_wait();
  griddep_launch();
  if (rw.slot < 0) return;
  const int nqkv = (dm.n_heads + 2 * dm.n_kv) * hd;
  const float4* w4 = reinterpret_cast<const float4*>(ws + static_cast<int64_t>(r) * nqkv);
  const int64_t ss4 = split_stride / 4;
  const int off = rw.pos % dm.page_size;
  const float2* rp = rope + static_cast<int64_t>(rw.pos) * half;
  // rotated heads (q then k): thread handles 4 consecutive pair indices i..i+3;
  // gridDim.y CTAs share a row (interleaved items) for more loads in flight
  for (int it = threadIdx.x + 256 * blockIdx.y; it < n_items; it += cta_stride) {
    const int head = it / q4, i = (it % q4) * 4;
    const int c1 = (head * hd + i) / 4, c2 = (head * hd + i + half) / 4;
    float4 a = sum_splits4(w4, splits, ss4, c1);
    float4 b = sum_splits4(w4, splits, ss4, c2);
    if (bias != nullptr) {  // Qwen2-style q|k|v bias, added after the split-K sum
      a = add4(a, reinterpret_cast<const float4*>(bias)[c1]);
      b = add4(b, reinterpret_cast<const float4*>(bias)[c2]);
    }
    const float x1[4] = {a.x, a.y, a.z, a.w}, x2[4] = {b.x, b.y, b.z, b.w};
    float o1[4], o2[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 cs = it == it0 ? cs0[e] : rp[i + e];
      o1[e] = __fsub_rn(__fmul_rn(x1[e], cs.x), __fmul_rn(x2[e], cs.y));
      o2[e] = __fadd_rn(__fmul_rn(x2[e], cs.x), __fmul_rn(x1[e], cs.y));
    }
    bf16* dst;
    if (head < dm.n_heads) {
      dst = q_out + (static_cast<int64_t>(r) * dm.n_heads + head) * hd;
    } else {
      const int kvh = head - dm.n_heads;
      dst = kc + ((static_cast<int64_t>(page) * dm.n_kv + kvh) * dm.page_size + off) * hd;
    }
    store_bf16x4(dst + i, o1[0], o1[1], o1[2], o1[3]);
    store_bf16x4(dst + i + half, o2[0], o2[1], o2[2], o2[3]);
  }
  const int vbase4 = (dm.n_heads + dm.n_kv) * hd / 4;
  const int hd4 = hd / 4;
  // V head-pages are stored TRANSPOSED ([hd][page_size]) so the attention PV
  // mma reads 4 consecutive tokens of one dim as a single 8-byte load
  for (int e = threadIdx.x + 256 * blockIdx.y; e < dm.n_kv * hd4; e += cta_stride) {
    float4 v = sum_splits4(w4, splits, ss4, vbase4 + e);
    if (bias != nullptr) v = add4(v, reinterpret_cast<const float4*>(bias)[vbase4 + e]);
    const int kvh = e / hd4, dd = (e % hd4) * 4;
    bf16* vt = vc + ((static_cast<int64_t>(page) * dm.n_kv + kvh) * hd + dd) * dm.page_size + off;
    vt[0] = __float2bfloat16_rn(v.x);
    vt[dm.page_size] = __float2bfloat16_rn(v.y);
    vt[2 * dm.page_size] = __float2bfloat16_rn(v.z);
    vt[3 * dm.page_size] = __float2bfloat16_rn(v.w);
  }
}

void launch_qkv_rope_append(const RowDev* rows, int n, const float* ws, const float* bias, int splits,
                            int64_t split_stride, const LmDims& dm, const float2* rope,
                            const int* page_table, bf16* kc, bf16* vc, bf16* q_out,
                            cudaStream_t st) {
  // CTAs per row: two while that keeps the grid within two per SM (64 / 128 rows:
  // 1% faster steps than one), one beyond (224 rows: 448 CTAs left a third of them
  // starting up to 6 us after the QKV GEMM ended; one per row is 1% faster); 8 for
  // <= 32 rows measured no different from 2
  const int gy = n <= vox_sm_budget() ? 2 : 1;
  launch_k(qkv_rope_append_kernel, dim3(n, gy), dim3(256), 0, st, rows, ws, bias, splits, split_stride, dm,
           rope, page_table, kc, vc, q_out);
}

// ---------------------------------------------------------------------------
// split-K reduce + residual add + RMSNorm (optionally compacting output rows)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(768)
    resid_norm_kernel(const RowDev* __restrict__ rows, const float* __restrict__ ws, int splits,
                      int64_t split_stride, int d, float eps, float* __restrict__ h,
                      const float* __restrict__ nw, bf16* __restrict__ x_out,
                      const int* __restrict__ out_index) {
  VOX_TRACE(kTrResidNorm);
  __shared__ float red[33];
  const int r = blockIdx.x;
  const int d4 = d / 4, nt = blockDim.x;
  if (d4 > 4 * nt) {  // wide rows: the generic path
    griddep_wait();
    griddep_launch();
    if (rows[r].slot < 0) return;
    resid_norm_row(r, ws, splits, split_stride, d, eps, h, nw, x_out, out_index ? out_index[r] : r, red);
    return;
  }
  // h (written >= 2 launches upstream: every kernel of the step launches its
  // dependents only after its own griddep_wait) and the norm weights do not
  // depend on the preceding GEMM: load them before waiting for it
  const bool live = rows[r].slot >= 0;
  const int orow = out_index ? out_index[r] : r;
  float4* h4 = reinterpret_cast<float4*>(h + static_cast<int64_t>(r) * d);
  const float4* n4 = reinterpret_cast<const float4*>(nw);
  float4 hv[4], nv[4];
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int i = threadIdx.x + k * nt;
    if (live && i < d4) {
      hv[k] = h4[i];
      nv[k] = n4[i];
    }
  }
  griddep_wait();
  griddep_launch();
  if (!live) return;
  const float4* w4 = reinterpret_cast<const float4*>(ws + static_cast<int64_t>(r) * d);
  const int64_t ss4 = split_stride / 4;
  float ss = 0.f;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int i = threadIdx.x + k * nt;
    if (i < d4) {
      hv[k] = add4(hv[k], sum_splits4(w4, splits, ss4, i));
      h4[i] = hv[k];
      ss = fmaf(hv[k].x, hv[k].x, ss);
      ss = fmaf(hv[k].y, hv[k].y, ss);
      ss = fmaf(hv[k].z, hv[k].z, ss);
      ss = fmaf(hv[k].w, hv[k].w, ss);
    }
  }
  ss = block_sum_any(ss, red);
  if (orow < 0) return;
  const float inv = 1.0f / sqrtf(ss / static_cast<float>(d) + eps);
  bf16* xr = x_out + static_cast<int64_t>(orow) * d;
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const int i = threadIdx.x + k * nt;
    if (i < d4) norm_store4(xr + 4 * i, hv[k], inv, nv[k]);
  }
}

void launch_resid_norm(const RowDev* rows, int n, const float* ws, int splits,
                       int64_t split_stride, const LmDims& dm, float* h, const float* norm_w,
                       bf16* x_out, const int* out_index, cudaStream_t st) {
  // few rows: more threads per row shorten each row's dependent-load chain; many
  // rows: 256-thread CTAs co-reside with the PDL-launched GEMM CTAs (768 threads
  // measured slower at 224 rows, profiles/gemm_mc_ab_r01.txt)
  int nt = 256;
  if (n <= 32) {  // one float4 per thread (d = 3072: 768 threads)
    nt = (dm.d / 4 + 31) / 32 * 32;
    nt = nt < 256 ? 256 : (nt > 768 ? 768 : nt);
  }
  launch_k(resid_norm_kernel, dim3(n), dim3(nt), 0, st, rows, ws, splits, split_stride, dm.d,
           dm.eps, h, norm_w, x_out, out_index);
}

// ---------------------------------------------------------------------------
// split-K reduce of gate|up + SiLU(gate) * up
// ---------------------------------------------------------------------------
VOX_DEV float silu_mul1(float g, float u) {
  return __fmul_rn(__fdiv_rn(g, __fadd_rn(1.0f, expf(-g))), u);
}

__global__ void __launch_bounds__(256)
    silu_mul_kernel(const RowDev* __restrict__ rows, const float* __restrict__ ws, int splits,
                    int64_t split_stride, int dff, bf16* __restrict__ a_out) {
  VOX_TRACE(kTrSilu);
  griddep_wait();
  griddep_launch();
  const int r = blockIdx.x;
  if (rows[r].slot < 0) return;
  const float4* w4 = reinterpret_cast<const float4*>(ws + static_cast<int64_t>(r) * 2 * dff);
  const int64_t ss4 = split_stride / 4;
  const int f4 = dff / 4;
  bf16* ar = a_out + static_cast<int64_t>(r) * dff;
  // gate|up columns are interleaved per 128 (the packed weight tiles): feature
  // f's gate at column 128 (f / 64) + f % 64, its up 64 columns later
#pragma unroll 4
  for (int j = threadIdx.x; j < f4; j += 256) {
    const int f = 4 * j;
    const int cg = ((f >> 6) << 7) + (f & 63);
    const float4 g = sum_splits4(w4, splits, ss4, cg / 4);
    const float4 u = sum_splits4(w4, splits, ss4, (cg + 64) / 4);
    store_bf16x4(ar + 4 * j, silu_mul1(g.x, u.x), silu_mul1(g.y, u.y), silu_mul1(g.z, u.z),
                 silu_mul1(g.w, u.w));
  }
}

void launch_silu_mul(const RowDev* rows, int n, const float* ws, int splits, int64_t split_stride,
                     const LmDims& dm, bf16* a_out, cudaStream_t st) {
  launch_k(silu_mul_kernel, dim3(n), dim3(256), 0, st, rows, ws, splits, split_stride, dm.dff,
           a_out);
}

}  // namespace vox
