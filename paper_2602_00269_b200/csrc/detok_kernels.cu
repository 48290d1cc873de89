// detok_kernels.cu — K4: causal SNAC-24kHz-style decoder, stencil/elementwise part.
//
// The decoder runs on a ragged batch of requests (DetokReq).  Every dense
// contraction (1x1 convs, transposed convs) is an implicit GEMM on the
// tcgen05 kernel (gemm_tc.cu); the kernels here do the VQ-decode gather,
// Snake activations, depthwise dilated causal convs and the output conv, and
// maintain each request's cached LEFT CONTEXT so a chunk decodes only its new
// frames (no history recompute):
//   history buffers [H][C] fp32 per slot, double-buffered by chunk parity:
//   read state[parity], write state[1-parity].
// Row r of a level with cumulative upsampling `up` belongs to request i with
// reqs[i].lat_off*up <= r < (reqs[i].lat_off + 4*reqs[i].nf)*up.
#include "common.cuh"
#include "kernels.h"

namespace vox {
VOX_TRACE_TU(trace_set_detok)


struct ReqHdr {  // first bytes of the uploaded detok staging block
  int32_t n_req, n_lat;
};

VOX_DEV int find_req(const DetokReq* reqs, int n_req, int lat_row) {
  int lo = 0, hi = n_req - 1;
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (reqs[mid].lat_off <= lat_row) lo = mid; else hi = mid - 1;
  }
  return lo;
}

VOX_DEV float snake(float x, float a) {
  const float s = snake_sin(__fmul_rn(a, x));
  return __fadd_rn(x, __fmul_rn(__fdiv_rn(1.0f, __fadd_rn(a, 1e-9f)), __fmul_rn(s, s)));
}

VOX_DEV float* slot_state(float* state, const DetokDims& dd, int slot, int parity) {
  return state + (static_cast<int64_t>(slot) * 2 + parity) * dd.state_floats;
}

// Orpheus frame layout: position k of 7 -> (codebook, sub-index)
//   k: 0->(0,0) 1->(1,0) 2->(2,0) 3->(2,1) 4->(1,1) 5->(2,2) 6->(2,3)
VOX_DEV int frame_code(const int* ts_slot, const DetokReq& q, const DetokDims& dd, int f, int k) {
  const int g = f * dd.frame_tokens + k;  // generated-token index
  if (g >= q.n_tokens) return 0;          // partial final frame: pad with code 0
  int c = ts_slot[q.prompt_len + g] - dd.audio_base - k * dd.cb_size;
  return c < 0 ? 0 : (c >= dd.cb_size ? dd.cb_size - 1 : c);
}

VOX_DEV float vq_latent(const int* ts_slot, const DetokReq& q, const DetokDims& dd,
                        const bf16* tabs, int t_local, int ch) {
  const int f = q.f0 + (t_local >> 2), j = t_local & 3;
  const int c0 = frame_code(ts_slot, q, dd, f, 0);
  const int c1 = frame_code(ts_slot, q, dd, f, j < 2 ? 1 : 4);
  const int k2 = (j == 0) ? 2 : (j == 1) ? 3 : (j == 2) ? 5 : 6;
  const int c2 = frame_code(ts_slot, q, dd, f, k2);
  const int64_t tab = static_cast<int64_t>(dd.cb_size) * dd.latent;
  const float a = __bfloat162float(tabs[static_cast<int64_t>(c0) * dd.latent + ch]);
  const float b = __bfloat162float(tabs[tab + static_cast<int64_t>(c1) * dd.latent + ch]);
  const float c = __bfloat162float(tabs[2 * tab + static_cast<int64_t>(c2) * dd.latent + ch]);
  return __fadd_rn(__fadd_rn(a, b), c);
}

// VQ decode (3 projected-codebook gathers, repeat x4/x2/x1) + depthwise causal
// k7 conv over the latent sequence.  grid: latent rows, block: 256.
__global__ void __launch_bounds__(256)
    vq_dwconv_kernel(const ReqHdr* hdr, const DetokReq* __restrict__ reqs,
                     const int* __restrict__ token_store, const bf16* __restrict__ tabs,
                     const float* __restrict__ dw_w, const float* __restrict__ dw_b,
                     float* __restrict__ state, DetokDims dd, bf16* __restrict__ out) {
  VOX_TRACE(kTrDetok);
  griddep_wait();
  griddep_launch();
  // grid: (latent rows, channel blocks of 256): each thread owns one channel of one row
  const int row = blockIdx.x;
  if (row >= hdr->n_lat) return;
  const int ri = find_req(reqs, hdr->n_req, row);
  const DetokReq q = reqs[ri];
  const int t = row - q.lat_off;
  const int n = 4 * q.nf;
  const int C = dd.latent, H = 6;
  const int ch = blockIdx.y * 256 + threadIdx.x;
  if (ch >= C) return;
  const int* ts = token_store + static_cast<int64_t>(q.slot) * dd.max_ctx;
  const float* hin = slot_state(state, dd, q.slot, q.parity) + dd.off_in;
  float* hout = slot_state(state, dd, q.slot, q.parity ^ 1) + dd.off_in;
  // the 7 taps' latents first (independent gathers in flight), then the conv
  float z[7];
#pragma unroll
  for (int k = 0; k < 7; ++k) {
    const int tt = t - 6 + k;
    z[k] = tt >= 0 ? vq_latent(ts, q, dd, tabs, tt, ch) : hin[(H + tt) * C + ch];
  }
  float acc = dw_b[ch];
#pragma unroll
  for (int k = 0; k < 7; ++k) acc = fmaf(dw_w[ch * 7 + k], z[k], acc);
  out[static_cast<int64_t>(row) * C + ch] = __float2bfloat16_rn(acc);
  if (t >= n - H) hout[(t - (n - H)) * C + ch] = z[6];  // vq_latent at t (tap 6)
  for (int hh = t; hh < H - n; hh += n) hout[hh * C + ch] = hin[(hh + n) * C + ch];
}

void launch_vq_dwconv(const DetokReq* reqs, int n_req, int n_lat, const int* token_store,
                      const bf16* tabs, const float* dw_w, const float* dw_b, float* state,
                      const DetokDims& dd, bf16* out_bf16, cudaStream_t st) {
  const ReqHdr* hdr = reinterpret_cast<const ReqHdr*>(reqs) - 1;
  (void)n_req;
  launch_k(vq_dwconv_kernel, dim3(n_lat, (dd.latent + 255) / 256), dim3(256), 0, st, hdr, reqs, token_store, tabs,
           dw_w, dw_b, state, dd, out_bf16);
}

// Snake + build the transposed-conv GEMM operand [s(x_t) | s(x_{t-1})] (bf16),
// history = 1 frame of s(x).  grid: rows of this level.
__global__ void __launch_bounds__(256)
    snake_upcat_kernel(const ReqHdr* hdr, const DetokReq* __restrict__ reqs, int up,
                       const float* __restrict__ x, int C, const float* __restrict__ alpha,
                       float* __restrict__ state, int64_t st_off, DetokDims dd,
                       bf16* __restrict__ out) {
  VOX_TRACE(kTrDetok);
  griddep_wait();
  griddep_launch();
  const int row = blockIdx.x;
  if (row >= hdr->n_lat * up) return;
  const int ri = find_req(reqs, hdr->n_req, row / up);
  const DetokReq q = reqs[ri];
  const int t = row - q.lat_off * up;
  const int n = 4 * q.nf * up;
  const float* hin = slot_state(state, dd, q.slot, q.parity) + st_off;
  float* hout = slot_state(state, dd, q.slot, q.parity ^ 1) + st_off;
  const float* xr = x + static_cast<int64_t>(row) * C;
  bf16* o = out + static_cast<int64_t>(row) * 2 * C;
  for (int ch = threadIdx.x; ch < C; ch += 256) {
    const float a = alpha[ch];
    const float cur = snake(xr[ch], a);
    const float prev = t > 0 ? snake(xr[ch - C], a) : hin[ch];
    o[ch] = __float2bfloat16_rn(cur);
    o[C + ch] = __float2bfloat16_rn(prev);
    if (t == n - 1) hout[ch] = cur;
  }
}

void launch_snake_upcat(const DetokReq* reqs, int n_req, int rows, int up_before,
                        const float* x, int C, const float* alpha, float* state, int64_t st_off,
                        const DetokDims& dd, bf16* out_cat, cudaStream_t st) {
  const ReqHdr* hdr = reinterpret_cast<const ReqHdr*>(reqs) - 1;
  (void)n_req;
  launch_k(snake_upcat_kernel, dim3(rows), dim3(256), 0, st, hdr, reqs, up_before, x, C, alpha, state, st_off, dd,
                                           out_cat);
}

// Residual-unit prologue: y1 = snake1(x); u = dwconv7_dil(y1) (causal, history
// 6*dil frames of y1); out = bf16(snake2(u)) -> 1x1 GEMM (+bias +x residual).
__global__ void __launch_bounds__(128)
    ru_prep_kernel(const ReqHdr* hdr, const DetokReq* __restrict__ reqs, int up,
                   const float* __restrict__ x, int C, int dil, const float* __restrict__ alpha1,
                   const float* __restrict__ dw_w, const float* __restrict__ dw_b,
                   const float* __restrict__ alpha2, float* __restrict__ state, int64_t st_off,
                   DetokDims dd, bf16* __restrict__ out) {
  VOX_TRACE(kTrDetok);
  griddep_wait();
  griddep_launch();
  const int row = blockIdx.x;
  if (row >= hdr->n_lat * up) return;
  const int ri = find_req(reqs, hdr->n_req, row / up);
  const DetokReq q = reqs[ri];
  const int t = row - q.lat_off * up;
  const int n = 4 * q.nf * up;
  const int H = 6 * dil;
  const float* hin = slot_state(state, dd, q.slot, q.parity) + st_off;
  float* hout = slot_state(state, dd, q.slot, q.parity ^ 1) + st_off;
  const int64_t base = static_cast<int64_t>(q.lat_off) * up;  // first row of this request
  for (int ch = threadIdx.x; ch < C; ch += 128) {
    const float a1 = alpha1[ch];
    float acc = dw_b[ch];
#pragma unroll
    for (int k = 0; k < 7; ++k) {
      const int tt = t - (6 - k) * dil;
      const float y = tt >= 0 ? snake(x[(base + tt) * C + ch], a1) : hin[(H + tt) * C + ch];
      acc = fmaf(dw_w[ch * 7 + k], y, acc);
    }
    out[static_cast<int64_t>(row) * C + ch] = __float2bfloat16_rn(snake(acc, alpha2[ch]));
    if (t >= n - H) hout[(t - (n - H)) * C + ch] = snake(x[(base + t) * C + ch], a1);
    for (int hh = t; hh < H - n; hh += n) hout[hh * C + ch] = hin[(hh + n) * C + ch];
  }
}

void launch_ru_prep(const DetokReq* reqs, int n_req, int rows, int up, const float* x, int C,
                    int dil, const float* alpha1, const float* dw_w, const float* dw_b,
                    const float* alpha2, float* state, int64_t st_off, const DetokDims& dd,
                    bf16* out, cudaStream_t st) {
  const ReqHdr* hdr = reinterpret_cast<const ReqHdr*>(reqs) - 1;
  (void)n_req;
  launch_k(ru_prep_kernel, dim3(rows), dim3(128), 0, st, hdr, reqs, up, x, C, dil, alpha1, dw_w, dw_b, alpha2,
                                       state, st_off, dd, out);
}

// Output head: snake -> causal conv k7 (C -> 1) -> tanh -> PCM.  One warp per
// output sample; history = 6 frames of snake(x).
__global__ void __launch_bounds__(256)
    detok_out_kernel(const ReqHdr* hdr, const DetokReq* __restrict__ reqs, int up,
                     const float* __restrict__ x, int C, const float* __restrict__ alpha,
                     const float* __restrict__ w, float b, float* __restrict__ state,
                     int64_t st_off, DetokDims dd, float* __restrict__ pcm) {
  VOX_TRACE(kTrDetok);
  griddep_wait();
  griddep_launch();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int row = blockIdx.x * 8 + warp;
  if (row >= hdr->n_lat * up) return;
  const int ri = find_req(reqs, hdr->n_req, row / up);
  const DetokReq q = reqs[ri];
  const int t = row - q.lat_off * up;
  const int n = 4 * q.nf * up;
  const int H = 6;
  const float* hin = slot_state(state, dd, q.slot, q.parity) + st_off;
  float* hout = slot_state(state, dd, q.slot, q.parity ^ 1) + st_off;
  const int64_t base = static_cast<int64_t>(q.lat_off) * up;
  float acc = 0.f;
  for (int ch = lane; ch < C; ch += 32) {
    const float a = alpha[ch];
#pragma unroll
    for (int k = 0; k < 7; ++k) {
      const int tt = t - 6 + k;
      const float y = tt >= 0 ? snake(x[(base + tt) * C + ch], a) : hin[(H + tt) * C + ch];
      acc = fmaf(w[ch * 7 + k], y, acc);
    }
    if (t >= n - H) hout[(t - (n - H)) * C + ch] = snake(x[(base + t) * C + ch], a);
    for (int hh = t; hh < H - n; hh += n) hout[hh * C + ch] = hin[(hh + n) * C + ch];
  }
  acc = warp_sum(acc);
  if (lane == 0 && t < q.n_samples) pcm[q.pcm_off + t] = tanhf(acc + b);
}

void launch_detok_out(const DetokReq* reqs, int n_req, int rows, int up, const float* x, int C,
                      const float* alpha, const float* w, float b, float* state, int64_t st_off,
                      const DetokDims& dd, float* pcm, cudaStream_t st) {
  const ReqHdr* hdr = reinterpret_cast<const ReqHdr*>(reqs) - 1;
  (void)n_req;
  launch_k(detok_out_kernel, dim3((rows + 7) / 8), dim3(256), 0, st, hdr, reqs, up, x, C, alpha, w, b, state,
                                                   st_off, dd, pcm);
}

}  // namespace vox
