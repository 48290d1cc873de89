// detok_fused.cu — K4 fine levels: one kernel per residual unit, and a tiled
// output head.
//
// At the fine decoder levels (C = 64 / 128 channels, 2^17..2^18 rows per
// steady-state detok call) the residual unit
//     y1 = Snake(x; a1);  u = b + dwconv7_dil(y1) (causal);  v = Snake(u; a2)
//     x' = x + pw_b + v . W^T                                  (1x1 conv)
// is memory/latency bound, not FLOP bound (K = C is tiny).  ru_fused_kernel
// does it in one pass over a 128-row tile:
//   1. y1 for rows [r0 - 6*dil, r0 + 128) into shared memory (Snake computed
//      once per element; rows before the request's first row come from its
//      cached left context, state[parity]; the new context is written to
//      state[parity ^ 1]),
//   2. v = Snake(dwconv(y1)) for the tile's 128 rows, rounded to bf16 straight
//      into the 128B-swizzled K-major UMMA operand layout in shared memory,
//   3. one elected thread issues tcgen05.mma (M = 128 rows, N = C, K = C;
//      W^T staged in shared memory in the same layout), accumulator in TMEM,
//   4. tcgen05.ld -> shared staging -> coalesced x + pw_b + acc -> y.
// The intermediate v never touches global memory and the unit is one launch
// instead of two.  A tile never straddles two requests: request row ranges
// are multiples of 4*up rows and 4*up >= 1024 at these levels (host checks).
// Arithmetic and rounding points are those of ru_prep_kernel + the GEMM
// (oracle/snac.py: bf16 GEMM operands, fp32 everything else).
#include "common.cuh"
#include "kernels.h"

namespace vox {
VOX_TRACE_TU(trace_set_detok_fused)


namespace {

struct ReqHdrF {
  int32_t n_req, n_lat;
};

// warp-cooperative lookup (lat_row uniform across the warp): the last request
// whose lat_off <= lat_row, one coalesced round of loads per 32 requests
// instead of log2(n_req) dependent loads
VOX_DEV int find_req_w(const DetokReq* reqs, int n_req, int lat_row) {
  const int lane = threadIdx.x & 31;
  int best = 0;
  for (int base = 0; base < n_req; base += 32) {
    const int i = base + lane;
    const unsigned m = __ballot_sync(0xffffffffu, i < n_req && reqs[i].lat_off <= lat_row);
    if (m == 0) break;
    best = base + 31 - __clz(m);
    if (m != 0xffffffffu) break;
  }
  return best;
}


VOX_DEV float snake_f(float x, float a) {
  const float s = snake_sin(__fmul_rn(a, x));
  return __fadd_rn(x, __fmul_rn(__fdiv_rn(1.0f, __fadd_rn(a, 1e-9f)), __fmul_rn(s, s)));
}
// same value with the per-channel reciprocal 1 / (a + 1e-9) precomputed
VOX_DEV float snake_r(float x, float a, float inv) {
  const float s = snake_sin(__fmul_rn(a, x));
  return __fadd_rn(x, __fmul_rn(inv, __fmul_rn(s, s)));
}
VOX_DEV float snake_inv(float a) { return __fdiv_rn(1.0f, __fadd_rn(a, 1e-9f)); }

VOX_DEV float* slot_state_f(float* state, const DetokDims& dd, int slot, int parity) {
  return state + (static_cast<int64_t>(slot) * 2 + parity) * dd.state_floats;
}

// byte offset of element (row r, k) in a K-major SWIZZLE_128B operand whose
// 64-element k-regions are stored one after another (rows x 128 B each)
VOX_DEV uint32_t swz_off(int r, int k, int rows) {
  const int kr = k >> 6, kk = k & 63;
  const int chunk = (kk >> 3) ^ (r & 7);
  return static_cast<uint32_t>(kr * rows * 128 + r * 128 + chunk * 16 + (kk & 7) * 2);
}

}  // namespace

constexpr int kRuRows = 128;  // rows per tile (UMMA M)
// threads: 8 threads per channel (C = 128 runs 1 CTA per SM, so it gets 32
// warps to hide the Snake / dwconv latency chains)
template <int C>
__host__ __device__ constexpr int ru_threads() { return C == 64 ? 512 : 1024; }

template <int C>
struct RuSmem {
  static constexpr int kMaxHalo = 6 * 9;
  static constexpr int kY1Floats = (kRuRows + kMaxHalo) * C;
  static constexpr int kStage = kRuRows * (C + 1);  // epilogue staging (reuses y1)
  static constexpr int kY1Bytes = (kY1Floats > kStage ? kY1Floats : kStage) * 4;
  static constexpr int kABytes = kRuRows * C * 2;
  static constexpr int kBBytes = C * C * 2;
  static constexpr int kAOff = (kY1Bytes + 1023) / 1024 * 1024;
  static constexpr int kBOff = kAOff + kABytes;
  static constexpr int kBarOff = kBOff + kBBytes;
  static constexpr int kBytes = kBarOff + 64 + 1024;  // + alignment slack
};

template <int C>
__global__ void __launch_bounds__(ru_threads<C>())
    ru_fused_kernel(const ReqHdrF* hdr, const DetokReq* __restrict__ reqs, int up,
                    const float* __restrict__ x, float* __restrict__ y, int dil,
                    const float* __restrict__ alpha1, const float* __restrict__ dw_w,
                    const float* __restrict__ dw_b, const float* __restrict__ alpha2,
                    const bf16* __restrict__ pw_w, const float* __restrict__ pw_b,
                    float* __restrict__ state, int64_t st_off, DetokDims dd) {
  VOX_TRACE(kTrDetok);
  using L = RuSmem<C>;
  constexpr int kRuThreads = ru_threads<C>();
  extern __shared__ uint8_t smem_raw[];
  // align to 1024 B by pointer arithmetic on the __shared__ array (an
  // integer round-trip would turn every smem access into a generic LD/ST)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  float* y1s = reinterpret_cast<float*>(smem);
  uint8_t* sa = smem + L::kAOff;
  uint8_t* sb = smem + L::kBOff;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + L::kBarOff);
  uint64_t* xbar = bar + 1;  // bulk copy of the x tile
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar + 2);

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int r0 = blockIdx.x * kRuRows;

  // weights do not depend on the preceding kernel: stage W (K-major, swizzled)
  for (int e = tid; e < C * C / 8; e += kRuThreads) {
    const int n = e / (C / 8), k = (e % (C / 8)) * 8;
    *reinterpret_cast<uint4*>(sb + swz_off(n, k, C)) =
        *reinterpret_cast<const uint4*>(pw_w + static_cast<int64_t>(n) * C + k);
  }
  if (tid == 0) {
    mbar_init(bar, 1);
    mbar_init(xbar, 1);
    fence_mbar_init();
  }
  if (warp == 0) tmem_alloc(tmem_slot, C);
  __syncthreads();  // barriers initialised before thread 0 arms xbar
  griddep_wait();
  griddep_launch();
  const int n_rows = hdr->n_lat * up;
  const bool active = r0 < n_rows;

  // ---------------- 1. y1 = Snake(x) for the tile + causal halo ----------------
  // The tile's x rows (and, for a request's first tile, the cached Snake'd
  // left context) arrive by 1-D bulk copies into y1s -- one transfer instead of
  // ~12 rounds of dependent per-thread loads -- then Snake runs in place.
  const int H = 6 * dil;
  constexpr int kRowStep = kRuThreads / C;      // rows between a thread's elements
  constexpr int kResRows = kRuRows / kRowStep;  // epilogue rows per thread
  int t0 = 0, n = 0;
  const float* hin = nullptr;
  float* hout = nullptr;
  float xres[kResRows];  // residual x of the rows this thread stores in the epilogue
  if (active) {
    const DetokReq q = reqs[find_req_w(reqs, hdr->n_req, r0 / up)];
    t0 = r0 - q.lat_off * up;  // local row of the tile's first row
    n = 4 * q.nf * up;         // rows of this request at this level
    hin = slot_state_f(state, dd, q.slot, q.parity) + st_off;
    hout = slot_state_f(state, dd, q.slot, q.parity ^ 1) + st_off;
    const int nr = kRuRows + H;
    const int i_first = t0 >= H ? 0 : H - t0;  // halo rows [0, i_first) come from the context
    if (tid == 0) {
      const uint32_t bx = static_cast<uint32_t>((nr - i_first) * C * 4);
      const uint32_t bh = static_cast<uint32_t>(i_first * C * 4);
      mbar_arrive_expect_tx(xbar, bx + bh);
      const uint64_t pol = policy_evict_first();
      bulk_load(y1s + i_first * C, x + static_cast<int64_t>(r0 - H + i_first) * C, bx, xbar, pol);
      if (bh) bulk_load(y1s, hin + static_cast<int64_t>(t0) * C, bh, xbar, pol);
    }
    mbar_wait(xbar, 0);
    const int ch = tid % C;
#pragma unroll
    for (int k = 0; k < kResRows; ++k) xres[k] = y1s[(H + tid / C + k * kRowStep) * C + ch];
    __syncthreads();  // every residual read before Snake overwrites in place
    const float a1 = alpha1[ch], inv1 = snake_inv(a1);
#pragma unroll 4
    for (int i = i_first + tid / C; i < nr; i += kRowStep) {
      const float v = snake_r(y1s[i * C + ch], a1, inv1);
      const int t = t0 - H + i;
      if (i >= H && t >= n - H) hout[(t - (n - H)) * C + ch] = v;  // new left context
      y1s[i * C + ch] = v;
    }
    // short requests (n < H): shift the old context
    for (int e = tid; e < kRuRows * C; e += kRuThreads) {
      const int i = e / C, c2 = e % C, t = t0 + i;
      for (int hh = t; hh < H - n; hh += n) hout[hh * C + c2] = hin[(hh + n) * C + c2];
    }
  } else {
    __syncthreads();
  }
  __syncthreads();

  // ---------------- 2. v = Snake(dwconv(y1)) -> bf16 UMMA operand ----------------
  if (active) {
    // each thread owns a channel pair (kRuThreads % (C / 2) == 0)
    constexpr int kRowStep2 = kRuThreads / (C / 2);
    const int ch = (tid % (C / 2)) * 2;
    float w0[7], w1[7];
#pragma unroll
    for (int k = 0; k < 7; ++k) {
      w0[k] = dw_w[ch * 7 + k];
      w1[k] = dw_w[(ch + 1) * 7 + k];
    }
    const float b0 = dw_b[ch], b1 = dw_b[ch + 1];
    const float a20 = alpha2[ch], a21 = alpha2[ch + 1];
    const float i20 = snake_inv(a20), i21 = snake_inv(a21);
#pragma unroll 2
    for (int i = tid / (C / 2); i < kRuRows; i += kRowStep2) {
      float acc0 = b0, acc1 = b1;
#pragma unroll
      for (int k = 0; k < 7; ++k) {
        const float* yr = y1s + (H + i - (6 - k) * dil) * C + ch;
        acc0 = fmaf(w0[k], yr[0], acc0);
        acc1 = fmaf(w1[k], yr[1], acc1);
      }
      const __nv_bfloat162 pr = __floats2bfloat162_rn(snake_r(acc0, a20, i20), snake_r(acc1, a21, i21));
      *reinterpret_cast<__nv_bfloat162*>(sa + swz_off(i, ch, kRuRows)) = pr;
    }
  }
  fence_proxy_async();  // generic-proxy smem writes -> visible to tcgen05 (async proxy)
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  // ---------------- 3. tcgen05.mma: acc[128 x C] = v[128 x C] . W^T ----------------
  if (active && tid == 0) {
    constexpr uint32_t idesc = make_idesc_bf16(128, C);
    const uint32_t a0 = smem_u32(sa), b0 = smem_u32(sb);
#pragma unroll
    for (int kr = 0; kr < C / 64; ++kr)
#pragma unroll
      for (int k = 0; k < 4; ++k)
        umma_bf16(tmem, make_desc_k128(a0 + kr * kRuRows * 128 + k * 32),
                  make_desc_k128(b0 + kr * C * 128 + k * 32), idesc, (kr | k) ? 1u : 0u);
    umma_commit(bar);
  }
  if (active) {
    mbar_wait(bar, 0);
    tc_fence_after();
    // ---------------- 4. epilogue: TMEM -> smem staging -> coalesced y ----------------
    float* stg = y1s;  // y1 is dead now
    const int quarter = warp & 3, part = warp >> 2;  // 32 columns per part
    const int row = quarter * 32 + lane;
    if (part * 32 < C) {  // warp-uniform: C / 32 parts x 4 lane quarters
      const int col = part * 32;
      uint32_t r[32];
      tmem_ld_32x32b_x32(tmem + (static_cast<uint32_t>(quarter * 32) << 16) + col, r);
      tmem_ld_wait();
#pragma unroll
      for (int j = 0; j < 32; ++j) stg[row * (C + 1) + col + j] = __uint_as_float(r[j]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (active) {
    const float* stg = y1s;
    const int ch = tid % C;
    const float pb = pw_b[ch];
#pragma unroll
    for (int k = 0; k < kResRows; ++k) {
      const int i = tid / C + k * kRowStep;
      y[static_cast<int64_t>(r0 + i) * C + ch] = (stg[i * (C + 1) + ch] + pb) + xres[k];
    }
  }
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, C);
  }
}

template <int C>
static void ru_fused_launch(const DetokReq* reqs, int rows, int up, const float* x, float* y,
                            int dil, const float* a1, const float* dw_w, const float* dw_b,
                            const float* a2, const bf16* pw_w, const float* pw_b, float* state,
                            int64_t st_off, const DetokDims& dd, cudaStream_t st) {
  const ReqHdrF* hdr = reinterpret_cast<const ReqHdrF*>(reqs) - 1;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(ru_fused_kernel<C>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         RuSmem<C>::kBytes);
    attr = true;
  }
  launch_k(ru_fused_kernel<C>, dim3((rows + kRuRows - 1) / kRuRows), dim3(ru_threads<C>()),
           RuSmem<C>::kBytes, st, hdr, reqs, up, x, y, dil, a1, dw_w, dw_b, a2, pw_w, pw_b, state,
           st_off, dd);
}

bool ru_fused_supported(int C, int up) { return (C == 64 || C == 128) && (4 * up) % kRuRows == 0; }

void launch_ru_fused(const DetokReq* reqs, int rows, int up, const float* x, float* y, int C,
                     int dil, const float* alpha1, const float* dw_w, const float* dw_b,
                     const float* alpha2, const bf16* pw_w, const float* pw_b, float* state,
                     int64_t st_off, const DetokDims& dd, cudaStream_t st) {
  if (C == 64)
    ru_fused_launch<64>(reqs, rows, up, x, y, dil, alpha1, dw_w, dw_b, alpha2, pw_w, pw_b, state,
                        st_off, dd, st);
  else
    ru_fused_launch<128>(reqs, rows, up, x, y, dil, alpha1, dw_w, dw_b, alpha2, pw_w, pw_b, state,
                         st_off, dd, st);
}

// ---------------------------------------------------------------------------
// Output head, tiled: Snake once per element into shared memory (tile + 6-row
// causal halo from the cached context), then one thread per output sample:
// pcm[t] = tanh(b + sum_{c,k} w[c][k] * s[t-6+k][c]).
// ---------------------------------------------------------------------------
constexpr int kOutRows = 128;

template <int C>
struct OutSmem {
  static constexpr int kS = (kOutRows + 6) * (C + 1);  // Snake'd rows, padded (conflict-free taps)
  static constexpr int kW = C * 7;
  static constexpr int kX = (kOutRows + 6) * C;        // raw x rows (bulk copy target)
  static constexpr int kXOff = (kS + kW + 3) / 4 * 4;  // 16-byte aligned
  static constexpr int kBytes = (kXOff + kX) * 4 + 16;
};

template <int C>
__global__ void __launch_bounds__(kOutRows)
    detok_out_tiled_kernel(const ReqHdrF* hdr, const DetokReq* __restrict__ reqs, int up,
                           const float* __restrict__ x, const float* __restrict__ alpha,
                           const float* __restrict__ w, float b, float* __restrict__ state,
                           int64_t st_off, DetokDims dd, float* __restrict__ pcm) {
  VOX_TRACE(kTrDetok);
  using L = OutSmem<C>;
  extern __shared__ __align__(16) float osm[];
  float* s = osm;
  float* ws = osm + L::kS;
  float* xs = osm + L::kXOff;
  uint64_t* bar = reinterpret_cast<uint64_t*>(xs + L::kX);
  const int tid = threadIdx.x;
  for (int e = tid; e < C * 7; e += kOutRows) ws[e] = w[e];
  if (tid == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  __syncthreads();
  griddep_wait();
  griddep_launch();
  const int r0 = blockIdx.x * kOutRows;
  if (r0 >= hdr->n_lat * up) return;
  const DetokReq q = reqs[find_req_w(reqs, hdr->n_req, r0 / up)];
  const int t0 = r0 - q.lat_off * up;
  const int n = 4 * q.nf * up;
  constexpr int H = 6;
  const float* hin = slot_state_f(state, dd, q.slot, q.parity) + st_off;
  float* hout = slot_state_f(state, dd, q.slot, q.parity ^ 1) + st_off;
  // the tile's x rows (+ halo rows inside the request) in one bulk copy; halo
  // rows before the request start come from the cached (Snake'd) context
  const int i_first = t0 >= H ? 0 : H - t0;
  if (tid == 0) {
    const uint32_t bx = static_cast<uint32_t>((kOutRows + H - i_first) * C * 4);
    mbar_arrive_expect_tx(bar, bx);
    bulk_load(xs + i_first * C, x + static_cast<int64_t>(r0 - H + i_first) * C, bx, bar, policy_evict_first());
  }
  const int chx = tid % C;
  const float ax = alpha[chx], ix = snake_inv(ax);
  for (int e = tid; e < i_first * C; e += kOutRows) {
    const int i = e / C;
    s[i * (C + 1) + chx] = hin[(t0 + i) * C + chx];
  }
  mbar_wait(bar, 0);
#pragma unroll 4
  for (int e = i_first * C + tid; e < (kOutRows + H) * C; e += kOutRows) {
    const int i = e / C;  // kOutRows % C == 0: fixed channel per thread
    const int t = t0 - H + i;
    const float v = snake_r(xs[e], ax, ix);
    if (i >= H && t >= n - H) hout[(t - (n - H)) * C + chx] = v;
    s[i * (C + 1) + chx] = v;
  }
  for (int e = tid; e < kOutRows * C; e += kOutRows) {
    const int i = e / C, ch = e % C, t = t0 + i;
    for (int hh = t; hh < H - n; hh += n) hout[hh * C + ch] = hin[(hh + n) * C + ch];
  }
  __syncthreads();
  const int t = t0 + tid;
  // 4 interleaved partial sums (channel c -> c % 4): short FMA chains, few registers
  float part[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll 8
  for (int ch = 0; ch < C; ++ch) {
    float a = part[ch & 3];
#pragma unroll
    for (int k = 0; k < 7; ++k) a = fmaf(ws[ch * 7 + k], s[(tid + k) * (C + 1) + ch], a);
    part[ch & 3] = a;
  }
  const float acc = (part[0] + part[1]) + (part[2] + part[3]);
  if (t < q.n_samples && t < n) pcm[q.pcm_off + t] = tanhf(acc + b);
}

void launch_detok_out_tiled(const DetokReq* reqs, int rows, int up, const float* x, int C,
                            const float* alpha, const float* w, float b, float* state,
                            int64_t st_off, const DetokDims& dd, float* pcm, cudaStream_t st) {
  const ReqHdrF* hdr = reinterpret_cast<const ReqHdrF*>(reqs) - 1;
  if (C == 64) {
    static bool attr = false;
    if (!attr) {
      cudaFuncSetAttribute(detok_out_tiled_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           OutSmem<64>::kBytes);
      attr = true;
    }
    launch_k(detok_out_tiled_kernel<64>, dim3((rows + kOutRows - 1) / kOutRows), dim3(kOutRows),
             OutSmem<64>::kBytes, st, hdr, reqs, up, x, alpha, w, b, state, st_off, dd, pcm);
  }
}

bool detok_out_tiled_supported(int C, int up) { return C == 64 && (4 * up) % kOutRows == 0; }

// ---------------------------------------------------------------------------
// Snake + transposed-conv operand [s(x_t) | s(x_{t-1})] (bf16), tiled: a CTA
// walks R consecutive rows of one request, each thread owning channels, so
// Snake is evaluated once per element (s(x_{t-1}) is carried in a register)
// and every access is coalesced along channels.  History = 1 row of s(x).
// ---------------------------------------------------------------------------
template <int CPT>  // channels per thread
__global__ void __launch_bounds__(256)
    snake_upcat_tiled_kernel(const ReqHdrF* hdr, const DetokReq* __restrict__ reqs, int up, int R,
                             const float* __restrict__ x, int C, const float* __restrict__ alpha,
                             float* __restrict__ state, int64_t st_off, DetokDims dd,
                             bf16* __restrict__ out) {
  VOX_TRACE(kTrDetok);
  const int tid = threadIdx.x;
  float a[CPT], inv[CPT];
#pragma unroll
  for (int k = 0; k < CPT; ++k) {
    const int ch = tid + k * blockDim.x;
    a[k] = ch < C ? alpha[ch] : 1.f;
    inv[k] = snake_inv(a[k]);
  }
  griddep_wait();
  griddep_launch();
  const int r0 = blockIdx.x * R;
  if (r0 >= hdr->n_lat * up) return;
  const DetokReq q = reqs[find_req_w(reqs, hdr->n_req, r0 / up)];
  const int t0 = r0 - q.lat_off * up;
  const int n = 4 * q.nf * up;
  const float* hin = slot_state_f(state, dd, q.slot, q.parity) + st_off;
  float* hout = slot_state_f(state, dd, q.slot, q.parity ^ 1) + st_off;
  float prev[CPT];
#pragma unroll
  for (int k = 0; k < CPT; ++k) {
    const int ch = tid + k * blockDim.x;
    if (ch < C)
      prev[k] = t0 > 0 ? snake_r(x[static_cast<int64_t>(r0 - 1) * C + ch], a[k], inv[k]) : hin[ch];
  }
  constexpr int kMaxR = 16;
#pragma unroll
  for (int i0 = 0; i0 < kMaxR; i0 += 8) {
    if (i0 >= R) break;
    float xv[8][CPT];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int k = 0; k < CPT; ++k) {
        const int ch = tid + k * blockDim.x;
        xv[i][k] = (i0 + i < R && ch < C) ? x[static_cast<int64_t>(r0 + i0 + i) * C + ch] : 0.f;
      }
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      if (i0 + i >= R) break;
      const int r = r0 + i0 + i;
      bf16* o = out + static_cast<int64_t>(r) * 2 * C;
#pragma unroll
      for (int k = 0; k < CPT; ++k) {
        const int ch = tid + k * blockDim.x;
        if (ch < C) {
          const float cur = snake_r(xv[i][k], a[k], inv[k]);
          o[ch] = __float2bfloat16_rn(cur);
          o[C + ch] = __float2bfloat16_rn(prev[k]);
          if (t0 + i0 + i == n - 1) hout[ch] = cur;
          prev[k] = cur;
        }
      }
    }
  }
}

bool snake_upcat_tiled_supported(int up_before) { return up_before >= 1; }

// ---------------------------------------------------------------------------
// Residual-unit prologue for the wide levels (C >= 256), tiled: a CTA owns TR
// rows x 64 channels of one request; y1 = Snake(x) for the rows plus the
// 6*dil causal halo is computed once into shared memory (ru_prep_kernel
// recomputes it for each of the 7 taps), then v = bf16(Snake(dwconv(y1))) is
// written for the 1x1 GEMM.  Cached left context as in ru_prep_kernel.
// ---------------------------------------------------------------------------
constexpr int kPrepCh = 64;

__global__ void __launch_bounds__(256)
    ru_prep_tiled_kernel(const ReqHdrF* hdr, const DetokReq* __restrict__ reqs, int up, int TR,
                         const float* __restrict__ x, int C, int dil,
                         const float* __restrict__ alpha1, const float* __restrict__ dw_w,
                         const float* __restrict__ dw_b, const float* __restrict__ alpha2,
                         float* __restrict__ state, int64_t st_off, DetokDims dd,
                         bf16* __restrict__ out) {
  VOX_TRACE(kTrDetok);
  extern __shared__ float y1s[];  // [TR + 6 dil][kPrepCh]
  const int tid = threadIdx.x;
  const int cl = tid % kPrepCh;                 // channel within the tile
  const int ch = blockIdx.y * kPrepCh + cl;     // channel
  const int rstep = 256 / kPrepCh;              // rows per pass
  const float a1 = alpha1[ch], i1 = snake_inv(a1);
  const float a2 = alpha2[ch], i2 = snake_inv(a2);
  float w[7];
#pragma unroll
  for (int k = 0; k < 7; ++k) w[k] = dw_w[ch * 7 + k];
  const float bias = dw_b[ch];
  griddep_wait();
  griddep_launch();
  const int r0 = blockIdx.x * TR;
  if (r0 >= hdr->n_lat * up) return;
  const DetokReq q = reqs[find_req_w(reqs, hdr->n_req, r0 / up)];
  const int t0 = r0 - q.lat_off * up;
  const int n = 4 * q.nf * up;
  const int H = 6 * dil;
  const float* hin = slot_state_f(state, dd, q.slot, q.parity) + st_off;
  float* hout = slot_state_f(state, dd, q.slot, q.parity ^ 1) + st_off;
  const int nr = TR + H;
  for (int i0 = tid / kPrepCh; i0 < nr; i0 += 8 * rstep) {
    float xv[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int i = i0 + u * rstep, t = t0 - H + i;
      xv[u] = 0.f;
      if (i < nr) xv[u] = t >= 0 ? x[static_cast<int64_t>(r0 - H + i) * C + ch] : hin[(H + t) * C + ch];
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int i = i0 + u * rstep, t = t0 - H + i;
      if (i < nr) {
        const float v = t >= 0 ? snake_r(xv[u], a1, i1) : xv[u];
        if (t >= 0 && i >= H && t >= n - H) hout[(t - (n - H)) * C + ch] = v;
        y1s[i * kPrepCh + cl] = v;
      }
    }
  }
  for (int i = tid / kPrepCh; i < TR; i += rstep) {  // short requests (n < H)
    const int t = t0 + i;
    for (int hh = t; hh < H - n; hh += n) hout[hh * C + ch] = hin[(hh + n) * C + ch];
  }
  __syncthreads();
#pragma unroll 4
  for (int i = tid / kPrepCh; i < TR; i += rstep) {
    float acc = bias;
#pragma unroll
    for (int k = 0; k < 7; ++k) acc = fmaf(w[k], y1s[(H + i - (6 - k) * dil) * kPrepCh + cl], acc);
    out[static_cast<int64_t>(r0 + i) * C + ch] = __float2bfloat16_rn(snake_r(acc, a2, i2));
  }
}

bool ru_prep_tiled_supported(int C, int up) { return C % kPrepCh == 0 && C >= 256 && 4 * up >= 16; }

void launch_ru_prep_tiled(const DetokReq* reqs, int rows, int up, const float* x, int C, int dil,
                          const float* alpha1, const float* dw_w, const float* dw_b,
                          const float* alpha2, float* state, int64_t st_off, const DetokDims& dd,
                          bf16* out, cudaStream_t st) {
  const ReqHdrF* hdr = reinterpret_cast<const ReqHdrF*>(reqs) - 1;
  const int TR = 4 * up < 64 ? 4 * up : 64;  // a request spans 4 * nf * up rows
  const size_t smem = static_cast<size_t>(TR + 6 * dil) * kPrepCh * 4;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(ru_prep_tiled_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    attr = true;
  }
  launch_k(ru_prep_tiled_kernel, dim3((rows + TR - 1) / TR, C / kPrepCh), dim3(256), smem, st, hdr,
           reqs, up, TR, x, C, dil, alpha1, dw_w, dw_b, alpha2, state, st_off, dd, out);
}

void launch_snake_upcat_tiled(const DetokReq* reqs, int rows, int up_before, const float* x, int C,
                              const float* alpha, float* state, int64_t st_off, const DetokDims& dd,
                              bf16* out_cat, cudaStream_t st) {
  const ReqHdrF* hdr = reinterpret_cast<const ReqHdrF*>(reqs) - 1;
  // rows per CTA: a request spans 4 * nf * up_before rows at this level
  const int R = (4 * up_before) < 16 ? 4 * up_before : 16;
  const int threads = C < 256 ? C : 256;
  const int cpt = (C + threads - 1) / threads;
  const dim3 grid((rows + R - 1) / R);
  if (cpt <= 1)
    launch_k(snake_upcat_tiled_kernel<1>, grid, dim3(threads), 0, st, hdr, reqs, up_before, R, x, C,
             alpha, state, st_off, dd, out_cat);
  else if (cpt <= 2)
    launch_k(snake_upcat_tiled_kernel<2>, grid, dim3(threads), 0, st, hdr, reqs, up_before, R, x, C,
             alpha, state, st_off, dd, out_cat);
  else
    launch_k(snake_upcat_tiled_kernel<4>, grid, dim3(threads), 0, st, hdr, reqs, up_before, R, x, C,
             alpha, state, st_off, dd, out_cat);
}

}  // namespace vox
