// gemm_tc.cu — tcgen05/TMEM/TMA bf16 GEMM for sm_100a.
//
//   out[n, m] = sum_k W[m, k] * X[n, k]   (+ bias[m]) (+ resid[n, m])
//
// W is a weight matrix [M, K] (nn.Linear layout, K-major), X the activation
// rows [N, K] (K-major).  "Swap-AB" orientation for decode: the weights fill
// the 128-row UMMA M dimension and the (small) batch of rows is UMMA N, so a
// decode step with B = 1..256 rows is a single UMMA N tile.  Split-K over
// blockIdx.z writes fp32 partials that the following fused elementwise
// kernel reduces (deterministic, no atomics).
//
// Warp roles (128 threads): warp0/lane0 = TMA producer, warp1/lane0 = MMA
// issuer (tcgen05.mma, accumulator in TMEM), warp2 = TMEM allocator; all four
// warps run the epilogue (tcgen05.ld 32x32b -> registers -> coalesced stores).
#include "common.cuh"
#include "kernels.h"
#include <cstdlib>

namespace vox {
VOX_TRACE_TU(trace_set_gemm)


template <int BN, int MT>
struct GemmCfg {
  // MT = 128-row weight sub-tiles per CTA (1 or 2).  MT = 2 computes a 256 x BN
  // output tile as two M=128 UMMAs that share one activation (B) stage: the
  // activation slab is re-read from L2 half as often (it is re-read once per
  // weight tile), which is what bounds the swap-AB decode GEMM at large batch.
  static constexpr int kABytes = MT * 128 * 64 * 2;
  static constexpr int kBBytes = BN * 64 * 2;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kBudget = MT == 2 ? 192 * 1024 : 96 * 1024;
  static constexpr int kStages0 = kBudget / kStageBytes > 8 ? 8 : kBudget / kStageBytes;
  static constexpr int kStages = (MT == 1 && BN >= 256) ? 4 : kStages0;
  static constexpr int kTmemCols0 = MT * BN < 32 ? 32 : MT * BN;
  // power of two >= 32 (tcgen05.alloc granularity)
  static constexpr int kTmemCols = kTmemCols0 <= 32 ? 32 : kTmemCols0 <= 64 ? 64 : kTmemCols0 <= 128 ? 128 : kTmemCols0 <= 256 ? 256 : 512;
  static constexpr int kSmemBytes = kStages * kStageBytes + 1024 + 256;
};

// ---------------------------------------------------------------------------
// Epilogue shared by the GEMM kernels: TMEM accumulator (128 lanes = weight
// rows m, BN columns = activation rows n) -> registers -> smem (transposed)
// -> 16-byte coalesced global stores.  `smem` is the idle pipeline ring.
// ---------------------------------------------------------------------------
VOX_DEV float gelu_erf(float v) { return 0.5f * v * (1.f + erff(v * 0.70710678118654752f)); }
VOX_DEV void store_gelu4(bf16* dst, float4 v) {
  const __nv_bfloat162 lo = __floats2bfloat162_rn(gelu_erf(v.x), gelu_erf(v.y));
  const __nv_bfloat162 hi = __floats2bfloat162_rn(gelu_erf(v.z), gelu_erf(v.w));
  uint2 u;
  u.x = *reinterpret_cast<const uint32_t*>(&lo);
  u.y = *reinterpret_cast<const uint32_t*>(&hi);
  *reinterpret_cast<uint2*>(dst) = u;
}

template <int BN, int MT>
__device__ __forceinline__ void gemm_epilogue(const GemmArgs& p, uint8_t* smem, uint32_t tmem,
                                              int warp, int lane, int m0, int n0, int split,
                                              uint64_t* done_bar) {
  if (MT == 1 && p.epi == 1) {
    if (done_bar != nullptr) {
      mbar_wait(done_bar, 0);
      tc_fence_after();
    }
    // fused SiLU(gate) * up: TMEM lanes 0-63 hold gate, 64-127 up of features
    // f = 64 * tile + (lane % 64).  32 accumulator columns (rows n) at a time are
    // staged transposed in the idle pipeline smem, then each thread turns 8
    // features of one row into 8 bf16 and writes them with one 16-byte store.
    float* stg = reinterpret_cast<float*>(smem);  // [32][128 + 4]
    constexpr int kSt = 128 + 4;
    const int f0 = (m0 / 128) * 64;
#pragma unroll 1
    for (int c = 0; c < BN; c += 32) {
      uint32_t r[32];
      tmem_ld_32x32b_x32(tmem + (static_cast<uint32_t>(warp * 32) << 16) + c, r);
      tmem_ld_wait();
      const int ml = warp * 32 + lane;
#pragma unroll
      for (int j = 0; j < 32; ++j) stg[j * kSt + ml] = __uint_as_float(r[j]);
      __syncthreads();
#pragma unroll 2
      for (int e = threadIdx.x; e < 32 * 8; e += 128) {
        const int j = e >> 3, q = (e & 7) * 8;
        const int n = n0 + c + j;
        if ((c + j) < BN && n < p.N) {
          uint32_t pk[4];
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            float o[2];
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              const float g = stg[j * kSt + q + 2 * t + h];
              const float u = stg[j * kSt + 64 + q + 2 * t + h];
              o[h] = __fmul_rn(__fdiv_rn(g, __fadd_rn(1.0f, expf(-g))), u);
            }
            const __nv_bfloat162 b2 = __floats2bfloat162_rn(o[0], o[1]);
            pk[t] = *reinterpret_cast<const uint32_t*>(&b2);
          }
          *reinterpret_cast<uint4*>(p.act + static_cast<int64_t>(n) * p.ld_act + f0 + q) =
              make_uint4(pk[0], pk[1], pk[2], pk[3]);
        }
      }
      __syncthreads();
    }
    return;
  }
  if (MT == 1 && p.epi == 2) {
    // act = bf16(GELU(acc + bias)) (the codec FFN's fc1; codec_gelu_kernel's
    // arithmetic), staged like the fp32 epilogue below; kept out of that loop so
    // the erf sequence does not bloat every GEMM's unrolled store loop
    if (done_bar != nullptr) {
      mbar_wait(done_bar, 0);
      tc_fence_after();
    }
    float* stg = reinterpret_cast<float*>(smem);
    constexpr int kSt = 128 + 4;
#pragma unroll 1
    for (int c = 0; c < BN; c += 32) {
      uint32_t r[32];
      tmem_ld_32x32b_x32(tmem + (static_cast<uint32_t>(warp * 32) << 16) + c, r);
      tmem_ld_wait();
#pragma unroll
      for (int j = 0; j < 32; ++j) stg[j * kSt + warp * 32 + lane] = __uint_as_float(r[j]);
      __syncthreads();
#pragma unroll 1
      for (int e = threadIdx.x; e < 32 * 32; e += 128) {
        const int j = e >> 5, q = (e & 31) * 4;
        const int n = n0 + c + j, m = m0 + q;
        if ((c + j) < BN && n < p.N && m + 3 < p.m_valid) {
          float4 v = *reinterpret_cast<const float4*>(&stg[j * kSt + q]);
          if (p.bias != nullptr) {
            const float4 b4 = *reinterpret_cast<const float4*>(p.bias + m);
            v.x += b4.x; v.y += b4.y; v.z += b4.z; v.w += b4.w;
          }
          store_gelu4(p.act + static_cast<int64_t>(n) * p.ld_act + m, v);
        }
      }
      __syncthreads();
    }
    return;
  }
  float* outp = p.out + static_cast<int64_t>(split) * p.split_stride;
  // Staged epilogue: 32 accumulator columns (= 32 output rows n) at a time go
  // TMEM -> registers -> shared memory (transposed to [n][m]) -> 16-byte
  // coalesced stores along m.  (Thread-per-m scalar stores issue 4x the store
  // instructions and serialise on the per-SM store path.)  The bias / residual
  // operands of a chunk are loaded before its TMEM read and barrier (all 8 per
  // thread in flight; chunk 0's before the accumulator is complete), so the
  // residual read is not a dependent round trip per store.
  float* stg = reinterpret_cast<float*>(smem);  // [32][128 + 4], pipeline smem is idle now
  constexpr int kSt = 128 + 4;
  float4 rr[8];
  auto prefetch = [&](int mb, int c, bool full_m) {
    if (!full_m || (p.resid == nullptr && p.bias == nullptr)) return;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int e = threadIdx.x + i * 128;
      const int j = e >> 5, q = (e & 31) * 4;
      const int n = n0 + c + j;
      float4 a = make_float4(0.f, 0.f, 0.f, 0.f);
      if ((c + j) < BN && n < p.N && p.resid != nullptr && mb + q < p.m_valid)
        a = *reinterpret_cast<const float4*>(p.resid + static_cast<int64_t>(n) * p.ldr + mb + q);
      rr[i] = a;
    }
  };
  // float4 path whenever every 4-column group is wholly valid or wholly past
  // m_valid (M % 4 == 0: e.g. the 32/64-channel codec convs that fill only part
  // of the 128-row weight tile) and the rows are 16-byte aligned
  auto is_full = [&](int mb) {
    (void)mb;
    return (p.m_valid & 3) == 0 && (p.ldo & 3) == 0 && (p.resid == nullptr || (p.ldr & 3) == 0) &&
           (reinterpret_cast<uintptr_t>(outp) & 15) == 0;
  };
  prefetch(m0, 0, is_full(m0));
  if (done_bar != nullptr) {
    mbar_wait(done_bar, 0);
    tc_fence_after();
  }
#pragma unroll 1
  for (int mt = 0; mt < MT; ++mt) {
    const int mb = m0 + mt * 128;
    const bool full_m = is_full(mb);
#pragma unroll 1
    for (int c = 0; c < BN; c += 32) {
      if (c > 0 || mt > 0) prefetch(mb, c, full_m);
      uint32_t r[32];
      tmem_ld_32x32b_x32(tmem + (static_cast<uint32_t>(warp * 32) << 16) + mt * BN + c, r);
      tmem_ld_wait();
      const int ml = warp * 32 + lane;
#pragma unroll
      for (int j = 0; j < 32; ++j) stg[j * kSt + ml] = __uint_as_float(r[j]);
      __syncthreads();
      // 32 rows n x 128 m: 1024 float4, 8 per thread
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const int e = threadIdx.x + i * 128;
        const int j = e >> 5, q = (e & 31) * 4;
        const int n = n0 + c + j;
        if ((c + j) < BN && n < p.N) {
          float4 v = *reinterpret_cast<const float4*>(&stg[j * kSt + q]);
          const int m = mb + q;
          if (full_m) {
            if (m >= p.m_valid) continue;
            if (p.bias != nullptr) {
              const float4 b4 = *reinterpret_cast<const float4*>(p.bias + m);
              v.x += b4.x; v.y += b4.y; v.z += b4.z; v.w += b4.w;
            }
            if (p.resid != nullptr) {
              const float4 r4 = rr[i];
              v.x += r4.x; v.y += r4.y; v.z += r4.z; v.w += r4.w;
            }
            *reinterpret_cast<float4*>(outp + static_cast<int64_t>(n) * p.ldo + m) = v;
          } else {
            const float vv[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int t = 0; t < 4; ++t) {
              if (m + t < p.m_valid) {
                float o = vv[t];
                if (p.bias != nullptr) o += p.bias[m + t];
                if (p.resid != nullptr) o += p.resid[static_cast<int64_t>(n) * p.ldr + m + t];
                outp[static_cast<int64_t>(n) * p.ldo + m + t] = o;
              }
            }
          }
        }
      }
      __syncthreads();
    }
  }
}

template <int BN, int MT>
__global__ void __launch_bounds__(128, 1)
    gemm_bf16_tc_kernel(const __grid_constant__ CUtensorMap tmW,
                        const __grid_constant__ CUtensorMap tmX, GemmArgs p) {
  VOX_TRACE(kTrGemm);
  using C = GemmCfg<BN, MT>;
  extern __shared__ uint8_t smem_raw[];
  // align to 1024 B by pointer arithmetic on the __shared__ array (an
  // integer round-trip would turn every smem access into a generic LD/ST)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::kStages * C::kStageBytes);
  uint64_t* empty = full + C::kStages;
  uint64_t* done = empty + C::kStages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  // n-tiles vary fastest so the CTAs that share a weight tile run in the same
  // wave: each weight byte comes from HBM once (then L2) per split.
  const int m0 = blockIdx.y * (128 * MT);
  const int n0 = blockIdx.x * BN;
  const int split = blockIdx.z;
  const int kb0 = split * p.kb_per_split;
  const int kb1 = min(p.n_kb, kb0 + p.kb_per_split);
  const int nkb = kb1 - kb0;  // host guarantees >= 1
  // k-block visiting order rotated per weight tile: the CTAs of one launch
  // then read different activation k-blocks at any instant instead of all
  // hammering the same L2 lines (each activation line is read by every CTA)
  const int krot = p.k_rotate ? static_cast<int>((blockIdx.y * 7u) % static_cast<unsigned>(nkb)) : 0;
  auto kbi = [&](int i) { const int t = i + krot; return kb0 + (t >= nkb ? t - nkb : t); };
  // activations in the packed tile layout: the BN rows of one k-block are
  // contiguous (BN * 128 B) inside a 128-row tile, so one bulk copy per 128 rows
  auto load_x_packed = [&](uint8_t* dst, int kb, uint64_t* bar, uint64_t pol) {
#pragma unroll
    for (int h = 0; h < (BN + 127) / 128; ++h) {
      const int nr = n0 + h * 128;
      const int rows = BN < 128 ? BN : 128;
      bulk_load(dst + h * 16384,
                p.x_packed + (static_cast<int64_t>(nr / 128) * p.n_kb + kb) * 8192 + (nr % 128) * 64,
                rows * 128, bar, pol);
    }
  };

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmW);
    tma_prefetch_desc(&tmX);
    for (int s = 0; s < C::kStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(done, 1);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, C::kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  // Dependents launch only after this grid passed its own griddep_wait (the
  // producer's, below): every kernel of the step follows wait-then-launch, so a
  // kernel may read data written two or more launches upstream BEFORE its own
  // griddep_wait (resid_norm prefetches h that way).
  if (warp == 0 && lane == 0) {
    // ---------------- TMA producer ----------------
    const uint64_t pol_w = policy_evict_first();  // weights: streamed once per step
    const uint64_t pol_x = policy_evict_last();   // activations: re-read by every CTA
    // Weights do not depend on the preceding kernel: fill the first stages'
    // weight tiles BEFORE the grid-dependency wait (overlaps the previous
    // kernel's tail), then load the activation tiles.
    const int pre = nkb < C::kStages ? nkb : C::kStages;
    for (int i = 0; i < pre; ++i) {
      mbar_arrive_expect_tx(&full[i], C::kStageBytes);
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        if (p.w_packed != nullptr)
          bulk_load(smem + i * C::kStageBytes + mt * 16384,
                    p.w_packed + (static_cast<int64_t>(m0 / 128 + mt) * p.n_kb + kbi(i)) * 8192,
                    16384, &full[i], pol_w);
        else
          tma_load_2d(smem + i * C::kStageBytes + mt * 16384, &tmW, &full[i], kbi(i) * 64,
                      m0 + mt * 128, pol_w);
      }
    }
    griddep_wait();
    griddep_launch();
    for (int i = 0; i < pre; ++i)
      if (p.x_packed != nullptr)
        load_x_packed(smem + i * C::kStageBytes + C::kABytes, kbi(i), &full[i], pol_x);
      else
        tma_load_2d(smem + i * C::kStageBytes + C::kABytes, &tmX, &full[i], kbi(i) * 64, n0,
                  pol_x);
    for (int i = pre; i < nkb; ++i) {
      const int s = i % C::kStages;
      mbar_wait(&empty[s], ((i / C::kStages) - 1) & 1);
      uint8_t* st = smem + s * C::kStageBytes;
      mbar_arrive_expect_tx(&full[s], C::kStageBytes);
      const int kx = kbi(i) * 64;
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) {
        if (p.w_packed != nullptr)
          bulk_load(st + mt * 16384,
                    p.w_packed + (static_cast<int64_t>(m0 / 128 + mt) * p.n_kb + kbi(i)) * 8192,
                    16384, &full[s], pol_w);
        else
          tma_load_2d(st + mt * 16384, &tmW, &full[s], kx, m0 + mt * 128, pol_w);
      }
      if (p.x_packed != nullptr)
        load_x_packed(st + C::kABytes, kbi(i), &full[s], pol_x);
      else
        tma_load_2d(st + C::kABytes, &tmX, &full[s], kx, n0, pol_x);
    }
  } else if (warp == 1 && lane == 0) {
    // ---------------- MMA issuer (single thread) ----------------
    constexpr uint32_t idesc = make_idesc_bf16(128, BN);
    for (int i = 0; i < nkb; ++i) {
      const int s = i % C::kStages;
      mbar_wait(&full[s], (i / C::kStages) & 1);
      tc_fence_after();
      const uint32_t a_addr = smem_u32(smem + s * C::kStageBytes);
      const uint32_t b_addr = a_addr + C::kABytes;
#pragma unroll
      for (int k = 0; k < 4; ++k) {  // 4 x UMMA_K(16) per 64-wide k-block
#pragma unroll
        for (int mt = 0; mt < MT; ++mt)  // accumulator mt lives at TMEM columns [mt*BN, mt*BN+BN)
          umma_bf16(tmem + mt * BN, make_desc_k128(a_addr + mt * 16384 + k * 32),
                    make_desc_k128(b_addr + k * 32), idesc, (i > 0 || k > 0) ? 1u : 0u);
      }
      umma_commit(&empty[s]);  // frees the smem stage once these MMAs retire
    }
    umma_commit(done);  // accumulator complete
  }
  __syncwarp();

  // ---------------- epilogue: TMEM -> registers -> global ----------------
  griddep_wait();  // outputs may alias buffers the preceding kernel was reading
  griddep_launch();
  gemm_epilogue<BN, MT>(p, smem, tmem, warp, lane, m0, n0, split, done);  // waits for `done`

  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, C::kTmemCols);
  }
}

// ---------------------------------------------------------------------------
// Decode-step GEMM ("mc" kernel: one n-tile covering every row of the step).
//
// One CTA covers ALL activation rows of the step (BN = the row bucket, a single
// n-tile), so every weight byte is read from HBM exactly once; the 1-CTA kernel
// above tiles the rows (BN <= 128) and re-reads each weight tile per n-tile.
// One CTA per SM with a deep ring (~200 KB): measured per-CTA phase stamps
// (VOX_GEMM_DBG, profiles/gemm_mc_phases_r01.txt) show the k-loop streaming
// weights at ~6.2 TB/s aggregate; what remains is the first-load latency and
// the epilogue.  (Round 1 also measured, and dropped, cluster multicast of the
// activation k-blocks, split-K reduced through DSMEM, a fused RMSNorm prologue
// and L2 prefetch of later weight k-blocks: all slower on the serving step,
// profiles/gemm_mc_sweep_r01.txt, gemm_mc_ab_r01.txt, gemm_l2_prefetch_ab_r01.txt.)
// ---------------------------------------------------------------------------
// Direct epilogue of the decode kernel (8 warps).  TMEM lane = weight row
// m, so for one accumulator column (activation row n) the 32 lanes of a warp
// hold 32 consecutive m: each column is one fully coalesced 128-byte warp
// store straight from registers -- no smem staging, no block barriers.  Warps
// w and w + 4 read the same TMEM lane quarter (w % 4) and split the 32-column
// chunks between them.  The loop body is kept to a compare, a store and a
// pointer bump: with one or two warps per SMSP the epilogue is bound by the
// issue latency of its instruction chain (ncu: the first version spent ~37
// instructions per store on 64-bit index math and per-element guards and took
// longer than the whole k-loop).
// epi == 1 (fused SiLU(gate) * up, gate|up rows interleaved per tile): gate
// (lanes 0-63) and up (lanes 64-127) are parked in smem [n][64] fp32, then
// each warp forms bf16(SiLU(g) * u) for whole rows: 32 threads x 2 features
// = one 128-byte store per row.
template <int BN>
__device__ __forceinline__ void mc_epilogue(const GemmArgs& p, uint8_t* smem, uint32_t tmem,
                                            int warp, int lane, int m0, int n0, int split) {
  constexpr int kChunks = (BN + 31) / 32;
  const int q = warp & 3, h = warp >> 2;
  const uint32_t tbase = tmem + (static_cast<uint32_t>(q * 32) << 16);
  const int nv = min(BN, p.N - n0);  // valid columns of this tile
  if (p.epi == 1) {
    // [kChunks*32][64] gate, then the same for up: whole 32-column chunks are
    // parked (BN = 16 still loads 32 TMEM columns)
    constexpr int kRowsP = kChunks * 32;
    float* sg = reinterpret_cast<float*>(smem);
    float* dst = sg + (q >= 2 ? kRowsP * 64 : 0) + (q & 1) * 32 + lane;
#pragma unroll 1
    for (int ch = h; ch < kChunks; ch += 2) {
      uint32_t r[32];
      tmem_ld_32x32b_x32(tbase + ch * 32, r);
      tmem_ld_wait();
      float* d = dst + ch * 32 * 64;
#pragma unroll
      for (int j = 0; j < 32; ++j) d[j * 64] = __uint_as_float(r[j]);
    }
    __syncthreads();
    const float* su = sg + kRowsP * 64;
    const int fp = lane * 2;
    __nv_bfloat162* out = reinterpret_cast<__nv_bfloat162*>(p.act + static_cast<int64_t>(n0) * p.ld_act +
                                                            (m0 / 128) * 64 + fp);
    const int64_t step = p.ld_act / 2;  // in bf16x2 units
#pragma unroll 4
    for (int j = warp; j < nv; j += 8) {
      const float2 g = *reinterpret_cast<const float2*>(&sg[j * 64 + fp]);
      const float2 u = *reinterpret_cast<const float2*>(&su[j * 64 + fp]);
      const float o0 = __fmul_rn(__fdiv_rn(g.x, __fadd_rn(1.0f, expf(-g.x))), u.x);
      const float o1 = __fmul_rn(__fdiv_rn(g.y, __fadd_rn(1.0f, expf(-g.y))), u.y);
      out[j * step] = __floats2bfloat162_rn(o0, o1);
    }
    return;
  }
  const int m = m0 + q * 32 + lane;
  const bool mok = m < p.m_valid;
  float* o = p.out + static_cast<int64_t>(split) * p.split_stride + static_cast<int64_t>(n0) * p.ldo + m;
  const int64_t ldo = p.ldo;
  if (p.bias == nullptr && p.resid == nullptr) {
#pragma unroll 1
    for (int ch = h; ch < kChunks; ch += 2) {
      uint32_t r[32];
      tmem_ld_32x32b_x32(tbase + ch * 32, r);
      tmem_ld_wait();
      if (!mok) continue;
      float* oc = o + ch * 32 * ldo;
      const int lim = nv - ch * 32;
      if (lim >= 32) {
#pragma unroll
        for (int j = 0; j < 32; ++j) { *oc = __uint_as_float(r[j]); oc += ldo; }
      } else {
#pragma unroll
        for (int j = 0; j < 32; ++j) { if (j < lim) *oc = __uint_as_float(r[j]); oc += ldo; }
      }
    }
    return;
  }
  const float b = (p.bias != nullptr && mok) ? p.bias[m] : 0.f;
#pragma unroll 1
  for (int ch = h; ch < kChunks; ch += 2) {
    uint32_t r[32];
    tmem_ld_32x32b_x32(tbase + ch * 32, r);
    tmem_ld_wait();
    if (!mok) continue;
#pragma unroll 4
    for (int j = 0; j < 32; ++j) {
      const int n = ch * 32 + j;
      if (n < nv) {
        float v = __uint_as_float(r[j]) + b;
        if (p.resid != nullptr) v += p.resid[static_cast<int64_t>(n0 + n) * p.ldr + m];
        o[n * ldo] = v;
      }
    }
  }
}

static int gemm_mc_budget_kb() {
  static int b = -1;
  if (b < 0) {
    const char* e = getenv("VOX_GEMM_MC_BUDGET_KB");
    // measured on the (GC-free) serving step at 224 rows: 220 KB (5 x 44 KB stages) 773-776,
    // 200 KB 757-769, 150 KB 739-745, 100 KB 580 audio-s/s (profiles/gemm_mc_ab_r01.txt)
    b = e ? atoi(e) : 220;
    if (b < 32) b = 32;
    if (b > 220) b = 220;
  }
  return b;
}

template <int BN>
struct McCfg {
  static constexpr int kABytes = 128 * 64 * 2;
  static constexpr int kBBytes = BN * 64 * 2;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kTmemCols = BN <= 32 ? 32 : BN <= 64 ? 64 : BN <= 128 ? 128 : BN <= 256 ? 256 : 512;
  // BN > 256 (decode rows plus a prefill burst): two MMAs per k-step over one
  // weight stage, N = 256 on activation rows [0, 256) and N = BN - 256 on the rest
  static constexpr int kN2 = BN > 256 ? BN - 256 : 0;
  // ring depth from a smem budget (KB): ~200 = one CTA per SM, deep; ~100 lets
  // the next kernel's CTA co-reside (PDL prologue overlap)
  static int stages(int budget_kb) {
    // narrow tiles (few rows): a ~100 KB ring still holds 4-5 weight stages and
    // lets two CTAs share an SM (one wave for e.g. the 224-tile LM head)
    static const int small_kb = getenv("VOX_GEMM_MC_SMALL_KB") ? atoi(getenv("VOX_GEMM_MC_SMALL_KB")) : 100;
    if (BN <= 32 && small_kb > 0) budget_kb = small_kb;
    else if (BN <= 64 && budget_kb > 150) budget_kb = 150;  // B=64: 2.53 ms at 220 KB vs 2.47 at 150
    int n = budget_kb * 1024 / kStageBytes;
    return n > 8 ? 8 : (n < 2 ? 2 : n);
  }
  // the fused-SiLU epilogue parks gate and up ([BN][64] fp32 each) in the ring
  __host__ __device__ static int ring_bytes(int st, int epi) {
    const int r = st * kStageBytes, e = epi == 1 ? 2 * ((BN + 31) / 32 * 32) * 64 * 4 : 0;
    return r > e ? r : e;
  }
  static int smem_bytes(int st, int epi) { return ring_bytes(st, epi) + 1024 + 256; }
  // dynamic smem cap: 227 KB minus the static smem of the fused-norm prologue
  static constexpr int kSmemMax = 8 * kStageBytes + 1024 + 256 > 226 * 1024 ? 226 * 1024 : 8 * kStageBytes + 1024 + 256;
};

template <int BN>
__global__ void __launch_bounds__(256, 1)
    gemm_mc_kernel(const __grid_constant__ CUtensorMap tmX, const __grid_constant__ CUtensorMap tmX2,
                   GemmArgs p) {
  VOX_TRACE(kTrGemmMc);
  using C = McCfg<BN>;
  const long long t_entry = clock64();
  unsigned long long g_entry;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_entry));
  const int nst = p.stages;  // ring depth (runtime: smem budget chosen by the host)
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::ring_bytes(nst, p.epi));
  uint64_t* empty = full + nst;
  uint64_t* done = empty + nst;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int m0 = blockIdx.y * 128;
  const int n0 = blockIdx.x * BN;
  const int split = blockIdx.z;
  const int kb0 = split * p.kb_per_split;
  const int kb1 = min(p.n_kb, kb0 + p.kb_per_split);
  const int nkb = kb1 - kb0;  // host guarantees >= 1
  // k-block order rotated per weight tile: the CTAs read different activation
  // k-blocks at any instant instead of all hammering the same L2 lines
  const int krot = p.k_rotate ? static_cast<int>((blockIdx.y * 7u) % static_cast<unsigned>(nkb)) : 0;
  auto kbi = [&](int i) { const int t = i + krot; return kb0 + (t >= nkb ? t - nkb : t); };
  const bf16* wt = p.w_packed + static_cast<int64_t>(m0 / 128) * p.n_kb * 8192;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmX);
    if (C::kN2 > 0) tma_prefetch_desc(&tmX2);
    for (int s = 0; s < nst; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    mbar_init(done, 1);
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, C::kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const long long t_setup = clock64();
  long long t_first = 0, t_lastmma = 0;

  if (warp == 0 && lane == 0) {
    // ---------------- producer ----------------
    const uint64_t pol_w = policy_evict_first(), pol_x = policy_evict_last();
    const int pre = nkb < nst ? nkb : nst;
    for (int i = 0; i < pre; ++i) {  // weights do not depend on the preceding kernel
      mbar_arrive_expect_tx(&full[i], C::kStageBytes);
      bulk_load(smem + i * C::kStageBytes, wt + static_cast<int64_t>(kbi(i)) * 8192, 16384, &full[i],
                pol_w);
    }
    // activation k-block: one box of BN rows, or 256 + (BN - 256) rows (TMA box <= 256)
    auto load_x = [&](uint8_t* dst, int kb, uint64_t* bar) {
      tma_load_2d(dst, &tmX, bar, kb * 64, n0, pol_x);
      if (C::kN2 > 0) tma_load_2d(dst + 256 * 128, &tmX2, bar, kb * 64, n0 + 256, pol_x);
    };
    griddep_wait();
    griddep_launch();  // wait-then-launch (see gemm_bf16_tc_kernel)
    for (int i = 0; i < pre; ++i) load_x(smem + i * C::kStageBytes + C::kABytes, kbi(i), &full[i]);
    for (int i = pre; i < nkb; ++i) {
      const int s = i % nst;
      mbar_wait(&empty[s], ((i / nst) - 1) & 1);
      uint8_t* st = smem + s * C::kStageBytes;
      mbar_arrive_expect_tx(&full[s], C::kStageBytes);
      bulk_load(st, wt + static_cast<int64_t>(kbi(i)) * 8192, 16384, &full[s], pol_w);
      load_x(st + C::kABytes, kbi(i), &full[s]);
    }
  } else if (warp == 1 && lane == 0) {
    // ---------------- MMA issuer ----------------
    constexpr uint32_t idesc = make_idesc_bf16(128, BN > 256 ? 256 : BN);
    constexpr uint32_t idesc2 = make_idesc_bf16(128, C::kN2 > 0 ? C::kN2 : 16);
    for (int i = 0; i < nkb; ++i) {
      const int s = i % nst;
      mbar_wait(&full[s], (i / nst) & 1);
      if (i == 0) t_first = clock64();
      tc_fence_after();
      const uint32_t a_addr = smem_u32(smem + s * C::kStageBytes);
      const uint32_t b_addr = a_addr + C::kABytes;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        umma_bf16(tmem, make_desc_k128(a_addr + k * 32), make_desc_k128(b_addr + k * 32), idesc,
                  (i > 0 || k > 0) ? 1u : 0u);
        if (C::kN2 > 0)
          umma_bf16(tmem + 256, make_desc_k128(a_addr + k * 32), make_desc_k128(b_addr + 256 * 128 + k * 32),
                    idesc2, (i > 0 || k > 0) ? 1u : 0u);
      }
      if (i == nkb - 1) t_lastmma = clock64();
      umma_commit(&empty[s]);
    }
    umma_commit(done);
  }
  __syncwarp();

  griddep_wait();
  griddep_launch();
  mbar_wait(done, 0);
  const long long t_done = clock64();
  tc_fence_after();
  mc_epilogue<BN>(p, smem, tmem, warp, lane, m0, n0, split);
  if (p.dbg != nullptr) {
    const int cta = (blockIdx.z * gridDim.y + blockIdx.y) * gridDim.x + blockIdx.x;
    unsigned long long* d = p.dbg + cta * 8;
    if (threadIdx.x == 32) { d[2] = t_first - t_entry; d[3] = t_lastmma - t_entry; }
    if (threadIdx.x == 0) {
      unsigned long long gt;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
      d[0] = g_entry; d[1] = t_setup - t_entry; d[4] = t_done - t_entry; d[5] = clock64() - t_entry;
      d[6] = gt;
      uint32_t smid;
      asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
      d[7] = smid;
    }
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, C::kTmemCols);
  }
}

// ---------------------------------------------------------------------------
// Persistent GEMM for many-tile activation streams (the codec detokenizers'
// transformer / conv GEMMs: tens of thousands of rows, K = 256..2048).
//
// One CTA per SM loops over 128 x BN output tiles (n-tiles fastest, so the CTAs
// of a wave share each weight tile in L2).  Warp 0 / lane 0 streams W and X
// k-blocks by TMA through one ring that runs on across tiles, warp 1 / lane 0
// issues tcgen05.mma into one of two TMEM accumulators, and warps 4..11 drain
// the other accumulator straight to global (TMEM lane = output channel m, so a
// warp's 32 lanes write 32 consecutive channels of one row: 128-byte stores, no
// smem staging) -- tile t's epilogue overlaps tile t+1's loads and MMAs,
// instead of one load -> MMA -> epilogue per CTA lifetime.
// Epilogues: fp32 out (+ bias[m]) (+ resid[n][m]); epi == 2: bf16(GELU(acc + b)).
// ---------------------------------------------------------------------------
constexpr int kPersistThreads = 384;
template <int BN, int MT>
struct PersistCfg {
  static constexpr int kABytes = MT * 128 * 64 * 2;  // MT weight sub-tiles share one X stage
  static constexpr int kStageBytes = kABytes + BN * 64 * 2;
  static constexpr int kStages = (200 * 1024) / kStageBytes > 8 ? 8 : (200 * 1024) / kStageBytes;
  static constexpr int kCols = MT * (BN <= 32 ? 32 : BN <= 64 ? 64 : BN <= 128 ? 128 : 256);  // per buffer
  static constexpr int kSmem = 1024 + kStages * kStageBytes + 256;
};

template <int BN, int MT>
__global__ void __launch_bounds__(kPersistThreads, 1)
    gemm_persist_kernel(const __grid_constant__ CUtensorMap tmW, const __grid_constant__ CUtensorMap tmX,
                        GemmArgs p) {
  VOX_TRACE(kTrGemm);
  using C = PersistCfg<BN, MT>;
  constexpr int ST = C::kStages;
  constexpr int kSub = C::kCols / MT;  // TMEM columns of one weight sub-tile
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + ST * C::kStageBytes);
  uint64_t* empty = full + ST;
  uint64_t* tfull = empty + ST;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n_nt = (p.N + BN - 1) / BN, n_mt = (p.M + 128 * MT - 1) / (128 * MT);
  const int ntiles = n_nt * n_mt;
  const int nkb = p.n_kb;

  if (threadIdx.x == 0) {
    tma_prefetch_desc(&tmW);
    tma_prefetch_desc(&tmX);
    for (int s = 0; s < ST; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    for (int b = 0; b < 2; ++b) { mbar_init(&tfull[b], 1); mbar_init(&tempty[b], 8); }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, 2 * C::kCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      const uint64_t pol_w = policy_evict_last(), pol_x = policy_evict_first();
      griddep_wait();  // X is the preceding kernel's output
      griddep_launch();
      int g = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x) {
        const int m0 = (t / n_nt) * 128 * MT, n0 = (t % n_nt) * BN;
        for (int i = 0; i < nkb; ++i, ++g) {
          const int s = g % ST;
          if (g >= ST) mbar_wait(&empty[s], ((g / ST) - 1) & 1);
          uint8_t* st = smem + s * C::kStageBytes;
          mbar_arrive_expect_tx(&full[s], C::kStageBytes);
#pragma unroll
          for (int mt = 0; mt < MT; ++mt) tma_load_2d(st + mt * 16384, &tmW, &full[s], i * 64, m0 + mt * 128, pol_w);
          tma_load_2d(st + C::kABytes, &tmX, &full[s], i * 64, n0, pol_x);
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {
      constexpr uint32_t idesc = make_idesc_bf16(128, BN);
      int g = 0, u = 0;
      for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++u) {
        const int b = u & 1;
        if (u >= 2) mbar_wait(&tempty[b], ((u >> 1) - 1) & 1);
        tc_fence_after();
        const uint32_t d = tmem + b * C::kCols;
        for (int i = 0; i < nkb; ++i, ++g) {
          const int s = g % ST;
          mbar_wait(&full[s], (g / ST) & 1);
          tc_fence_after();
          const uint32_t a_addr = smem_u32(smem + s * C::kStageBytes);
          const uint32_t b_addr = a_addr + C::kABytes;
#pragma unroll
          for (int k = 0; k < 4; ++k)
#pragma unroll
            for (int mt = 0; mt < MT; ++mt)
              umma_bf16(d + mt * kSub, make_desc_k128(a_addr + mt * 16384 + k * 32), make_desc_k128(b_addr + k * 32),
                        idesc, (i > 0 || k > 0) ? 1u : 0u);
          umma_commit(&empty[s]);
        }
        umma_commit(&tfull[b]);
      }
    }
    __syncwarp();
  } else if (warp >= 4) {
    // MT == 1: warps w and w + 4 split the tile's 32-column chunks; MT == 2: warps
    // 4..7 drain weight sub-tile 0, warps 8..11 sub-tile 1
    const int q = warp & 3, h = (warp - 4) >> 2;
    const int sub = MT == 2 ? h : 0, c0 = MT == 2 ? 0 : h, cstep = MT == 2 ? 1 : 2;
    griddep_wait();  // outputs may alias buffers the preceding kernel was reading
    griddep_launch();
    constexpr int kChunks = (BN + 31) / 32;
    int u = 0;
    for (int t = blockIdx.x; t < ntiles; t += gridDim.x, ++u) {
      const int m0 = (t / n_nt) * 128 * MT + sub * 128, n0 = (t % n_nt) * BN;
      const int b = u & 1;
      const int m = m0 + q * 32 + lane;
      const bool mok = m < p.m_valid;
      const float bias = (p.bias != nullptr && mok) ? p.bias[m] : 0.f;
      const int nv = min(BN, p.N - n0);
      mbar_wait(&tfull[b], (u >> 1) & 1);
      tc_fence_after();
      const uint32_t tbase = tmem + (static_cast<uint32_t>(q * 32) << 16) + b * C::kCols + sub * kSub;
#pragma unroll 1
      for (int ch = c0; ch < kChunks; ch += cstep) {
        uint32_t r[32];
        tmem_ld_32x32b_x32(tbase + ch * 32, r);
        tmem_ld_wait();
        if (!mok) continue;
        const int lim = nv - ch * 32;
        const int64_t n = n0 + ch * 32;
        if (p.epi == 2) {
          bf16* o = p.act + n * p.ld_act + m;
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if (j < lim) o[j * p.ld_act] = __float2bfloat16_rn(gelu_erf(__uint_as_float(r[j]) + bias));
        } else if (p.resid != nullptr) {
          const float* rs = p.resid + n * p.ldr + m;
          float rv[32];
#pragma unroll
          for (int j = 0; j < 32; ++j) rv[j] = j < lim ? rs[j * p.ldr] : 0.f;
          float* o = p.out + n * p.ldo + m;
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if (j < lim) o[j * p.ldo] = (__uint_as_float(r[j]) + bias) + rv[j];
        } else {
          float* o = p.out + n * p.ldo + m;
#pragma unroll
          for (int j = 0; j < 32; ++j)
            if (j < lim) o[j * p.ldo] = __uint_as_float(r[j]) + bias;
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[b]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, 2 * C::kCols);
  }
}

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
static PFN_cuTensorMapEncodeTiled_v12000 g_encode = nullptr;

static bool load_encode() {
  if (g_encode) return true;
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) !=
          cudaSuccess ||
      fn == nullptr)
    return false;
  g_encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
  return true;
}

bool make_tmap_bf16(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer,
                    uint64_t row_stride_bytes, uint32_t box_outer) {
  if (!load_encode()) return false;
  cuuint64_t dims[2] = {inner, outer};
  cuuint64_t strides[1] = {row_stride_bytes};
  cuuint32_t box[2] = {64, box_outer};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = g_encode(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims,
                        strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

template <int BN, int MT>
static cudaError_t launch_bn(const CUtensorMap& tw, const CUtensorMap& tx, const GemmArgs& a,
                             int splits, cudaStream_t st) {
  using C = GemmCfg<BN, MT>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(gemm_bf16_tc_kernel<BN, MT>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         C::kSmemBytes);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  dim3 grid((a.N + BN - 1) / BN, (a.M + 128 * MT - 1) / (128 * MT), splits);
  return launch_k(gemm_bf16_tc_kernel<BN, MT>, grid, dim3(128), C::kSmemBytes, st, tw, tx, a);
}

template <int BN>
static cudaError_t launch_mc(const CUtensorMap& tx, const CUtensorMap& tx2, const GemmArgs& a, int splits,
                            cudaStream_t st) {
  using C = McCfg<BN>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(gemm_mc_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         C::kSmemMax);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  GemmArgs a2 = a;
  a2.stages = C::stages(gemm_mc_budget_kb());
  const dim3 grid((a.N + BN - 1) / BN, (a.M + 127) / 128, splits);
  return launch_k(gemm_mc_kernel<BN>, grid, dim3(256), C::smem_bytes(a2.stages, a2.epi), st, tx, tx2, a2);
}

// CTAs of gemm_mc_kernel<BN> that can be co-resident (one per SM at the deep
// ring, two at the 100 KB ring of <= 32-row tiles).  Queried once per width.
static int g_sm_budget = kNumSMs;
void vox_set_sm_budget(int sms) { g_sm_budget = (sms > 0 && sms <= kNumSMs) ? sms : kNumSMs; }
int vox_sm_budget() { return g_sm_budget; }

template <int BN>
static int mc_capacity_t() {
  static int per_sm_c = 0;
  if (per_sm_c == 0) {
    using C = McCfg<BN>;
    cudaFuncSetAttribute(gemm_mc_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmemMax);
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, gemm_mc_kernel<BN>, 256,
                                                      C::smem_bytes(C::stages(gemm_mc_budget_kb()), 0)) !=
            cudaSuccess ||
        per_sm <= 0) {
      cudaGetLastError();
      per_sm = 1;
    }
    per_sm_c = per_sm;
  }
  return per_sm_c * g_sm_budget;
}
int gemm_mc_capacity(int bn) {
  switch (bn) {
    case 16: return mc_capacity_t<16>();
    case 32: return mc_capacity_t<32>();
    case 64: return mc_capacity_t<64>();
    case 96: return mc_capacity_t<96>();
    case 128: return mc_capacity_t<128>();
    case 160: return mc_capacity_t<160>();
    case 192: return mc_capacity_t<192>();
    case 224: return mc_capacity_t<224>();
    case 288: return mc_capacity_t<288>();
    case 320: return mc_capacity_t<320>();
    case 384: return mc_capacity_t<384>();
    default: return mc_capacity_t<256>();
  }
}

// BN in {16, 32, 64, 96, 128, 160, 192, 224, 256, 288, 320, 384}; tx = activation map
// with box rows min(BN, 256), tx2 = box rows BN - 256 (BN > 256 only)
cudaError_t gemm_launch_mc(const CUtensorMap& tx, const CUtensorMap& tx2, GemmArgs a, int splits, int bn,
                           cudaStream_t st) {
  if (a.w_packed == nullptr) return cudaErrorInvalidValue;
  a.n_kb = a.K / 64;
  a.kb_per_split = (a.n_kb + splits - 1) / splits;
  splits = (a.n_kb + a.kb_per_split - 1) / a.kb_per_split;
  switch (bn) {
    case 16: return launch_mc<16>(tx, tx2, a, splits, st);
    case 32: return launch_mc<32>(tx, tx2, a, splits, st);
    case 64: return launch_mc<64>(tx, tx2, a, splits, st);
    case 96: return launch_mc<96>(tx, tx2, a, splits, st);
    case 128: return launch_mc<128>(tx, tx2, a, splits, st);
    case 160: return launch_mc<160>(tx, tx2, a, splits, st);
    case 192: return launch_mc<192>(tx, tx2, a, splits, st);
    case 224: return launch_mc<224>(tx, tx2, a, splits, st);
    case 256: return launch_mc<256>(tx, tx2, a, splits, st);
    case 288: return launch_mc<288>(tx, tx2, a, splits, st);
    case 320: return launch_mc<320>(tx, tx2, a, splits, st);
    case 384: return launch_mc<384>(tx, tx2, a, splits, st);
    default: return cudaErrorInvalidValue;
  }
}

int gemm_bn_for_rows(int rows) {
  if (rows <= 16) return 16;
  if (rows <= 32) return 32;
  if (rows <= 64) return 64;
  if (rows <= 128) return 128;
  return 256;
}

// Tile plan for out[rows, M] = X[rows, K] W[M, K]^T.
// One 128 x BN tile per CTA (BN = rows rounded up to a power of two, capped at
// 128; 64 for the d_model-wide outputs at >= 128 rows), ~2 CTAs per SM and
// split-K to fill the machine: at decode sizes the GEMM streams weights, and
// every SM must keep loads in flight (measured, profiles/gemm_sweep_r01.txt:
// 256 x 256 tiles (MT = 2) leave SMs idle and lose 2x at 224 rows).
GemmPlan gemm_plan_1cta(int M, int rows, int K) {
  GemmPlan g{};
  const int n_kb = K / 64;
  g.mc = 0;
  g.bn = gemm_bn_for_rows(rows);
  if (g.bn > 128) g.bn = 128;
  if (rows >= 128 && M <= 4096) g.bn = 64;
  g.mt = 1;
  if (const char* e = getenv("VOX_GEMM_BN_TEST")) {  // microbenchmarks only
    const int f = atoi(e);
    if (f == 16 || f == 32 || f == 64 || f == 128 || f == 256) g.bn = f;
  }
  if (const char* e = getenv("VOX_GEMM_MT_TEST")) g.mt = atoi(e) == 2 ? 2 : 1;
  const int tiles = ((M + 128 * g.mt - 1) / (128 * g.mt)) * ((rows + g.bn - 1) / g.bn);
  const int slots = (g.mt == 2 ? 1 : 2) * g_sm_budget;
  int best = 1;
  for (int s = 1; s <= kGemmMaxSplits; ++s) {
    const int per = (n_kb + s - 1) / s;
    if (per < 2) break;
    if ((n_kb + per - 1) / per != s) continue;  // every split non-empty
    if (tiles * s > slots) break;
    best = s;
  }
  g.splits = best;
  if (const char* e = getenv("VOX_GEMM_SPLITS_TEST")) g.splits = atoi(e) < 1 ? 1 : atoi(e);
  return g;
}

GemmPlan gemm_plan(int M, int rows, int K) {
  GemmPlan g{};
  const int n_kb = K / 64;
  // Decode-sized row counts: the mc kernel (one n-tile covering every row, so
  // each weight byte is read once; split-K to fill the co-resident CTA slots).
  // Callers fall back to the plan below when the weights are not packed.
  if (rows <= 512 && K % 64 == 0) {
    // <= 384 rows (decode plus a burst of prefill rows): one n-tile, so every
    // weight byte is read once (BN > 256 runs two MMAs per k-step); 385..512
    // rows: two n-tiles of half the rows each
    const int ntiles = rows > 384 ? 2 : 1;
    const int per_tile = (rows + ntiles - 1) / ntiles;
    int bn = 256;
    for (int b : {16, 32, 64, 96, 128, 160, 192, 224, 256, 288, 320, 384})
      if (per_tile <= b) { bn = b; break; }
    const int mtiles = (M + 127) / 128 * ntiles;  // CTAs per split
    const int cap = gemm_mc_capacity(bn);
    int best = 1;
    for (int s2 = 1; s2 <= kGemmMaxSplits; ++s2) {
      const int per = (n_kb + s2 - 1) / s2;
      if (per < 2) break;
      if ((n_kb + per - 1) / per != s2) continue;  // every split non-empty
      if (mtiles * s2 > cap) break;
      best = s2;
    }
    g.mc = 1;
    g.bn = bn;
    g.mt = 1;
    g.splits = best;
    if (const char* e = getenv("VOX_GEMM_SPLITS_TEST")) g.splits = atoi(e) < 1 ? 1 : atoi(e);
    return g;
  }
  return gemm_plan_1cta(M, rows, K);
}

cudaError_t gemm_launch(const CUtensorMap& tw, const CUtensorMap& tx, GemmArgs a, int splits,
                        int bn, int mt, cudaStream_t st) {
  a.n_kb = a.K / 64;
  a.kb_per_split = (a.n_kb + splits - 1) / splits;
  splits = (a.n_kb + a.kb_per_split - 1) / a.kb_per_split;
  if (mt == 2) {
    switch (bn) {
      case 16: return launch_bn<16, 2>(tw, tx, a, splits, st);
      case 32: return launch_bn<32, 2>(tw, tx, a, splits, st);
      case 64: return launch_bn<64, 2>(tw, tx, a, splits, st);
      case 128: return launch_bn<128, 2>(tw, tx, a, splits, st);
      default: return launch_bn<256, 2>(tw, tx, a, splits, st);
    }
  }
  switch (bn) {
    case 16: return launch_bn<16, 1>(tw, tx, a, splits, st);
    case 32: return launch_bn<32, 1>(tw, tx, a, splits, st);
    case 64: return launch_bn<64, 1>(tw, tx, a, splits, st);
    case 128: return launch_bn<128, 1>(tw, tx, a, splits, st);
    default: return launch_bn<256, 1>(tw, tx, a, splits, st);
  }
}

template <int BN, int MT>
static cudaError_t launch_persist(const CUtensorMap& tw, const CUtensorMap& tx, const GemmArgs& a, cudaStream_t st) {
  using C = PersistCfg<BN, MT>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(gemm_persist_kernel<BN, MT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         C::kSmem);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  const int tiles = ((a.N + BN - 1) / BN) * ((a.M + 128 * MT - 1) / (128 * MT));
  const int grid = tiles < g_sm_budget ? tiles : g_sm_budget;
  return launch_k(gemm_persist_kernel<BN, MT>, dim3(grid), dim3(kPersistThreads), C::kSmem, st, tw, tx, a);
}

// one split; tx = activation map with box rows bn (128); mt = 2: 256-row weight
// tiles sharing each activation stage (activations read from L2 half as often)
cudaError_t gemm_launch_persist(const CUtensorMap& tw, const CUtensorMap& tx, GemmArgs a, int bn, int mt,
                                cudaStream_t st) {
  a.n_kb = a.K / 64;
  a.kb_per_split = a.n_kb;
  if (a.epi == 2 && a.resid != nullptr) return cudaErrorInvalidValue;
  if (bn != 128) return cudaErrorInvalidValue;
  return mt == 2 ? launch_persist<128, 2>(tw, tx, a, st) : launch_persist<128, 1>(tw, tx, a, st);
}

}  // namespace vox
