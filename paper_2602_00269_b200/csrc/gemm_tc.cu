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

namespace vox {

template <int BN>
struct GemmCfg {
  static constexpr int kABytes = 128 * 64 * 2;
  static constexpr int kBBytes = BN * 64 * 2;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kStages =
      BN >= 256 ? 4 : (96 * 1024 / kStageBytes > 8 ? 8 : 96 * 1024 / kStageBytes);
  static constexpr int kTmemCols = BN < 32 ? 32 : BN;
  static constexpr int kSmemBytes = kStages * kStageBytes + 1024 + 256;
};

template <int BN>
__global__ void __launch_bounds__(128, 1)
    gemm_bf16_tc_kernel(const __grid_constant__ CUtensorMap tmW,
                        const __grid_constant__ CUtensorMap tmX, GemmArgs p) {
  using C = GemmCfg<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + C::kStages * C::kStageBytes);
  uint64_t* empty = full + C::kStages;
  uint64_t* done = empty + C::kStages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(done + 1);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int m0 = blockIdx.x * 128;
  const int n0 = blockIdx.y * BN;
  const int split = blockIdx.z;
  const int kb0 = split * p.kb_per_split;
  const int kb1 = min(p.n_kb, kb0 + p.kb_per_split);
  const int nkb = kb1 - kb0;  // host guarantees >= 1

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

  griddep_launch();  // let the next kernel start its own prologue
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
      tma_load_2d(smem + i * C::kStageBytes, &tmW, &full[i], (kb0 + i) * 64, m0, pol_w);
    }
    griddep_wait();
    for (int i = 0; i < pre; ++i)
      tma_load_2d(smem + i * C::kStageBytes + C::kABytes, &tmX, &full[i], (kb0 + i) * 64, n0,
                  pol_x);
    for (int i = pre; i < nkb; ++i) {
      const int s = i % C::kStages;
      mbar_wait(&empty[s], ((i / C::kStages) - 1) & 1);
      uint8_t* st = smem + s * C::kStageBytes;
      mbar_arrive_expect_tx(&full[s], C::kStageBytes);
      const int kx = (kb0 + i) * 64;
      tma_load_2d(st, &tmW, &full[s], kx, m0, pol_w);
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
        umma_bf16(tmem, make_desc_k128(a_addr + k * 32), make_desc_k128(b_addr + k * 32), idesc,
                  (i > 0 || k > 0) ? 1u : 0u);
      }
      umma_commit(&empty[s]);  // frees the smem stage once these MMAs retire
    }
    umma_commit(done);  // accumulator complete
  }
  __syncwarp();

  // ---------------- epilogue: TMEM -> registers -> global ----------------
  griddep_wait();  // outputs may alias buffers the preceding kernel was reading
  mbar_wait(done, 0);
  tc_fence_after();
  const int m = m0 + warp * 32 + lane;
  float* outp = p.out + static_cast<int64_t>(split) * p.split_stride;
  const bool m_ok = m < p.m_valid;
  const float b = (p.bias != nullptr && m_ok) ? p.bias[m] : 0.f;
#pragma unroll 1
  for (int c = 0; c < BN; c += 32) {
    uint32_t r[32];
    tmem_ld_32x32b_x32(tmem + (static_cast<uint32_t>(warp * 32) << 16) + c, r);
    tmem_ld_wait();
    if (m_ok) {
#pragma unroll
      for (int j = 0; j < 32; ++j) {
        const int n = n0 + c + j;
        if ((c + j) < BN && n < p.N) {
          float v = __uint_as_float(r[j]) + b;
          if (p.resid != nullptr) v += p.resid[static_cast<int64_t>(n) * p.ldr + m];
          outp[static_cast<int64_t>(n) * p.ldo + m] = v;
        }
      }
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

template <int BN>
static cudaError_t launch_bn(const CUtensorMap& tw, const CUtensorMap& tx, const GemmArgs& a,
                             int splits, cudaStream_t st) {
  using C = GemmCfg<BN>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(gemm_bf16_tc_kernel<BN>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         C::kSmemBytes);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  dim3 grid((a.M + 127) / 128, (a.N + BN - 1) / BN, splits);
  return launch_k(gemm_bf16_tc_kernel<BN>, grid, dim3(128), C::kSmemBytes, st, tw, tx, a);
}

int gemm_bn_for_rows(int rows) {
  if (rows <= 16) return 16;
  if (rows <= 32) return 32;
  if (rows <= 64) return 64;
  if (rows <= 128) return 128;
  return 256;
}

// Tile width over the activation rows (UMMA N).  Measured on B200 at the
// Orpheus-3B shapes (scripts/gemm_sweep.py, profiles/gemm_sweep_r01.txt):
// one 256-wide tile is L2/latency-limited (every CTA re-reads the whole
// activation slab), so large batches use 128-wide tiles, and 64-wide ones
// when the weight matrix has few 128-row tiles (d_model outputs).
int gemm_plan_bn(int M, int rows) {
  int bn = gemm_bn_for_rows(rows);
  if (bn > 128) bn = 128;
  if (rows >= 128 && M <= 4096) bn = 64;
  return bn;
}

// Split-K factor: ~2 CTAs per SM (2 x 148 slots), each split >= 2 k-blocks.
int gemm_pick_splits(int M, int N, int K, int max_splits) {
  const int bn = gemm_plan_bn(M, N);
  const int tiles = ((M + 127) / 128) * ((N + bn - 1) / bn);
  const int n_kb = K / 64;
  int best = 1;
  const int target = 2 * kNumSMs;
  for (int s = 1; s <= max_splits; ++s) {
    const int per = (n_kb + s - 1) / s;
    if (per < 2) break;
    if ((n_kb + per - 1) / per != s) continue;  // every split non-empty
    if (tiles * s > target) break;
    best = s;
  }
  return best;
}

cudaError_t gemm_launch(const CUtensorMap& tw, const CUtensorMap& tx, GemmArgs a, int splits,
                        int bn, cudaStream_t st) {
  a.n_kb = a.K / 64;
  a.kb_per_split = (a.n_kb + splits - 1) / splits;
  splits = (a.n_kb + a.kb_per_split - 1) / a.kb_per_split;
  switch (bn) {
    case 16: return launch_bn<16>(tw, tx, a, splits, st);
    case 32: return launch_bn<32>(tw, tx, a, splits, st);
    case 64: return launch_bn<64>(tw, tx, a, splits, st);
    case 128: return launch_bn<128>(tw, tx, a, splits, st);
    default: return launch_bn<256>(tw, tx, a, splits, st);
  }
}

}  // namespace vox
