// attn.cu — K2: paged GQA decode attention (HBM-bound) + split-KV combine.
//
// One CTA (4 warps) per (row, kv head, kv split).  The G = H/KV query heads
// that share a kv head are processed together, so every K/V byte is read from
// HBM exactly once per step.
//
// Data movement: thread 0 streams whole head-pages (K page [ps][hd] and the
// TRANSPOSED V page [hd][ps], 4 KB each at ps=16, hd=128) into a 3-stage
// shared-memory ring with 1-D bulk copies (cp.async.bulk + mbarrier
// transaction counts), 4 pages (64 tokens, 32 KB) per stage, so ~96 KB per CTA
// is in flight independent of registers.
//
// Math on tensor cores (mma.sync m16n8k16 bf16 -> fp32), one page per warp per
// stage, fragments loaded with single vector loads thanks to consistent
// permutations (a dot product is invariant to permuting its reduction index):
//   QK^T: A = q (rows = the G heads, padded to 16), B = K^T.  Lane (n=lane/4,
//         j=lane%4) loads dims 32m+8j..+7 of its token row (16 B): k-block 2m
//         uses the first 4 of those dims, 2m+1 the last 4; q uses the same map.
//         Two n-tiles cover the page; tile t holds token 4(n>>1)+2t+(n&1), so
//         lane j ends up owning the scores of tokens 4j..4j+3.
//   PV:   A = P straight from the QK accumulators (tokens 4j..4j+3 are lane j's
//         k-slots 2j,2j+1,2j+8,2j+9), B = V: with V^T stored per page, lane j
//         reads V^T[dim][4j..4j+3] as one 8-byte load per 8-dim n-tile.
// Online softmax in exp2 (scores scaled by log2(e)/sqrt(hd) in fp32); P is
// rounded to bf16 for the PV product.  Small batches split the context across
// blockIdx.z (fixed split count per launch -> graph-capturable) and a combine
// pass merges the partial (m, l, acc) triples.
#include "common.cuh"
#include "kernels.h"
#include <cstdlib>

namespace vox {

constexpr int kAttnStages = 3;
constexpr int kAttnPagesPerStage = 4;  // one page per warp
constexpr int kAttnPtSmem = 512;       // page ids staged in smem (8192 tokens at ps 16)

template <int HD>
__host__ __device__ constexpr int attn_stage_bytes(int ps) {
  return kAttnPagesPerStage * 2 * ps * HD * 2;
}

VOX_DEV void mma_bf16_16816(float (&d)[4], uint32_t a0, uint32_t a2, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(0u), "r"(a2), "r"(0u), "r"(b0), "r"(b1));
}

VOX_DEV uint32_t pack_bf16x2(float lo, float hi) {
  __nv_bfloat162 v = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&v);
}

template <int HD, int G>
__global__ void __launch_bounds__(128)
    attn_decode_kernel(const RowDev* __restrict__ rows, const bf16* __restrict__ q,
                       const bf16* __restrict__ kc, const bf16* __restrict__ vc,
                       const int* __restrict__ page_table, LmDims dm, bf16* __restrict__ out,
                       float* __restrict__ ws, int n_split) {
  static_assert(G <= 8, "GQA group must fit the mma row tile");
  constexpr int NB = HD / 32;  // 32-dim blocks (2 k-blocks each)
  constexpr int NT = HD / 8;   // PV n-tiles
  extern __shared__ __align__(128) uint8_t stage_raw[];
  __shared__ uint64_t full[kAttnStages], empty[kAttnStages];
  __shared__ float s_m[4][8], s_l[4][8];
  // the 4 warps' partial outputs are merged through the (then idle) K/V ring
  float (*s_acc)[8][HD] = reinterpret_cast<float (*)[8][HD]>(stage_raw);

  // rows / page table are uploaded before the step's first kernel and K/V of
  // positions < pos were appended by earlier steps: none of it depends on the
  // preceding kernel, so the prologue and the first K/V copies overlap its
  // tail (PDL); only q and the page holding `pos` wait for griddep_wait.
  const int r = blockIdx.x, kvh = blockIdx.y, z = blockIdx.z;
  const RowDev rw = rows[r];
  if (rw.slot < 0) {
    griddep_wait();
    griddep_launch();
    return;
  }
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int gn = lane >> 2, j = lane & 3;  // mma row/col group, k-slot group
  const int ps = dm.page_size;
  const int L = rw.pos + 1;
  const int n_pages = (L + ps - 1) / ps;
  const int pps = (n_pages + n_split - 1) / n_split;
  const int p_begin = z * pps;
  const int p_end = min(n_pages, p_begin + pps);
  const int n_rounds = p_end > p_begin ? (p_end - p_begin + kAttnPagesPerStage - 1) / kAttnPagesPerStage : 0;
  const int page_elems = ps * HD;
  const int stage_bytes = attn_stage_bytes<HD>(ps);
  const int* pt_g = page_table + static_cast<int64_t>(rw.slot) * dm.max_pages_per_slot;
  // this split's page ids, staged once (a dependent global load per bulk copy
  // would serialise the issue loop on load latency)
  __shared__ int s_pt[kAttnPtSmem];
  const bool pt_in_smem = (p_end - p_begin) <= kAttnPtSmem;
  if (pt_in_smem)
    for (int i = tid; i < p_end - p_begin; i += 128) s_pt[i] = pt_g[p_begin + i];
  auto page_id = [&](int pg) { return pt_in_smem ? s_pt[pg - p_begin] : pt_g[pg]; };

  if (tid == 0) {
    for (int s = 0; s < kAttnStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 4);
    }
    fence_mbar_init();
  }
  __syncthreads();
  auto stage_ptr = [&](int s, int jp, int kv) -> const bf16* {
    return reinterpret_cast<const bf16*>(stage_raw + static_cast<size_t>(s) * stage_bytes) +
           (jp * 2 + kv) * page_elems;
  };
  uint64_t pol = 0;
  auto issue = [&](int rr) {
    const int s = rr % kAttnStages;
    const int pa = p_begin + rr * kAttnPagesPerStage;
    const int np = min(kAttnPagesPerStage, p_end - pa);
    mbar_arrive_expect_tx(&full[s], static_cast<uint32_t>(np * 2 * page_elems * 2));
    for (int jp = 0; jp < np; ++jp) {
      const int64_t base = (static_cast<int64_t>(page_id(pa + jp)) * dm.n_kv + kvh) * page_elems;
      bulk_load(const_cast<bf16*>(stage_ptr(s, jp, 0)), kc + base, page_elems * 2, &full[s], pol);
      bulk_load(const_cast<bf16*>(stage_ptr(s, jp, 1)), vc + base, page_elems * 2, &full[s], pol);
    }
  };
  // stages whose pages all precede the first page this forward appends to
  // (rw.fresh, written by the preceding kernel) are issued before the
  // grid-dependency wait
  const int last_page = rw.fresh / ps;
  const int pre = min(kAttnStages, n_rounds);
  int n_early = 0;
  while (n_early < pre && p_begin + (n_early + 1) * kAttnPagesPerStage - 1 < last_page &&
         p_begin + (n_early + 1) * kAttnPagesPerStage <= p_end)
    ++n_early;
  if (tid == 0) {
    pol = policy_evict_first();  // K/V are read once per step
    for (int rr = 0; rr < n_early; ++rr) issue(rr);
  }
  griddep_wait();
  griddep_launch();
  if (tid == 0)
    for (int rr = n_early; rr < pre; ++rr) issue(rr);

  // q A-fragments: head gn (< G), dims 32m + 8j .. +7 (zero rows beyond G)
  uint4 qa[NB];
#pragma unroll
  for (int m = 0; m < NB; ++m) {
    if (gn < G)
      qa[m] = *reinterpret_cast<const uint4*>(
          q + (static_cast<int64_t>(r) * dm.n_heads + kvh * G + gn) * HD + 32 * m + 8 * j);
    else
      qa[m] = make_uint4(0u, 0u, 0u, 0u);
  }
  const float qscale = 1.4426950408889634f / sqrtf(static_cast<float>(HD));
  float mrow = -INFINITY, lrow = 0.f;  // head gn, lane-partial l
  float acc[NT][4];
#pragma unroll
  for (int t = 0; t < NT; ++t) acc[t][0] = acc[t][1] = acc[t][2] = acc[t][3] = 0.f;

  for (int rr = 0; rr < n_rounds; ++rr) {
    const int s = rr % kAttnStages;
    mbar_wait(&full[s], (rr / kAttnStages) & 1);
    const int page_idx = p_begin + rr * kAttnPagesPerStage + warp;
    if (page_idx < p_end) {
      const bf16* kp = stage_ptr(s, warp, 0);
      const bf16* vp = stage_ptr(s, warp, 1);
      // ---- S = q K^T over the 16 tokens of this page (two n-tiles)
      float sacc[2][4];
#pragma unroll
      for (int t = 0; t < 2; ++t) {
        sacc[t][0] = sacc[t][1] = sacc[t][2] = sacc[t][3] = 0.f;
        const int tok = 4 * (gn >> 1) + 2 * t + (gn & 1);
        const bf16* krow = kp + tok * HD + 8 * j;
        // Odd rows LOAD the 32-dim blocks in XOR-1 order so the two token rows
        // of an 8-lane shared-memory phase hit disjoint banks; the mma then
        // consumes block m on every lane (the k->dim map must be lane-uniform)
        const int odd = gn & 1;
        uint4 kb[NB];
#pragma unroll
        for (int i = 0; i < NB; ++i) kb[i] = *reinterpret_cast<const uint4*>(krow + 32 * (i ^ odd));
#pragma unroll
        for (int m = 0; m < NB; ++m) {
          const uint4 ku = odd ? kb[m ^ 1] : kb[m];
          mma_bf16_16816(sacc[t], qa[m].x, qa[m].y, ku.x, ku.y);
          mma_bf16_16816(sacc[t], qa[m].z, qa[m].w, ku.z, ku.w);
        }
      }
      // lane j owns tokens 4j..4j+3 of row gn: (sacc[0][0], sacc[0][1], sacc[1][0], sacc[1][1])
      const int tok0 = page_idx * ps + 4 * j;
      float sv[4] = {sacc[0][0] * qscale, sacc[0][1] * qscale, sacc[1][0] * qscale,
                     sacc[1][1] * qscale};
#pragma unroll
      for (int e = 0; e < 4; ++e)
        if (tok0 + e >= L) sv[e] = -INFINITY;
      float cm = fmaxf(fmaxf(sv[0], sv[1]), fmaxf(sv[2], sv[3]));
      cm = fmaxf(cm, __shfl_xor_sync(0xffffffffu, cm, 1));
      cm = fmaxf(cm, __shfl_xor_sync(0xffffffffu, cm, 2));
      const float nm = fmaxf(mrow, cm);  // finite: the page's first token is valid
      const float corr = exp2f(mrow - nm);
      float p[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) p[e] = exp2f(sv[e] - nm);
      mrow = nm;
      lrow = lrow * corr + (p[0] + p[1]) + (p[2] + p[3]);
      // P as a bf16 hi + lo pair (~16-bit mantissa): two PV mmas keep the
      // probabilities at near-fp32 accuracy (the oracle weights V in fp32)
      const __nv_bfloat162 h01 = __floats2bfloat162_rn(p[0], p[1]);
      const __nv_bfloat162 h23 = __floats2bfloat162_rn(p[2], p[3]);
      const uint32_t pa0 = *reinterpret_cast<const uint32_t*>(&h01);
      const uint32_t pa2 = *reinterpret_cast<const uint32_t*>(&h23);
      const uint32_t pl0 = pack_bf16x2(p[0] - __low2float(h01), p[1] - __high2float(h01));
      const uint32_t pl2 = pack_bf16x2(p[2] - __low2float(h23), p[3] - __high2float(h23));
      // ---- O += P V  (B = V^T rows: dim 8t + gn, tokens 4j..4j+3)
#pragma unroll
      for (int t = 0; t < NT; ++t) {
        acc[t][0] *= corr;
        acc[t][1] *= corr;
        const uint2 vu = *reinterpret_cast<const uint2*>(vp + (8 * t + gn) * ps + 4 * j);
        mma_bf16_16816(acc[t], pa0, pa2, vu.x, vu.y);
        mma_bf16_16816(acc[t], pl0, pl2, vu.x, vu.y);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    if (tid == 0 && rr + kAttnStages < n_rounds) {
      mbar_wait(&empty[s], (rr / kAttnStages) & 1);  // all 4 warps released this stage
      issue(rr + kAttnStages);
    }
  }
  // row sums: reduce the 4 lane partials of each row
  lrow += __shfl_xor_sync(0xffffffffu, lrow, 1);
  lrow += __shfl_xor_sync(0xffffffffu, lrow, 2);
  // ------------------------------------------------ merge the 4 warps
  __syncthreads();  // every warp is done reading the ring before it is reused
  if (j == 0) {
    s_m[warp][gn] = mrow;
    s_l[warp][gn] = lrow;
  }
#pragma unroll
  for (int t = 0; t < NT; ++t) {
    s_acc[warp][gn][8 * t + 2 * j] = acc[t][0];
    s_acc[warp][gn][8 * t + 2 * j + 1] = acc[t][1];
  }
  __syncthreads();
  for (int idx = tid; idx < G * HD; idx += 128) {
    const int g = idx / HD, dd = idx % HD;
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < 4; ++w) M = fmaxf(M, s_m[w][g]);
    float Ls = 0.f, A = 0.f;
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      const float f = (s_m[w][g] == -INFINITY) ? 0.f : exp2f(s_m[w][g] - M);
      Ls += s_l[w][g] * f;
      A += s_acc[w][g][dd] * f;
    }
    if (n_split == 1) {
      out[(static_cast<int64_t>(r) * dm.n_heads + kvh * G + g) * HD + dd] =
          __float2bfloat16_rn(A / Ls);
    } else {
      float* wp = ws + ((static_cast<int64_t>(r) * dm.n_kv + kvh) * n_split + z) * G * (HD + 2);
      wp[g * (HD + 2) + dd] = A;
      if (dd == 0) {
        wp[g * (HD + 2) + HD] = M;
        wp[g * (HD + 2) + HD + 1] = Ls;
      }
    }
  }
}

template <int HD, int G>
__global__ void __launch_bounds__(128)
    attn_combine_kernel(const RowDev* __restrict__ rows, const float* __restrict__ ws, LmDims dm,
                        int n_split, bf16* __restrict__ out) {
  griddep_wait();
  griddep_launch();
  const int r = blockIdx.x, kvh = blockIdx.y;
  if (rows[r].slot < 0) return;
  const float* base = ws + (static_cast<int64_t>(r) * dm.n_kv + kvh) * n_split * G * (HD + 2);
  for (int idx = threadIdx.x; idx < G * HD; idx += 128) {
    const int g = idx / HD, dd = idx % HD;
    float M = -INFINITY;
    for (int zz = 0; zz < n_split; ++zz) M = fmaxf(M, base[zz * G * (HD + 2) + g * (HD + 2) + HD]);
    float Ls = 0.f, A = 0.f;
    for (int zz = 0; zz < n_split; ++zz) {
      const float* p = base + zz * G * (HD + 2) + g * (HD + 2);
      const float f = (p[HD] == -INFINITY) ? 0.f : exp2f(p[HD] - M);
      Ls += p[HD + 1] * f;
      A += p[dd] * f;
    }
    out[(static_cast<int64_t>(r) * dm.n_heads + kvh * G + g) * HD + dd] = __float2bfloat16_rn(A / Ls);
  }
}

template <int HD, int G>
static void attn_launch(const RowDev* rows, int n, const bf16* q, const bf16* kc, const bf16* vc,
                        const int* pt, const LmDims& dm, bf16* out, float* ws, int n_split,
                        cudaStream_t st) {
  const int smem = kAttnStages * attn_stage_bytes<HD>(dm.page_size);  // 96 KB at ps 16, hd 128
  static int attr_bytes = 0;
  if (smem > attr_bytes) {
    cudaFuncSetAttribute(attn_decode_kernel<HD, G>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         smem);
    attr_bytes = smem;
  }
  launch_k(attn_decode_kernel<HD, G>, dim3(n, dm.n_kv, n_split), dim3(128), smem, st, rows, q, kc,
           vc, pt, dm, out, ws, n_split);
  if (n_split > 1)
    launch_k(attn_combine_kernel<HD, G>, dim3(n, dm.n_kv), dim3(128), 0, st, rows, ws, dm, n_split,
             out);
}

template <int HD>
static void attn_dispatch_g(const RowDev* rows, int n, const bf16* q, const bf16* kc,
                            const bf16* vc, const int* pt, const LmDims& dm, bf16* out, float* ws,
                            int n_split, cudaStream_t st) {
  switch (dm.n_heads / dm.n_kv) {
    case 1: attn_launch<HD, 1>(rows, n, q, kc, vc, pt, dm, out, ws, n_split, st); break;
    case 2: attn_launch<HD, 2>(rows, n, q, kc, vc, pt, dm, out, ws, n_split, st); break;
    case 3: attn_launch<HD, 3>(rows, n, q, kc, vc, pt, dm, out, ws, n_split, st); break;
    case 4: attn_launch<HD, 4>(rows, n, q, kc, vc, pt, dm, out, ws, n_split, st); break;
    default: break;  // rejected at vox_create
  }
}

int attn_pick_splits(int n_rows, int n_kv) {
  if (const char* e = getenv("VOX_ATTN_SPLITS_TEST")) return atoi(e) < 1 ? 1 : atoi(e);  // debug
  const int ctas = n_rows * n_kv;
  int s = (2 * kNumSMs + ctas - 1) / ctas;
  if (s > kAttnMaxSplits) s = kAttnMaxSplits;
  if (n_rows > kAttnSplitRows) s = 1;
  return s < 1 ? 1 : s;
}

void launch_attn_decode(const RowDev* rows, int n, const bf16* q, const bf16* kc, const bf16* vc,
                        const int* page_table, const LmDims& dm, bf16* out, float* ws, int n_split,
                        cudaStream_t st) {
  if (dm.hd == 64)
    attn_dispatch_g<64>(rows, n, q, kc, vc, page_table, dm, out, ws, n_split, st);
  else
    attn_dispatch_g<128>(rows, n, q, kc, vc, page_table, dm, out, ws, n_split, st);
}

}  // namespace vox
