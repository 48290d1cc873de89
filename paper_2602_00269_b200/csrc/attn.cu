// attn.cu — K2: paged GQA decode attention (HBM-bound) + split-KV combine.
//
// Work item = (row, kv head, kv split).  The G = H/KV query heads that share a
// kv head are processed together, so every K/V byte is read from HBM exactly
// once per step.  Persistent CTAs (two per SM) pull items from a device counter
// (see the producer below for the look-ahead rule).
//
// Data movement: one producer warp streams whole head-pages (K page [ps][hd] and
// the TRANSPOSED V page [hd][ps], 4 KB each at ps=16, hd=128) into a 3-stage
// shared-memory ring with 1-D bulk copies (cp.async.bulk + mbarrier transaction
// counts), one page per consumer warp per stage: 4 pages (64 tokens, 32 KB) at
// hd 128, 8 pages at hd 64, so the loads in flight do not depend on registers.
// Pages that precede the position appended by this step are issued before
// griddepcontrol.wait (PDL).
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
// Online softmax in exp2 (scores scaled by log2(e)/sqrt(hd) in fp32); P enters
// the PV product as a bf16 hi + lo pair (near-fp32 probabilities).  The warps'
// partial (m, l, acc) are merged per item in shared memory.  Small batches with
// long contexts split each item's pages (fixed split count per launch ->
// graph-capturable) and a combine launch merges the partials.
#include "common.cuh"
#include "kernels.h"
#include <cstdlib>

namespace vox {
VOX_TRACE_TU(trace_set_attn)


// K/V ring depth: 3 stages of 32 KB at hd 128 (4 pages); 2 at hd 64 (8 pages), whose
// 8-warp merge buffers (14 KB static) would otherwise leave room for only one CTA
// per SM (measured: 108 of 256 CTAs in a second wave at 128 rows x 2 kv heads)
template <int HD>
__host__ __device__ constexpr int attn_stages() {
  return HD == 64 ? 2 : 3;
}
// consumer warps = K/V head-pages per stage (one page per warp): 4 at hd 128;
// 8 at hd 64, whose per-page math is a short latency chain, so a lone item (as
// many items as CTA slots, e.g. 128 rows x 2 kv heads) needs more pages in flight
template <int HD>
__host__ __device__ constexpr int attn_warps() {
  return HD == 64 ? 8 : 4;
}
constexpr int kAttnQSlot = 1024;       // per-stage q slot (G * hd * 2 <= 1 KB)

template <int HD>
__host__ __device__ constexpr int attn_stage_bytes(int ps) {
  return attn_warps<HD>() * 2 * ps * HD * 2;
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

// Work item = (row, kv head, kv split), item = ((row * n_kv) + kvh) * n_split + z.
// Persistent CTAs (2 per SM), warp-specialised: warps 0..NW-1 consume one K/V
// head-page each per stage; warp NW is the producer.  The producer pulls items
// from a device counter ONE ITEM AHEAD when there are more items than CTAs
// (counter, row descriptor and the item's page ids, loaded lane-parallel into
// shared memory, are ready before they are needed) and walks a flat sequence of
// stages across items, so the ring keeps streaming through item boundaries.  Everything the consumers need about an
// item travels in the stage descriptor (no global loads on their side).
struct StageMeta {
  int item;  // -1: no more work
  int rr;    // round within the item
  int np;    // pages in this stage (0: empty split)
  int last;  // last round of the item
  int row, kvh, z;
  int L;      // context length (pos + 1)
  int begin;  // first page of this item's split
  int pad_[3];
};

struct AttnItem {
  int item, row, kvh, z, slot, L, begin, end, nr, rr;
};

VOX_DEV void attn_item_decode(int item, int n_kv, int n_split, int& r, int& kvh, int& z) {
  z = item % n_split;
  const int t = item / n_split;
  kvh = t % n_kv;
  r = t / n_kv;
}

template <int NW>
VOX_DEV void named_bar_consumers() { asm volatile("bar.sync 1, %0;" ::"n"(32 * NW) : "memory"); }

template <int HD>
__host__ __device__ constexpr int attn_threads() {
  return 32 * (attn_warps<HD>() + 1);
}
constexpr int kAttnItemPages = 64;  // page ids staged per item (1024 tokens at ps 16)

template <int HD, int G>
__global__ void __launch_bounds__(attn_threads<HD>(), 2)
    attn_decode_kernel(const RowDev* __restrict__ rows, const bf16* __restrict__ q,
                       const bf16* __restrict__ kc, const bf16* __restrict__ vc,
                       const int* __restrict__ page_table, LmDims dm, bf16* __restrict__ out,
                       float* __restrict__ ws, int n_split, int n_items, int* __restrict__ sched) {
  VOX_TRACE(kTrAttn);
  static_assert(G <= 8, "GQA group must fit the mma row tile");
  constexpr int NB = HD / 32;  // 32-dim blocks (2 k-blocks each)
  constexpr int NT = HD / 8;   // PV n-tiles
  constexpr int kP = attn_warps<HD>();
  constexpr int NW = kP;  // consumer warps
  constexpr int kQBytes = G * HD * 2;
  constexpr int kAttnStages = attn_stages<HD>();
  extern __shared__ __align__(128) uint8_t stage_raw[];
  __shared__ uint64_t full[kAttnStages], empty[kAttnStages];
  __shared__ __align__(16) StageMeta meta[kAttnStages];
  __shared__ float s_m[NW][G], s_l[NW][G];
  __shared__ __align__(16) float s_acc[NW][G][HD];
  __shared__ int s_pt[2][kAttnItemPages];

  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int ps = dm.page_size;
  const int page_elems = ps * HD;
  const int stage_bytes = attn_stage_bytes<HD>(ps);

  if (tid == 0) {
    for (int s = 0; s < kAttnStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NW);
    }
    fence_mbar_init();
  }
  __syncthreads();
  auto stage_ptr = [&](int s, int jp, int kv) -> bf16* {
    return reinterpret_cast<bf16*>(stage_raw + static_cast<size_t>(s) * stage_bytes) +
           (jp * 2 + kv) * page_elems;
  };
  auto q_slot = [&](int s) -> bf16* {
    return reinterpret_cast<bf16*>(stage_raw + static_cast<size_t>(kAttnStages) * stage_bytes +
                                   static_cast<size_t>(s) * kAttnQSlot);
  };

  if (warp == NW) {
    // ====================== producer warp ======================
    // The counter is zeroed by the last CTA of the previous launch; every kernel
    // between two attention launches does griddep_wait before griddep_launch,
    // so the previous attention grid has completed when this one starts.
    const uint64_t pol = policy_evict_first();  // K/V are read once per step
    auto fetch = [&](AttnItem& it, int buf) {
      int v[9] = {-1, 0, 0, 0, 0, 0, 0, 0, 0};
      if (lane == 0) {
        for (;;) {
          const int idx = atomicAdd(&sched[0], 1);
          if (idx >= n_items) break;
          int r, kvh, z;
          attn_item_decode(idx, dm.n_kv, n_split, r, kvh, z);
          r = rows[r].attn_row;  // longest contexts first
          const RowDev rw = rows[r];
          if (rw.slot < 0) continue;  // bucket padding
          const int n_pages = (rw.pos + 1 + ps - 1) / ps;
          const int pps = (n_pages + n_split - 1) / n_split;
          const int b = min(n_pages, z * pps);
          const int e = min(n_pages, b + pps);
          v[0] = idx; v[1] = r; v[2] = kvh; v[3] = z; v[4] = rw.slot; v[5] = rw.pos + 1;
          v[6] = b; v[7] = e; v[8] = max(1, (e - b + kP - 1) / kP);
          break;
        }
      }
#pragma unroll
      for (int k = 0; k < 9; ++k) v[k] = __shfl_sync(0xffffffffu, v[k], 0);
      it = AttnItem{v[0], v[1], v[2], v[3], v[4], v[5], v[6], v[7], v[8], 0};
      if (it.item >= 0) {
        const int* pt = page_table + static_cast<int64_t>(it.slot) * dm.max_pages_per_slot + it.begin;
        const int n = min(it.end - it.begin, kAttnItemPages);
        for (int i = lane; i < n; i += 32) s_pt[buf][i] = pt[i];
      }
      __syncwarp();
    };
    AttnItem cur, nxt;
    int buf = 0;
    // Look one item ahead (the ring streams through item boundaries) when there are
    // more items than CTAs; with at most one item per CTA a look-ahead claim lets
    // early CTAs hoard a second item while late ones get none (128 rows x 2 kv
    // heads: half the CTAs did two items, half none), so each CTA then claims its
    // next item only as cur's last stage goes out (finding none).  A mixed policy
    // (look-ahead until fewer items than CTAs remain) measured slower at 64-224 rows.
    const bool ahead = n_items > static_cast<int>(gridDim.x);
    bool have_nxt = false;
    fetch(cur, 0);
    if (ahead) {
      fetch(nxt, 1);
      have_nxt = true;
    }
    // issue the next stage of `cur` into slot s (q optionally deferred)
    auto issue = [&](int s, bool with_q) {
      if (cur.item < 0) {
        if (lane == 0) {
          meta[s] = StageMeta{-1, 0, 0, 0, 0, 0, 0, 0, 0, {0, 0, 0}};
          mbar_arrive(&full[s]);  // terminator: completes the phase without data
        }
        return;
      }
      const int pa = cur.begin + cur.rr * kP;
      const int np = max(0, min(kP, cur.end - pa));
      if (lane == 0) {
        meta[s] = StageMeta{cur.item, cur.rr, np, cur.rr == cur.nr - 1, cur.row, cur.kvh, cur.z,
                            cur.L, cur.begin, {cur.end, 0, 0}};
        const uint32_t q_bytes = cur.rr == 0 ? kQBytes : 0u;
        mbar_arrive_expect_tx(&full[s], static_cast<uint32_t>(np * 2 * page_elems * 2) + q_bytes);
      }
      __syncwarp();
      // lanes 0..np-1 copy K pages, lanes 4..4+np-1 the matching V pages, lane 8 q
      if (lane < 2 * kP && (lane & (kP - 1)) < np) {
        const int jp = lane & (kP - 1), kv = lane / kP;
        const int off = pa - cur.begin + jp;
        const int pid = off < kAttnItemPages
                            ? s_pt[buf][off]
                            : page_table[static_cast<int64_t>(cur.slot) * dm.max_pages_per_slot + pa + jp];
        const int64_t base = (static_cast<int64_t>(pid) * dm.n_kv + cur.kvh) * page_elems;
        bulk_load(stage_ptr(s, jp, kv), (kv ? vc : kc) + base, page_elems * 2, &full[s], pol);
      } else if (lane == 2 * kP && cur.rr == 0 && with_q) {
        bulk_load(q_slot(s), q + (static_cast<int64_t>(cur.row) * dm.n_heads + cur.kvh * G) * HD,
                  kQBytes, &full[s], pol);
      }
      __syncwarp();
      if (!have_nxt && cur.rr == cur.nr - 1) {
        fetch(nxt, buf ^ 1);
        have_nxt = true;
      }
      if (++cur.rr == cur.nr) {
        cur = nxt;
        buf ^= 1;
        have_nxt = false;
        if (ahead) {
          fetch(nxt, buf ^ 1);
          have_nxt = true;
        }
      }
    };
    // ---- prologue: stages of the first item whose pages all precede the first
    // page this forward appends to (RowDev::fresh; written by the preceding
    // kernel) go out before griddep_wait; q (written by it) after it.
    int g = 0, deferred_q = -1;
    if (cur.item >= 0) {
      const int fresh_page = rows[cur.row].fresh / ps;
      const int first = cur.item;
      while (g < kAttnStages && cur.item == first) {
        const int pa = cur.begin + cur.rr * kP;
        const int np = max(0, min(kP, cur.end - pa));
        if (np == 0 || pa + np > fresh_page) break;
        if (cur.rr == 0) deferred_q = g;
        issue(g++, false);
      }
    }
    griddep_wait();
    griddep_launch();
    if (deferred_q >= 0 && lane == 0) {
      const StageMeta m = meta[deferred_q];
      bulk_load(q_slot(deferred_q), q + (static_cast<int64_t>(m.row) * dm.n_heads + m.kvh * G) * HD,
                kQBytes, &full[deferred_q], pol);
    }
    for (;; ++g) {
      const int s = g % kAttnStages;
      if (g >= kAttnStages) mbar_wait(&empty[s], ((g / kAttnStages) - 1) & 1);
      const bool done = cur.item < 0;
      issue(s, true);
      if (done) break;
    }
  } else {
    // ====================== consumer warps 0..NW-1 ======================
    griddep_wait();
    griddep_launch();
    const int gn = lane >> 2, j = lane & 3;  // mma row/col group, k-slot group
    const float qscale = 1.4426950408889634f / sqrtf(static_cast<float>(HD));
    uint4 qa[NB];
    float mrow = -INFINITY, lrow = 0.f;  // head gn, lane-partial l
    float acc[NT][4];
    for (int g = 0;; ++g) {
      const int s = g % kAttnStages;
      mbar_wait(&full[s], (g / kAttnStages) & 1);
      const StageMeta m = meta[s];
      if (m.item < 0) break;
      if (m.rr == 0) {  // new item: q from the stage, reset the online softmax
        const bf16* qs = q_slot(s);
#pragma unroll
        for (int mb = 0; mb < NB; ++mb)
          qa[mb] = gn < G ? *reinterpret_cast<const uint4*>(qs + gn * HD + 32 * mb + 8 * j)
                          : make_uint4(0u, 0u, 0u, 0u);
        mrow = -INFINITY;
        lrow = 0.f;
#pragma unroll
        for (int t = 0; t < NT; ++t) acc[t][0] = acc[t][1] = acc[t][2] = acc[t][3] = 0.f;
      }
      if (warp < m.np) {
        const int page_idx = m.begin + m.rr * kP + warp;
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
          for (int mb = 0; mb < NB; ++mb) {
            const uint4 ku = odd ? kb[mb ^ 1] : kb[mb];
            mma_bf16_16816(sacc[t], qa[mb].x, qa[mb].y, ku.x, ku.y);
            mma_bf16_16816(sacc[t], qa[mb].z, qa[mb].w, ku.z, ku.w);
          }
        }
        // lane j owns tokens 4j..4j+3 of row gn: (sacc[0][0], sacc[0][1], sacc[1][0], sacc[1][1])
        const int tok0 = page_idx * ps + 4 * j;
        float sv[4] = {sacc[0][0] * qscale, sacc[0][1] * qscale, sacc[1][0] * qscale,
                       sacc[1][1] * qscale};
#pragma unroll
        for (int e = 0; e < 4; ++e)
          if (tok0 + e >= m.L) sv[e] = -INFINITY;
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
      if (m.last) {
        // ---------------- finalize the item: merge the 4 warps ----------------
        float lr = lrow;
        lr += __shfl_xor_sync(0xffffffffu, lr, 1);
        lr += __shfl_xor_sync(0xffffffffu, lr, 2);
        if (gn < G) {
          if (j == 0) {
            s_m[warp][gn] = mrow;
            s_l[warp][gn] = lr;
          }
#pragma unroll
          for (int t = 0; t < NT; ++t) {
            s_acc[warp][gn][8 * t + 2 * j] = acc[t][0];
            s_acc[warp][gn][8 * t + 2 * j + 1] = acc[t][1];
          }
        }
        named_bar_consumers<NW>();
        for (int idx = tid; idx < G * HD; idx += 32 * NW) {
          const int gg = idx / HD, dd = idx % HD;
          float M = -INFINITY;
#pragma unroll
          for (int w = 0; w < NW; ++w) M = fmaxf(M, s_m[w][gg]);
          float Ls = 0.f, A = 0.f;
#pragma unroll
          for (int w = 0; w < NW; ++w) {
            const float f = (s_m[w][gg] == -INFINITY) ? 0.f : exp2f(s_m[w][gg] - M);
            Ls += s_l[w][gg] * f;
            A += s_acc[w][gg][dd] * f;
          }
          if (n_split == 1) {
            out[(static_cast<int64_t>(m.row) * dm.n_heads + m.kvh * G + gg) * HD + dd] =
                __float2bfloat16_rn(A / Ls);
          } else {
            float* wp =
                ws + ((static_cast<int64_t>(m.row) * dm.n_kv + m.kvh) * n_split + m.z) * G * (HD + 2);
            wp[gg * (HD + 2) + dd] = A;
            if (dd == 0) {
              wp[gg * (HD + 2) + HD] = M;
              wp[gg * (HD + 2) + HD + 1] = Ls;
            }
          }
        }
        named_bar_consumers<NW>();  // s_acc / s_m / s_l are reused by the next item
      }
    }
  }
  // self-resetting scheduler: the last CTA to finish zeroes the counters
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    if (atomicAdd(&sched[1], 1) == static_cast<int>(gridDim.x) - 1) {
      sched[0] = 0;
      sched[1] = 0;
      __threadfence();
    }
  }
}

template <int HD, int G>
__global__ void __launch_bounds__(128)
    attn_combine_kernel(const RowDev* __restrict__ rows, const float* __restrict__ ws, LmDims dm,
                        int n_split, bf16* __restrict__ out) {
  VOX_TRACE(kTrAttnCombine);
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
                        int* sched, cudaStream_t st) {
  // K/V ring + one q slot per stage (96 KB + 3 KB at ps 16, hd 128): 2 CTAs per SM
  const int smem = attn_stages<HD>() * (attn_stage_bytes<HD>(dm.page_size) + kAttnQSlot);
  static int attr_bytes = 0;
  if (smem > attr_bytes) {
    cudaFuncSetAttribute(attn_decode_kernel<HD, G>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         smem);
    attr_bytes = smem;
  }
  const int n_items = n * dm.n_kv * n_split;
  const int sms = vox_sm_budget();
  const int grid = n_items < 2 * sms ? n_items : 2 * sms;
  // (merging the splits in the last split's CTA instead of a combine launch, and L2
  // prefetch of pages beyond the smem ring, both measured slower and were removed:
  // DESIGN.md section 9)
  launch_k(attn_decode_kernel<HD, G>, dim3(grid), dim3(attn_threads<HD>()), smem, st, rows, q, kc, vc, pt, dm,
           out, ws, n_split, n_items, sched);
  if (n_split > 1)
    launch_k(attn_combine_kernel<HD, G>, dim3(n, dm.n_kv), dim3(128), 0, st, rows, ws, dm, n_split,
             out);
}

template <int HD>
static void attn_dispatch_g(const RowDev* rows, int n, const bf16* q, const bf16* kc,
                            const bf16* vc, const int* pt, const LmDims& dm, bf16* out, float* ws,
                            int n_split, int* sched, cudaStream_t st) {
  switch (dm.n_heads / dm.n_kv) {
    case 1: attn_launch<HD, 1>(rows, n, q, kc, vc, pt, dm, out, ws, n_split, sched, st); break;
    case 2: attn_launch<HD, 2>(rows, n, q, kc, vc, pt, dm, out, ws, n_split, sched, st); break;
    case 3: attn_launch<HD, 3>(rows, n, q, kc, vc, pt, dm, out, ws, n_split, sched, st); break;
    case 4: attn_launch<HD, 4>(rows, n, q, kc, vc, pt, dm, out, ws, n_split, sched, st); break;
    default:
      if constexpr (HD == 64) {  // wider GQA groups (Qwen2.5-0.5B: 14 q / 2 kv heads)
        switch (dm.n_heads / dm.n_kv) {
          case 5: attn_launch<HD, 5>(rows, n, q, kc, vc, pt, dm, out, ws, n_split, sched, st); break;
          case 6: attn_launch<HD, 6>(rows, n, q, kc, vc, pt, dm, out, ws, n_split, sched, st); break;
          case 7: attn_launch<HD, 7>(rows, n, q, kc, vc, pt, dm, out, ws, n_split, sched, st); break;
          case 8: attn_launch<HD, 8>(rows, n, q, kc, vc, pt, dm, out, ws, n_split, sched, st); break;
          default: break;  // rejected at vox_create
        }
      }
      break;
  }
}

// Split-KV (+ a combine launch) only pays for long contexts: at the contexts of
// these serving configs (<= 768 tokens) one item per (row, kv head) is faster at
// every batch size (traced decode step: B=1 2.01 -> 1.92 ms, B=16 2.13 -> 1.99 ms
// unsplit; CosyVoice2 LM at 128 rows 1.38 -> 1.19 ms), so split only when
// contexts can exceed 1024 tokens and the items leave half the CTA slots idle.
int attn_pick_splits(int n_rows, int n_kv, int max_ctx) {
  if (const char* e = getenv("VOX_ATTN_SPLITS_TEST")) {  // debug; the partials workspace holds
    const int f = atoi(e) < 1 ? 1 : (atoi(e) > kAttnMaxSplits ? kAttnMaxSplits : atoi(e));  // kAttnSplitRows
    return n_rows > kAttnSplitRows ? 1 : f;
  }
  if (max_ctx < 1024) return 1;
  const int ctas = n_rows * n_kv;
  int s = (2 * vox_sm_budget()) / ctas;
  if (s > kAttnMaxSplits) s = kAttnMaxSplits;
  if (n_rows > kAttnSplitRows) s = 1;
  return s < 1 ? 1 : s;
}

void launch_attn_decode(const RowDev* rows, int n, const bf16* q, const bf16* kc, const bf16* vc,
                        const int* page_table, const LmDims& dm, bf16* out, float* ws, int n_split,
                        int* sched, cudaStream_t st) {
  if (dm.hd == 64)
    attn_dispatch_g<64>(rows, n, q, kc, vc, page_table, dm, out, ws, n_split, sched, st);
  else
    attn_dispatch_g<128>(rows, n, q, kc, vc, page_table, dm, out, ws, n_split, sched, st);
}

}  // namespace vox
