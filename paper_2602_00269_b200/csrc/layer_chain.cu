// layer_chain.cu — K6: the persistent per-layer decode chain (sm_100a).
//
// One launch runs everything of a decoder layer between two attention
// launches, as a list of jobs over ONE persistent grid (one CTA per SM):
//
//   O proj -> residual + RMSNorm -> gate|up (+ SiLU) -> down -> residual +
//   RMSNorm -> next layer's q|k|v proj -> q|k|v reduce + RoPE + KV append
//
// Why: at decode sizes every projection is a weight stream (6.2 GB per step at
// the Orpheus-3B shape) and the per-kernel design paid ~2.5 us first-data
// latency + ~2 us epilogue + ~1.5 us tail per GEMM launch plus two elementwise
// launches per layer (~78 us exposed per layer vs ~31 us of HBM time for its
// 200 MB of weights).  Here the weight stream never stops at a job boundary:
// weights do not depend on activations, so the producer keeps bulk-copying
// the NEXT units' weight tiles into a deep ring while the current job's
// epilogue, the grid-wide dependency and the row-wise norm/RoPE work finish.
//
// Warp roles (384 threads):
//   warp 0 lane 0   producer: claims GEMM units, streams weight k-blocks (1-D
//                   bulk copies of packed 16 KB tiles) as far ahead as the W
//                   ring allows, and activation k-blocks (TMA, 128B swizzle)
//                   once the unit's job dependency is met
//   warp 1 lane 0   MMA issuer: tcgen05.mma 128 x BN x 16 per k step into one
//                   of two TMEM accumulators (double-buffered across units)
//   warp 2          TMEM allocator
//   warps 4..11     epilogue + elementwise group (256 threads): TMEM -> fp32
//                   split planes or fused SiLU(gate)*up -> bf16; the norm and
//                   RoPE jobs (rows claimed dynamically)
//
// Work is CLAIMED (atomic counters per job), never statically assigned, so the
// chain completes even when not all of its CTAs are resident (another context's
// kernels on the same GPU): a unit is only ever waited for after a running CTA
// claimed it, and claims are taken in job order.  Completion counters (units or
// rows done) carry release/acquire ordering; TMA reads of generic-proxy writes
// are preceded by fence.proxy.async.global.  The last CTA to exit zeroes the
// launch's counters (one counter block per layer).
//
// Numerics are those of the per-kernel path: the same split-K factors and
// k-block rotation per tile (bit-identical fp32 planes), the reduction order of
// resid_norm_kernel at 256 threads and qkv_rope_append_kernel's per-element
// arithmetic, and the mc GEMM's SiLU epilogue.
#include "common.cuh"
#include "kernels.h"
#include "rownorm.cuh"
#include <cstdlib>

namespace vox {
VOX_TRACE_TU(trace_set_chain)

namespace {

constexpr int kQN = 8;            // unit queue depth (producer -> MMA / epilogue)
constexpr int kEpiThreads = 256;  // warps 4..11
constexpr int kThreads = 384;
constexpr int kParkBytes = 32768; // SiLU: gate + up of a 32-column chunk, per half group (2 x 16 KB)

VOX_DEV int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
VOX_DEV void red_release_add(int* p, int v) {
  asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
VOX_DEV bool mbar_test(uint64_t* bar, uint32_t parity) {
  uint32_t ok;
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n"
      "selp.u32 %0, 1, 0, p;\n"
      "}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
VOX_DEV void named_bar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
VOX_DEV void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }

// diagnostics (vox_trace armed): per-CTA event records {tag | cta << 8, smid, t0, t1}
// tag 32 + j: producer, job j's inputs ready (t0 = CTA entry); 40 + j: MMA of one
// unit of job j (first issue, last commit); 48 + j: epilogue of one unit / the
// CTA's rows of elementwise job j (start, signalled).  scripts/trace_chain.py
enum : uint32_t { kEvDep = 32, kEvMma = 40, kEvEpi = 48, kEvWait = 56 };
VOX_DEV void chain_mark(uint32_t ev, unsigned long long t0, unsigned long long t1) {
  unsigned long long* buf = g_vox_trace;
  if (buf == nullptr) return;
  const unsigned long long i = atomicAdd(buf, 1ull);
  if (i < buf[1]) {
    uint32_t sm;
    asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
    TraceRec* r = reinterpret_cast<TraceRec*>(buf + 2) + i;
    r->tag = ev | (blockIdx.x << 8);
    r->smid = sm;
    r->t0 = t0;
    r->t1 = t1;
  }
}

// a claimed GEMM unit: weight tile and k-block range (the mc kernel's rotation)
struct Unit {
  int job, tile, split, kb0, nkb, krot;
};
VOX_DEV Unit decode_unit(const ChainJob& j, int ji, int u, int k_rotate) {
  Unit x;
  x.job = ji;
  x.tile = u % j.m_tiles;
  x.split = u / j.m_tiles;
  x.kb0 = x.split * j.kb_per_split;
  x.nkb = min(j.n_kb, x.kb0 + j.kb_per_split) - x.kb0;
  x.krot = k_rotate ? static_cast<int>((static_cast<unsigned>(x.tile) * 7u) % static_cast<unsigned>(x.nkb)) : 0;
  return x;
}
VOX_DEV int unit_kb(const Unit& x, int i) {
  const int t = i + x.krot;
  return x.kb0 + (t >= x.nkb ? t - x.nkb : t);
}
VOX_DEV int job_units(const ChainArgs& a, int j) {
  return a.job[j].kind == kChGemm ? a.job[j].m_tiles * a.job[j].splits : a.nrows;
}

// ---- elementwise jobs (epilogue group, 256 threads, rows read through L2) ----
VOX_DEV float4 ldcg4(const float* p) { return __ldcg(reinterpret_cast<const float4*>(p)); }
// resid_norm_row at 256 threads (same accumulation and reduction order) for up
// to kPar rows at once: every row's loads are in flight together and the rows
// share one set of block barriers; each thread keeps its h values in registers
constexpr int kPar = 1;
constexpr int kMaxD4PerThread = 3;  // d <= 3072 (host: chain_bn_for_rows)
VOX_DEV void chain_norm_rows(const ChainJob& j, const RowDev* rows, int r0, int nr, int d, float eps,
                             int eg, float* red) {
  const int d4 = d / 4;
  float4 v[kPar][kMaxD4PerThread];
  float ss[kPar];
  bool live[kPar];
#pragma unroll
  for (int p = 0; p < kPar; ++p) {
    live[p] = p < nr && rows[r0 + p].slot >= 0;
    ss[p] = 0.f;
  }
  // split-major: every (row, k) load of one plane is in flight at once, so the
  // L2 round trips are one per plane (h rides with plane 0), not one per
  // (row, k, plane); the per-element sum order is still h + (p0 + p1 + ...)
  float4 hv[kPar][kMaxD4PerThread];
#pragma unroll
  for (int k = 0; k < kMaxD4PerThread; ++k) {
    const int i = eg + k * kEpiThreads;
#pragma unroll
    for (int p = 0; p < kPar; ++p) {
      if (live[p] && i < d4) {
        const int64_t ro = static_cast<int64_t>(r0 + p) * d;
        hv[p][k] = ldcg4(j.h + ro + 4 * i);
        v[p][k] = ldcg4(j.ws + ro + 4 * i);
      }
    }
  }
  for (int s = 1; s < j.nsplits; s += 2) {  // two planes per round trip
    const bool two = s + 1 < j.nsplits;
    float4 t[kPar][kMaxD4PerThread], u[kPar][kMaxD4PerThread];
#pragma unroll
    for (int k = 0; k < kMaxD4PerThread; ++k) {
      const int i = eg + k * kEpiThreads;
#pragma unroll
      for (int p = 0; p < kPar; ++p)
        if (live[p] && i < d4) {
          const float* src = j.ws + s * j.ss + static_cast<int64_t>(r0 + p) * d + 4 * i;
          t[p][k] = ldcg4(src);
          if (two) u[p][k] = ldcg4(src + j.ss);
        }
    }
#pragma unroll
    for (int k = 0; k < kMaxD4PerThread; ++k) {
      const int i = eg + k * kEpiThreads;
#pragma unroll
      for (int p = 0; p < kPar; ++p)
        if (live[p] && i < d4) {
          v[p][k] = add4(v[p][k], t[p][k]);
          if (two) v[p][k] = add4(v[p][k], u[p][k]);
        }
    }
  }
#pragma unroll
  for (int k = 0; k < kMaxD4PerThread; ++k) {
    const int i = eg + k * kEpiThreads;
#pragma unroll
    for (int p = 0; p < kPar; ++p)
      if (live[p] && i < d4) v[p][k] = add4(hv[p][k], v[p][k]);
  }
#pragma unroll
  for (int k = 0; k < kMaxD4PerThread; ++k) {
    const int i = eg + k * kEpiThreads;
#pragma unroll
    for (int p = 0; p < kPar; ++p) {
      if (live[p] && i < d4) {
        reinterpret_cast<float4*>(j.h + static_cast<int64_t>(r0 + p) * d)[i] = v[p][k];
        ss[p] = fmaf(v[p][k].x, v[p][k].x, ss[p]);
        ss[p] = fmaf(v[p][k].y, v[p][k].y, ss[p]);
        ss[p] = fmaf(v[p][k].z, v[p][k].z, ss[p]);
        ss[p] = fmaf(v[p][k].w, v[p][k].w, ss[p]);
      }
    }
  }
  const int w = eg >> 5, l = eg & 31;
#pragma unroll
  for (int p = 0; p < kPar; ++p) {
    ss[p] = warp_sum(ss[p]);
    if (l == 0) red[p * 8 + w] = ss[p];
  }
  named_bar(1, kEpiThreads);
  if (eg < 32) {
#pragma unroll
    for (int p = 0; p < kPar; ++p) {
      float t = (l < kEpiThreads / 32) ? red[p * 8 + l] : 0.f;
      t = warp_sum(t);
      if (l == 0) red[16 + p] = t;
    }
  }
  named_bar(1, kEpiThreads);
#pragma unroll
  for (int p = 0; p < kPar; ++p) ss[p] = red[16 + p];
  named_bar(1, kEpiThreads);  // red is reused by the next rows
  const float4* n4 = reinterpret_cast<const float4*>(j.nw);
#pragma unroll
  for (int p = 0; p < kPar; ++p) {
    if (!live[p]) continue;
    const int orow = j.out_index != nullptr ? j.out_index[r0 + p] : r0 + p;
    if (orow < 0) continue;
    const float inv = 1.0f / sqrtf(ss[p] / static_cast<float>(d) + eps);
    bf16* xr = j.x + static_cast<int64_t>(orow) * d;
#pragma unroll
    for (int k = 0; k < kMaxD4PerThread; ++k) {
      const int i = eg + k * kEpiThreads;
      if (i < d4) norm_store4(xr + 4 * i, v[p][k], inv, n4[i]);
    }
  }
}

// qkv_rope_append_kernel's per-element arithmetic for rows r0..r0+nr-1 at 256
// threads (the rows' items interleaved so all their loads are in flight)
VOX_DEV void chain_rope_rows(const ChainJob& j, const RowDev* rows, int r0, int nr, const LmDims& dm,
                             const float2* __restrict__ rope, int eg) {
  const int hd = dm.hd, half = hd / 2;
  const int nqkv = (dm.n_heads + 2 * dm.n_kv) * hd;
  const int q4 = half / 4;
  const int n_items = (dm.n_heads + dm.n_kv) * q4;
  // kRB items per thread per pass, their plane loads issued split-major (one L2
  // round trip per plane for all of them) together with the rope / page-table
  // loads; the per-element arithmetic is the per-kernel path's
  constexpr int kRB = 2;
  for (int t0 = eg; t0 < nr * n_items; t0 += kRB * kEpiThreads) {
    bool ok[kRB];
    float4 xa[kRB], xb[kRB];
    const float* pa[kRB];  // plane-0 address of the item's first half (second: + half)
#pragma unroll
    for (int m = 0; m < kRB; ++m) {
      const int t = t0 + m * kEpiThreads;
      ok[m] = t < nr * n_items;
      const int r = r0 + (ok[m] ? t / n_items : 0), it = ok[m] ? t % n_items : 0;
      ok[m] = ok[m] && rows[r].slot >= 0;
      pa[m] = j.ws + static_cast<int64_t>(r) * nqkv + (it / q4) * hd + (it % q4) * 4;
      if (ok[m]) {
        xa[m] = ldcg4(pa[m]);
        xb[m] = ldcg4(pa[m] + half);
      }
    }
    for (int s = 1; s < j.nsplits; ++s) {
      float4 ta[kRB], tb[kRB];
#pragma unroll
      for (int m = 0; m < kRB; ++m)
        if (ok[m]) {
          ta[m] = ldcg4(pa[m] + s * j.ss);
          tb[m] = ldcg4(pa[m] + s * j.ss + half);
        }
#pragma unroll
      for (int m = 0; m < kRB; ++m)
        if (ok[m]) {
          xa[m] = add4(xa[m], ta[m]);
          xb[m] = add4(xb[m], tb[m]);
        }
    }
#pragma unroll
    for (int m = 0; m < kRB; ++m) {
      if (!ok[m]) continue;
      const int t = t0 + m * kEpiThreads;
      const int r = r0 + t / n_items, it = t % n_items;
      const RowDev rw = rows[r];
      const int head = it / q4, i = (it % q4) * 4;
      const int c1 = (head * hd + i) / 4, c2 = (head * hd + i + half) / 4;
      float4 av = xa[m], bv = xb[m];
      if (j.bias != nullptr) {
        av = add4(av, reinterpret_cast<const float4*>(j.bias)[c1]);
        bv = add4(bv, reinterpret_cast<const float4*>(j.bias)[c2]);
      }
      const float2* rp = rope + static_cast<int64_t>(rw.pos) * half;
      const float x1[4] = {av.x, av.y, av.z, av.w}, x2[4] = {bv.x, bv.y, bv.z, bv.w};
      float o1[4], o2[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const float2 cs = rp[i + e];
        o1[e] = __fsub_rn(__fmul_rn(x1[e], cs.x), __fmul_rn(x2[e], cs.y));
        o2[e] = __fadd_rn(__fmul_rn(x2[e], cs.x), __fmul_rn(x1[e], cs.y));
      }
      bf16* dst;
      if (head < dm.n_heads) {
        dst = j.q + (static_cast<int64_t>(r) * dm.n_heads + head) * hd;
      } else {
        const int page = j.page_table[static_cast<int64_t>(rw.slot) * dm.max_pages_per_slot + rw.pos / dm.page_size];
        const int kvh = head - dm.n_heads;
        dst = j.kc + ((static_cast<int64_t>(page) * dm.n_kv + kvh) * dm.page_size + rw.pos % dm.page_size) * hd;
      }
      store_bf16x4(dst + i, o1[0], o1[1], o1[2], o1[3]);
      store_bf16x4(dst + i + half, o2[0], o2[1], o2[2], o2[3]);
    }
  }
  const int vbase4 = (dm.n_heads + dm.n_kv) * hd / 4;
  const int hd4 = hd / 4;
  const int nv = dm.n_kv * hd4;
  for (int t0 = eg; t0 < nr * nv; t0 += kRB * kEpiThreads) {
    bool ok[kRB];
    float4 xv[kRB];
    const float* wp[kRB];
#pragma unroll
    for (int m = 0; m < kRB; ++m) {
      const int t = t0 + m * kEpiThreads;
      ok[m] = t < nr * nv;
      const int r = r0 + (ok[m] ? t / nv : 0), e = ok[m] ? t % nv : 0;
      ok[m] = ok[m] && rows[r].slot >= 0;
      wp[m] = j.ws + static_cast<int64_t>(r) * nqkv + 4 * (vbase4 + e);
      if (ok[m]) xv[m] = ldcg4(wp[m]);
    }
    for (int s = 1; s < j.nsplits; ++s) {
      float4 tv[kRB];
#pragma unroll
      for (int m = 0; m < kRB; ++m)
        if (ok[m]) tv[m] = ldcg4(wp[m] + s * j.ss);
#pragma unroll
      for (int m = 0; m < kRB; ++m)
        if (ok[m]) xv[m] = add4(xv[m], tv[m]);
    }
#pragma unroll
    for (int m = 0; m < kRB; ++m) {
      if (!ok[m]) continue;
      const int t = t0 + m * kEpiThreads;
      const int e = t % nv;
      const RowDev rw = rows[r0 + t / nv];
      float4 v = xv[m];
      if (j.bias != nullptr) v = add4(v, reinterpret_cast<const float4*>(j.bias)[vbase4 + e]);
      const int page = j.page_table[static_cast<int64_t>(rw.slot) * dm.max_pages_per_slot + rw.pos / dm.page_size];
      const int kvh = e / hd4, dd = (e % hd4) * 4;
      bf16* vt = j.vc + ((static_cast<int64_t>(page) * dm.n_kv + kvh) * hd + dd) * dm.page_size + rw.pos % dm.page_size;
      vt[0] = __float2bfloat16_rn(v.x);
      vt[dm.page_size] = __float2bfloat16_rn(v.y);
      vt[2 * dm.page_size] = __float2bfloat16_rn(v.z);
      vt[3 * dm.page_size] = __float2bfloat16_rn(v.w);
    }
  }
}

}  // namespace

template <int BN>
struct ChainCfg {
  static constexpr int kWBytes = 128 * 64 * 2;  // one packed weight k-block
  static constexpr int kXBytes = BN * 64 * 2;   // one activation k-block (BN rows)
  static constexpr int kCols = BN <= 32 ? 32 : BN <= 64 ? 64 : BN <= 128 ? 128 : 256;
  static constexpr int kBarBytes = 1024;
  static int smem(int wst, int xst) { return 1024 + wst * kWBytes + xst * kXBytes + kParkBytes + kBarBytes; }
};

template <int BN>
__global__ void __launch_bounds__(kThreads, 1)
    layer_chain_kernel(const __grid_constant__ CUtensorMap mx0, const __grid_constant__ CUtensorMap mx1,
                       const __grid_constant__ CUtensorMap mx2, const __grid_constant__ ChainArgs a) {
  VOX_TRACE(kTrChain);
  using C = ChainCfg<BN>;
  const int WST = a.wst, XST = a.xst;  // ring depths (host: chain_smem_bytes)
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* wring = smem;
  uint8_t* xring = wring + WST * C::kWBytes;
  float* park = reinterpret_cast<float*>(xring + XST * C::kXBytes);
  uint64_t* bars = reinterpret_cast<uint64_t*>(reinterpret_cast<uint8_t*>(park) + kParkBytes);
  uint64_t* wfull = bars;
  uint64_t* wempty = wfull + WST;
  uint64_t* xfull = wempty + WST;
  uint64_t* xempty = xfull + XST;
  uint64_t* tfull = xempty + XST;
  uint64_t* tempty = tfull + 2;
  uint64_t* qfull = tempty + 2;
  uint64_t* qempty = qfull + kQN;
  int* qbuf = reinterpret_cast<int*>(qempty + kQN);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(qbuf + kQN);
  int* claim_bc = reinterpret_cast<int*>(tmem_slot + 1);
  float* red = reinterpret_cast<float*>(claim_bc + 1);  // 18 floats

  // one counter per 128-byte line: [j] claims, [8 + j] completions, [16] exits
  auto claim_ctr = [&](int j) { return a.ctr + j * kChainCtrStride; };
  auto done_ctr = [&](int j) { return a.ctr + (kChainMaxJobs + j) * kChainCtrStride; };
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const unsigned long long t_entry = vox_now();

  if (threadIdx.x == 0) {
    for (int s = 0; s < WST; ++s) { mbar_init(&wfull[s], 1); mbar_init(&wempty[s], 1); }
    for (int s = 0; s < XST; ++s) { mbar_init(&xfull[s], 1); mbar_init(&xempty[s], 1); }
    for (int b = 0; b < 2; ++b) { mbar_init(&tfull[b], 1); mbar_init(&tempty[b], 1); }
    // queue slot consumers: the producer's X cursor, the MMA issuer, 8 epilogue warps
    for (int s = 0; s < kQN; ++s) { mbar_init(&qfull[s], 1); mbar_init(&qempty[s], 10); }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc(tmem_slot, 2 * C::kCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ======================= W producer =======================
      // claims GEMM units in job order, publishes them to the queue, streams
      // their weight k-blocks (weights never wait for a job's inputs)
      const uint64_t pol_w = policy_evict_first();
      int wj = 0, wk = 0, wg = 0;
      for (;;) {
        int u = -1;
        while (wj < a.njobs) {
          if (a.job[wj].kind == kChGemm) {
            u = atomicAdd(claim_ctr(wj), 1);
            if (u < job_units(a, wj)) break;
          }
          ++wj;
        }
        const int qs = wk % kQN;
        if (wk >= kQN) mbar_wait(&qempty[qs], ((wk / kQN) - 1) & 1);
        qbuf[qs] = wj < a.njobs ? ((wj << 24) | u) : -1;
        mbar_arrive(&qfull[qs]);
        ++wk;
        if (wj >= a.njobs) break;
        const Unit wu = decode_unit(a.job[wj], wj, u, a.k_rotate);
        const bf16* wsrc = a.job[wj].w + static_cast<int64_t>(wu.tile) * a.job[wj].n_kb * 8192;
        for (int i = 0; i < wu.nkb; ++i, ++wg) {
          const int s = wg % WST;
          if (wg >= WST) mbar_wait(&wempty[s], ((wg / WST) - 1) & 1);
          mbar_arrive_expect_tx(&wfull[s], C::kWBytes);
          bulk_load(wring + s * C::kWBytes, wsrc + static_cast<int64_t>(unit_kb(wu, i)) * 8192, C::kWBytes,
                    &wfull[s], pol_w);
        }
      }
    }
    __syncwarp();
  } else if (warp == 3) {
    if (lane == 0) {
      // ======================= X producer =======================
      // follows the queue; a unit's activation k-blocks go out once its job's
      // inputs are complete (the preceding kernel, or an earlier job's counter)
      tma_prefetch_desc(&mx0);
      tma_prefetch_desc(&mx1);
      tma_prefetch_desc(&mx2);
      const uint64_t pol_x = policy_evict_last();
      int xg = 0, dep_ok_job = -1;
      bool gdw = false;
      for (int k = 0;; ++k) {
        const int qs = k % kQN;
        mbar_wait(&qfull[qs], (k / kQN) & 1);
        const int e = qbuf[qs];
        mbar_arrive(&qempty[qs]);
        if (e < 0) break;
        const int jj = e >> 24;
        const Unit xu = decode_unit(a.job[jj], jj, e & 0xFFFFFF, a.k_rotate);
        if (jj != dep_ok_job) {
          const int dj = a.job[jj].dep;
          if (dj < 0) {
            if (!gdw) griddep_wait();
            gdw = true;
          } else {
            const int need = job_units(a, dj);
            while (ld_acquire(done_ctr(dj)) < need) __nanosleep(64);
            fence_proxy_async_global();  // generic-proxy writes -> TMA reads
          }
          chain_mark(kEvDep + jj, t_entry, vox_now());
          dep_ok_job = jj;
        }
        const int m = a.job[jj].xmap;
        const CUtensorMap* xmap = m == 0 ? &mx0 : (m == 1 ? &mx1 : &mx2);
        for (int i = 0; i < xu.nkb; ++i, ++xg) {
          const int s = xg % XST;
          if (xg >= XST) mbar_wait(&xempty[s], ((xg / XST) - 1) & 1);
          mbar_arrive_expect_tx(&xfull[s], C::kXBytes);
          tma_load_2d(xring + s * C::kXBytes, xmap, &xfull[s], unit_kb(xu, i) * 64, 0, pol_x);
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {
      // ======================= MMA issuer =======================
      constexpr uint32_t idesc = make_idesc_bf16(128, BN);
      int k = 0, g = 0, uidx = 0;
      for (;;) {
        const int qs = k % kQN;
        mbar_wait(&qfull[qs], (k / kQN) & 1);
        const int e = qbuf[qs];
        mbar_arrive(&qempty[qs]);
        ++k;
        if (e < 0) break;
        const int jj = e >> 24;
        const Unit u = decode_unit(a.job[jj], jj, e & 0xFFFFFF, 0);
        const int b = uidx & 1;
        if (uidx >= 2) mbar_wait(&tempty[b], ((uidx >> 1) - 1) & 1);
        tc_fence_after();
        const uint32_t d = tmem + b * C::kCols;
        unsigned long long tm0 = 0, wait_w = 0, wait_x = 0;
        for (int i = 0; i < u.nkb; ++i, ++g) {
          const int sw = g % WST, sx = g % XST;
          const unsigned long long tw0 = vox_now();
          mbar_wait(&wfull[sw], (g / WST) & 1);
          const unsigned long long tw1 = vox_now();
          mbar_wait(&xfull[sx], (g / XST) & 1);
          const unsigned long long tw2 = vox_now();
          if (i > 0) { wait_w += tw1 - tw0; wait_x += tw2 - tw1; }
          tc_fence_after();
          if (i == 0) tm0 = vox_now();
          const uint32_t a_addr = smem_u32(wring + sw * C::kWBytes);
          const uint32_t b_addr = smem_u32(xring + sx * C::kXBytes);
#pragma unroll
          for (int kk = 0; kk < 4; ++kk)
            umma_bf16(d, make_desc_k128(a_addr + kk * 32), make_desc_k128(b_addr + kk * 32), idesc,
                      (i > 0 || kk > 0) ? 1u : 0u);
          umma_commit(&wempty[sw]);
          umma_commit(&xempty[sx]);
        }
        umma_commit(&tfull[b]);
        chain_mark(kEvMma + jj, tm0, vox_now());
        chain_mark(kEvWait + jj, tm0, (wait_w << 32) | (wait_x & 0xFFFFFFFFull));
        ++uidx;
      }
    }
    __syncwarp();
  } else if (warp >= 4) {
    // ======================= epilogue / elementwise group =======================
    const int eg = threadIdx.x - 128;
    const int q = warp & 3, hh = (warp - 4) >> 2;  // TMEM lane quarter, chunk parity
    griddep_wait();
    griddep_launch();
    int k = 0, uidx = 0, cur = 0;
    for (;;) {
      const int qs = k % kQN;
      mbar_wait(&qfull[qs], (k / kQN) & 1);
      const int e = qbuf[qs];
      __syncwarp();
      if (lane == 0) mbar_arrive(&qempty[qs]);
      ++k;
      const int jj = e < 0 ? a.njobs : (e >> 24);
      // elementwise jobs ordered before this unit's job
      for (; cur < jj; ++cur) {
        const ChainJob& ej = a.job[cur];
        if (ej.kind == kChGemm) continue;
        // claim the first rows before the inputs are ready (claims need no data)
        const int chunk = (a.nrows + gridDim.x - 1) / gridDim.x;
        if (eg == 0) {
          *claim_bc = atomicAdd(claim_ctr(cur), chunk);
          const int need = job_units(a, ej.dep);
          while (ld_acquire(done_ctr(ej.dep)) < need) __nanosleep(100);
        }
        named_bar(1, kEpiThreads);
        const unsigned long long te0 = vox_now();
        for (;;) {
          const int r0 = *claim_bc;
          named_bar(1, kEpiThreads);
          if (r0 >= a.nrows) break;
          const int r1 = min(a.nrows, r0 + chunk);
          if (ej.kind == kChNorm) {
            for (int r = r0; r < r1; r += kPar) chain_norm_rows(ej, a.rows, r, min(kPar, r1 - r), a.dm.d, a.dm.eps, eg, red);
          } else {
            chain_rope_rows(ej, a.rows, r0, r1 - r0, a.dm, a.rope, eg);
          }
          __threadfence();
          named_bar(1, kEpiThreads);
          if (eg == 0) {
            red_release_add(done_ctr(cur), r1 - r0);
            if (r1 < a.nrows) *claim_bc = atomicAdd(claim_ctr(cur), chunk);
          }
          if (r1 >= a.nrows) break;
          named_bar(1, kEpiThreads);
        }
        if (eg == 0) chain_mark(kEvEpi + cur, te0, vox_now());
      }
      if (e < 0) break;
      // ---- drain one GEMM unit
      const ChainJob& gj = a.job[jj];
      const Unit u = decode_unit(gj, jj, e & 0xFFFFFF, 0);
      const int b = uidx & 1;
      mbar_wait(&tfull[b], (uidx >> 1) & 1);
      tc_fence_after();
      const unsigned long long te0 = vox_now();
      const uint32_t tbase = tmem + (static_cast<uint32_t>(q * 32) << 16) + b * C::kCols;
      constexpr int kChunks = (BN + 31) / 32;
      const int nv = min(BN, a.nrows);
      const int m0 = u.tile * 128;
      if (gj.epi == 1) {
        // lanes 0-63 = gate, 64-127 = up of the tile's 64 features: the half's
        // four warps park gate and up of a 32-column chunk in smem, then each
        // warp forms bf16(SiLU(g) * u) for whole rows (2 features per lane ->
        // one 128-byte store per row), the mc epilogue's arithmetic
        float* pk = park + hh * (2 * 32 * 64);
        const int fo = (q & 1) * 32 + lane + (q >= 2 ? 32 * 64 : 0);
        __nv_bfloat162* act = reinterpret_cast<__nv_bfloat162*>(gj.act + (m0 / 128) * 64 + 2 * lane);
        const int64_t step2 = gj.ld_act / 2;
#pragma unroll 1
        for (int ch = hh; ch < kChunks; ch += 2) {
          uint32_t r[32];
          tmem_ld_32x32b_x32(tbase + ch * 32, r);
          tmem_ld_wait();
#pragma unroll
          for (int jx = 0; jx < 32; ++jx) pk[jx * 64 + fo] = __uint_as_float(r[jx]);
          named_bar(2 + hh, 128);
#pragma unroll 2
          for (int jx = q; jx < 32; jx += 4) {
            const int n = ch * 32 + jx;
            if (n < nv) {
              const float2 g = *reinterpret_cast<const float2*>(&pk[jx * 64 + 2 * lane]);
              const float2 uu = *reinterpret_cast<const float2*>(&pk[32 * 64 + jx * 64 + 2 * lane]);
              const float o0 = __fmul_rn(__fdiv_rn(g.x, __fadd_rn(1.0f, expf(-g.x))), uu.x);
              const float o1 = __fmul_rn(__fdiv_rn(g.y, __fadd_rn(1.0f, expf(-g.y))), uu.y);
              act[n * step2] = __floats2bfloat162_rn(o0, o1);
            }
          }
          named_bar(2 + hh, 128);
        }
      } else {
        const int m = m0 + q * 32 + lane;
        const bool mok = m < gj.m_valid;
        float* o = gj.out + static_cast<int64_t>(u.split) * gj.split_stride + m;
        const int64_t ldo = gj.ldo;
#pragma unroll 1
        for (int ch = hh; ch < kChunks; ch += 2) {
          uint32_t r[32];
          tmem_ld_32x32b_x32(tbase + ch * 32, r);
          tmem_ld_wait();
          if (!mok) continue;
          float* oc = o + static_cast<int64_t>(ch * 32) * ldo;
          const int lim = nv - ch * 32;
          if (lim >= 32) {
#pragma unroll
            for (int jx = 0; jx < 32; ++jx) { *oc = __uint_as_float(r[jx]); oc += ldo; }
          } else {
#pragma unroll
            for (int jx = 0; jx < 32; ++jx) { if (jx < lim) *oc = __uint_as_float(r[jx]); oc += ldo; }
          }
        }
      }
      tc_fence_before();
      __threadfence();
      named_bar(1, kEpiThreads);
      if (eg == 0) {
        mbar_arrive(&tempty[b]);
        red_release_add(done_ctr(jj), 1);
        chain_mark(kEvEpi + jj, te0, vox_now());
      }
      ++uidx;
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    tmem_dealloc(tmem, 2 * C::kCols);
  }
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(a.ctr + 2 * kChainMaxJobs * kChainCtrStride, 1) == static_cast<int>(gridDim.x) - 1) {
      for (int i = 0; i <= 2 * kChainMaxJobs; ++i) a.ctr[i * kChainCtrStride] = 0;
      __threadfence();
    }
  }
}

template <int BN>
static cudaError_t launch_chain_bn(const CUtensorMap& m0, const CUtensorMap& m1, const CUtensorMap& m2,
                                   const ChainArgs& a, cudaStream_t st) {
  using C = ChainCfg<BN>;
  static bool attr = false;
  if (!attr) {
    cudaError_t e = cudaFuncSetAttribute(layer_chain_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         227 * 1024);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const int smem = C::smem(a.wst, a.xst);
  if (smem > 227 * 1024 || a.wst < 2 || a.xst < 2 || a.wst > 16 || a.xst > 8) return cudaErrorInvalidValue;
  return launch_k(layer_chain_kernel<BN>, dim3(vox_sm_budget()), dim3(kThreads), smem, st, m0, m1, m2, a);
}

// ring depths for a tile width: X (activation, L2-resident) stages first, then as
// many 16 KB weight stages as fit (<= 16)
void chain_stages(int bn, int* wst, int* xst) {
  static const int xe = getenv("VOX_CHAIN_XST") ? atoi(getenv("VOX_CHAIN_XST")) : 0;
  int x = xe > 0 ? xe : (bn <= 128 ? 4 : 3);
  if (x > 8) x = 8;
  const int xb = bn * 128;
  int w = (227 * 1024 - 1024 - 1024 - kParkBytes - x * xb) / 16384;
  if (w > 16) w = 16;
  *wst = w;
  *xst = x;
}

bool chain_supported_bn(int bn) {
  switch (bn) {
    case 16: case 32: case 64: case 96: case 128: case 160: case 192: case 224: case 256: return true;
    default: return false;
  }
}

cudaError_t launch_layer_chain(const CUtensorMap& m0, const CUtensorMap& m1, const CUtensorMap& m2,
                               const ChainArgs& a, int bn, cudaStream_t st) {
  switch (bn) {
    case 16: return launch_chain_bn<16>(m0, m1, m2, a, st);
    case 32: return launch_chain_bn<32>(m0, m1, m2, a, st);
    case 64: return launch_chain_bn<64>(m0, m1, m2, a, st);
    case 96: return launch_chain_bn<96>(m0, m1, m2, a, st);
    case 128: return launch_chain_bn<128>(m0, m1, m2, a, st);
    case 160: return launch_chain_bn<160>(m0, m1, m2, a, st);
    case 192: return launch_chain_bn<192>(m0, m1, m2, a, st);
    case 224: return launch_chain_bn<224>(m0, m1, m2, a, st);
    case 256: return launch_chain_bn<256>(m0, m1, m2, a, st);
    default: return cudaErrorInvalidValue;
  }
}

}  // namespace vox
