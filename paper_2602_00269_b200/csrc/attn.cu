// attn.cu — K2: paged GQA decode attention (HBM-bound) + split-KV combine.
//
// One CTA (4 warps) per (row, kv head, kv split).  The G = H/KV query heads
// that share a kv head are processed together, so every K/V byte is read from
// HBM exactly once per step.  A warp consumes chunks of 8 tokens (a chunk
// never straddles a page since page_size % 8 == 0), two chunks per iteration
// so ~8 KB of K/V loads are in flight per warp:
//   * QK: 4 lanes per token, 4 x 16-byte K segments per lane (the warp reads
//     8 consecutive 256-byte token rows of the head-page = fully used
//     sectors); q is staged once in fp32 shared memory pre-scaled by
//     log2(e)/sqrt(hd) (segment offsets 32*i + 8*ks -> conflict-free LDS.128);
//     2 shuffles reduce the dot, 3 give the chunk max (online softmax, exp2);
//   * PV: lane owns hd/32 output dims for all 8 tokens (8-byte V loads, one
//     256-byte row per warp instruction); p is broadcast through 96 bytes of
//     per-warp shared memory instead of 24 shuffles.
// Low register count (no q / K-row register arrays) -> 4+ CTAs per SM.
// Small batches split the context across blockIdx.z (fixed split count per
// launch, so the step stays graph-capturable) and a combine pass merges the
// partial (m, l, acc) triples.
#include "common.cuh"
#include "kernels.h"

namespace vox {

template <int HD, int G>
__global__ void __launch_bounds__(128)
    attn_decode_kernel(const RowDev* __restrict__ rows, const bf16* __restrict__ q,
                       const bf16* __restrict__ kc, const bf16* __restrict__ vc,
                       const int* __restrict__ page_table, LmDims dm, bf16* __restrict__ out,
                       float* __restrict__ ws, int n_split) {
  griddep_wait();
  griddep_launch();
  constexpr int KSEG = HD / 32;  // 16-byte K segments per lane
  constexpr int VPL = HD / 32;   // output dims per lane
  __shared__ __align__(16) float s_q[G][HD];
  __shared__ __align__(16) float s_p[4][G][8];
  __shared__ float s_m[4][G], s_l[4][G];
  __shared__ __align__(16) float s_acc[4][G][HD];

  const int r = blockIdx.x, kvh = blockIdx.y, z = blockIdx.z;
  const RowDev rw = rows[r];
  if (rw.slot < 0) return;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int t8 = lane >> 2, ks = lane & 3;
  const int L = rw.pos + 1;
  const int n_chunks = (L + 7) >> 3;
  const int cps = (n_chunks + n_split - 1) / n_split;
  const int c_begin = z * cps;
  const int c_end = min(n_chunks, c_begin + cps);
  const float qscale = 1.4426950408889634f / sqrtf(static_cast<float>(HD));

  for (int i = tid; i < G * HD; i += 128)
    s_q[i / HD][i % HD] =
        __bfloat162float(q[(static_cast<int64_t>(r) * dm.n_heads + kvh * G + i / HD) * HD + i % HD]) *
        qscale;
  __syncthreads();

  float m[G], l[G], acc[G][VPL];
#pragma unroll
  for (int g = 0; g < G; ++g) {
    m[g] = -INFINITY;
    l[g] = 0.f;
#pragma unroll
    for (int d = 0; d < VPL; ++d) acc[g][d] = 0.f;
  }
  const int* pt = page_table + static_cast<int64_t>(rw.slot) * dm.max_pages_per_slot;
  const int ps = dm.page_size;
  const int64_t head_stride = static_cast<int64_t>(ps) * HD;  // elements per (page, head)

  auto chunk_base = [&](int c) -> int64_t {  // element offset of the chunk's first token row
    const int tok = c * 8;
    const int page = pt[tok / ps];
    return (static_cast<int64_t>(page) * dm.n_kv + kvh) * head_stride +
           static_cast<int64_t>(tok % ps) * HD;
  };

  for (int c0 = c_begin + warp; c0 < c_end; c0 += 8) {
    const int cB = c0 + 4;
    const bool hasB = cB < c_end;
    // ------------------------------------------------ loads (two chunks)
    uint4 kA[KSEG], kB[KSEG];
    uint2 vA[8], vB[8];
    {
      const int64_t bA = chunk_base(c0);
      const bf16* kp = kc + bA + t8 * HD + 8 * ks;
#pragma unroll
      for (int i = 0; i < KSEG; ++i) kA[i] = *reinterpret_cast<const uint4*>(kp + 32 * i);
      const bf16* vp = vc + bA + lane * VPL;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if constexpr (VPL == 4) vA[j] = *reinterpret_cast<const uint2*>(vp + j * HD);
        else vA[j] = make_uint2(*reinterpret_cast<const uint32_t*>(vp + j * HD), 0u);
      }
    }
    if (hasB) {
      const int64_t bB = chunk_base(cB);
      const bf16* kp = kc + bB + t8 * HD + 8 * ks;
#pragma unroll
      for (int i = 0; i < KSEG; ++i) kB[i] = *reinterpret_cast<const uint4*>(kp + 32 * i);
      const bf16* vp = vc + bB + lane * VPL;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if constexpr (VPL == 4) vB[j] = *reinterpret_cast<const uint2*>(vp + j * HD);
        else vB[j] = make_uint2(*reinterpret_cast<const uint32_t*>(vp + j * HD), 0u);
      }
    }
    // ------------------------------------------------ compute
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      if (half == 1 && !hasB) break;
      const int c = half ? cB : c0;
      const uint4* kk = half ? kB : kA;
      const uint2* vv = half ? vB : vA;
      const bool valid = c * 8 + t8 < L;
      float s[G];
#pragma unroll
      for (int g = 0; g < G; ++g) s[g] = 0.f;
#pragma unroll
      for (int i = 0; i < KSEG; ++i) {
        const bf16* kb = reinterpret_cast<const bf16*>(&kk[i]);
        float kf[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) kf[e] = __bfloat162float(kb[e]);
#pragma unroll
        for (int g = 0; g < G; ++g) {
          const float4 q0 = *reinterpret_cast<const float4*>(&s_q[g][32 * i + 8 * ks]);
          const float4 q1 = *reinterpret_cast<const float4*>(&s_q[g][32 * i + 8 * ks + 4]);
          s[g] = fmaf(q0.x, kf[0], s[g]);
          s[g] = fmaf(q0.y, kf[1], s[g]);
          s[g] = fmaf(q0.z, kf[2], s[g]);
          s[g] = fmaf(q0.w, kf[3], s[g]);
          s[g] = fmaf(q1.x, kf[4], s[g]);
          s[g] = fmaf(q1.y, kf[5], s[g]);
          s[g] = fmaf(q1.z, kf[6], s[g]);
          s[g] = fmaf(q1.w, kf[7], s[g]);
        }
      }
#pragma unroll
      for (int g = 0; g < G; ++g) {
        s[g] += __shfl_xor_sync(0xffffffffu, s[g], 1);
        s[g] += __shfl_xor_sync(0xffffffffu, s[g], 2);
        if (!valid) s[g] = -INFINITY;
        float cm = fmaxf(s[g], __shfl_xor_sync(0xffffffffu, s[g], 4));
        cm = fmaxf(cm, __shfl_xor_sync(0xffffffffu, cm, 8));
        cm = fmaxf(cm, __shfl_xor_sync(0xffffffffu, cm, 16));
        const float nm = fmaxf(m[g], cm);  // finite: token c*8 is always valid
        const float corr = exp2f(m[g] - nm);
        const float p = valid ? exp2f(s[g] - nm) : 0.f;
        if (ks == 0) s_p[warp][g][t8] = p;
        m[g] = nm;
        l[g] *= corr;
#pragma unroll
        for (int d = 0; d < VPL; ++d) acc[g][d] *= corr;
      }
      __syncwarp();
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const float4 p0 = *reinterpret_cast<const float4*>(&s_p[warp][g][0]);
        const float4 p1 = *reinterpret_cast<const float4*>(&s_p[warp][g][4]);
        const float pj[8] = {p0.x, p0.y, p0.z, p0.w, p1.x, p1.y, p1.z, p1.w};
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          l[g] += pj[j];
          const bf16* vb = reinterpret_cast<const bf16*>(&vv[j]);
#pragma unroll
          for (int d = 0; d < VPL; ++d) acc[g][d] = fmaf(pj[j], __bfloat162float(vb[d]), acc[g][d]);
        }
      }
      __syncwarp();
    }
  }
  // ------------------------------------------------ merge the 4 warps
#pragma unroll
  for (int g = 0; g < G; ++g) {
    if (lane == 0) {
      s_m[warp][g] = m[g];
      s_l[warp][g] = l[g];
    }
#pragma unroll
    for (int d = 0; d < VPL; ++d) s_acc[warp][g][lane * VPL + d] = acc[g][d];
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
  dim3 grid(n, dm.n_kv, n_split);
  launch_k(attn_decode_kernel<HD, G>, dim3(grid), dim3(128), 0, st, rows, q, kc, vc, pt, dm, out, ws, n_split);
  if (n_split > 1)
    launch_k(attn_combine_kernel<HD, G>, dim3(n, dm.n_kv), dim3(128), 0, st, rows, ws, dm, n_split, out);
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
  const int ctas = n_rows * n_kv;
  int s = (4 * kNumSMs + ctas - 1) / ctas;
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
