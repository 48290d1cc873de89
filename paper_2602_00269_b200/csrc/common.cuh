// common.cuh — shared device helpers for the sm_100a kernels.
#pragma once
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#define VOX_DEV __device__ __forceinline__

namespace vox {

constexpr int kNumSMs = 148;

// ---------------------------------------------------------------------------
// splitmix64 — the reference's counter mixer (model_api.py:39-51).  Used for
// seeded random-init weights, synthetic prompt ids and the per-request
// sampling RNG so CPU oracle and GPU agree bit-for-bit on inputs.
// ---------------------------------------------------------------------------
constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ull;

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x += kGolden;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

// per-tensor init key (oracle/weights.py:tensor_key mirrors this)
__host__ __device__ __forceinline__ uint64_t tensor_key(uint64_t seed, uint64_t tid,
                                                        uint64_t layer) {
  return mix64(mix64(seed ^ (tid * 0xD1B54A32D192ED03ull)) ^ (layer * 0x8CB92BA72F3D8DD7ull));
}

// uniform in [-1, 1) with 24 random bits: exact in fp32 on both sides.
__host__ __device__ __forceinline__ float unit_pm1(uint64_t h) {
  return (float)(int32_t)(h >> 40) * (1.0f / 8388608.0f) - 1.0f;
}

// uniform in (0, 1) with 24 bits, never 0 (for -log(u)).
VOX_DEV float unit_open01(uint64_t h) {
  return ((float)(uint32_t)(h >> 40) + 0.5f) * (1.0f / 16777216.0f);
}

// sin(x) for the Snake activations: one Cody-Waite reduction to [-pi, pi]
// (two FMAs with a split 2*pi) and the SFU sine.  Absolute error ~1e-6 for
// |x| < 1e4 (vs ~2 ulp for libdevice sinf at ~8x the instruction count); far
// below the bf16 rounding of the GEMM operands that follow.
VOX_DEV float snake_sin(float x) {
  const float k = rintf(x * 0.15915494309189535f);
  float r = fmaf(-k, 6.28318548202514648f, x);
  r = fmaf(-k, -1.7484556e-07f, r);
  return __sinf(r);
}

VOX_DEV float bf16_to_f32(__nv_bfloat16 v) { return __bfloat162float(v); }
VOX_DEV __nv_bfloat16 f32_to_bf16(float v) { return __float2bfloat16_rn(v); }

VOX_DEV float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
VOX_DEV float warp_max(float v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// ---------------------------------------------------------------------------
// mbarrier / TMA / tcgen05 PTX wrappers (sm_100a)
// ---------------------------------------------------------------------------
VOX_DEV uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

VOX_DEV void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
VOX_DEV void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
VOX_DEV void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

VOX_DEV void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
VOX_DEV void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
VOX_DEV void mbar_wait(uint64_t* bar, uint32_t parity) {
  uint32_t addr = smem_u32(bar);
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(addr),
      "r"(parity)
      : "memory");
}

// 2D TMA tile load into shared memory, completion on an mbarrier, with an L2
// cache-policy hint (evict-first for streamed weights, evict-last for reused
// activations).
VOX_DEV void tma_load_2d(void* dst, const CUtensorMap* map, uint64_t* bar, int x, int y,
                         uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_"
      "hint [%0], [%1, {%2, %3}], [%4], %5;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(x), "r"(y), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
// 1-D bulk copy global -> shared (no tensor map), completion on an mbarrier.
// bytes % 16 == 0, both addresses 16-byte aligned.
VOX_DEV void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
      "[%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(src)), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}
// Bulk prefetch of global memory into L2 (no shared memory, no completion).
VOX_DEV void prefetch_l2_bulk(const void* src, uint32_t bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(reinterpret_cast<uint64_t>(src)),
               "r"(bytes)
               : "memory");
}
VOX_DEV void tma_prefetch_desc(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(map)) : "memory");
}
VOX_DEV uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
VOX_DEV uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// TMEM allocation (one warp), power-of-two columns >= 32.
VOX_DEV void tmem_alloc(uint32_t* dst_smem, uint32_t ncols) {
  asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                   smem_u32(dst_smem)),
               "r"(ncols));
  asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
}
VOX_DEV void tmem_dealloc(uint32_t taddr, uint32_t ncols) {
  asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(taddr), "r"(ncols));
}
VOX_DEV void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
VOX_DEV void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// D[tmem] (+)= A[smem] * B[smem]^T, bf16 inputs, fp32 accumulate, 1 CTA.
VOX_DEV void umma_bf16(uint32_t tmem_d, uint64_t desc_a, uint64_t desc_b, uint32_t idesc,
                       uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(desc_a), "l"(desc_b), "r"(idesc), "r"(accumulate));
}
// Arrive on an mbarrier when all previously issued tcgen05.mma have completed.
VOX_DEV void umma_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(bar))
      : "memory");
}

// K-major, 128B-swizzled shared-memory matrix descriptor (sm100 format):
// start>>4 in [0,14), LBO (unused for swizzled K-major, 1) in [16,30),
// SBO = 1024B (8 rows x 128B) in [32,46), version 1 at bit 46,
// layout SWIZZLE_128B (2) in [61,64).
VOX_DEV uint64_t make_desc_k128(uint32_t smem_addr) {
  uint64_t d = 0;
  d |= (uint64_t)((smem_addr >> 4) & 0x3FFF);
  d |= (uint64_t)1 << 16;
  d |= (uint64_t)(1024 >> 4) << 32;
  d |= (uint64_t)1 << 46;
  d |= (uint64_t)2 << 61;
  return d;
}

// Instruction descriptor: kind::f16, A=B=bf16, D=f32, both K-major.
__host__ __device__ constexpr uint32_t make_idesc_bf16(int M, int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) |
         ((uint32_t)(M >> 4) << 24);
}

// TMEM -> registers: 32 lanes x 32 columns (thread i gets lane base+i).
VOX_DEV void tmem_ld_32x32b_x32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
}
VOX_DEV void tmem_ld_wait() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// Programmatic dependent launch: wait for the preceding grid's completion
// (and memory flush) / allow the next grid to start its prologue.
VOX_DEV void griddep_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
VOX_DEV void griddep_launch() { asm volatile("griddepcontrol.launch_dependents;" :::); }

VOX_DEV bool elect_one() {
  uint32_t pred = 0;
  asm volatile(
      "{\n"
      ".reg .pred P;\n"
      "elect.sync _|P, 0xffffffff;\n"
      "selp.b32 %0, 1, 0, P;\n"
      "}\n"
      : "=r"(pred));
  return pred != 0;
}


// ---------------------------------------------------------------------------
// In-graph kernel tracer (diagnostics, vox_trace_*): when a trace buffer is
// armed, thread 0 of every CTA of an instrumented kernel appends
// {tag, smid, globaltimer at CTA start, at CTA end}.  buf[0] is the record
// counter, records start at buf[2].  One pointer per translation unit
// (no relocatable device code); off = one predicated global load per CTA.
// ---------------------------------------------------------------------------
struct TraceRec {
  uint32_t tag, smid;
  unsigned long long t0, t1;
};
#define VOX_TRACE_TU(setter)                                                              \
  static __device__ unsigned long long* g_vox_trace = nullptr;                            \
  void setter(unsigned long long* buf) {                                                  \
    cudaMemcpyToSymbol(g_vox_trace, &buf, sizeof(buf));                                    \
  }
VOX_DEV unsigned long long vox_now() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
struct TraceScope {
  unsigned long long* buf;
  unsigned long long t0;
  uint32_t tag;
  // tag | (CTAs in the grid << 8): separates back-to-back launches of one kernel
  __device__ __forceinline__ TraceScope(unsigned long long* b, uint32_t tg)
      : buf(b), t0(0), tag(tg | ((gridDim.x * gridDim.y * gridDim.z) << 8)) {
    if (buf != nullptr && threadIdx.x == 0) t0 = vox_now();
  }
  __device__ __forceinline__ ~TraceScope() {
    if (buf != nullptr && threadIdx.x == 0) {
      const unsigned long long t1 = vox_now();
      const unsigned long long i = atomicAdd(buf, 1ull);
      if (i < buf[1]) {
        uint32_t sm;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
        TraceRec* r = reinterpret_cast<TraceRec*>(buf + 2) + i;
        r->tag = tag;
        r->smid = sm;
        r->t0 = t0;
        r->t1 = t1;
      }
    }
  }
};
#define VOX_TRACE(tag) TraceScope vox_trace_scope_(g_vox_trace, (tag))
enum TraceTag : uint32_t {
  kTrGemm = 1, kTrGemmMc = 2, kTrAttn = 3, kTrAttnCombine = 4, kTrQkvRope = 5, kTrResidNorm = 6,
  kTrEmbedNorm = 7, kTrSilu = 8, kTrSampler = 9, kTrDetok = 10, kTrChain = 11
};

}  // namespace vox
