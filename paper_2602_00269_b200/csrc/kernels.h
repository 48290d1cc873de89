// kernels.h — internal launcher declarations shared by the .cu translation units.
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/voxb200.h"

namespace vox {

using bf16 = __nv_bfloat16;

// Launch with programmatic stream serialization (PDL): the kernel may start
// while its predecessor drains; every kernel calls griddep_wait() before it
// touches data produced upstream.  Captured into CUDA graphs as programmatic
// dependency edges.
template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                            cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kernel, static_cast<KArgs>(args)...);
}

// ---------------------------------------------------------------- GEMM
struct GemmArgs {
  int M, N, K;            // out features, rows, reduction
  int n_kb, kb_per_split; // filled by gemm_launch
  float* out;             // fp32 output / split-K partials
  int64_t ldo;            // row stride of out (elements)
  int64_t split_stride;   // elements between split partial planes
  const float* bias;      // [M] or null (only with 1 split)
  const float* resid;     // [N, ldr] or null (only with 1 split)
  int64_t ldr;
  int m_valid;            // columns m >= m_valid are not stored
  int k_rotate;           // rotate each CTA's k-block order by its weight tile
  // epi == 1 (gate|up GEMM, 1 split, interleaved weight tiles): instead of fp32
  // out, write act[n][f] = bf16(SiLU(gate) * up) for the tile's 64 features
  int epi;
  bf16* act;
  int64_t ld_act;
  const bf16* x_packed;   // non-null: activations in the packed tile layout (bulk copies)
  int stages;             // mc kernel: smem ring depth (set by the launcher)
  unsigned long long* dbg; // gemm_test only: per-CTA clock64 stamps (VOX_GEMM_DBG=1)
  const bf16* w_packed;   // non-null: W in the packed tile layout (init.cu), 1-D bulk
                          // copies of contiguous 16 KB tiles instead of the tensor map
};

bool make_tmap_bf16(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer,
                    uint64_t row_stride_bytes, uint32_t box_outer);
int gemm_bn_for_rows(int rows);
constexpr int kGemmMaxSplits = 16;
struct GemmPlan {
  int bn;      // activation rows per tile (UMMA N)
  int mt;      // 128-row weight sub-tiles per CTA (1 or 2)
  int splits;  // split-K factor (fp32 partial planes)
  int mc;      // 1: decode kernel (one n-tile of bn >= rows, packed weights)
};
GemmPlan gemm_plan(int M, int rows, int K);
GemmPlan gemm_plan_1cta(int M, int rows, int K);  // the 1-CTA kernel only
cudaError_t gemm_launch(const CUtensorMap& tw, const CUtensorMap& tx, GemmArgs a, int splits,
                        int bn, int mt, cudaStream_t st);
// persistent many-tile GEMM (codec detokenizers): one split, bn 128, mt 1 or 2
cudaError_t gemm_launch_persist(const CUtensorMap& tw, const CUtensorMap& tx, GemmArgs a, int bn, int mt,
                                cudaStream_t st);
// decode kernel: tx = activation map with box rows bn
cudaError_t gemm_launch_mc(const CUtensorMap& tx, const CUtensorMap& tx2, GemmArgs a, int splits, int bn,
                           cudaStream_t st);
int gemm_mc_capacity(int bn);
// SMs the LM stream's kernels may use (kNumSMs unless the context split the GPU
// into LM / detok partitions): grids and split-K plans are sized to it
void vox_set_sm_budget(int sms);
int vox_sm_budget();

// ---------------------------------------------------------------- init
// w[i] = bf16(unit_pm1(mix64(key + i)) * scale); key per tensor (host-derived).
void launch_init_bf16(bf16* w, int64_t n, uint64_t key, float scale, cudaStream_t st);
// packed-tile variant (see init.cu); buffer holds roundup(M, 128) * K elements
void launch_init_bf16_packed(bf16* w, int64_t M, int64_t K, int64_t row0, uint64_t key,
                             float scale, cudaStream_t st, int64_t interleave_half = 0);
void launch_pack_bf16(const bf16* src, bf16* dst, int64_t M, int64_t K, cudaStream_t st);
// rows padded to 256 (two 128-row tiles) so a tile never reads past the buffer
inline int64_t packed_elems(int64_t M, int64_t K) { return (M + 255) / 256 * 256 * K; }
void launch_l2_flush(const void* buf, size_t bytes, uint32_t* sink, cudaStream_t st);
// fp32 variant: w[i] = offset + unit_pm1(mix64(key+i)) * scale rounded through bf16.
void launch_init_f32(float* w, int64_t n, uint64_t key, float scale, float offset,
                     cudaStream_t st);

// ---------------------------------------------------------------- LM step
struct RowDev {
  int32_t slot, pos, token, sample;
  int32_t fresh;  // lowest position of this slot whose K/V this forward appends: pages
                  // below fresh / page_size are complete before the forward starts
  int32_t attn_row;  // attention work order: the i-th row to schedule is rows[rows[i].attn_row]
                     // (longest context first, so the persistent grid's tail is short)
  int32_t pad_[2];
};

struct LmDims {
  int d, n_heads, n_kv, hd, dff, vocab;
  float eps;
  int page_size, max_pages_per_slot, n_pages, max_ctx;
};

// frame (nullable): [slot][max_ctx][nfc] extra codebook ids summed into the
// embedding; ext (nullable): fp32 [rows][d] inputs of token == -2 rows
void launch_link_tokens(const int* links, int n, const int* src_ts, int src_max_ctx, int* dst,
                        int dst_max_ctx, int nfc, int offset, int mode, cudaStream_t st);
void launch_advance_rows(RowDev* rows, int n, cudaStream_t st);
void launch_embed_norm(const RowDev* rows, int n, int* token_store, const int* frame, int nfc,
                       const float* ext, int max_ctx, const bf16* emb,
                       const float* norm_w, const LmDims& dm, float* h, bf16* x, cudaStream_t st);
void launch_qkv_rope_append(const RowDev* rows, int n, const float* ws, const float* bias, int splits,
                            int64_t split_stride, const LmDims& dm, const float2* rope,
                            const int* page_table, bf16* kc, bf16* vc, bf16* q_out,
                            cudaStream_t st);
constexpr int kAttnMaxSplits = 8;    // split-KV factor cap
constexpr int kAttnSplitRows = 128;  // split-KV only for batches up to this many rows
int attn_pick_splits(int n_rows, int n_kv, int max_ctx);
// ws: split-KV partials [rows][kv][n_split][G][hd + 2] (unused when n_split == 1)
// sched: 2 zeroed ints (work counter, done counter), self-resetting per launch
void launch_attn_decode(const RowDev* rows, int n, const bf16* q, const bf16* kc, const bf16* vc,
                        const int* page_table, const LmDims& dm, bf16* out, float* ws, int n_split,
                        int* sched, cudaStream_t st);
void launch_resid_norm(const RowDev* rows, int n, const float* ws, int splits,
                       int64_t split_stride, const LmDims& dm, float* h, const float* norm_w,
                       bf16* x_out, const int* out_index, cudaStream_t st);
void launch_silu_mul(const RowDev* rows, int n, const float* ws, int splits, int64_t split_stride,
                     const LmDims& dm, bf16* a_out, cudaStream_t st);

// ---------------------------------------------------------------- layer chain (K6)
// One persistent launch per decoder layer runs a list of jobs (layer_chain.cu).
enum ChainKind { kChGemm = 0, kChNorm = 1, kChRope = 2 };
constexpr int kChainMaxJobs = 8;
constexpr int kChainCtrStride = 32;  // one counter per 128-byte line
constexpr int kChainCtrInts = (2 * kChainMaxJobs + 1) * kChainCtrStride;  // claim[8], done[8], exit
struct ChainJob {
  int kind;
  int dep;  // job whose outputs this job reads; -1 = the preceding kernel (griddep_wait)
  // GEMM (packed weight tiles, activations via tensor map `xmap`: 0 x, 1 attn, 2 act)
  const bf16* w;
  int xmap, m_tiles, n_kb, splits, kb_per_split;
  int epi;                 // 0: fp32 split planes, 1: act = bf16(SiLU(gate) * up)
  float* out;
  int64_t ldo, split_stride;
  int m_valid;
  bf16* act;
  int64_t ld_act;
  // NORM (split planes + residual -> h; bf16 RMSNorm rows -> x[out_index[r] or r])
  // and ROPE (q|k|v planes (+ bias) -> RoPE -> q, K/V page append)
  const float* ws;
  int nsplits;
  int64_t ss;
  float* h;
  const float* nw;
  bf16* x;
  const int* out_index;
  const float* bias;
  const int* page_table;
  bf16* kc;
  bf16* vc;
  bf16* q;
};
struct ChainArgs {
  ChainJob job[kChainMaxJobs];
  int njobs;
  const RowDev* rows;
  int nrows;
  LmDims dm;
  const float2* rope;
  int* ctr;  // kChainCtrInts zeroed ints (self-resetting)
  int k_rotate;
  int wst, xst;  // weight / activation ring depths (chain_stages)
};
void chain_stages(int bn, int* wst, int* xst);
bool chain_supported_bn(int bn);
cudaError_t launch_layer_chain(const CUtensorMap& mx, const CUtensorMap& mattn, const CUtensorMap& mact,
                               const ChainArgs& a, int bn, cudaStream_t st);

// ---------------------------------------------------------------- sampler (K1)
struct SampRowDesc {
  int64_t logit_off;  // element offset of this row's column 0
  int32_t col_base;   // vocab id of column 0
  int32_t lo, hi;     // candidate vocab-id range [lo, hi)
  int32_t wlen, woff; // window ids at window_ids[woff .. woff+wlen)
  int32_t out_index;
  uint64_t seed, step;
  VoxSampling params;
};

struct SampFusedArgs {
  const RowDev* rows;
  const int* sample_rows;  // [n_sample] indices into rows
  int n_sample;
  const float* logits;     // [n_sample, ld]
  int64_t ld;
  int col_base;            // vocab id of logits column 0
  int* token_store;
  int max_ctx;
  const int* slot_prompt_len;
  const uint64_t* slot_seed;
  const VoxSampling* slot_params;
  int audio_base, codebook_size, frame_tokens, vocab;
  int* tokens_out;         // [n_sample]
  int* err_flag;
};

void launch_sample_fused(const SampFusedArgs& a, cudaStream_t st);
void launch_sample_desc(const float* logits, const SampRowDesc* rows, int n,
                        const int* window_ids, int* tokens_out, int* err_flag, int max_span,
                        cudaStream_t st);

// ---------------------------------------------------------------- detokenizer (K4)
struct DetokReq {      // one request of a detok batch (device copy)
  int32_t slot;
  int32_t f0;          // first token frame to decode (generated-token frame index)
  int32_t nf;          // token frames to decode
  int32_t lat_off;     // latent-frame row offset of this request in the batch
  int32_t parity;      // state buffer to read (write 1-parity)
  int32_t prompt_len;
  int32_t n_tokens;    // generated tokens available for the last (maybe partial) frame
  int32_t pcm_off;     // sample offset in the pcm output
  int32_t n_samples;   // samples to emit
};

struct DetokDims {
  int latent, dec, n_rates, rates[4], ch[5];
  int cb_size, frame_tokens, audio_base, max_ctx;
  int64_t state_floats;  // per slot per parity
  int64_t off_in;        // state offsets (floats) within a slot's state
  int64_t off_up[4];
  int64_t off_ru[4][3];
  int64_t off_out;
};

void launch_vq_dwconv(const DetokReq* reqs, int n_req, int n_lat, const int* token_store,
                      const bf16* tabs, const float* dw_w, const float* dw_b, float* state,
                      const DetokDims& dd, bf16* out_bf16, cudaStream_t st);
void launch_snake_upcat(const DetokReq* reqs, int n_req, int rows, int up_before,
                        const float* x, int C, const float* alpha, float* state, int64_t st_off,
                        const DetokDims& dd, bf16* out_cat, cudaStream_t st);
void launch_ru_prep(const DetokReq* reqs, int n_req, int rows, int up, const float* x, int C,
                    int dil, const float* alpha1, const float* dw_w, const float* dw_b,
                    const float* alpha2, float* state, int64_t st_off, const DetokDims& dd,
                    bf16* out, cudaStream_t st);
void launch_detok_out(const DetokReq* reqs, int n_req, int rows, int up, const float* x, int C,
                      const float* alpha, const float* w, float b, float* state, int64_t st_off,
                      const DetokDims& dd, float* pcm, cudaStream_t st);

// fused residual unit / tiled output head (detok_fused.cu)
bool ru_fused_supported(int C, int up);
void launch_ru_fused(const DetokReq* reqs, int rows, int up, const float* x, float* y, int C,
                     int dil, const float* alpha1, const float* dw_w, const float* dw_b,
                     const float* alpha2, const bf16* pw_w, const float* pw_b, float* state,
                     int64_t st_off, const DetokDims& dd, cudaStream_t st);
bool detok_out_tiled_supported(int C, int up);
bool snake_upcat_tiled_supported(int up_before);
bool ru_prep_tiled_supported(int C, int up);
void launch_ru_prep_tiled(const DetokReq* reqs, int rows, int up, const float* x, int C, int dil,
                          const float* alpha1, const float* dw_w, const float* dw_b,
                          const float* alpha2, float* state, int64_t st_off, const DetokDims& dd,
                          bf16* out, cudaStream_t st);
void launch_snake_upcat_tiled(const DetokReq* reqs, int rows, int up_before, const float* x, int C,
                              const float* alpha, float* state, int64_t st_off, const DetokDims& dd,
                              bf16* out_cat, cudaStream_t st);
void launch_detok_out_tiled(const DetokReq* reqs, int rows, int up, const float* x, int C,
                            const float* alpha, const float* w, float b, float* state,
                            int64_t st_off, const DetokDims& dd, float* pcm, cudaStream_t st);

}  // namespace vox
