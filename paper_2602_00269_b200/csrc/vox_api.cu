// vox_api.cu — the C-ABI runtime: one context per GPU owning weights, the
// paged KV pool, the device token store, detokenizer state, workspaces and
// per-bucket CUDA graphs of the decode step.  See include/voxb200.h.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <tuple>
#include <vector>

#include "common.cuh"
#include "kernels.h"

using namespace vox;

namespace {

std::mutex g_err_mu;
std::string g_err;

// Tensor ids for the counter-based init (oracle/weights.py mirrors these).
enum TensorId : uint64_t {
  T_EMB = 1,
  T_NORM_ATTN = 2,
  T_NORM_MLP = 3,
  T_NORM_FINAL = 4,
  T_QKV = 5,
  T_O = 6,
  T_GU = 7,
  T_DOWN = 8,
  T_QKV_BIAS = 9,
  T_PROJ = 10,  // ext input projector [d_model, ext_dim] (CSM depth decoder)
  // detokenizer
  T_VQ_TAB = 20,
  T_IN_DW_W = 21,
  T_IN_DW_B = 22,
  T_IN_PW_W = 23,
  T_IN_PW_B = 24,
  T_UP_ALPHA = 30,  // + block
  T_UP_W = 34,
  T_UP_B = 38,
  T_RU_A1 = 50,  // + block*3 + unit
  T_RU_DW_W = 70,
  T_RU_DW_B = 90,
  T_RU_A2 = 110,
  T_RU_PW_W = 130,
  T_RU_PW_B = 150,
  T_OUT_ALPHA = 170,
  T_OUT_W = 171,
  T_OUT_B = 172,
};

// decode-step row buckets (one CUDA graph each): steps of 32 rows between 64
// and 320 so a step pays at most 31 padding rows of tensor work -- at ~224 rows
// the projections are at the tensor/HBM ridge; 257..384 rows
// (decode rows plus a prefill burst) still run as one GEMM n-tile
constexpr int kBuckets[] = {16, 32, 64, 96, 128, 160, 192, 224, 256, 288, 320, 384, 448, 512, 1024, 2048};
constexpr int kTicketRing = 32;  // in-flight detok calls (VOX_TICKET_RING in voxb200.h)

struct TimingRec {
  std::string cls;
  cudaEvent_t a, b;
  double bytes;
};

struct Ticket {
  int64_t id = -1;
  cudaEvent_t ev = nullptr;
  float* pcm_host = nullptr;
  uint8_t* stage_host = nullptr;  // ReqHdr + DetokReq[] (pinned), reused after ev
  int32_t total = 0;
};

struct AdmitStage {  // pinned admission staging (page-table row, prompt, slot meta)
  uint8_t* host = nullptr;
  cudaEvent_t ev = nullptr;
  bool in_flight = false;
};

struct FwdStage {  // pinned per-call staging; reused only after `ev` completed
  RowDev* rows = nullptr;
  int* sample_rows = nullptr;
  int* out_index = nullptr;
  int* tokens = nullptr;
  int* err = nullptr;
  cudaEvent_t ev = nullptr;
  bool in_flight = false;
};

struct DetokW {  // detokenizer weights
  bf16* tabs = nullptr;          // [3][cb][latent]
  float *in_dw_w = nullptr, *in_dw_b = nullptr;
  bf16* in_pw_w = nullptr;       // [dec][latent]
  float* in_pw_b = nullptr;
  float* up_alpha[4] = {};
  bf16* up_w[4] = {};            // [s*Cout][2*Cin]
  float* up_b[4] = {};           // expanded [s*Cout]
  float* ru_a1[4][3] = {};
  float* ru_dw_w[4][3] = {};
  float* ru_dw_b[4][3] = {};
  float* ru_a2[4][3] = {};
  bf16* ru_pw_w[4][3] = {};      // [C][C]
  float* ru_pw_b[4][3] = {};
  float* out_alpha = nullptr;
  float* out_w = nullptr;        // [64][7]
  float out_b = 0.f;
  CUtensorMap tm_in_pw, tm_up[4], tm_ru[4][3];
};

}  // namespace

struct VoxCtx {
  int device = 0;
  VoxModelCfg cfg{};
  uint64_t seed = 0;
  std::string err;
  cudaStream_t s_lm = nullptr, s_dt = nullptr;
  // optional spatial split (VOX_DETOK_SMS): green contexts owning the LM / detok SMs
  CUgreenCtx green_lm = nullptr, green_dt = nullptr;
  int lm_sms = kNumSMs, dt_sms = 0;
  cudaEvent_t epoch = nullptr;
  LmDims dm{};
  int nqkv = 0, max_pages_per_slot = 0;

  // ---- backbone weights
  bf16* emb = nullptr;
  float *norm_attn = nullptr, *norm_mlp = nullptr, *norm_final = nullptr;
  float* b_qkv = nullptr;  // [L][nqkv] fp32 when cfg.qkv_bias (Qwen2-style)
  int* frame_store = nullptr;  // [slot][max_ctx][n_codebooks - 1] when n_codebooks > 1
  int nfc = 0;                 // n_codebooks - 1
  float* ext = nullptr;        // [max_rows][d] projected external inputs (ext_dim > 0)
  bf16* w_proj = nullptr;      // packed [d, ext_dim]
  std::map<const void*, std::map<int, CUtensorMap>> ext_maps;  // src final-hidden maps
  int* d_links = nullptr;      // [8][max_rows * 4] vox_link_tokens device staging
  int* h_links = nullptr;      // pinned twin (ring of 8, reused once its event completed)
  cudaEvent_t ev_links[8] = {};
  int64_t link_seq = 0;
  cudaEvent_t ev_xfer = nullptr;
  bf16 *w_qkv = nullptr, *w_o = nullptr, *w_gu = nullptr, *w_down = nullptr;
  float* inv_freq = nullptr;
  float2* rope_tab = nullptr;  // [max_ctx][hd/2] (cos, sin)
  bf16* w_head_audio = nullptr;  // packed copy of the tied head's audio rows
  CUtensorMap tm_head_full{};  // full-vocab (parity) head over the logical embedding
  int head_audio_rows = 0;

  // ---- activations [max_rows, ...]
  float* h = nullptr;
  bf16 *x = nullptr, *q = nullptr, *attn = nullptr, *act = nullptr, *xf = nullptr;
  float* ws = nullptr;
  size_t ws_elems = 0;
  float* attn_ws = nullptr;  // split-KV partials
  float* logits = nullptr;
  size_t logits_elems = 0;
  int last_logit_rows = 0, last_logit_ld = 0, last_logit_base = 0;  // vox_read_logits
  std::map<int, CUtensorMap> tm_x, tm_attn, tm_act, tm_xf;  // by BN

  // ---- KV / tokens / slots
  bf16 *kc = nullptr, *vc = nullptr;
  int* token_store = nullptr;
  int* page_table = nullptr;
  int* slot_prompt = nullptr;
  uint64_t* slot_seed = nullptr;
  VoxSampling* slot_params = nullptr;
  std::vector<int> free_pages;  // LIFO stack
  std::vector<std::vector<int>> slot_pages;
  std::vector<int> slot_used, h_prompt, h_target, slot_chunks, slot_covered;
  std::vector<int64_t> slot_last_fwd;
  std::vector<uint64_t> h_seed;

  // ---- per-step staging
  RowDev* d_rows = nullptr;
  int* attn_sched = nullptr;  // persistent attention work counters (self-resetting)
  int* chain_ctr = nullptr;   // layer-chain job counters: [n_layers + 1][kChainCtrInts]
  // VOX_CHAIN=1: decode steps of <= 256 rows run each layer's projections + norms +
  // RoPE as ONE persistent layer-chain launch (layer_chain.cu).  Opt-in: bit-identical
  // to the per-kernel path but measured slower at the serving shape (224 rows: 136 vs
  // ~78 us per layer; profiles/chain_timeline_r02.txt) -- the activation k-blocks
  // (28 KB from L2, ~1.7 us under load) need the ring depth the per-kernel GEMM gives
  // them, and the in-kernel norm / RoPE phases are latency chains as long as kernels
  bool chain_on = getenv("VOX_CHAIN") && atoi(getenv("VOX_CHAIN")) == 1;
  int* d_sample_rows = nullptr;
  int* d_out_index = nullptr;
  int* d_tokens = nullptr;
  int* d_err = nullptr;
  std::vector<FwdStage> stages;  // ring
  std::vector<AdmitStage> admit_stages;
  int64_t admit_seq = 0;
  size_t admit_seed_off = 0, admit_par_off = 0;
  int64_t stage_seq = 0;
  FwdStage* cur = nullptr;       // staging of the call being enqueued
  double step_attn_bytes = 0;    // per layer, for timing/roofline

  // ---- graphs keyed by (row bucket, sample bucket)
  // key = (row bucket, sample bucket, head frame slot or -1)
  std::map<std::tuple<int, int, int>, cudaGraphExec_t> graphs;
  // vox_forward_steps: steps 1.. of a multi-step decode as ONE graph, keyed by
  // (row bucket, sample bucket, first head frame slot, steps, sampler on)
  std::map<std::tuple<int, int, int, int, int>, cudaGraphExec_t> step_graphs;
  std::map<std::tuple<int, int, int, int, int>, int64_t> step_graph_launches;
  std::map<std::tuple<int, int, int>, int64_t> graph_launches;
  int64_t fwd_seq = 0;
  std::vector<cudaEvent_t> fwd_events;  // ring
  std::vector<int64_t> fwd_event_seq;

  // ---- detokenizer
  DetokW dw;
  DetokDims dd{};
  float* dstate = nullptr;
  float *dx = nullptr, *dy = nullptr;
  bf16* dbf = nullptr;
  size_t dx_elems = 0, dbf_elems = 0;
  uint8_t* d_dstage = nullptr;  // ReqHdr + DetokReq[]
  float* d_pcm = nullptr;
  size_t pcm_cap = 0;
  std::vector<Ticket> tickets;
  int64_t next_ticket = 0;
  std::map<int, cudaGraphExec_t> detok_graphs;  // by latent-frame bucket
  std::map<int, int64_t> detok_graph_launches;

  int detok_stop = 1 << 30;  // debug: stop the detok pipeline after this many stages
  bool detok_unfused = getenv("VOX_DETOK_UNFUSED") != nullptr;  // A/B: two-kernel residual units
  int gemm_k_rotate = getenv("VOX_GEMM_KROT") ? atoi(getenv("VOX_GEMM_KROT")) : 1;
  const bf16* test_x_packed = nullptr;  // gemm_test only: packed activations
  unsigned long long* test_dbg = nullptr;  // gemm_test only: per-CTA stamps
  unsigned long long* trace_buf = nullptr;  // vox_trace_*: [count, cap, records...]
  int64_t trace_cap = 0;
  bool no_graphs = getenv("VOX_NO_GRAPH") != nullptr;  // debug: eager decode steps
  bool silu_unfused = getenv("VOX_SILU_UNFUSED") != nullptr;  // A/B: separate SiLU kernel
  float* dbg_last = nullptr;  // debug: buffer holding the last stage's fp32 output

  // ---- timing / counting
  bool timing = false;
  bool capturing = false;
  std::vector<TimingRec> trecs;
  int64_t launches = 0;
};

// ---------------------------------------------------------------------------
// helpers
// ---------------------------------------------------------------------------
static int fail(VoxCtx* c, int code, const std::string& msg) {
  if (c) c->err = msg;
  std::lock_guard<std::mutex> g(g_err_mu);
  g_err = msg;
  return code;
}

#define CK(call)                                                                          \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess)                                                                \
      return fail(c, VOX_ERR_CUDA, std::string(#call) + ": " + cudaGetErrorString(e_));   \
  } while (0)

template <typename T>
static cudaError_t dalloc(T** p, size_t n) {
  return cudaMalloc(reinterpret_cast<void**>(p), std::max<size_t>(n, 1) * sizeof(T));
}

static int bucket_of(int n) {
  for (int b : kBuckets)
    if (n <= b) return b;
  return -1;
}

struct TimedLaunch {  // RAII event pair around a launch (eager + timing only)
  VoxCtx* c;
  cudaStream_t st;
  const char* cls;
  double bytes;
  cudaEvent_t a = nullptr, b = nullptr;
  TimedLaunch(VoxCtx* c_, cudaStream_t s, const char* k, double by, int n_kernels = 1)
      : c(c_), st(s), cls(k), bytes(by) {
    c->launches += n_kernels;
    if (c->timing && !c->capturing) {
      cudaEventCreate(&a);
      cudaEventCreate(&b);
      cudaEventRecord(a, st);
    }
  }
  ~TimedLaunch() {
    if (a) {
      cudaEventRecord(b, st);
      c->trecs.push_back({cls, a, b, bytes});
    }
  }
};

static bool make_act_maps(VoxCtx* c, std::map<int, CUtensorMap>& m, const bf16* base, int K,
                          int rows) {
  // box rows: the decode GEMM's row buckets and the 1-CTA kernel's tile widths
  for (int bn : {16, 32, 64, 96, 128, 160, 192, 224, 256}) {
    CUtensorMap t;
    if (!make_tmap_bf16(&t, base, K, rows, static_cast<uint64_t>(K) * 2, bn)) return false;
    m[bn] = t;
  }
  return true;
}

// GEMM over `rows` activation rows of buffer map set `xm`.
// `wp` non-null: W is in the packed tile layout (init.cu) and `tw` is unused;
static int run_gemm(VoxCtx* c, const CUtensorMap& tw, std::map<int, CUtensorMap>& xm, int M,
                    int rows, int K, float* out, int64_t ldo, int splits, const float* bias,
                    const float* resid, int64_t ldr, int m_valid, cudaStream_t st,
                    const char* cls = "gemm", const bf16* wp = nullptr,
                    bf16* act_out = nullptr,
                    int64_t ld_act = 0) {
  GemmPlan plan = gemm_plan(M, rows, K);  // tile shape (splits are the caller's)
  {
    // the effective split count: every split gets ceil(n_kb / splits) k-blocks, so a
    // requested count that leaves trailing splits empty launches (and leaves) fewer planes
    const int n_kb = K / 64;
    const int per = (n_kb + splits - 1) / splits;
    splits = (n_kb + per - 1) / per;
  }
  if (plan.mc && wp == nullptr) plan = gemm_plan_1cta(M, rows, K);  // mc streams packed tiles only
  const int bn = plan.bn;
  GemmArgs a{};
  a.M = M;
  a.N = rows;
  a.K = K;
  a.out = out;
  a.ldo = ldo;
  a.split_stride = static_cast<int64_t>(rows) * ldo;
  a.bias = bias;
  a.resid = resid;
  a.ldr = ldr;
  a.m_valid = m_valid;
  a.w_packed = wp;
  a.x_packed = c->test_x_packed;
  a.dbg = c->test_dbg;
  a.k_rotate = c->gemm_k_rotate;
  a.epi = act_out != nullptr ? 1 : 0;
  a.act = act_out;
  a.ld_act = ld_act;
  if (a.epi == 1 && (splits != 1 || plan.mt != 1))
    return fail(c, VOX_ERR_INVALID, "fused SiLU epilogue needs one split, 1-CTA tiles");
  const double bytes = static_cast<double>(m_valid) * K * 2 + static_cast<double>(rows) * K * 2 +
                       static_cast<double>(rows) * m_valid * 4 * splits;
  TimedLaunch tl(c, st, cls, bytes);
  cudaError_t e = plan.mc     ? gemm_launch_mc(xm.at(bn > 256 ? 256 : bn), xm.at(bn > 256 ? bn - 256 : bn), a,
                                               splits, bn, st)
                              : gemm_launch(tw, xm.at(bn), a, splits, bn, plan.mt, st);
  if (e != cudaSuccess) return fail(c, VOX_ERR_CUDA, std::string("gemm: ") + cudaGetErrorString(e));
  return VOX_OK;
}

// ---------------------------------------------------------------------------
// weights
// ---------------------------------------------------------------------------
static int init_bf16(VoxCtx* c, bf16* w, int64_t n, uint64_t tid, uint64_t layer, float scale) {
  launch_init_bf16(w, n, tensor_key(c->seed, tid, layer), scale, c->s_lm);
  CK(cudaGetLastError());
  return VOX_OK;
}
static int init_f32(VoxCtx* c, float* w, int64_t n, uint64_t tid, uint64_t layer, float scale,
                    float offset) {
  launch_init_f32(w, n, tensor_key(c->seed, tid, layer), scale, offset, c->s_lm);
  CK(cudaGetLastError());
  return VOX_OK;
}

#define RET(x)                  \
  do {                          \
    int r_ = (x);               \
    if (r_ != VOX_OK) return r_; \
  } while (0)

static int create_backbone(VoxCtx* c) {
  const VoxModelCfg& g = c->cfg;
  const int L = g.n_layers, d = g.d_model, hd = g.head_dim, H = g.n_heads, KV = g.n_kv_heads;
  const int dff = g.d_ff, V = g.vocab;
  c->nqkv = (H + 2 * KV) * hd;
  // projection weights live in the packed tile layout (init.cu) the GEMM streams
  const int64_t n_qkv = packed_elems(c->nqkv, d), n_o = packed_elems(d, H * hd);
  const int64_t n_gu = packed_elems(2 * dff, d), n_dn = packed_elems(d, dff);
  CK(dalloc(&c->emb, static_cast<size_t>(V) * d));
  CK(dalloc(&c->norm_attn, static_cast<size_t>(L) * d));
  CK(dalloc(&c->norm_mlp, static_cast<size_t>(L) * d));
  CK(dalloc(&c->norm_final, static_cast<size_t>(d)));
  CK(dalloc(&c->w_qkv, static_cast<size_t>(L * n_qkv)));
  CK(dalloc(&c->w_o, static_cast<size_t>(L * n_o)));
  CK(dalloc(&c->w_gu, static_cast<size_t>(L * n_gu)));
  CK(dalloc(&c->w_down, static_cast<size_t>(L * n_dn)));
  RET(init_bf16(c, c->emb, static_cast<int64_t>(V) * d, T_EMB, 0, g.embed_scale));
  auto packed = [&](bf16* w, int64_t M, int64_t K, int64_t row0, uint64_t tid, uint64_t layer,
                    float scale, int64_t interleave_half = 0) {
    launch_init_bf16_packed(w, M, K, row0, tensor_key(c->seed, tid, layer), scale, c->s_lm,
                            interleave_half);
    return cudaGetLastError() == cudaSuccess ? VOX_OK : fail(c, VOX_ERR_CUDA, "init packed");
  };
  for (int l = 0; l < L; ++l) {
    RET(init_f32(c, c->norm_attn + static_cast<int64_t>(l) * d, d, T_NORM_ATTN, l, 0.25f, 1.0f));
    RET(init_f32(c, c->norm_mlp + static_cast<int64_t>(l) * d, d, T_NORM_MLP, l, 0.25f, 1.0f));
    RET(packed(c->w_qkv + l * n_qkv, c->nqkv, d, 0, T_QKV, l, std::sqrt(3.0f / d)));
    RET(packed(c->w_o + l * n_o, d, H * hd, 0, T_O, l, std::sqrt(3.0f / (H * hd))));
    // gate|up rows interleaved per 128-row tile (64 gate + the same 64 up rows)
    RET(packed(c->w_gu + l * n_gu, 2 * dff, d, 0, T_GU, l, std::sqrt(3.0f / d), dff));
    RET(packed(c->w_down + l * n_dn, d, dff, 0, T_DOWN, l, std::sqrt(3.0f / dff)));
  }
  if (g.audio_base >= 0) {  // packed copy of the audio rows of the tied head
    const int rows = g.frame_tokens * g.codebook_size;
    CK(dalloc(&c->w_head_audio, static_cast<size_t>(packed_elems(rows, d))));
    RET(packed(c->w_head_audio, rows, d, g.audio_base, T_EMB, 0, g.embed_scale));
  }
  RET(init_f32(c, c->norm_final, d, T_NORM_FINAL, 0, 0.25f, 1.0f));
  if (g.qkv_bias) {
    CK(dalloc(&c->b_qkv, static_cast<size_t>(L) * c->nqkv));
    for (int l = 0; l < L; ++l)
      RET(init_f32(c, c->b_qkv + static_cast<int64_t>(l) * c->nqkv, c->nqkv, T_QKV_BIAS, l, 0.5f, 0.0f));
  }
  // RoPE inverse frequencies, fp64 -> fp32 (oracle: identical table)
  std::vector<float> inv(hd / 2);
  for (int i = 0; i < hd / 2; ++i)
    inv[i] = static_cast<float>(1.0 / std::pow(static_cast<double>(g.rope_theta),
                                               (2.0 * i) / static_cast<double>(hd)));
  CK(dalloc(&c->inv_freq, inv.size()));
  CK(cudaMemcpy(c->inv_freq, inv.data(), inv.size() * 4, cudaMemcpyHostToDevice));
  // (cos, sin) table: angle = float(pos) * inv_freq[i] in fp32, trig in fp64,
  // rounded to fp32 (oracle/llama.py:rope computes the identical values)
  {
    std::vector<float2> tab(static_cast<size_t>(g.max_ctx) * (hd / 2));
    for (int p = 0; p < g.max_ctx; ++p)
      for (int i = 0; i < hd / 2; ++i) {
        const float ang = static_cast<float>(p) * inv[i];
        tab[static_cast<size_t>(p) * (hd / 2) + i] =
            make_float2(static_cast<float>(std::cos(static_cast<double>(ang))),
                        static_cast<float>(std::sin(static_cast<double>(ang))));
      }
    CK(dalloc(&c->rope_tab, tab.size()));
    CK(cudaMemcpy(c->rope_tab, tab.data(), tab.size() * sizeof(float2), cudaMemcpyHostToDevice));
  }

  if (!make_tmap_bf16(&c->tm_head_full, c->emb, d, V, d * 2ull, 128))
    return fail(c, VOX_ERR_CUDA, "tensor map (lm head)");
  if (g.audio_base >= 0) {
    c->head_audio_rows = g.frame_tokens * g.codebook_size;

  }
  return VOX_OK;
}

static int create_buffers(VoxCtx* c) {
  const VoxModelCfg& g = c->cfg;
  const int R = g.max_rows, d = g.d_model, dff = g.d_ff;
  CK(dalloc(&c->h, static_cast<size_t>(R) * d));
  CK(dalloc(&c->x, static_cast<size_t>(R) * d));
  CK(dalloc(&c->xf, static_cast<size_t>(R) * d));
  CK(dalloc(&c->q, static_cast<size_t>(R) * g.n_heads * g.head_dim));
  CK(dalloc(&c->attn, static_cast<size_t>(R) * g.n_heads * g.head_dim));
  CK(dalloc(&c->act, static_cast<size_t>(R) * dff));
  CK(cudaMemset(c->x, 0, static_cast<size_t>(R) * d * 2));
  CK(cudaMemset(c->xf, 0, static_cast<size_t>(R) * d * 2));
  CK(cudaMemset(c->attn, 0, static_cast<size_t>(R) * g.n_heads * g.head_dim * 2));
  CK(cudaMemset(c->act, 0, static_cast<size_t>(R) * dff * 2));
  // split-K workspace: worst case splits * rows * max(N)
  const int maxN = std::max({c->nqkv, d, 2 * dff});
  c->ws_elems = static_cast<size_t>(16) * R * maxN;
  {
    const int grp = g.n_heads / g.n_kv_heads;
    const size_t n = static_cast<size_t>(std::min(R, kAttnSplitRows)) * g.n_kv_heads *
                     kAttnMaxSplits * grp * (g.head_dim + 2);
    CK(dalloc(&c->attn_ws, n));
  }
  CK(dalloc(&c->ws, c->ws_elems));
  const int head_cols = g.audio_base >= 0 ? c->head_audio_rows : g.vocab;
  const int full_rows = std::min(R, 256);
  c->logits_elems = std::max(static_cast<size_t>(R) * head_cols,
                             static_cast<size_t>(full_rows) * g.vocab);
  CK(dalloc(&c->logits, c->logits_elems));
  if (!make_act_maps(c, c->tm_x, c->x, d, R) || !make_act_maps(c, c->tm_xf, c->xf, d, R) ||
      !make_act_maps(c, c->tm_attn, c->attn, g.n_heads * g.head_dim, R) ||
      !make_act_maps(c, c->tm_act, c->act, dff, R))
    return fail(c, VOX_ERR_CUDA, "tensor map (activations)");

  // KV pool
  c->max_pages_per_slot = (g.max_ctx + g.page_size - 1) / g.page_size;
  const size_t kv_elems = static_cast<size_t>(g.n_layers) * g.n_pages * g.n_kv_heads *
                          g.page_size * g.head_dim;
  CK(dalloc(&c->kc, kv_elems));
  CK(dalloc(&c->vc, kv_elems));
  CK(cudaMemset(c->kc, 0, kv_elems * 2));
  CK(cudaMemset(c->vc, 0, kv_elems * 2));
  CK(dalloc(&c->token_store, static_cast<size_t>(g.max_slots) * g.max_ctx));
  CK(cudaMemset(c->token_store, 0, static_cast<size_t>(g.max_slots) * g.max_ctx * 4));
  c->nfc = g.n_codebooks > 1 ? g.n_codebooks - 1 : 0;
  if (c->nfc > 0) {
    const size_t nf = static_cast<size_t>(g.max_slots) * g.max_ctx * c->nfc;
    CK(dalloc(&c->frame_store, nf));
    CK(cudaMemset(c->frame_store, 0xFF, nf * 4));  // -1: no id
  }
  if (g.ext_dim > 0) {
    CK(dalloc(&c->ext, static_cast<size_t>(g.max_rows) * g.d_model));
    CK(cudaMemset(c->ext, 0, static_cast<size_t>(g.max_rows) * g.d_model * 4));
    CK(dalloc(&c->w_proj, static_cast<size_t>(packed_elems(g.d_model, g.ext_dim))));
    launch_init_bf16_packed(c->w_proj, g.d_model, g.ext_dim, 0, tensor_key(c->seed, T_PROJ, 0),
                            std::sqrt(3.0f / g.ext_dim), c->s_lm);
    CK(cudaGetLastError());
  }
  CK(dalloc(&c->d_links, static_cast<size_t>(g.max_rows) * 4 * 8));
  CK(cudaHostAlloc(&c->h_links, static_cast<size_t>(g.max_rows) * 4 * 8 * 4, cudaHostAllocDefault));
  for (auto& e : c->ev_links) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&c->ev_xfer, cudaEventDisableTiming));
  CK(dalloc(&c->page_table, static_cast<size_t>(g.max_slots) * c->max_pages_per_slot));
  CK(cudaMemset(c->page_table, 0, static_cast<size_t>(g.max_slots) * c->max_pages_per_slot * 4));
  CK(dalloc(&c->slot_prompt, static_cast<size_t>(g.max_slots)));
  CK(dalloc(&c->slot_seed, static_cast<size_t>(g.max_slots)));
  CK(dalloc(&c->slot_params, static_cast<size_t>(g.max_slots)));
  c->free_pages.clear();
  for (int p = g.n_pages - 1; p >= 0; --p) c->free_pages.push_back(p);  // pop -> 0,1,2..
  c->slot_pages.assign(g.max_slots, {});
  c->slot_used.assign(g.max_slots, 0);
  c->h_prompt.assign(g.max_slots, 0);
  c->h_target.assign(g.max_slots, 0);
  c->slot_chunks.assign(g.max_slots, 0);
  c->slot_covered.assign(g.max_slots, 0);
  c->slot_last_fwd.assign(g.max_slots, -1);
  c->h_seed.assign(g.max_slots, 0);

  CK(dalloc(&c->d_rows, static_cast<size_t>(R)));
  // [0..1] persistent work counters, [2 + row * n_kv + kvh] split arrival counters
  // (the last split of a (row, kv head) combines the partials; all self-resetting)
  {
    const size_t ns = 2 + static_cast<size_t>(R) * g.n_kv_heads;
    CK(dalloc(&c->attn_sched, ns));
    CK(cudaMemset(c->attn_sched, 0, ns * sizeof(int)));
  }
  CK(dalloc(&c->chain_ctr, static_cast<size_t>(g.n_layers + 1) * kChainCtrInts));
  CK(cudaMemset(c->chain_ctr, 0, static_cast<size_t>(g.n_layers + 1) * kChainCtrInts * sizeof(int)));
  CK(dalloc(&c->d_sample_rows, static_cast<size_t>(R)));
  CK(dalloc(&c->d_out_index, static_cast<size_t>(R)));
  CK(dalloc(&c->d_tokens, static_cast<size_t>(R)));
  CK(dalloc(&c->d_err, 1));
  CK(cudaMemset(c->d_err, 0, 4));
  c->stages.resize(8);
  for (auto& s : c->stages) {
    CK(cudaHostAlloc(&s.rows, sizeof(RowDev) * R, cudaHostAllocDefault));
    CK(cudaHostAlloc(&s.sample_rows, sizeof(int) * R, cudaHostAllocDefault));
    CK(cudaHostAlloc(&s.out_index, sizeof(int) * R, cudaHostAllocDefault));
    CK(cudaHostAlloc(&s.tokens, sizeof(int) * R, cudaHostAllocDefault));
    CK(cudaHostAlloc(&s.err, sizeof(int), cudaHostAllocDefault));
    *s.err = 0;
    CK(cudaEventCreateWithFlags(&s.ev, cudaEventDisableTiming));
  }
  {
    const size_t ints = static_cast<size_t>(c->max_pages_per_slot) + g.max_ctx + 1;
    c->admit_seed_off = (ints * 4 + 15) / 16 * 16;
    c->admit_par_off = c->admit_seed_off + 16;
    const size_t bytes = c->admit_par_off + sizeof(VoxSampling);
    c->admit_stages.resize(64);
    for (auto& a : c->admit_stages) {
      CK(cudaHostAlloc(&a.host, bytes, cudaHostAllocDefault));
      CK(cudaEventCreateWithFlags(&a.ev, cudaEventDisableTiming));
    }
  }
  c->fwd_events.resize(64);
  c->fwd_event_seq.assign(64, -1);
  for (auto& e : c->fwd_events) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  return VOX_OK;
}

// ---------------------------------------------------------------------------
// detokenizer weights + state layout
// ---------------------------------------------------------------------------
static int create_detok(VoxCtx* c) {
  const VoxModelCfg& g = c->cfg;
  DetokDims& dd = c->dd;
  DetokW& w = c->dw;
  dd.latent = g.latent_dim;
  dd.dec = g.decoder_dim;
  dd.n_rates = g.n_rates;
  for (int b = 0; b < 4; ++b) dd.rates[b] = g.rates[b];
  dd.ch[0] = g.decoder_dim;
  for (int b = 0; b < 4; ++b) dd.ch[b + 1] = dd.ch[b] / 2;
  dd.cb_size = g.codebook_size;
  dd.frame_tokens = g.frame_tokens;
  dd.audio_base = g.audio_base;
  dd.max_ctx = g.max_ctx;
  // state layout (floats): in-dwconv history 6*latent; per block: 1 frame of
  // Cin (transposed conv), RU histories 6*d*Cout for d in {1,3,9}; out 6*C4
  int64_t off = 0;
  dd.off_in = off;
  off += 6LL * dd.latent;
  const int dils[3] = {1, 3, 9};
  for (int b = 0; b < 4; ++b) {
    dd.off_up[b] = off;
    off += dd.ch[b];
    for (int u = 0; u < 3; ++u) {
      dd.off_ru[b][u] = off;
      off += 6LL * dils[u] * dd.ch[b + 1];
    }
  }
  dd.off_out = off;
  off += 6LL * dd.ch[4];
  dd.state_floats = (off + 63) / 64 * 64;
  CK(dalloc(&c->dstate, static_cast<size_t>(g.max_slots) * 2 * dd.state_floats));
  CK(cudaMemset(c->dstate, 0, static_cast<size_t>(g.max_slots) * 2 * dd.state_floats * 4));

  const int L = dd.latent, D0 = dd.dec, cb = dd.cb_size;
  CK(dalloc(&w.tabs, static_cast<size_t>(3) * cb * L));
  RET(init_bf16(c, w.tabs, 3LL * cb * L, T_VQ_TAB, 0, 0.866f));
  CK(dalloc(&w.in_dw_w, static_cast<size_t>(L) * 7));
  CK(dalloc(&w.in_dw_b, static_cast<size_t>(L)));
  RET(init_f32(c, w.in_dw_w, 7LL * L, T_IN_DW_W, 0, std::sqrt(3.0f / 7.0f), 0.f));
  RET(init_f32(c, w.in_dw_b, L, T_IN_DW_B, 0, 0.05f, 0.f));
  CK(dalloc(&w.in_pw_w, static_cast<size_t>(D0) * L));
  CK(dalloc(&w.in_pw_b, static_cast<size_t>(D0)));
  RET(init_bf16(c, w.in_pw_w, static_cast<int64_t>(D0) * L, T_IN_PW_W, 0, std::sqrt(3.0f / L)));
  RET(init_f32(c, w.in_pw_b, D0, T_IN_PW_B, 0, 0.05f, 0.f));
  if (!make_tmap_bf16(&w.tm_in_pw, w.in_pw_w, L, D0, L * 2ull, 128))
    return fail(c, VOX_ERR_CUDA, "tmap detok in");
  for (int b = 0; b < 4; ++b) {
    const int Ci = dd.ch[b], Co = dd.ch[b + 1], s = dd.rates[b];
    CK(dalloc(&w.up_alpha[b], static_cast<size_t>(Ci)));
    RET(init_f32(c, w.up_alpha[b], Ci, T_UP_ALPHA + b, 0, 0.5f, 1.0f));
    CK(dalloc(&w.up_w[b], static_cast<size_t>(s) * Co * 2 * Ci));
    RET(init_bf16(c, w.up_w[b], static_cast<int64_t>(s) * Co * 2 * Ci, T_UP_W + b, 0,
                  std::sqrt(3.0f / (2.0f * Ci))));
    std::vector<float> bias_small(Co), bias_ext(static_cast<size_t>(s) * Co);
    float* tmp;
    CK(dalloc(&tmp, static_cast<size_t>(Co)));
    RET(init_f32(c, tmp, Co, T_UP_B + b, 0, 0.05f, 0.f));
    CK(cudaStreamSynchronize(c->s_lm));  // init ran on the non-blocking LM stream
    CK(cudaMemcpy(bias_small.data(), tmp, Co * 4, cudaMemcpyDeviceToHost));
    cudaFree(tmp);
    for (int j = 0; j < s; ++j)
      for (int o = 0; o < Co; ++o) bias_ext[static_cast<size_t>(j) * Co + o] = bias_small[o];
    CK(dalloc(&w.up_b[b], bias_ext.size()));
    CK(cudaMemcpy(w.up_b[b], bias_ext.data(), bias_ext.size() * 4, cudaMemcpyHostToDevice));
    if (!make_tmap_bf16(&w.tm_up[b], w.up_w[b], 2 * Ci, static_cast<uint64_t>(s) * Co,
                        2ull * Ci * 2, 128))
      return fail(c, VOX_ERR_CUDA, "tmap detok up");
    for (int u = 0; u < 3; ++u) {
      const uint64_t li = static_cast<uint64_t>(b * 3 + u);
      CK(dalloc(&w.ru_a1[b][u], static_cast<size_t>(Co)));
      CK(dalloc(&w.ru_a2[b][u], static_cast<size_t>(Co)));
      CK(dalloc(&w.ru_dw_w[b][u], static_cast<size_t>(Co) * 7));
      CK(dalloc(&w.ru_dw_b[b][u], static_cast<size_t>(Co)));
      CK(dalloc(&w.ru_pw_w[b][u], static_cast<size_t>(Co) * Co));
      CK(dalloc(&w.ru_pw_b[b][u], static_cast<size_t>(Co)));
      RET(init_f32(c, w.ru_a1[b][u], Co, T_RU_A1, li, 0.5f, 1.0f));
      RET(init_f32(c, w.ru_a2[b][u], Co, T_RU_A2, li, 0.5f, 1.0f));
      RET(init_f32(c, w.ru_dw_w[b][u], 7LL * Co, T_RU_DW_W, li, std::sqrt(3.0f / 7.0f), 0.f));
      RET(init_f32(c, w.ru_dw_b[b][u], Co, T_RU_DW_B, li, 0.05f, 0.f));
      RET(init_bf16(c, w.ru_pw_w[b][u], static_cast<int64_t>(Co) * Co, T_RU_PW_W, li,
                    0.25f * std::sqrt(3.0f / Co)));
      RET(init_f32(c, w.ru_pw_b[b][u], Co, T_RU_PW_B, li, 0.05f, 0.f));
      if (!make_tmap_bf16(&w.tm_ru[b][u], w.ru_pw_w[b][u], Co, Co, Co * 2ull, 128))
        return fail(c, VOX_ERR_CUDA, "tmap detok ru");
    }
  }
  const int C4 = dd.ch[4];
  CK(dalloc(&w.out_alpha, static_cast<size_t>(C4)));
  CK(dalloc(&w.out_w, static_cast<size_t>(C4) * 7));
  RET(init_f32(c, w.out_alpha, C4, T_OUT_ALPHA, 0, 0.5f, 1.0f));
  // residual branches at 1/4 gain and a 0.15-gain output conv keep the random
  // decoder contractive (well-conditioned for bf16 parity; pre-tanh rms ~0.3)
  RET(init_f32(c, w.out_w, 7LL * C4, T_OUT_W, 0, 0.15f * std::sqrt(3.0f / (7.0f * C4)), 0.f));
  {
    float* tmp;
    CK(dalloc(&tmp, 1));
    RET(init_f32(c, tmp, 1, T_OUT_B, 0, 0.05f, 0.f));
    CK(cudaStreamSynchronize(c->s_lm));
    CK(cudaMemcpy(&w.out_b, tmp, 4, cudaMemcpyDeviceToHost));
    cudaFree(tmp);
  }
  // activation buffers sized by the largest level: rows*channels
  const int64_t F = g.max_detok_frames;
  int64_t mx = F * D0;
  int64_t mbf = F * L;
  int up = 1;
  for (int b = 0; b < 4; ++b) {
    mbf = std::max<int64_t>(mbf, F * up * 2 * dd.ch[b]);  // upcat operand
    up *= dd.rates[b];
    mx = std::max<int64_t>(mx, F * up * dd.ch[b + 1]);
    mbf = std::max<int64_t>(mbf, F * up * dd.ch[b + 1]);
  }
  c->dx_elems = static_cast<size_t>(mx);
  c->dbf_elems = static_cast<size_t>(mbf);
  CK(dalloc(&c->dx, c->dx_elems));
  CK(dalloc(&c->dy, c->dx_elems));
  CK(dalloc(&c->dbf, c->dbf_elems));
  CK(cudaMemset(c->dbf, 0, c->dbf_elems * 2));
  const size_t stage_bytes = 8 + sizeof(DetokReq) * (F / 4 + 8);
  CK(dalloc(&c->d_dstage, stage_bytes));
  c->pcm_cap = static_cast<size_t>(F) * up;
  CK(dalloc(&c->d_pcm, c->pcm_cap));
  c->tickets.resize(kTicketRing);
  for (auto& t : c->tickets) {
    CK(cudaEventCreate(&t.ev));
    CK(cudaHostAlloc(&t.pcm_host, c->pcm_cap * 4, cudaHostAllocDefault));
    CK(cudaHostAlloc(&t.stage_host, stage_bytes, cudaHostAllocDefault));
  }
  return VOX_OK;
}

// ---------------------------------------------------------------------------
// the decoder layers as persistent layer-chain launches (layer_chain.cu):
//   chain(-1) = [QKV_0, RoPE_0]; per layer l: attention_l, then
//   chain(l)  = [O_l, norm, gate|up_l (+SiLU), down_l, norm, QKV_l+1, RoPE_l+1]
// (the last layer's second norm is the final norm into xf).  Split-K factors
// and k-block rotation are the per-kernel path's, so the fp32 planes, h, x and
// the KV pages are bit-identical to it.
// ---------------------------------------------------------------------------
static int chain_bn_for_rows(int rows) {
  for (int b : {16, 32, 64, 96, 128, 160, 192, 224, 256})
    if (rows <= b) return b;
  return -1;
}

static int enqueue_layers_chain(VoxCtx* c, int nrows, int bn, cudaStream_t st) {
  const VoxModelCfg& g = c->cfg;
  const LmDims& dm = c->dm;
  const int L = g.n_layers, d = g.d_model, dff = g.d_ff, Hhd = g.n_heads * g.head_dim;
  const size_t kv_layer = static_cast<size_t>(g.n_pages) * g.n_kv_heads * g.page_size * g.head_dim;
  const int64_t n_qkv = packed_elems(c->nqkv, d), n_o = packed_elems(d, Hhd);
  const int64_t n_gu = packed_elems(2 * dff, d), n_dn = packed_elems(d, dff);
  const int sp_qkv = gemm_plan(c->nqkv, nrows, d).splits, sp_o = gemm_plan(d, nrows, Hhd).splits;
  const int sp_dn = gemm_plan(d, nrows, dff).splits;
  auto gemm_job = [&](const bf16* w, int xmap, int M, int K, int splits, int dep, int epi) {
    ChainJob j{};
    j.kind = kChGemm;
    j.dep = dep;
    j.w = w;
    j.xmap = xmap;
    j.m_tiles = (M + 127) / 128;
    j.n_kb = K / 64;
    const int per = (j.n_kb + splits - 1) / splits;  // every split non-empty (as run_gemm)
    j.splits = (j.n_kb + per - 1) / per;
    j.kb_per_split = per;
    j.epi = epi;
    j.out = c->ws;
    j.ldo = M;
    j.split_stride = static_cast<int64_t>(nrows) * M;
    j.m_valid = M;
    j.act = c->act;
    j.ld_act = dff;
    return j;
  };
  auto planes = [](const ChainJob& j) { return j.splits; };
  auto norm_job = [&](int dep, int nspl, const float* nw, bf16* x, const int* oi) {
    ChainJob j{};
    j.kind = kChNorm;
    j.dep = dep;
    j.ws = c->ws;
    j.nsplits = nspl;
    j.ss = static_cast<int64_t>(nrows) * d;
    j.h = c->h;
    j.nw = nw;
    j.x = x;
    j.out_index = oi;
    return j;
  };
  auto rope_job = [&](int dep, int nspl, int l) {
    ChainJob j{};
    j.kind = kChRope;
    j.dep = dep;
    j.ws = c->ws;
    j.nsplits = nspl;
    j.ss = static_cast<int64_t>(nrows) * c->nqkv;
    j.bias = c->b_qkv ? c->b_qkv + static_cast<int64_t>(l) * c->nqkv : nullptr;
    j.page_table = c->page_table;
    j.kc = c->kc + l * kv_layer;
    j.vc = c->vc + l * kv_layer;
    j.q = c->q;
    return j;
  };
  ChainArgs a{};
  a.rows = c->d_rows;
  a.nrows = nrows;
  a.dm = dm;
  a.rope = c->rope_tab;
  a.k_rotate = c->gemm_k_rotate;
  chain_stages(bn, &a.wst, &a.xst);
  const CUtensorMap &mx = c->tm_x.at(bn), &ma = c->tm_attn.at(bn), &mf = c->tm_act.at(bn);
  const double act_b = static_cast<double>(nrows) * 2;
  auto launch = [&](int slot, double bytes) -> int {
    a.ctr = c->chain_ctr + static_cast<int64_t>(slot) * kChainCtrInts;
    TimedLaunch tl(c, st, "chain", bytes);
    cudaError_t e = launch_layer_chain(mx, ma, mf, a, bn, st);
    if (e != cudaSuccess) return fail(c, VOX_ERR_CUDA, std::string("layer chain: ") + cudaGetErrorString(e));
    return VOX_OK;
  };
  const double w_qkv = 2.0 * c->nqkv * d, w_o = 2.0 * d * Hhd, w_gu = 4.0 * dff * d, w_dn = 2.0 * d * dff;
  // chain(-1): layer 0's q|k|v projection + RoPE/KV append
  a.job[0] = gemm_job(c->w_qkv, 0, c->nqkv, d, sp_qkv, -1, 0);
  a.job[1] = rope_job(0, planes(a.job[0]), 0);
  a.njobs = 2;
  RET(launch(L, w_qkv + act_b * d + act_b * 2 * c->nqkv));
  for (int l = 0; l < L; ++l) {
    {
      const int asp = attn_pick_splits(nrows, g.n_kv_heads, g.max_ctx);
      TimedLaunch tl(c, st, "attn", c->step_attn_bytes, asp > 1 ? 2 : 1);
      launch_attn_decode(c->d_rows, nrows, c->q, c->kc + l * kv_layer, c->vc + l * kv_layer,
                         c->page_table, dm, c->attn, c->attn_ws, asp, c->attn_sched, st);
    }
    const bool last = (l == L - 1);
    a.job[0] = gemm_job(c->w_o + l * n_o, 1, d, Hhd, sp_o, -1, 0);
    a.job[1] = norm_job(0, planes(a.job[0]), c->norm_mlp + static_cast<int64_t>(l) * d, c->x, nullptr);
    a.job[2] = gemm_job(c->w_gu + l * n_gu, 0, 2 * dff, d, 1, 1, 1);
    a.job[3] = gemm_job(c->w_down + l * n_dn, 2, d, dff, sp_dn, 2, 0);
    a.job[4] = norm_job(3, planes(a.job[3]), last ? c->norm_final : c->norm_attn + static_cast<int64_t>(l + 1) * d,
                        last ? c->xf : c->x, last ? c->d_out_index : nullptr);
    a.njobs = 5;
    double bytes = w_o + w_gu + w_dn + act_b * (Hhd + d + dff) + act_b * 2 * (d + dff + d);
    if (!last) {
      a.job[5] = gemm_job(c->w_qkv + (l + 1) * n_qkv, 0, c->nqkv, d, sp_qkv, 4, 0);
      a.job[6] = rope_job(5, planes(a.job[5]), l + 1);
      a.njobs = 7;
      bytes += w_qkv + act_b * d + act_b * 2 * c->nqkv;
    }
    RET(launch(l, bytes));
  }
  return VOX_OK;
}

// ---------------------------------------------------------------------------
// the decode step (eager or captured)
// ---------------------------------------------------------------------------
// hslot >= 0: every sampled row is at the same frame slot, so the LM head runs
// over that slot's codebook rows only (CSM depth decoder: 1 of 31 codebook heads)
// Grids and split-K plans follow the partition of the stream being enqueued to:
// the LM stream's SMs for forwards, the detok partition for detok calls (the
// budget is process-wide state, so every enqueue sets its own).
struct SmBudgetScope {
  int prev;
  explicit SmBudgetScope(int sms) : prev(vox_sm_budget()) {
    if (sms > 0) vox_set_sm_budget(sms);
  }
  ~SmBudgetScope() { vox_set_sm_budget(prev); }
};

static int enqueue_forward(VoxCtx* c, int nrows, int nsamp, bool full_logits, int hslot = -1,
                           bool run_sampler = true) {
  SmBudgetScope sms(c->lm_sms);
  const VoxModelCfg& g = c->cfg;
  const LmDims& dm = c->dm;
  cudaStream_t st = c->s_lm;
  const int L = g.n_layers, d = g.d_model, dff = g.d_ff, Hhd = g.n_heads * g.head_dim;
  {
    TimedLaunch tl(c, st, "norm", static_cast<double>(nrows) * d * 8);
    launch_embed_norm(c->d_rows, nrows, c->token_store, c->frame_store, c->nfc, c->ext, g.max_ctx,
                      c->emb, c->norm_attn, dm, c->h, c->x, st);
  }
  const GemmPlan qkv_plan = gemm_plan(c->nqkv, nrows, d), o_plan = gemm_plan(d, nrows, Hhd);
  const GemmPlan dn_plan = gemm_plan(d, nrows, dff);
  const int sp_qkv = qkv_plan.splits, sp_o = o_plan.splits;
  // fp32 planes the consumers reduce (1 when the GEMM reduced its splits in-cluster)
  const int pl_qkv = qkv_plan.splits, pl_o = o_plan.splits, pl_dn = dn_plan.splits;
  const GemmPlan gu_plan = gemm_plan(2 * dff, nrows, d);
  const int sp_gu = gu_plan.splits;
  const int sp_dn = dn_plan.splits;
  // gate|up CTAs (1 split, mc kernel) all co-resident -> norm fusable
  const size_t kv_layer = static_cast<size_t>(g.n_pages) * g.n_kv_heads * g.page_size * g.head_dim;
  const int64_t n_qkv = packed_elems(c->nqkv, d), n_o = packed_elems(d, Hhd);
  const int64_t n_gu = packed_elems(2 * dff, d), n_dn = packed_elems(d, dff);
  const CUtensorMap& tw_unused = c->tm_head_full;  // packed weights: the W map is not read
  const int cbn = c->chain_on ? chain_bn_for_rows(nrows) : -1;
  if (cbn > 0) RET(enqueue_layers_chain(c, nrows, cbn, st));
  for (int l = 0; l < L && cbn < 0; ++l) {
    RET(run_gemm(c, tw_unused, c->tm_x, c->nqkv, nrows, d, c->ws, c->nqkv, sp_qkv, nullptr,
                 nullptr, 0, c->nqkv, st, "gemm", c->w_qkv + l * n_qkv));
    {
      TimedLaunch tl(c, st, "qkv_rope", static_cast<double>(nrows) * c->nqkv * 4 * pl_qkv);
      launch_qkv_rope_append(c->d_rows, nrows, c->ws,
                             c->b_qkv ? c->b_qkv + static_cast<int64_t>(l) * c->nqkv : nullptr, pl_qkv,
                             static_cast<int64_t>(nrows) * c->nqkv, dm, c->rope_tab,
                             c->page_table, c->kc + l * kv_layer, c->vc + l * kv_layer, c->q, st);
    }
    {
      const int asp = attn_pick_splits(nrows, g.n_kv_heads, g.max_ctx);
      TimedLaunch tl(c, st, "attn", c->step_attn_bytes, asp > 1 ? 2 : 1);
      launch_attn_decode(c->d_rows, nrows, c->q, c->kc + l * kv_layer, c->vc + l * kv_layer,
                         c->page_table, dm, c->attn, c->attn_ws, asp, c->attn_sched, st);
    }
    RET(run_gemm(c, tw_unused, c->tm_attn, d, nrows, Hhd, c->ws, d, sp_o, nullptr, nullptr, 0, d,
                 st, "gemm", c->w_o + l * n_o));
    {
      TimedLaunch tl(c, st, "norm", static_cast<double>(nrows) * d * (4.0 * pl_o + 10));
      launch_resid_norm(c->d_rows, nrows, c->ws, pl_o, static_cast<int64_t>(nrows) * d, dm, c->h,
                        c->norm_mlp + static_cast<int64_t>(l) * d, c->x, nullptr, st);
    }
    if (sp_gu == 1 && !c->silu_unfused) {  // SiLU(gate) * up in the epilogue
      RET(run_gemm(c, tw_unused, c->tm_x, 2 * dff, nrows, d, c->ws, 2 * dff, 1, nullptr, nullptr,
                   0, 2 * dff, st, "gemm", c->w_gu + l * n_gu, c->act, dff));
    } else {
      RET(run_gemm(c, tw_unused, c->tm_x, 2 * dff, nrows, d, c->ws, 2 * dff, sp_gu, nullptr,
                   nullptr, 0, 2 * dff, st, "gemm", c->w_gu + l * n_gu));
      TimedLaunch tl(c, st, "silu", static_cast<double>(nrows) * dff * (8.0 * sp_gu + 2));
      launch_silu_mul(c->d_rows, nrows, c->ws, sp_gu, static_cast<int64_t>(nrows) * 2 * dff, dm,
                      c->act, st);
    }
    RET(run_gemm(c, tw_unused, c->tm_act, d, nrows, dff, c->ws, d, sp_dn, nullptr, nullptr, 0,
                 d, st, "gemm", c->w_down + l * n_dn));
    {
      const bool last = (l == L - 1);
      TimedLaunch tl(c, st, "norm", static_cast<double>(nrows) * d * (4.0 * pl_dn + 10));
      launch_resid_norm(c->d_rows, nrows, c->ws, pl_dn, static_cast<int64_t>(nrows) * d, dm, c->h,
                        last ? c->norm_final : c->norm_attn + static_cast<int64_t>(l + 1) * d,
                        last ? c->xf : c->x, last ? c->d_out_index : nullptr, st);
    }
  }
  if (nsamp > 0) {
    const bool audio = (g.audio_base >= 0) && !full_logits;
    const bool one_slot = audio && hslot >= 0;
    const int M = one_slot ? g.codebook_size : (audio ? c->head_audio_rows : g.vocab);
    const bf16* wh = audio ? c->w_head_audio : nullptr;
    if (one_slot)  // packed 128-row tiles: slot k starts at tile k * codebook_size / 128
      wh += static_cast<int64_t>(hslot) * (g.codebook_size / 128) * (d / 64) * 8192;
    RET(run_gemm(c, c->tm_head_full, c->tm_xf, M, nsamp, d, c->logits, M, 1, nullptr, nullptr, 0,
                 M, st, "lm_head", wh));
    SampFusedArgs a{};
    a.rows = c->d_rows;
    a.sample_rows = c->d_sample_rows;
    a.n_sample = nsamp;
    a.logits = c->logits;
    a.ld = M;
    a.col_base = audio ? g.audio_base + (one_slot ? hslot * g.codebook_size : 0) : 0;
    a.token_store = c->token_store;
    a.max_ctx = g.max_ctx;
    a.slot_prompt_len = c->slot_prompt;
    a.slot_seed = c->slot_seed;
    a.slot_params = c->slot_params;
    a.audio_base = g.audio_base;
    a.codebook_size = g.codebook_size;
    a.frame_tokens = g.frame_tokens;
    a.vocab = g.vocab;
    a.tokens_out = c->d_tokens;
    a.err_flag = c->d_err;
    if (run_sampler) {
      const int span = g.audio_base >= 0 ? g.codebook_size : g.vocab;
      TimedLaunch tl(c, st, "sampler", static_cast<double>(nsamp) * span * 4);
      launch_sample_fused(a, st);
    }
  }
  CK(cudaGetLastError());
  return VOX_OK;
}

static int check_err_value(VoxCtx* c, int e) {
  if (e == 0) return VOX_OK;
  if (e == VOX_ERR_NONFINITE) return fail(c, e, "logits must not contain NaN or +inf");
  if (e == VOX_ERR_DEGENERATE) return fail(c, e, "all logits are -inf after truncation");
  return fail(c, e, "device error flag " + std::to_string(e));
}

// ---------------------------------------------------------------------------
// C-ABI
// ---------------------------------------------------------------------------
extern "C" {

int vox_abi_version(void) { return VOX_ABI_VERSION; }

const char* vox_last_error(const VoxCtx* ctx) {
  if (ctx) return ctx->err.c_str();
  return g_err.c_str();
}

static int validate_cfg(const VoxModelCfg* g) {
  if (g->n_layers < 1 || g->d_model % 64 || g->d_ff % 64 || g->head_dim % 2) return 0;
  if (!(g->head_dim == 64 || g->head_dim == 128)) return 0;
  if (g->n_heads % g->n_kv_heads) return 0;
  const int grp = g->n_heads / g->n_kv_heads;
  // GQA group: the q slot of the attention ring holds G * hd bf16 <= 1 KB
  if (grp < 1 || grp > 8 || grp * g->head_dim > 512) return 0;
  if ((g->n_heads * g->head_dim) % 64) return 0;
  // 8-token chunks; the attention smem ring holds 6 x 2 head-pages (<= 192 KB)
  // the attention kernel's mma tiling is built for 16-token pages
  if (g->page_size != 16 || g->max_rows < 1 || g->max_rows > 2048) return 0;
  if (g->n_codebooks < 0 || g->n_codebooks > 64 || g->ext_dim < 0 || g->ext_dim % 64) return 0;
  if (g->max_slots < 1 || g->n_pages < 1 || g->max_ctx < 2) return 0;
  if (g->detok_enabled) {
    if (g->audio_base < 0 || g->n_rates != 4 || g->latent_dim % 64 || g->decoder_dim % 1024)
      return 0;
    if (g->max_detok_frames < 4) return 0;
  }
  return 1;
}

static bool make_partition_streams(VoxCtx* c, int dt_want, int prio_lm, int prio_dt);

int vox_create(int device, const VoxModelCfg* cfg, uint64_t weight_seed, VoxCtx** out) {
  VoxCtx* c = nullptr;
  if (!cfg || !out) return fail(nullptr, VOX_ERR_INVALID, "null argument");
  if (!validate_cfg(cfg)) return fail(nullptr, VOX_ERR_INVALID, "invalid VoxModelCfg");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || device >= ndev)
    return fail(nullptr, VOX_ERR_NO_DEVICE, "no CUDA device");
  cudaDeviceProp prop;
  cudaGetDeviceProperties(&prop, device);
  if (prop.major != 10) return fail(nullptr, VOX_ERR_NO_DEVICE, "needs an sm_100 (B200) device");
  c = new VoxCtx();
  c->device = device;
  c->cfg = *cfg;
  c->seed = weight_seed;
  CK(cudaSetDevice(device));
  // The LM step is the throughput-critical path (every live stream waits on it);
  // detokenization has a chunk of playback time as slack.  With the LM stream
  // at the higher priority the CTA scheduler fills SMs from it first and detok
  // CTAs soak up the gaps (VOX_STREAM_PRIO=0: equal priorities, for A/B).
  int prio_lo = 0, prio_hi = 0;
  CK(cudaDeviceGetStreamPriorityRange(&prio_lo, &prio_hi));
  const bool prio = !(getenv("VOX_STREAM_PRIO") && atoi(getenv("VOX_STREAM_PRIO")) == 0);
  // Contexts that detokenize split the GPU by default: 16 SMs (two partition
  // granules) for the detok stream, the rest for the LM -- the serving step measured
  // 1.0-1.5% faster than sharing every SM (detok CTAs no longer hold SMs an LM
  // GEMM is waiting for; the LM step itself is as fast on 132 SMs).  VOX_DETOK_SMS=N
  // sets the size, 0 shares the whole GPU.  If the driver cannot make the partition
  // the default falls back to shared streams; an explicit request fails loudly.
  const char* dt_env = getenv("VOX_DETOK_SMS");
  const int dt_sms = dt_env ? atoi(dt_env) : (cfg->detok_enabled ? 16 : 0);
  if (dt_sms > 0 && make_partition_streams(c, dt_sms, prio ? prio_hi : prio_lo, prio_lo)) {
    // grids follow c->lm_sms / c->dt_sms per enqueue (SmBudgetScope)
  } else {
    if (dt_sms > 0 && dt_env) return fail(c, VOX_ERR_CUDA, "VOX_DETOK_SMS: green-context SM partition failed");
    CK(cudaStreamCreateWithPriority(&c->s_lm, cudaStreamNonBlocking, prio ? prio_hi : prio_lo));
    // (detokenizing on the LM stream, between decode steps, measured 4% slower than
    // this concurrent low-priority stream: profiles/detok_serial_ab_r02.txt)
    CK(cudaStreamCreateWithPriority(&c->s_dt, cudaStreamNonBlocking, prio_lo));
  }
  CK(cudaEventCreate(&c->epoch));
  c->dm.d = cfg->d_model;
  c->dm.n_heads = cfg->n_heads;
  c->dm.n_kv = cfg->n_kv_heads;
  c->dm.hd = cfg->head_dim;
  c->dm.dff = cfg->d_ff;
  c->dm.vocab = cfg->vocab;
  c->dm.eps = cfg->rms_eps;
  c->dm.page_size = cfg->page_size;
  c->dm.max_ctx = cfg->max_ctx;
  c->dm.n_pages = cfg->n_pages;
  int r = create_backbone(c);
  if (r == VOX_OK) r = create_buffers(c);
  c->dm.max_pages_per_slot = c->max_pages_per_slot;
  if (r == VOX_OK && cfg->detok_enabled) r = create_detok(c);
  if (r == VOX_OK) {
    cudaError_t e = cudaStreamSynchronize(c->s_lm);
    if (e != cudaSuccess) r = fail(c, VOX_ERR_CUDA, cudaGetErrorString(e));
  }
  if (r != VOX_OK) {
    std::string m = c->err;
    vox_destroy(c);
    return fail(nullptr, r, m);
  }
  CK(cudaEventRecord(c->epoch, c->s_lm));
  *out = c;
  return VOX_OK;
}

// Spatial split of the GPU between the LM step and detokenization: the detok
// stream gets a green context of `dt_want` SMs (rounded up to the partition
// granularity, 8 SMs on sm_90+), the LM stream one of the remaining SMs, so detok
// CTAs never hold SMs an LM kernel is waiting for.  CUDA graphs keep the partition
// of the stream they were captured on.  Returns false (and leaves the streams
// unset) when the driver lacks the API or the split fails.
static bool make_partition_streams(VoxCtx* c, int dt_want, int prio_lm, int prio_dt) {
  auto sym = [](const char* n) -> void* {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint(n, &fn, cudaEnableDefault, &q) != cudaSuccess || q != cudaDriverEntryPointSuccess)
      return nullptr;
    return fn;
  };
  auto getdev = reinterpret_cast<decltype(&cuDeviceGet)>(sym("cuDeviceGet"));
  auto getres = reinterpret_cast<decltype(&cuDeviceGetDevResource)>(sym("cuDeviceGetDevResource"));
  auto split = reinterpret_cast<decltype(&cuDevSmResourceSplitByCount)>(sym("cuDevSmResourceSplitByCount"));
  auto gendesc = reinterpret_cast<decltype(&cuDevResourceGenerateDesc)>(sym("cuDevResourceGenerateDesc"));
  auto mkctx = reinterpret_cast<decltype(&cuGreenCtxCreate)>(sym("cuGreenCtxCreate"));
  auto mkstream = reinterpret_cast<decltype(&cuGreenCtxStreamCreate)>(sym("cuGreenCtxStreamCreate"));
  if (!getdev || !getres || !split || !gendesc || !mkctx || !mkstream) return false;
  CUdevice dev;
  CUdevResource all{}, grp{}, rest{};
  unsigned nb = 1;
  if (getdev(&dev, c->device) != CUDA_SUCCESS || getres(dev, &all, CU_DEV_RESOURCE_TYPE_SM) != CUDA_SUCCESS ||
      split(&grp, &nb, &all, &rest, 0, static_cast<unsigned>(dt_want)) != CUDA_SUCCESS || nb != 1 ||
      rest.sm.smCount < 64)
    return false;
  CUdevResourceDesc d_dt, d_lm;
  if (gendesc(&d_dt, &grp, 1) != CUDA_SUCCESS || gendesc(&d_lm, &rest, 1) != CUDA_SUCCESS) return false;
  if (mkctx(&c->green_dt, d_dt, dev, CU_GREEN_CTX_DEFAULT_STREAM) != CUDA_SUCCESS ||
      mkctx(&c->green_lm, d_lm, dev, CU_GREEN_CTX_DEFAULT_STREAM) != CUDA_SUCCESS)
    return false;
  CUstream a = nullptr, b = nullptr;
  if (mkstream(&a, c->green_lm, CU_STREAM_NON_BLOCKING, prio_lm) != CUDA_SUCCESS ||
      mkstream(&b, c->green_dt, CU_STREAM_NON_BLOCKING, prio_dt) != CUDA_SUCCESS)
    return false;
  c->s_lm = reinterpret_cast<cudaStream_t>(a);
  c->s_dt = reinterpret_cast<cudaStream_t>(b);
  c->lm_sms = static_cast<int>(rest.sm.smCount);
  c->dt_sms = static_cast<int>(grp.sm.smCount);
  return true;
}

void vox_destroy(VoxCtx* c) {
  if (!c) return;
  cudaSetDevice(c->device);
  cudaDeviceSynchronize();
  for (auto& kv : c->graphs) cudaGraphExecDestroy(kv.second);
  for (auto& kv : c->step_graphs) cudaGraphExecDestroy(kv.second);
  for (auto& kv : c->detok_graphs) cudaGraphExecDestroy(kv.second);
  for (auto& t : c->tickets) {
    if (t.ev) cudaEventDestroy(t.ev);
    if (t.pcm_host) cudaFreeHost(t.pcm_host);
    if (t.stage_host) cudaFreeHost(t.stage_host);
  }
  for (auto& e : c->fwd_events) cudaEventDestroy(e);
  for (auto& t : c->trecs) {
    cudaEventDestroy(t.a);
    cudaEventDestroy(t.b);
  }
  void* dev_ptrs[] = {c->emb, c->norm_attn, c->norm_mlp, c->norm_final, c->w_qkv, c->w_o,
                      c->w_gu, c->w_down, c->w_head_audio, c->inv_freq, c->rope_tab, c->h, c->x, c->xf, c->q, c->attn, c->act,
                      c->ws, c->attn_ws, c->logits, c->kc, c->vc, c->token_store, c->page_table,
                      c->slot_prompt, c->slot_seed, c->slot_params, c->d_rows, c->attn_sched, c->d_sample_rows,
                      c->d_out_index, c->d_tokens, c->d_err, c->dstate, c->dx, c->dy, c->dbf,
                      c->d_dstage, c->d_pcm, c->dw.tabs, c->dw.in_dw_w, c->dw.in_dw_b,
                      c->dw.in_pw_w, c->dw.in_pw_b, c->dw.out_alpha, c->dw.out_w, c->b_qkv,
                      c->trace_buf, c->frame_store, c->ext, c->w_proj, c->d_links, c->chain_ctr};
  if (c->ev_xfer) cudaEventDestroy(c->ev_xfer);
  for (auto& e : c->ev_links)
    if (e) cudaEventDestroy(e);
  if (c->h_links) cudaFreeHost(c->h_links);
  for (void* p : dev_ptrs)
    if (p) cudaFree(p);
  if (c->cfg.detok_enabled && c->dw.tabs) {
    for (int b = 0; b < 4; ++b) {
      cudaFree(c->dw.up_alpha[b]);
      cudaFree(c->dw.up_w[b]);
      cudaFree(c->dw.up_b[b]);
      for (int u = 0; u < 3; ++u) {
        cudaFree(c->dw.ru_a1[b][u]);
        cudaFree(c->dw.ru_a2[b][u]);
        cudaFree(c->dw.ru_dw_w[b][u]);
        cudaFree(c->dw.ru_dw_b[b][u]);
        cudaFree(c->dw.ru_pw_w[b][u]);
        cudaFree(c->dw.ru_pw_b[b][u]);
      }
    }
  }
  for (auto& a : c->admit_stages) {
    if (a.host) cudaFreeHost(a.host);
    if (a.ev) cudaEventDestroy(a.ev);
  }
  for (auto& s : c->stages) {
    void* host_ptrs[] = {s.rows, s.sample_rows, s.out_index, s.tokens, s.err};
    for (void* p : host_ptrs)
      if (p) cudaFreeHost(p);
    if (s.ev) cudaEventDestroy(s.ev);
  }
  if (c->s_lm) cudaStreamDestroy(c->s_lm);
  if (c->s_dt && c->s_dt != c->s_lm) cudaStreamDestroy(c->s_dt);
  if (c->epoch) cudaEventDestroy(c->epoch);
  if (c->green_lm || c->green_dt) {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuGreenCtxDestroy", &fn, cudaEnableDefault, &q) == cudaSuccess && fn) {
      auto destroy = reinterpret_cast<decltype(&cuGreenCtxDestroy)>(fn);
      if (c->green_dt) destroy(c->green_dt);
      if (c->green_lm) destroy(c->green_lm);
    }
  }
  delete c;
}

// synthetic prompt id i of a request (oracle/workload.py: prompt_ids)
static int prompt_id(uint64_t req_seed, int i, int text_vocab) {
  return static_cast<int>(mix64(req_seed + 0x632BE59BD9B4E019ull * static_cast<uint64_t>(i + 1)) %
                          static_cast<uint64_t>(text_vocab));
}

int vox_admit(VoxCtx* c, uint64_t req_seed, int32_t prompt_len, int32_t target_len,
              const VoxSampling* params, int32_t* slot_out) {
  if (!c || !params || !slot_out) return fail(c, VOX_ERR_INVALID, "null argument");
  const VoxModelCfg& g = c->cfg;
  if (prompt_len < 1) return fail(c, VOX_ERR_INVALID_TOKEN_COUNT, "prompt_tokens must be >= 1");
  if (target_len < 1)
    return fail(c, VOX_ERR_INVALID_TOKEN_COUNT, "target_output_tokens must be >= 1");
  if (prompt_len + target_len > g.max_ctx)
    return fail(c, VOX_ERR_PROMPT_TOO_LONG, "prompt + target exceeds the context capacity");
  if (params->penalty_window < 0 || params->penalty_window > 256)
    return fail(c, VOX_ERR_INVALID, "penalty_window must be in [0, 256]");
  int slot = -1;
  for (int s = 0; s < g.max_slots; ++s)
    if (!c->slot_used[s]) {
      slot = s;
      break;
    }
  if (slot < 0) return fail(c, VOX_ERR_OUT_OF_MEMORY, "no free request slot");
  const int need = (prompt_len + target_len + g.page_size - 1) / g.page_size;
  if (need > static_cast<int>(c->free_pages.size()))
    return fail(c, VOX_ERR_OUT_OF_MEMORY, "KV page pool exhausted");
  std::vector<int> pages(need);
  for (int i = 0; i < need; ++i) {
    pages[i] = c->free_pages.back();
    c->free_pages.pop_back();
  }
  std::vector<int> pt(c->max_pages_per_slot, 0);
  std::copy(pages.begin(), pages.end(), pt.begin());
  std::vector<int> prompt(prompt_len);
  for (int i = 0; i < prompt_len; ++i) prompt[i] = prompt_id(req_seed, i, g.text_vocab);
  // Asynchronous admission: the slot's rows are copied from a pinned staging
  // ring in LM-stream order (before any forward that uses the slot), so an
  // arrival never stalls the host pipeline.
  cudaStream_t st = c->s_lm;
  AdmitStage& as = c->admit_stages[static_cast<size_t>(c->admit_seq++ %
                                                       static_cast<int64_t>(c->admit_stages.size()))];
  if (as.in_flight) CK(cudaEventSynchronize(as.ev));
  int* h_pt = reinterpret_cast<int*>(as.host);
  int* h_prompt = h_pt + c->max_pages_per_slot;
  std::copy(pt.begin(), pt.end(), h_pt);
  std::copy(prompt.begin(), prompt.end(), h_prompt);
  int* h_plen = h_prompt + g.max_ctx;
  *h_plen = prompt_len;
  uint64_t* h_seed = reinterpret_cast<uint64_t*>(as.host + c->admit_seed_off);
  *h_seed = req_seed;
  VoxSampling* h_par = reinterpret_cast<VoxSampling*>(as.host + c->admit_par_off);
  *h_par = *params;
  CK(cudaMemcpyAsync(c->page_table + static_cast<int64_t>(slot) * c->max_pages_per_slot, h_pt,
                     pt.size() * 4, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(c->token_store + static_cast<int64_t>(slot) * g.max_ctx, h_prompt,
                     prompt.size() * 4, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(c->slot_prompt + slot, h_plen, 4, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(c->slot_seed + slot, h_seed, 8, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(c->slot_params + slot, h_par, sizeof(VoxSampling), cudaMemcpyHostToDevice,
                     st));
  if (g.detok_enabled)
    CK(cudaMemsetAsync(c->dstate + static_cast<int64_t>(slot) * 2 * c->dd.state_floats, 0,
                       sizeof(float) * 2 * c->dd.state_floats, st));
  if (c->nfc > 0)
    CK(cudaMemsetAsync(c->frame_store + static_cast<int64_t>(slot) * g.max_ctx * c->nfc, 0xFF,
                       static_cast<size_t>(g.max_ctx) * c->nfc * 4, st));
  CK(cudaEventRecord(as.ev, st));
  as.in_flight = true;
  c->slot_used[slot] = 1;
  c->slot_pages[slot] = pages;
  c->h_prompt[slot] = prompt_len;
  c->h_target[slot] = target_len;
  c->slot_chunks[slot] = 0;
  c->slot_covered[slot] = 0;
  c->slot_last_fwd[slot] = -1;
  c->h_seed[slot] = req_seed;
  *slot_out = slot;
  return VOX_OK;
}

int vox_release(VoxCtx* c, int32_t slot) {
  if (!c || slot < 0 || slot >= c->cfg.max_slots || !c->slot_used[slot])
    return fail(c, VOX_ERR_CACHE_MISSING, "release of an unknown slot");
  auto& pages = c->slot_pages[slot];
  for (int i = static_cast<int>(pages.size()) - 1; i >= 0; --i) c->free_pages.push_back(pages[i]);
  pages.clear();
  c->slot_used[slot] = 0;
  return VOX_OK;
}

int vox_page_table(VoxCtx* c, int32_t slot, int32_t* out, int32_t cap, int32_t* n_out) {
  if (!c || slot < 0 || slot >= c->cfg.max_slots || !c->slot_used[slot])
    return fail(c, VOX_ERR_CACHE_MISSING, "unknown slot");
  const auto& pages = c->slot_pages[slot];
  const int n = static_cast<int>(pages.size());
  std::vector<int> dev(c->max_pages_per_slot);
  CK(cudaStreamSynchronize(c->s_lm));  // admission copies are stream-ordered
  CK(cudaMemcpy(dev.data(), c->page_table + static_cast<int64_t>(slot) * c->max_pages_per_slot,
                dev.size() * 4, cudaMemcpyDeviceToHost));
  for (int i = 0; i < n; ++i)
    if (dev[i] != pages[i]) return fail(c, VOX_ERR_CUDA, "device page table diverged from host");
  for (int i = 0; i < n && i < cap; ++i) out[i] = dev[i];
  if (n_out) *n_out = n;
  return VOX_OK;
}

int vox_read_tokens(VoxCtx* c, int32_t slot, int32_t pos, int32_t n, int32_t* out) {
  if (!c || slot < 0 || slot >= c->cfg.max_slots || pos < 0 || n < 0 || pos + n > c->cfg.max_ctx)
    return fail(c, VOX_ERR_INVALID, "bad token range");
  CK(cudaStreamSynchronize(c->s_lm));
  CK(cudaMemcpy(out, c->token_store + static_cast<int64_t>(slot) * c->cfg.max_ctx + pos,
                static_cast<size_t>(n) * 4, cudaMemcpyDeviceToHost));
  return VOX_OK;
}

int vox_write_tokens(VoxCtx* c, int32_t slot, int32_t pos, int32_t n, const int32_t* ids) {
  if (!c || !ids || slot < 0 || slot >= c->cfg.max_slots || !c->slot_used[slot] || pos < 0 ||
      n < 0 || pos + n > c->cfg.max_ctx)
    return fail(c, VOX_ERR_INVALID, "bad token range");
  for (int i = 0; i < n; ++i)
    if (ids[i] < 0 || ids[i] >= c->cfg.vocab) return fail(c, VOX_ERR_INVALID, "token id outside vocab");
  CK(cudaDeviceSynchronize());  // both streams may read the token store
  CK(cudaMemcpy(c->token_store + static_cast<int64_t>(slot) * c->cfg.max_ctx + pos, ids,
                static_cast<size_t>(n) * 4, cudaMemcpyHostToDevice));
  return VOX_OK;
}

int vox_write_frame(VoxCtx* c, int32_t slot, int32_t pos, int32_t n_pos, const int32_t* ids) {
  if (!c || !ids || c->nfc == 0 || slot < 0 || slot >= c->cfg.max_slots || !c->slot_used[slot] ||
      pos < 0 || n_pos < 0 || pos + n_pos > c->cfg.max_ctx)
    return fail(c, VOX_ERR_INVALID, "bad frame range");
  for (int i = 0; i < n_pos * c->nfc; ++i)
    if (ids[i] < -1 || ids[i] >= c->cfg.vocab) return fail(c, VOX_ERR_INVALID, "frame id outside vocab");
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(c->frame_store + (static_cast<int64_t>(slot) * c->cfg.max_ctx + pos) * c->nfc, ids,
                static_cast<size_t>(n_pos) * c->nfc * 4, cudaMemcpyHostToDevice));
  return VOX_OK;
}

int vox_read_frame(VoxCtx* c, int32_t slot, int32_t pos, int32_t n_pos, int32_t* out) {
  if (!c || !out || c->nfc == 0 || slot < 0 || slot >= c->cfg.max_slots || pos < 0 || n_pos < 0 ||
      pos + n_pos > c->cfg.max_ctx)
    return fail(c, VOX_ERR_INVALID, "bad frame range");
  CK(cudaStreamSynchronize(c->s_lm));
  CK(cudaMemcpy(out, c->frame_store + (static_cast<int64_t>(slot) * c->cfg.max_ctx + pos) * c->nfc,
                static_cast<size_t>(n_pos) * c->nfc * 4, cudaMemcpyDeviceToHost));
  return VOX_OK;
}

int vox_project_ext(VoxCtx* c, VoxCtx* src, int32_t n) {
  if (!c || !src || c->cfg.ext_dim <= 0 || src->cfg.d_model != c->cfg.ext_dim || n < 1 ||
      n > c->cfg.max_rows || n > src->cfg.max_rows || c->device != src->device)
    return fail(c, VOX_ERR_INVALID, "bad ext projection");
  auto& xm = c->ext_maps[src->xf];
  if (xm.empty() && !make_act_maps(c, xm, src->xf, src->cfg.d_model, src->cfg.max_rows))
    return fail(c, VOX_ERR_CUDA, "tensor map (ext source)");
  CK(cudaEventRecord(src->ev_xfer, src->s_lm));
  CK(cudaStreamWaitEvent(c->s_lm, src->ev_xfer, 0));
  const CUtensorMap& tw_unused = c->tm_head_full;
  const int M = c->cfg.d_model, K = c->cfg.ext_dim;
  // one split: the result lands as a single fp32 plane straight in ext[n][d]
  return run_gemm(c, tw_unused, xm, M, n, K, c->ext, M, 1, nullptr, nullptr, 0, M, c->s_lm, "gemm",
                  c->w_proj);
}

int vox_link_tokens(VoxCtx* dst, VoxCtx* src, const int32_t* links, int32_t n, int32_t offset,
                    int32_t mode) {
  VoxCtx* c = dst;  // error context of CK()
  if (!dst || !src || !links || n < 1 || n > dst->cfg.max_rows || (mode != 0 && mode != 1) ||
      (mode == 1 && dst->nfc == 0) || dst->device != src->device)
    return fail(dst, VOX_ERR_INVALID, "bad token links");
  for (int i = 0; i < n; ++i) {
    const int32_t* l = links + 4 * i;
    const int span = mode == 1 ? dst->nfc : 1;
    if (l[0] < 0 || l[0] >= dst->cfg.max_slots || l[1] < 0 || l[1] >= dst->cfg.max_ctx || l[2] < 0 ||
        l[2] >= src->cfg.max_slots || l[3] < 0 || l[3] + span > src->cfg.max_ctx)
      return fail(dst, VOX_ERR_INVALID, "token link out of range");
  }
  // pinned staging ring: no host sync (the entry is reused once its copy completed)
  const int e = static_cast<int>(dst->link_seq++ % 8);
  CK(cudaEventSynchronize(dst->ev_links[e]));
  int* hl = dst->h_links + static_cast<size_t>(e) * dst->cfg.max_rows * 4;
  int* dl = dst->d_links + static_cast<size_t>(e) * dst->cfg.max_rows * 4;
  std::memcpy(hl, links, static_cast<size_t>(n) * 16);
  CK(cudaEventRecord(src->ev_xfer, src->s_lm));
  CK(cudaStreamWaitEvent(dst->s_lm, src->ev_xfer, 0));
  CK(cudaMemcpyAsync(dl, hl, static_cast<size_t>(n) * 16, cudaMemcpyHostToDevice, dst->s_lm));
  launch_link_tokens(dl, n, src->token_store, src->cfg.max_ctx,
                     mode == 0 ? dst->token_store : dst->frame_store, dst->cfg.max_ctx, dst->nfc, offset, mode,
                     dst->s_lm);
  CK(cudaGetLastError());
  CK(cudaEventRecord(dst->ev_links[e], dst->s_lm));
  return VOX_OK;
}

// Disaggregated LM -> detok (reference engine.py:119-123,150-156): copy
// token-store spans of an LM context into a detokenizer context, possibly on another GPU,
// ordered after every forward already enqueued on the LM context and before the next
// work on the detok stream of `dst`.  Peer-accessible contexts (same device, or NVLink
// peers with access enabled here) use one gather kernel on the destination reading the
// source store through its device pointer; otherwise one cudaMemcpyPeerAsync per span.
int vox_copy_tokens(VoxCtx* dst, VoxCtx* src, const int32_t* spans, int32_t n) {
  VoxCtx* c = dst;
  if (!dst || !src || !spans || n < 1 || n > dst->cfg.max_rows) return fail(dst, VOX_ERR_INVALID, "bad token spans");
  for (int i = 0; i < n; ++i) {
    const int32_t* l = spans + 5 * i;
    if (l[0] < 0 || l[0] >= dst->cfg.max_slots || l[2] < 0 || l[2] >= src->cfg.max_slots || l[4] < 1 ||
        l[1] < 0 || l[1] + l[4] > dst->cfg.max_ctx || l[3] < 0 || l[3] + l[4] > src->cfg.max_ctx)
      return fail(dst, VOX_ERR_INVALID, "token span out of range");
  }
  bool peer = dst->device == src->device;
  if (!peer) {
    int can = 0;
    cudaDeviceCanAccessPeer(&can, dst->device, src->device);
    if (can) {
      CK(cudaSetDevice(dst->device));
      const cudaError_t pe = cudaDeviceEnablePeerAccess(src->device, 0);
      if (pe == cudaErrorPeerAccessAlreadyEnabled) cudaGetLastError();
      peer = pe == cudaSuccess || pe == cudaErrorPeerAccessAlreadyEnabled;
    }
  }
  CK(cudaSetDevice(src->device));
  CK(cudaEventRecord(src->ev_xfer, src->s_lm));
  CK(cudaSetDevice(dst->device));
  CK(cudaStreamWaitEvent(dst->s_dt, src->ev_xfer, 0));
  if (peer) {
    // one link per token (mode 0 of link_tokens_kernel), staged through the pinned ring
    const int e = static_cast<int>(dst->link_seq++ % 8);
    CK(cudaEventSynchronize(dst->ev_links[e]));
    int* hl = dst->h_links + static_cast<size_t>(e) * dst->cfg.max_rows * 4;
    int* dl = dst->d_links + static_cast<size_t>(e) * dst->cfg.max_rows * 4;
    int m = 0;
    for (int i = 0; i < n; ++i) {
      const int32_t* l = spans + 5 * i;
      for (int k = 0; k < l[4]; ++k) {
        if (m == dst->cfg.max_rows) return fail(dst, VOX_ERR_BATCH_TOO_LARGE, "more tokens than max_rows per copy");
        int* o = hl + 4 * m++;
        o[0] = l[0];
        o[1] = l[1] + k;
        o[2] = l[2];
        o[3] = l[3] + k;
      }
    }
    CK(cudaMemcpyAsync(dl, hl, static_cast<size_t>(m) * 16, cudaMemcpyHostToDevice, dst->s_dt));
    launch_link_tokens(dl, m, src->token_store, src->cfg.max_ctx, dst->token_store, dst->cfg.max_ctx, 0, 0, 0,
                       dst->s_dt);
    CK(cudaGetLastError());
    CK(cudaEventRecord(dst->ev_links[e], dst->s_dt));
    dst->launches++;
  } else {
    for (int i = 0; i < n; ++i) {
      const int32_t* l = spans + 5 * i;
      CK(cudaMemcpyPeerAsync(dst->token_store + static_cast<int64_t>(l[0]) * dst->cfg.max_ctx + l[1], dst->device,
                             src->token_store + static_cast<int64_t>(l[2]) * src->cfg.max_ctx + l[3], src->device,
                             static_cast<size_t>(l[4]) * 4, dst->s_dt));
    }
  }
  return VOX_OK;
}

int vox_slot_info(VoxCtx* c, int32_t slot, int32_t* prompt_len, int32_t* target_len) {
  if (!c || slot < 0 || slot >= c->cfg.max_slots || !c->slot_used[slot])
    return fail(c, VOX_ERR_CACHE_MISSING, "unknown slot");
  if (prompt_len) *prompt_len = c->h_prompt[slot];
  if (target_len) *target_len = c->h_target[slot];
  return VOX_OK;
}

int vox_forward(VoxCtx* c, const VoxRow* rows, int32_t n, uint32_t flags, float* logits_out,
                int32_t* tokens_out);

int vox_forward_steps(VoxCtx* c, const VoxRow* rows, int32_t n, int32_t steps, uint32_t flags) {
  if (!c || !rows || n <= 0 || steps < 1 || !(flags & VOX_FWD_SAMPLE) ||
      (flags & (VOX_FWD_FULL_LOGITS | VOX_FWD_SYNC)))
    return fail(c, VOX_ERR_INVALID, "bad multi-step forward");
  const VoxModelCfg& g = c->cfg;
  // every row: one distinct slot, sampled, the same step of the same prompt length
  // (the CSM depth decoder) -> steps 1.. run as one graph of [advance rows, step]
  bool uniform = steps > 1 && !(flags & VOX_FWD_NO_GRAPH) && !c->timing && !c->no_graphs;
  for (int i = 0; i < n && uniform; ++i) {
    const VoxRow& r = rows[i];
    if (!r.sample || r.slot < 0 || r.slot >= g.max_slots || !c->slot_used[r.slot]) uniform = false;
    else if (r.pos - c->h_prompt[r.slot] != rows[0].pos - c->h_prompt[rows[0].slot]) uniform = false;
    else {
      const int cap = static_cast<int>(c->slot_pages[r.slot].size()) * g.page_size;
      if (r.pos + steps - 1 >= cap || r.pos + steps >= g.max_ctx) uniform = false;
    }
  }
  if (uniform) {
    std::vector<int> sl(n);
    for (int i = 0; i < n; ++i) sl[i] = rows[i].slot;
    std::sort(sl.begin(), sl.end());
    for (int i = 1; i < n && uniform; ++i)
      if (sl[i] == sl[i - 1]) uniform = false;
  }
  if (!uniform) {
    std::vector<VoxRow> r(rows, rows + n);
    for (int k = 0; k < steps; ++k) {
      if (k > 0)
        for (auto& x : r) {
          ++x.pos;
          x.token = -1;  // the previous step's sample, from the token store
        }
      const int rc = vox_forward(c, r.data(), n, flags, nullptr, nullptr);
      if (rc != VOX_OK) return rc;
    }
    return VOX_OK;
  }
  // step 0 uploads the rows; steps 1.. advance them on the device
  int rc = vox_forward(c, rows, n, flags, nullptr, nullptr);
  if (rc != VOX_OK) return rc;
  int nrows = bucket_of(n);
  if (nrows < 0 || nrows > g.max_rows) nrows = n;
  int ns = bucket_of(n);
  if (ns < 0 || ns > nrows) ns = n;
  const bool run_sampler = true;
  auto hslot_of = [&](int k) {  // vox_forward's frame-slot rule at step k
    if (g.audio_base < 0 || g.frame_tokens <= 1 || g.codebook_size % 128) return -1;
    const int step = rows[0].pos + k + 1 - c->h_prompt[rows[0].slot];
    return ((step % g.frame_tokens) + g.frame_tokens) % g.frame_tokens;
  };
  cudaStream_t st = c->s_lm;
  auto key = std::make_tuple(nrows, ns, hslot_of(1), steps, run_sampler ? 1 : 0);
  auto it = c->step_graphs.find(key);
  if (it == c->step_graphs.end()) {
    const int64_t before = c->launches;
    cudaGraph_t graph;
    c->capturing = true;
    CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
    for (int k = 1; k < steps && rc == VOX_OK; ++k) {
      launch_advance_rows(c->d_rows, nrows, st);
      rc = enqueue_forward(c, nrows, ns, false, hslot_of(k), run_sampler);
    }
    cudaError_t ce = cudaStreamEndCapture(st, &graph);
    c->capturing = false;
    if (rc != VOX_OK) return rc;
    CK(ce);
    cudaGraphExec_t ex;
    CK(cudaGraphInstantiate(&ex, graph, 0));
    cudaGraphDestroy(graph);
    c->step_graph_launches[key] = c->launches - before;
    c->step_graphs[key] = ex;
    it = c->step_graphs.find(key);
    c->launches = before;
  }
  CK(cudaGraphLaunch(it->second, st));
  c->launches += c->step_graph_launches[key];
  {  // the logits buffer now holds the last step's head rows
    const int hs = hslot_of(steps - 1);
    c->last_logit_rows = n;
    c->last_logit_ld = hs >= 0 ? g.codebook_size : (g.audio_base >= 0 ? c->head_audio_rows : g.vocab);
    c->last_logit_base = g.audio_base >= 0 ? g.audio_base + (hs >= 0 ? hs * g.codebook_size : 0) : 0;
  }
  // error flag / ordering bookkeeping of one forward for the whole sequence
  FwdStage& sg = c->stages[static_cast<size_t>(c->stage_seq++ % static_cast<int64_t>(c->stages.size()))];
  if (sg.in_flight) {
    CK(cudaEventSynchronize(sg.ev));
    sg.in_flight = false;
    if (*sg.err) {
      const int e = *sg.err;
      *sg.err = 0;
      return check_err_value(c, e);
    }
  }
  CK(cudaMemcpyAsync(sg.err, c->d_err, sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(cudaMemsetAsync(c->d_err, 0, sizeof(int), st));
  CK(cudaEventRecord(sg.ev, st));
  sg.in_flight = true;
  const int64_t seq = ++c->fwd_seq;
  const int ei = static_cast<int>(seq % static_cast<int64_t>(c->fwd_events.size()));
  CK(cudaEventRecord(c->fwd_events[ei], st));
  c->fwd_event_seq[ei] = seq;
  for (int i = 0; i < n; ++i) c->slot_last_fwd[rows[i].slot] = seq;
  return VOX_OK;
}

int vox_forward(VoxCtx* c, const VoxRow* rows, int32_t n, uint32_t flags, float* logits_out,
                int32_t* tokens_out) {
  if (!c || (!rows && n > 0)) return fail(c, VOX_ERR_INVALID, "null argument");
  const VoxModelCfg& g = c->cfg;
  if (n <= 0) return fail(c, VOX_ERR_EMPTY_BATCH, "empty batch");
  if (n > g.max_rows) return fail(c, VOX_ERR_BATCH_TOO_LARGE, "batch exceeds max_rows");
  const bool want_logits = logits_out != nullptr;
  const bool full = (flags & VOX_FWD_FULL_LOGITS) != 0 || want_logits;
  if (want_logits && !(flags & VOX_FWD_FULL_LOGITS))
    return fail(c, VOX_ERR_INVALID, "logits_out requires VOX_FWD_FULL_LOGITS");
  int nsamp = 0;
  for (int i = 0; i < n; ++i) {
    const VoxRow& r = rows[i];
    if (r.slot < 0 || r.slot >= g.max_slots || !c->slot_used[r.slot])
      return fail(c, VOX_ERR_CACHE_MISSING, "row references an unknown slot");
    const int cap = static_cast<int>(c->slot_pages[r.slot].size()) * g.page_size;
    if (r.pos < 0 || r.pos + 1 >= g.max_ctx || r.pos >= cap)
      return fail(c, VOX_ERR_INVALID, "row position outside the reserved KV range");
    if (r.token >= g.vocab) return fail(c, VOX_ERR_INVALID, "token id outside the vocabulary");
    if (r.token == -2 && g.ext_dim <= 0)
      return fail(c, VOX_ERR_INVALID, "external input row on a ctx without an input projector");
    if (r.token < -2) return fail(c, VOX_ERR_INVALID, "bad token id");
    if (r.sample) {
      if (r.pos + 1 < c->h_prompt[r.slot])
        return fail(c, VOX_ERR_INVALID, "sampling row inside the prompt");
      ++nsamp;
    }
  }
  if (full && nsamp > std::min(g.max_rows, 256))
    return fail(c, VOX_ERR_BATCH_TOO_LARGE, "full-vocab logits limited to 256 rows");
  int nrows = full ? n : bucket_of(n);
  if (nrows < 0 || nrows > g.max_rows) nrows = n;  // no bucket fits: exact size
  int ns = nsamp == 0 ? 0 : (full ? nsamp : bucket_of(nsamp));
  if (ns < 0 || ns > nrows) ns = nsamp;
  // pinned staging ring entry (wait for its previous user)
  FwdStage& sg = c->stages[static_cast<size_t>(c->stage_seq++ % static_cast<int64_t>(c->stages.size()))];
  if (sg.in_flight) {
    CK(cudaEventSynchronize(sg.ev));
    sg.in_flight = false;
    if (*sg.err) {
      const int e = *sg.err;
      *sg.err = 0;
      return check_err_value(c, e);
    }
  }
  int k = 0;
  double attn_bytes = 0;
  // lowest position appended per slot in this forward (attention may read the
  // pages below it before the grid-dependency wait)
  std::map<int, int> fresh;
  for (int i = 0; i < n; ++i) {
    auto it = fresh.find(rows[i].slot);
    if (it == fresh.end()) fresh.emplace(rows[i].slot, rows[i].pos);
    else it->second = std::min(it->second, static_cast<int>(rows[i].pos));
  }
  for (int i = 0; i < nrows; ++i) {
    if (i < n) {
      sg.rows[i] = RowDev{rows[i].slot, rows[i].pos, rows[i].token, rows[i].sample,
                          fresh[rows[i].slot], i, {0, 0}};
      attn_bytes += static_cast<double>(rows[i].pos + 1) * g.n_kv_heads * g.head_dim * 4;
      if (rows[i].sample) {
        sg.sample_rows[k] = i;
        sg.out_index[i] = k++;
      } else {
        sg.out_index[i] = -1;
      }
    } else {
      sg.rows[i] = RowDev{-1, 0, -1, 0, 0, i, {0, 0}};
      sg.out_index[i] = -1;
    }
  }
  for (int j = k; j < ns; ++j) sg.sample_rows[j] = -1;  // sampler skips padding
  {  // attention order: longest context first (LPT), padding rows last
    std::vector<int> ord(n);
    for (int i = 0; i < n; ++i) ord[i] = i;
    std::stable_sort(ord.begin(), ord.end(),
                     [&](int a, int b) { return rows[a].pos > rows[b].pos; });
    for (int i = 0; i < n; ++i) sg.rows[i].attn_row = ord[i];
  }
  c->step_attn_bytes = attn_bytes;
  cudaStream_t st = c->s_lm;
  CK(cudaMemcpyAsync(c->d_rows, sg.rows, sizeof(RowDev) * nrows, cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(c->d_out_index, sg.out_index, sizeof(int) * nrows, cudaMemcpyHostToDevice,
                     st));
  if (ns > 0)
    CK(cudaMemcpyAsync(c->d_sample_rows, sg.sample_rows, sizeof(int) * ns,
                       cudaMemcpyHostToDevice, st));
  const bool use_graph = !(flags & VOX_FWD_NO_GRAPH) && !full && !c->timing && !c->no_graphs;
  // VOX_FWD_SAMPLE clear: the LM head still runs over the sampling rows (their
  // logits are the result), but K1 does not (the host samples: engine.py:294-303)
  const bool run_sampler = (flags & VOX_FWD_SAMPLE) != 0;
  // one frame slot for every sampled row -> that slot's head rows only
  int hslot = -1;
  if (!full && ns > 0 && g.audio_base >= 0 && g.frame_tokens > 1 && g.codebook_size % 128 == 0) {
    for (int i = 0; i < n; ++i) {
      if (!rows[i].sample) continue;
      const int step = rows[i].pos + 1 - c->h_prompt[rows[i].slot];
      const int k = ((step % g.frame_tokens) + g.frame_tokens) % g.frame_tokens;
      if (hslot == -1) hslot = k;
      else if (hslot != k) { hslot = -2; break; }
    }
    if (hslot < 0) hslot = -1;
  }
  int rc = VOX_OK;
  if (use_graph) {
    auto key = std::make_tuple(nrows, ns, hslot * 2 + (run_sampler ? 1 : 0));
    auto it = c->graphs.find(key);
    if (it == c->graphs.end()) {
      // eager pass (executes this step and sets kernel attributes), then capture
      rc = enqueue_forward(c, nrows, ns, false, hslot, run_sampler);
      if (rc != VOX_OK) return rc;
      CK(cudaStreamSynchronize(st));
      const int64_t before = c->launches;
      cudaGraph_t graph;
      c->capturing = true;
      CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
      rc = enqueue_forward(c, nrows, ns, false, hslot, run_sampler);
      cudaError_t ce = cudaStreamEndCapture(st, &graph);
      c->capturing = false;
      if (rc != VOX_OK) return rc;
      CK(ce);
      cudaGraphExec_t ex;
      CK(cudaGraphInstantiate(&ex, graph, 0));
      cudaGraphDestroy(graph);
      c->graph_launches[key] = c->launches - before;
      c->launches = before + c->graph_launches[key];  // the eager pass counted once
      c->graphs[key] = ex;
    } else {
      CK(cudaGraphLaunch(it->second, st));
      c->launches += c->graph_launches[key];
    }
  } else {
    rc = enqueue_forward(c, nrows, ns, full, full ? -1 : hslot, run_sampler);
    if (rc != VOX_OK) return rc;
  }
  {  // layout of the logits buffer this forward leaves behind (vox_read_logits)
    const bool audio = g.audio_base >= 0 && !full;
    const bool one_slot = audio && hslot >= 0;
    c->last_logit_rows = nsamp;
    c->last_logit_ld = one_slot ? g.codebook_size : (audio ? c->head_audio_rows : g.vocab);
    c->last_logit_base = audio ? g.audio_base + (one_slot ? hslot * g.codebook_size : 0) : 0;
  }
  if (nsamp > 0)
    CK(cudaMemcpyAsync(sg.tokens, c->d_tokens, sizeof(int) * nsamp, cudaMemcpyDeviceToHost, st));
  CK(cudaMemcpyAsync(sg.err, c->d_err, sizeof(int), cudaMemcpyDeviceToHost, st));
  // zero the flag in-stream: each forward's error is attributed to it alone
  CK(cudaMemsetAsync(c->d_err, 0, sizeof(int), st));
  CK(cudaEventRecord(sg.ev, st));
  sg.in_flight = true;
  const int64_t seq = ++c->fwd_seq;
  const int ei = static_cast<int>(seq % static_cast<int64_t>(c->fwd_events.size()));
  CK(cudaEventRecord(c->fwd_events[ei], st));
  c->fwd_event_seq[ei] = seq;
  for (int i = 0; i < n; ++i)
    if (rows[i].sample) c->slot_last_fwd[rows[i].slot] = seq;

  const bool sync = (flags & VOX_FWD_SYNC) || tokens_out || logits_out;
  if (sync) {
    CK(cudaEventSynchronize(sg.ev));
    sg.in_flight = false;
    const int e = *sg.err;
    *sg.err = 0;
    rc = check_err_value(c, e);
    if (rc != VOX_OK) return rc;
    if (tokens_out)
      for (int j = 0; j < nsamp; ++j) tokens_out[j] = sg.tokens[j];
    if (logits_out)
      CK(cudaMemcpy(logits_out, c->logits, sizeof(float) * static_cast<size_t>(nsamp) * g.vocab,
                    cudaMemcpyDeviceToHost));
  }
  return VOX_OK;
}

int vox_read_logits(VoxCtx* c, float* out, int32_t rows, int32_t cols, int32_t* n_rows,
                    int32_t* ld, int32_t* col_base) {
  if (!c) return fail(c, VOX_ERR_INVALID, "null ctx");
  if (n_rows) *n_rows = c->last_logit_rows;
  if (ld) *ld = c->last_logit_ld;
  if (col_base) *col_base = c->last_logit_base;
  if (!out) return VOX_OK;
  if (rows > c->last_logit_rows || cols != c->last_logit_ld)
    return fail(c, VOX_ERR_INVALID, "logits read outside the last forward's buffer");
  CK(cudaStreamSynchronize(c->s_lm));
  CK(cudaMemcpy(out, c->logits, sizeof(float) * static_cast<size_t>(rows) * cols,
                cudaMemcpyDeviceToHost));
  return VOX_OK;
}

int vox_forward_seq(VoxCtx* c, int64_t* seq) {
  if (!c || !seq) return fail(c, VOX_ERR_INVALID, "null argument");
  *seq = c->fwd_seq;
  return VOX_OK;
}

int vox_forward_wait(VoxCtx* c, int64_t seq) {
  if (!c) return fail(c, VOX_ERR_INVALID, "null ctx");
  if (seq <= 0) return VOX_OK;
  const int ei = static_cast<int>(seq % static_cast<int64_t>(c->fwd_events.size()));
  if (c->fwd_event_seq[ei] == seq) {
    CK(cudaEventSynchronize(c->fwd_events[ei]));
  } else if (seq > c->fwd_seq - static_cast<int64_t>(c->fwd_events.size())) {
    return fail(c, VOX_ERR_INVALID, "unknown forward sequence number");
  }  // older than the event ring: long complete (ring >> staging depth)
  return VOX_OK;
}

int vox_sample_logits(VoxCtx* c, const float* logits, int32_t n, int32_t vocab,
                      const VoxSampling* params, const int32_t* window_ids, int32_t wcap,
                      const int32_t* window_len, const uint64_t* seeds, const uint64_t* steps,
                      const int32_t* lo, const int32_t* hi, int32_t* tokens_out) {
  if (!c || !logits || !params || !seeds || !steps || !tokens_out)
    return fail(c, VOX_ERR_INVALID, "null argument");
  if (n <= 0) return fail(c, VOX_ERR_EMPTY_BATCH, "empty batch");
  if (wcap < 0 || wcap > 256) return fail(c, VOX_ERR_INVALID, "window capacity must be <= 256");
  float* d_log = nullptr;
  SampRowDesc* d_desc = nullptr;
  int *d_win = nullptr, *d_out = nullptr;
  std::vector<SampRowDesc> desc(n);
  int max_span = 1;
  for (int i = 0; i < n; ++i) {
    SampRowDesc& s = desc[i];
    s.logit_off = static_cast<int64_t>(i) * vocab;
    s.col_base = 0;
    s.lo = lo ? lo[i] : 0;
    s.hi = hi ? hi[i] : vocab;
    if (s.lo < 0 || s.hi > vocab || s.lo >= s.hi)
      return fail(c, VOX_ERR_INVALID, "bad candidate range");
    s.wlen = window_len ? std::min(window_len[i], wcap) : 0;
    s.woff = i * wcap;
    s.out_index = i;
    s.seed = seeds[i];
    s.step = steps[i];
    s.params = params[i];
    if (s.params.temperature < 0 || s.params.top_p <= 0 || s.params.top_p > 1 ||
        s.params.repetition_penalty < 1 || s.params.top_k < 0)
      return fail(c, VOX_ERR_INVALID, "invalid sampling parameters");
    max_span = std::max(max_span, s.hi - s.lo);
  }
  cudaStream_t st = c->s_lm;
  CK(dalloc(&d_log, static_cast<size_t>(n) * vocab));
  CK(dalloc(&d_desc, static_cast<size_t>(n)));
  CK(dalloc(&d_win, static_cast<size_t>(n) * std::max(wcap, 1)));
  CK(dalloc(&d_out, static_cast<size_t>(n)));
  CK(cudaMemcpyAsync(d_log, logits, sizeof(float) * n * static_cast<size_t>(vocab),
                     cudaMemcpyHostToDevice, st));
  CK(cudaMemcpyAsync(d_desc, desc.data(), sizeof(SampRowDesc) * n, cudaMemcpyHostToDevice, st));
  if (window_ids && wcap > 0)
    CK(cudaMemcpyAsync(d_win, window_ids, sizeof(int) * n * static_cast<size_t>(wcap),
                       cudaMemcpyHostToDevice, st));
  {
    TimedLaunch tl(c, st, "sampler", static_cast<double>(n) * max_span * 4);
    launch_sample_desc(d_log, d_desc, n, d_win, d_out, c->d_err, max_span, st);
  }
  CK(cudaGetLastError());
  CK(cudaMemcpyAsync(tokens_out, d_out, sizeof(int) * n, cudaMemcpyDeviceToHost, st));
  int errv = 0;
  CK(cudaMemcpyAsync(&errv, c->d_err, sizeof(int), cudaMemcpyDeviceToHost, st));
  CK(cudaMemsetAsync(c->d_err, 0, sizeof(int), st));
  CK(cudaStreamSynchronize(st));
  cudaFree(d_log);
  cudaFree(d_desc);
  cudaFree(d_win);
  cudaFree(d_out);
  return check_err_value(c, errv);
}

// ---------------------------------------------------------------------------
// detokenizer
// ---------------------------------------------------------------------------
static int enqueue_detok(VoxCtx* c, int n_req, int n_lat) {
  SmBudgetScope sms(c->dt_sms > 0 ? c->dt_sms : c->lm_sms);
  const DetokDims& dd = c->dd;
  DetokW& w = c->dw;
  cudaStream_t st = c->s_dt;
  const DetokReq* reqs = reinterpret_cast<const DetokReq*>(c->d_dstage + 8);
  const int L = dd.latent, D0 = dd.dec;
  int stage = 0;
#define DSTOP(buf)                                   \
  do {                                               \
    c->dbg_last = (buf);                             \
    if (++stage >= c->detok_stop) return VOX_OK;     \
  } while (0)
  {
    TimedLaunch tl(c, st, "detok_elt", static_cast<double>(n_lat) * L * 2);
    launch_vq_dwconv(reqs, n_req, n_lat, c->token_store, w.tabs, w.in_dw_w, w.in_dw_b, c->dstate,
                     dd, c->dbf, st);
  }
  DSTOP(nullptr);
  std::map<int, CUtensorMap> xm;
  if (!make_act_maps(c, xm, c->dbf, L, n_lat)) return fail(c, VOX_ERR_CUDA, "tmap detok act");
  RET(run_gemm(c, w.tm_in_pw, xm, D0, n_lat, L, c->dx, D0, 1, w.in_pw_b, nullptr, 0, D0, st,
               "detok_gemm"));
  DSTOP(c->dx);
  float* x = c->dx;
  float* y = c->dy;
  int up = 1;
  const int dils[3] = {1, 3, 9};
  for (int b = 0; b < 4; ++b) {
    const int Ci = dd.ch[b], Co = dd.ch[b + 1], s = dd.rates[b];
    const int rows = n_lat * up;
    {
      TimedLaunch tl(c, st, "detok_elt", static_cast<double>(rows) * Ci * 8);
      if (snake_upcat_tiled_supported(up) && !c->detok_unfused)
        launch_snake_upcat_tiled(reqs, rows, up, x, Ci, w.up_alpha[b], c->dstate, dd.off_up[b], dd,
                                 c->dbf, st);
      else
        launch_snake_upcat(reqs, n_req, rows, up, x, Ci, w.up_alpha[b], c->dstate, dd.off_up[b], dd,
                           c->dbf, st);
    }
    DSTOP(nullptr);
    std::map<int, CUtensorMap> um;
    if (!make_act_maps(c, um, c->dbf, 2 * Ci, rows)) return fail(c, VOX_ERR_CUDA, "tmap up");
    RET(run_gemm(c, w.tm_up[b], um, s * Co, rows, 2 * Ci, y, static_cast<int64_t>(s) * Co, 1,
                 w.up_b[b], nullptr, 0, s * Co, st, "detok_gemm"));
    std::swap(x, y);
    DSTOP(x);
    up *= s;
    const int rows2 = n_lat * up;
    std::map<int, CUtensorMap> rm;
    if (!make_act_maps(c, rm, c->dbf, Co, rows2)) return fail(c, VOX_ERR_CUDA, "tmap ru");
    for (int u = 0; u < 3; ++u) {
      if (ru_fused_supported(Co, up) && !c->detok_unfused) {
        TimedLaunch tl(c, st, "detok_ru", static_cast<double>(rows2) * Co * 8);
        launch_ru_fused(reqs, rows2, up, x, y, Co, dils[u], w.ru_a1[b][u], w.ru_dw_w[b][u],
                        w.ru_dw_b[b][u], w.ru_a2[b][u], w.ru_pw_w[b][u], w.ru_pw_b[b][u],
                        c->dstate, dd.off_ru[b][u], dd, st);
        std::swap(x, y);
        DSTOP(nullptr);
        DSTOP(x);
        continue;
      }
      {
        TimedLaunch tl(c, st, "detok_elt", static_cast<double>(rows2) * Co * 6);
        if (ru_prep_tiled_supported(Co, up) && !c->detok_unfused)
          launch_ru_prep_tiled(reqs, rows2, up, x, Co, dils[u], w.ru_a1[b][u], w.ru_dw_w[b][u],
                               w.ru_dw_b[b][u], w.ru_a2[b][u], c->dstate, dd.off_ru[b][u], dd,
                               c->dbf, st);
        else
          launch_ru_prep(reqs, n_req, rows2, up, x, Co, dils[u], w.ru_a1[b][u], w.ru_dw_w[b][u],
                         w.ru_dw_b[b][u], w.ru_a2[b][u], c->dstate, dd.off_ru[b][u], dd, c->dbf,
                         st);
      }
      DSTOP(nullptr);
      RET(run_gemm(c, w.tm_ru[b][u], rm, Co, rows2, Co, x, Co, 1, w.ru_pw_b[b][u], x, Co, Co, st,
                   "detok_gemm"));
      DSTOP(x);
    }
  }
  {
    const int rows = n_lat * up;
    TimedLaunch tl(c, st, "detok_elt", static_cast<double>(rows) * dd.ch[4] * 4);
    if (detok_out_tiled_supported(dd.ch[4], up) && !c->detok_unfused)
      launch_detok_out_tiled(reqs, rows, up, x, dd.ch[4], w.out_alpha, w.out_w, w.out_b,
                             c->dstate, dd.off_out, dd, c->d_pcm, st);
    else
      launch_detok_out(reqs, n_req, rows, up, x, dd.ch[4], w.out_alpha, w.out_w, w.out_b,
                       c->dstate, dd.off_out, dd, c->d_pcm, st);
  }
  CK(cudaGetLastError());
  return VOX_OK;
}

int vox_detok(VoxCtx* c, const VoxWindow* win, int32_t n, float* pcm_out, int32_t* n_samples,
              int64_t* ticket) {
  if (!c || (!win && n > 0)) return fail(c, VOX_ERR_INVALID, "null argument");
  const VoxModelCfg& g = c->cfg;
  if (!g.detok_enabled) return fail(c, VOX_ERR_INVALID, "detokenizer disabled in this context");
  if (n <= 0) return fail(c, VOX_ERR_EMPTY_BATCH, "empty detok batch");
  const int ft = g.frame_tokens;
  int hop = 1;
  for (int b = 0; b < 4; ++b) hop *= g.rates[b];
  const int frame_samples = 4 * hop;
  // ticket (its pinned staging/PCM buffers are reused only after its event)
  const int64_t tid = c->next_ticket;
  Ticket& tk = c->tickets[static_cast<size_t>(tid % static_cast<int64_t>(c->tickets.size()))];
  if (tk.id >= 0) CK(cudaEventSynchronize(tk.ev));
  int32_t* hdr = reinterpret_cast<int32_t*>(tk.stage_host);
  DetokReq* hr = reinterpret_cast<DetokReq*>(tk.stage_host + 8);
  int lat = 0, pcm = 0;
  int64_t wait_seq = -1;
  std::vector<int> seen;
  for (int i = 0; i < n; ++i) {
    const VoxWindow& w = win[i];
    if (w.slot < 0 || w.slot >= g.max_slots || !c->slot_used[w.slot])
      return fail(c, VOX_ERR_CACHE_MISSING, "detokenize without cache for request slot");
    if (std::find(seen.begin(), seen.end(), w.slot) != seen.end())
      return fail(c, VOX_ERR_INVALID, "a request appears twice in one detok batch");
    seen.push_back(w.slot);
    if (w.new_tokens < 1 || w.new_tokens > w.length || w.start < 0)
      return fail(c, VOX_ERR_WINDOW_RULE, "window new_tokens outside the window");
    const int g0 = w.start + w.length - w.new_tokens;
    if (g0 != c->slot_covered[w.slot] || g0 % ft != 0)
      return fail(c, VOX_ERR_WINDOW_RULE,
                  "stateful detokenizer needs in-order, frame-aligned windows");
    if (w.start + w.length > c->h_target[w.slot])
      return fail(c, VOX_ERR_WINDOW_RULE, "window beyond the request's generated tokens");
    DetokReq& q = hr[i];
    q.slot = w.slot;
    q.f0 = g0 / ft;
    q.nf = (w.new_tokens + ft - 1) / ft;
    q.lat_off = lat;
    q.parity = c->slot_chunks[w.slot] & 1;
    q.prompt_len = c->h_prompt[w.slot];
    q.n_tokens = w.start + w.length;
    q.pcm_off = pcm;
    q.n_samples = static_cast<int>((static_cast<int64_t>(w.new_tokens) * frame_samples) / ft);
    lat += 4 * q.nf;
    pcm += q.n_samples;
    wait_seq = std::max(wait_seq, c->slot_last_fwd[w.slot]);
    if (n_samples) n_samples[i] = q.n_samples;
  }
  if (lat > g.max_detok_frames)
    return fail(c, VOX_ERR_BATCH_TOO_LARGE, "detok batch exceeds max_detok_frames");
  hdr[0] = n;
  hdr[1] = lat;
  c->next_ticket++;
  // LM -> detok dependency: the forward that produced the windows' last tokens
  if (wait_seq >= 0) {
    const int ei = static_cast<int>(wait_seq % static_cast<int64_t>(c->fwd_events.size()));
    if (c->fwd_event_seq[ei] == wait_seq) CK(cudaStreamWaitEvent(c->s_dt, c->fwd_events[ei], 0));
    else CK(cudaStreamWaitEvent(c->s_dt, c->fwd_events[c->fwd_seq % c->fwd_events.size()], 0));
  }
  const size_t stage_bytes = 8 + sizeof(DetokReq) * n;
  CK(cudaMemcpyAsync(c->d_dstage, tk.stage_host, stage_bytes, cudaMemcpyHostToDevice, c->s_dt));
  // one CUDA graph per latent-frame bucket (power of two): the kernels read the
  // real request count / frame count from the staged header and skip padding
  int nb = 4;
  while (nb < lat) nb <<= 1;
  const bool use_graph = !c->timing && c->detok_stop >= (1 << 30) && nb <= g.max_detok_frames;
  if (use_graph) {
    auto it = c->detok_graphs.find(nb);
    if (it == c->detok_graphs.end()) {
      RET(enqueue_detok(c, n, nb));  // executes this call eagerly (sets kernel attributes)
      const int64_t before = c->launches;
      cudaGraph_t graph;
      c->capturing = true;
      CK(cudaStreamBeginCapture(c->s_dt, cudaStreamCaptureModeThreadLocal));
      const int rc = enqueue_detok(c, n, nb);
      const cudaError_t ce = cudaStreamEndCapture(c->s_dt, &graph);
      c->capturing = false;
      if (rc != VOX_OK) return rc;
      CK(ce);
      cudaGraphExec_t ex;
      CK(cudaGraphInstantiate(&ex, graph, 0));
      cudaGraphDestroy(graph);
      c->detok_graph_launches[nb] = c->launches - before;
      c->launches = before;
      c->detok_graphs[nb] = ex;
    } else {
      CK(cudaGraphLaunch(it->second, c->s_dt));
      c->launches += c->detok_graph_launches[nb];
    }
  } else {
    RET(enqueue_detok(c, n, lat));
  }
  CK(cudaMemcpyAsync(tk.pcm_host, c->d_pcm, sizeof(float) * pcm, cudaMemcpyDeviceToHost, c->s_dt));
  CK(cudaEventRecord(tk.ev, c->s_dt));
  tk.id = tid;
  tk.total = pcm;
  for (int i = 0; i < n; ++i) {
    c->slot_chunks[win[i].slot] += 1;
    c->slot_covered[win[i].slot] += win[i].new_tokens;
  }
  if (ticket) *ticket = tid;
  if (pcm_out) {
    CK(cudaEventSynchronize(tk.ev));
    std::memcpy(pcm_out, tk.pcm_host, sizeof(float) * pcm);
  }
  return VOX_OK;
}

int vox_ticket_query(VoxCtx* c, int64_t ticket, int32_t* done, double* t_ms) {
  if (!c) return fail(c, VOX_ERR_INVALID, "null ctx");
  Ticket& tk = c->tickets[static_cast<size_t>(ticket % static_cast<int64_t>(c->tickets.size()))];
  if (tk.id != ticket) return fail(c, VOX_ERR_INVALID, "stale ticket");
  cudaError_t e = cudaEventQuery(tk.ev);
  if (e == cudaErrorNotReady) {
    if (done) *done = 0;
    return VOX_OK;
  }
  CK(e);
  if (done) *done = 1;
  if (t_ms) {
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, c->epoch, tk.ev));
    *t_ms = ms;
  }
  return VOX_OK;
}

int vox_ticket_pcm(VoxCtx* c, int64_t ticket, const float** pcm, int32_t* total) {
  if (!c) return fail(c, VOX_ERR_INVALID, "null ctx");
  Ticket& tk = c->tickets[static_cast<size_t>(ticket % static_cast<int64_t>(c->tickets.size()))];
  if (tk.id != ticket) return fail(c, VOX_ERR_INVALID, "stale ticket");
  CK(cudaEventSynchronize(tk.ev));
  if (pcm) *pcm = tk.pcm_host;
  if (total) *total = tk.total;
  return VOX_OK;
}

int vox_clock_reset(VoxCtx* c) {
  if (!c) return fail(c, VOX_ERR_INVALID, "null ctx");
  CK(cudaEventRecord(c->epoch, c->s_lm));
  CK(cudaEventSynchronize(c->epoch));
  return VOX_OK;
}

int vox_synchronize(VoxCtx* c) {
  if (!c) return fail(c, VOX_ERR_INVALID, "null ctx");
  CK(cudaStreamSynchronize(c->s_lm));
  CK(cudaStreamSynchronize(c->s_dt));
  for (auto& s : c->stages) {
    if (s.in_flight) s.in_flight = false;
    if (*s.err) {
      const int e = *s.err;
      *s.err = 0;
      return check_err_value(c, e);
    }
  }
  return VOX_OK;
}

int vox_streams(VoxCtx* c, void** lm, void** dt) {
  if (!c) return fail(c, VOX_ERR_INVALID, "null ctx");
  if (lm) *lm = c->s_lm;
  if (dt) *dt = c->s_dt;
  return VOX_OK;
}

int vox_timing_enable(VoxCtx* c, int32_t on) {
  if (!c) return fail(c, VOX_ERR_INVALID, "null ctx");
  CK(cudaDeviceSynchronize());
  for (auto& t : c->trecs) {
    cudaEventDestroy(t.a);
    cudaEventDestroy(t.b);
  }
  c->trecs.clear();
  c->timing = on != 0;
  return VOX_OK;
}

int vox_timing_read(VoxCtx* c, const char* name, double* total_ms, int64_t* launches,
                    double* bytes) {
  if (!c || !name) return fail(c, VOX_ERR_INVALID, "null argument");
  CK(cudaDeviceSynchronize());
  double ms = 0, by = 0;
  int64_t cnt = 0;
  for (auto& t : c->trecs) {
    if (t.cls != name) continue;
    float e = 0.f;
    CK(cudaEventElapsedTime(&e, t.a, t.b));
    ms += e;
    by += t.bytes;
    ++cnt;
  }
  if (total_ms) *total_ms = ms;
  if (launches) *launches = cnt;
  if (bytes) *bytes = by;
  return VOX_OK;
}

}  // extern "C" (trace setters below are C++ symbols of the kernel TUs)
namespace vox {
void trace_set_attn(unsigned long long*);
void trace_set_chain(unsigned long long*);
void trace_set_detok_fused(unsigned long long*);
void trace_set_detok(unsigned long long*);
void trace_set_gemm(unsigned long long*);
void trace_set_lm(unsigned long long*);
void trace_set_sampler(unsigned long long*);
}  // namespace vox
static void trace_set_all(unsigned long long* b) {
  vox::trace_set_attn(b);
  vox::trace_set_chain(b);
  vox::trace_set_detok_fused(b);
  vox::trace_set_detok(b);
  vox::trace_set_gemm(b);
  vox::trace_set_lm(b);
  vox::trace_set_sampler(b);
}
extern "C" {

int vox_trace_arm(VoxCtx* c, int64_t capacity) {
  if (!c || capacity < 1) return fail(c, VOX_ERR_INVALID, "bad trace arguments");
  CK(cudaDeviceSynchronize());
  if (c->trace_buf) cudaFree(c->trace_buf);
  c->trace_cap = capacity;
  CK(cudaMalloc(&c->trace_buf, (2 + 3 * capacity) * 8));
  unsigned long long hdr[2] = {0ull, static_cast<unsigned long long>(capacity)};
  CK(cudaMemcpy(c->trace_buf, hdr, 16, cudaMemcpyHostToDevice));
  trace_set_all(c->trace_buf);
  return VOX_OK;
}

int vox_trace_read(VoxCtx* c, void* records, int64_t max_records, int64_t* n_records) {
  if (!c || !records || !n_records) return fail(c, VOX_ERR_INVALID, "null argument");
  if (!c->trace_buf) return fail(c, VOX_ERR_INVALID, "trace not armed");
  CK(cudaDeviceSynchronize());
  trace_set_all(nullptr);
  unsigned long long n = 0;
  CK(cudaMemcpy(&n, c->trace_buf, 8, cudaMemcpyDeviceToHost));
  n = std::min<unsigned long long>(n, static_cast<unsigned long long>(std::min(max_records, c->trace_cap)));
  CK(cudaMemcpy(records, c->trace_buf + 2, n * 24, cudaMemcpyDeviceToHost));
  *n_records = static_cast<int64_t>(n);
  cudaFree(c->trace_buf);
  c->trace_buf = nullptr;
  return VOX_OK;
}

int vox_launch_count(VoxCtx* c, int64_t* launches) {
  if (!c || !launches) return fail(c, VOX_ERR_INVALID, "null argument");
  *launches = c->launches;
  return VOX_OK;
}

int vox_sm_partition(VoxCtx* c, int32_t* lm_sms, int32_t* detok_sms) {
  if (!c || !lm_sms || !detok_sms) return fail(c, VOX_ERR_INVALID, "null argument");
  *lm_sms = c->lm_sms;
  *detok_sms = c->dt_sms;
  return VOX_OK;
}

int vox_debug_detok(VoxCtx* c, int32_t stop_after, float* out, size_t n_floats, uint16_t* bf_out,
                    size_t n_bf) {
  if (!c) return fail(c, VOX_ERR_INVALID, "null ctx");
  CK(cudaDeviceSynchronize());
  if (out && c->dbg_last) CK(cudaMemcpy(out, c->dbg_last, n_floats * 4, cudaMemcpyDeviceToHost));
  if (bf_out) CK(cudaMemcpy(bf_out, c->dbf, n_bf * 2, cudaMemcpyDeviceToHost));
  c->detok_stop = stop_after > 0 ? stop_after : (1 << 30);
  return VOX_OK;
}

int vox_gemm_test(VoxCtx* c, const uint16_t* w, const uint16_t* x, const float* bias, int32_t M,
                  int32_t N, int32_t K, int32_t splits, int32_t iters, float* out,
                  double* mean_ms) {
  if (!c || !w || !x || !out) return fail(c, VOX_ERR_INVALID, "null argument");
  if (M < 1 || N < 1 || K < 64 || K % 64 || splits < 1 || iters < 1)
    return fail(c, VOX_ERR_INVALID, "bad GEMM shape");
  bf16 *dw = nullptr, *dx = nullptr;
  float *dout = nullptr, *db = nullptr;
  CK(dalloc(&dw, static_cast<size_t>(M) * K));
  CK(dalloc(&dx, static_cast<size_t>(N) * K));
  CK(dalloc(&dout, static_cast<size_t>(splits) * N * M));
  CK(cudaMemset(dout, 0, static_cast<size_t>(splits) * N * M * 4));
  CK(cudaMemcpy(dw, w, static_cast<size_t>(M) * K * 2, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dx, x, static_cast<size_t>(N) * K * 2, cudaMemcpyHostToDevice));
  if (bias) {
    CK(dalloc(&db, static_cast<size_t>(M)));
    CK(cudaMemcpy(db, bias, static_cast<size_t>(M) * 4, cudaMemcpyHostToDevice));
  }
  CUtensorMap tw;
  std::map<int, CUtensorMap> xm;
  if (!make_tmap_bf16(&tw, dw, K, M, K * 2ull, 128) || !make_act_maps(c, xm, dx, K, N))
    return fail(c, VOX_ERR_CUDA, "tensor map (gemm test)");
  // Each timed iteration starts with L2 flushed (a 512 MB read between
  // iterations, outside the event pair): weights stream from HBM as they do
  // inside a decode step, where 6.6 GB of weights pass through a 126 MB L2.
  void* flush = nullptr;
  uint32_t* sink = nullptr;
  const size_t flush_bytes = 512ull << 20;
  CK(cudaMalloc(&flush, flush_bytes));
  CK(cudaMemset(flush, 0, flush_bytes));
  CK(cudaMalloc(&sink, 148 * 8 * 4));
  // VOX_GEMM_PACKED_TEST=1: stream W from the packed tile layout (the decode path)
  bf16* wpk = nullptr;
  bf16* xpk = nullptr;
  if (getenv("VOX_GEMM_XPACKED_TEST") && atoi(getenv("VOX_GEMM_XPACKED_TEST")) == 1) {
    CK(dalloc(&xpk, static_cast<size_t>(packed_elems(N, K))));
    launch_pack_bf16(dx, xpk, N, K, c->s_lm);
    CK(cudaStreamSynchronize(c->s_lm));
    c->test_x_packed = xpk;
  }
  if (getenv("VOX_GEMM_PACKED_TEST") && atoi(getenv("VOX_GEMM_PACKED_TEST")) == 1) {
    CK(dalloc(&wpk, static_cast<size_t>(packed_elems(M, K))));
    launch_pack_bf16(dw, wpk, M, K, c->s_lm);
    CK(cudaStreamSynchronize(c->s_lm));
  }
  unsigned long long* dbg = nullptr;
  const size_t dbg_n = 8ull * 4096;
  if (getenv("VOX_GEMM_DBG") && atoi(getenv("VOX_GEMM_DBG")) == 1) {
    CK(cudaMalloc(&dbg, dbg_n * 8));
    CK(cudaMemset(dbg, 0, dbg_n * 8));
    c->test_dbg = dbg;
  }
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  int rc = VOX_OK;
  // fp32 planes the GEMM leaves: every split gets ceil(n_kb / splits) k-blocks
  const int per_split = (K / 64 + splits - 1) / splits;
  const int planes = (K / 64 + per_split - 1) / per_split;
  double total_ms = 0.0;
  for (int it = 0; it < iters && rc == VOX_OK; ++it) {
    launch_l2_flush(flush, flush_bytes, sink, c->s_lm);  // clean L2 lines, not dirty ones
    CK(cudaEventRecord(a, c->s_lm));
    // VOX_GEMM_PERSIST_TEST=1|2: the codec detokenizers' persistent kernel (MT 1|2), one split
    const int pt = getenv("VOX_GEMM_PERSIST_TEST") ? atoi(getenv("VOX_GEMM_PERSIST_TEST")) : 0;
    if (pt == 1 || pt == 2) {
      CUtensorMap tx;
      if (splits != 1 || !make_tmap_bf16(&tx, dx, K, N, K * 2ull, 128))
        return fail(c, VOX_ERR_INVALID, "persistent GEMM test: one split, tensor map");
      GemmArgs ga{};
      ga.M = M;
      ga.N = N;
      ga.K = K;
      ga.out = dout;
      ga.ldo = M;
      ga.bias = db;
      ga.m_valid = M;
      const cudaError_t e = gemm_launch_persist(tw, tx, ga, 128, pt, c->s_lm);
      if (e != cudaSuccess) return fail(c, VOX_ERR_CUDA, std::string("persistent gemm: ") + cudaGetErrorString(e));
    } else {
      rc = run_gemm(c, tw, xm, M, N, K, dout, M, splits, splits == 1 ? db : nullptr, nullptr, 0, M,
                    c->s_lm, "gemm", wpk, nullptr, 0);
    }
    CK(cudaEventRecord(b, c->s_lm));
    CK(cudaEventSynchronize(b));
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, a, b));
    if (it > 0 || iters == 1) total_ms += ms;
  }
  if (mean_ms) *mean_ms = total_ms / (iters > 1 ? iters - 1 : 1);
  if (dbg) {  // per-CTA stamps of the last launch: mean deltas (cycles) + SM spread
    std::vector<unsigned long long> h(dbg_n);
    CK(cudaMemcpy(h.data(), dbg, dbg_n * 8, cudaMemcpyDeviceToHost));
    double sum[6] = {0}, ghz = 0;
    int n = 0;
    unsigned long long gmin = ~0ull, gmax = 0, dmax = 0, g0 = ~0ull;
    for (size_t i = 0; i < dbg_n / 8; ++i) {
      if (h[i * 8 + 6] == 0) continue;
      ++n;
      for (int k = 1; k < 6; ++k) sum[k] += static_cast<double>(h[i * 8 + k]);
      g0 = std::min(g0, h[i * 8]);
      ghz += static_cast<double>(h[i * 8 + 5]) / static_cast<double>(h[i * 8 + 6] - h[i * 8]);
      gmin = std::min(gmin, h[i * 8 + 6]);
      gmax = std::max(gmax, h[i * 8 + 6]);
      dmax = std::max(dmax, h[i * 8 + 5]);
    }
    if (n > 0)
      fprintf(stderr,
              "gemm dbg M=%d N=%d K=%d ctas=%d cyc: setup %.0f first_full %.0f last_mma %.0f "
              "done %.0f end %.0f (max end %llu); end spread %.2f us; first entry -> last end "
              "%.2f us; SM clock %.2f GHz\n",
              M, N, K, n, sum[1] / n, sum[2] / n, sum[3] / n, sum[4] / n, sum[5] / n, dmax,
              (gmax - gmin) * 1e-3, (gmax - g0) * 1e-3, ghz / n);
    cudaFree(dbg);
    c->test_dbg = nullptr;
  }
  cudaFree(flush);
  cudaFree(sink);
  if (wpk) cudaFree(wpk);
  if (xpk) cudaFree(xpk);
  c->test_x_packed = nullptr;
  if (rc == VOX_OK) {
    std::vector<float> tmp(static_cast<size_t>(splits) * N * M);
    CK(cudaMemcpy(tmp.data(), dout, tmp.size() * 4, cudaMemcpyDeviceToHost));
    for (size_t i = 0; i < static_cast<size_t>(N) * M; ++i) {
      float s = 0.f;
      for (int k = 0; k < planes; ++k) s += tmp[k * static_cast<size_t>(N) * M + i];
      out[i] = s;
    }
  }
  cudaEventDestroy(a);
  cudaEventDestroy(b);
  cudaFree(dw);
  cudaFree(dx);
  cudaFree(dout);
  if (db) cudaFree(db);
  return rc;
}

int vox_read_weight(VoxCtx* c, const char* name, int32_t layer, void* out, size_t bytes) {
  if (!c || !name || !out) return fail(c, VOX_ERR_INVALID, "null argument");
  const VoxModelCfg& g = c->cfg;
  const int d = g.d_model;
  const void* src = nullptr;
  size_t avail = 0;
  const std::string n(name);
  const int64_t n_qkv = static_cast<int64_t>(c->nqkv) * d;
  if (n == "emb") {
    src = c->emb;
    avail = static_cast<size_t>(g.vocab) * d * 2;
  } else if (n == "qkv") {  // stored packed (init.cu): unpack to the logical [nqkv, d]
    if (layer < 0 || layer >= g.n_layers) return fail(c, VOX_ERR_INVALID, "bad layer");
    const int64_t np = packed_elems(c->nqkv, d);
    std::vector<uint16_t> pk(static_cast<size_t>(np));
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(pk.data(), c->w_qkv + layer * np, np * 2, cudaMemcpyDeviceToHost));
    const size_t want = std::min(bytes, static_cast<size_t>(n_qkv) * 2) / 2;
    uint16_t* o = static_cast<uint16_t*>(out);
    const int n_kb = d / 64;
    for (size_t i = 0; i < want; ++i) {
      const int64_t m = static_cast<int64_t>(i) / d, k = static_cast<int64_t>(i) % d;
      const int64_t t = (m / 128) * n_kb + k / 64;
      const int r = static_cast<int>(m % 128), ch = static_cast<int>((k % 64) / 8) ^ (r & 7);
      o[i] = pk[static_cast<size_t>(t * 8192 + r * 64 + ch * 8 + k % 8)];
    }
    return VOX_OK;
  } else if (n == "qkv_bias" && c->b_qkv) {
    src = c->b_qkv + static_cast<int64_t>(layer) * c->nqkv;
    avail = static_cast<size_t>(c->nqkv) * 4;
  } else if (n == "norm_attn") {
    src = c->norm_attn + static_cast<int64_t>(layer) * d;
    avail = d * 4;
  } else if (n == "vq_tab" && g.detok_enabled) {
    src = c->dw.tabs;
    avail = static_cast<size_t>(3) * g.codebook_size * g.latent_dim * 2;
  } else {
    return fail(c, VOX_ERR_INVALID, "unknown weight name");
  }
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(out, src, std::min(bytes, avail), cudaMemcpyDeviceToHost));
  return VOX_OK;
}

int vox_read_kv(VoxCtx* c, int32_t layer, int32_t slot, int32_t pos, float* k_out,
                float* v_out) {
  if (!c || slot < 0 || slot >= c->cfg.max_slots || !c->slot_used[slot])
    return fail(c, VOX_ERR_CACHE_MISSING, "unknown slot");
  const VoxModelCfg& g = c->cfg;
  if (layer < 0 || layer >= g.n_layers || pos < 0 ||
      pos >= static_cast<int>(c->slot_pages[slot].size()) * g.page_size)
    return fail(c, VOX_ERR_INVALID, "bad kv coordinate");
  CK(cudaDeviceSynchronize());
  const int page = c->slot_pages[slot][pos / g.page_size], off = pos % g.page_size;
  const size_t kv_layer = static_cast<size_t>(g.n_pages) * g.n_kv_heads * g.page_size * g.head_dim;
  std::vector<bf16> tmp(g.head_dim);
  for (int h = 0; h < g.n_kv_heads; ++h) {
    const size_t idx = layer * kv_layer +
                       ((static_cast<size_t>(page) * g.n_kv_heads + h) * g.page_size + off) *
                           g.head_dim;
    CK(cudaMemcpy(tmp.data(), c->kc + idx, g.head_dim * 2, cudaMemcpyDeviceToHost));
    for (int e = 0; e < g.head_dim; ++e) k_out[h * g.head_dim + e] = __bfloat162float(tmp[e]);
    // V head-pages are transposed: [hd][page_size]
    std::vector<bf16> vpage(static_cast<size_t>(g.head_dim) * g.page_size);
    const size_t vidx = layer * kv_layer +
                        (static_cast<size_t>(page) * g.n_kv_heads + h) * g.page_size * g.head_dim;
    CK(cudaMemcpy(vpage.data(), c->vc + vidx, vpage.size() * 2, cudaMemcpyDeviceToHost));
    for (int e = 0; e < g.head_dim; ++e)
      v_out[h * g.head_dim + e] = __bfloat162float(vpage[static_cast<size_t>(e) * g.page_size + off]);
  }
  return VOX_OK;
}

}  // extern "C"
