// mimi.cu — K7: Mimi-style 12.5 Hz streaming detokenizer (BASELINE config 3, CSM-1B-style).
//
// Algorithm: [3P] transformers 5.5.0 MimiModel.decode (modeling_mimi.py:1613-1680),
// restated in oracle/mimi.py and pinned there against transformers itself.  Every
// layer is causal, so a stream decoded chunk by chunk with per-stream cached state
// (conv padding caches = the last k-1 input rows of every causal conv, the previous
// input row of every transposed conv, and a 250-position K/V ring per transformer
// layer) reproduces the full-sequence decode; this file is that stateful decoder.
//
// Replaces the reference's stub detokenizer (profiles.py:333-356) for a depth-stage
// profile (profiles.py:214-231, token_rate 12.5, stateful_detok).
//
// Per decode call over n streams with nf_i new frames each (rows are per-stream
// contiguous at every level; a level with u rows per frame holds stream i's rows at
// [f_off_i * u, (f_off_i + nf_i) * u)):
//   mimi_embed_up   codes -> sum of projected codebook tables (fp32) -> depthwise ConvT x2
//   8 x { mimi_ln -> QKV GEMM -> mimi_rope_kv (ring append) -> mimi_attn -> O GEMM ->
//         mimi_ln (h += ls1 * o) -> fc1 GEMM -> mimi_gelu -> fc2 GEMM -> (h += ls2 * .) }
//   SEANet: every conv = mimi_im2col (ELU + causal taps from the chunk or the cached
//   history, bf16 UMMA operand) + tcgen05 GEMM (gemm_tc.cu, bias / residual in the
//   epilogue) + mimi_hist (history for the next chunk, double-buffered by chunk parity);
//   transposed convs (k = 2s, stride s, right-trimmed) are the GEMM
//   [x_{t-1} | x_t] . W[(s * Cout), 2 * Cin] whose output rows ARE the s upsampled rows;
//   the last conv (64 -> 1) is mimi_out.
#include <cuda.h>

#include <algorithm>
#include <cmath>
#include <mutex>
#include <string>
#include <vector>

#include "codec_common.cuh"

namespace vox {
namespace {

// tensor ids (oracle/weights.py: T_MI_*)
enum : uint64_t {
  T_MI_EMB = 300, T_MI_PSEM = 301, T_MI_PAC = 302, T_MI_UP = 303,
  T_MI_LN1W = 310, T_MI_LN1B = 311, T_MI_LN2W = 312, T_MI_LN2B = 313,
  T_MI_QKV = 314, T_MI_O = 315, T_MI_FC1 = 316, T_MI_FC2 = 317, T_MI_LS1 = 318, T_MI_LS2 = 319,
  T_MI_C0W = 330, T_MI_C0B = 331, T_MI_UPW = 332, T_MI_UPB = 333,
  T_MI_R1W = 334, T_MI_R1B = 335, T_MI_R2W = 336, T_MI_R2B = 337, T_MI_OUTW = 338, T_MI_OUTB = 339,
};

constexpr int kMaxWin = 256;

// codes [F][n_q] -> h rows 2f, 2f+1 (25 Hz): x_f = sum_q T_q[code], depthwise ConvT
// (k 4, stride 2, right-trimmed): y[2t + j] = x_t * w[j] + x_{t-1} * w[j + 2]
__global__ void __launch_bounds__(128) mimi_embed_up_kernel(
    const int32_t* __restrict__ codes, const int32_t* __restrict__ frame_req,
    const SegDev* __restrict__ reqs, int n_q, int cb, int D, const float* __restrict__ tabs,
    const float4* __restrict__ up, StateView sv, int64_t off_up, float* __restrict__ h) {
  const int f = blockIdx.x;
  const SegDev q = reqs[frame_req[f]];
  const int t = f - q.f_off;
  for (int c = threadIdx.x; c < D; c += blockDim.x) {
    float x = 0.f, xp = 0.f;
    for (int k = 0; k < n_q; ++k) x += tabs[(static_cast<int64_t>(k) * cb + codes[f * n_q + k]) * D + c];
    if (t > 0) {
      for (int k = 0; k < n_q; ++k)
        xp += tabs[(static_cast<int64_t>(k) * cb + codes[(f - 1) * n_q + k]) * D + c];
    } else {
      xp = sv.in(q, off_up)[c];
    }
    const float4 w = up[c];
    h[static_cast<int64_t>(2 * f) * D + c] = x * w.x + xp * w.z;
    h[static_cast<int64_t>(2 * f + 1) * D + c] = x * w.y + xp * w.w;
    if (t == q.nf - 1) sv.out(q, off_up)[c] = x;
  }
}

// RoPE (rotate-half) on q and k of every row, append k, v to the stream's K/V ring
// kv[slot][layer][W][2][D] at pos % W; q -> qo (fp32).
__global__ void __launch_bounds__(128) mimi_rope_kv_kernel(
    const float* __restrict__ qkv, const int32_t* __restrict__ frame_req, const SegDev* __restrict__ reqs,
    int D, int hd, int W, int L, int layer, const float* __restrict__ inv_freq, float* __restrict__ kv,
    float* __restrict__ qo) {  // W = ring size
  const int64_t r = blockIdx.x;
  const SegDev q = reqs[frame_req[r >> 1]];
  const int pos = q.pos0 + static_cast<int>(r - 2LL * q.f_off);
  float* kvr = kv + ((static_cast<int64_t>(q.slot) * L + layer) * W + pos % W) * 2 * D;
  const float* src = qkv + r * 3 * D;
  const int half = hd / 2;
  for (int e = threadIdx.x; e < D; e += blockDim.x) {
    const int d = e % hd;
    const float ang = static_cast<float>(pos) * inv_freq[d % half];
    float sn, cs;
    sincosf(ang, &sn, &cs);
    const float pq = d < half ? -src[e + half] : src[e - half];
    const float pk = d < half ? -src[D + e + half] : src[D + e - half];
    qo[r * D + e] = src[e] * cs + pq * sn;
    kvr[e] = src[D + e] * cs + pk * sn;
    kvr[D + e] = src[2 * D + e];
  }
}

// Sliding-window causal attention, one CTA per (stream, head), 4 warps over the
// stream's new query rows; keys max(0, pos - W + 1) .. pos from the ring.  The ring
// holds Wr = W + 2 * max_chunk positions: a chunk of n new positions reads the
// W + n - 1 positions [P0 - W + 1, P0 + n - 1], none of which its own appends evict.
__global__ void __launch_bounds__(128) mimi_attn_kernel(const float* __restrict__ qi,
                                                        const SegDev* __restrict__ reqs,
                                                        const float* __restrict__ kv, int D, int hd, int W,
                                                        int Wr, int L, int layer, bf16* __restrict__ out) {
  __shared__ float p[4][kMaxWin];
  __shared__ float sq[4][128];
  const SegDev q = reqs[blockIdx.x];
  const int hh = blockIdx.y;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const float scale = rsqrtf(static_cast<float>(hd));
  const float* ring = kv + (static_cast<int64_t>(q.slot) * L + layer) * Wr * 2 * D;
  const int nq = 2 * q.nf;
  for (int t = warp; t < nq; t += 4) {
    const int64_t row = 2LL * q.f_off + t;
    const int pos = q.pos0 + t;
    const int lo = max(0, pos - W + 1), nk = pos - lo + 1;
    for (int d = lane; d < hd; d += 32) sq[warp][d] = qi[row * D + hh * hd + d];
    __syncwarp();
    float mx = -INFINITY;
    for (int j = lane; j < nk; j += 32) {
      const float* kr = ring + static_cast<int64_t>((lo + j) % Wr) * 2 * D + hh * hd;
      float s = 0.f;
      for (int d = 0; d < hd; d += 4) {
        const float4 k4 = *reinterpret_cast<const float4*>(kr + d);
        s += sq[warp][d] * k4.x + sq[warp][d + 1] * k4.y + sq[warp][d + 2] * k4.z + sq[warp][d + 3] * k4.w;
      }
      s *= scale;
      p[warp][j] = s;
      mx = fmaxf(mx, s);
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    float sum = 0.f;
    for (int j = lane; j < nk; j += 32) {
      const float e = __expf(p[warp][j] - mx);
      p[warp][j] = e;
      sum += e;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    __syncwarp();
    for (int d = lane; d < hd; d += 32) {
      float o = 0.f;
      for (int j = 0; j < nk; ++j) o += p[warp][j] * ring[static_cast<int64_t>((lo + j) % Wr) * 2 * D + D + hh * hd + d];
      out[row * D + hh * hd + d] = f32_to_bf16(o / sum);
    }
    __syncwarp();
  }
}

// last conv (C -> 1, k taps, ELU on the input), one thread per output sample
__global__ void mimi_out_kernel(const float* __restrict__ x, int C, int k, int u,
                                const int32_t* __restrict__ frame_req, const SegDev* __restrict__ reqs,
                                StateView sv, int64_t off, const float* __restrict__ w, float b, int64_t rows,
                                float* __restrict__ pcm) {
  const int64_t r = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= rows) return;
  const SegDev q = reqs[frame_req[r / u]];
  const int64_t t = r - static_cast<int64_t>(q.f_off) * u;
  float acc = 0.f;
  for (int j = 0; j < k; ++j) {
    const int64_t src = t - (k - 1) + j;
    const float* p = src >= 0 ? x + (r - t + src) * C : sv.in(q, off) + ((k - 1) + src) * C;
    for (int c = 0; c < C; c += 4) {
      const float4 a = *reinterpret_cast<const float4*>(p + c);
      acc += elu(a.x) * w[j * C + c] + elu(a.y) * w[j * C + c + 1] + elu(a.z) * w[j * C + c + 2] +
             elu(a.w) * w[j * C + c + 3];
    }
  }
  pcm[r] = acc + b;
}

// projected codebook tables T_q[code][o] = sum_c emb_q[code][c] * P[o][c] (one-time)
__global__ void mimi_tables_kernel(const float* __restrict__ emb, const bf16* __restrict__ P, int cd, int D,
                                   float* __restrict__ tab) {
  const int code = blockIdx.x;
  for (int o = threadIdx.x; o < D; o += blockDim.x) {
    float s = 0.f;
    for (int c = 0; c < cd; ++c) s += emb[static_cast<int64_t>(code) * cd + c] * bf16_to_f32(P[static_cast<int64_t>(o) * cd + c]);
    tab[static_cast<int64_t>(code) * D + o] = s;
  }
}

}  // namespace
}  // namespace vox

using namespace vox;

struct MimiLayerW {
  float *ln1w, *ln1b, *ln2w, *ln2b, *ls1, *ls2;
  bf16 *qkv, *o, *fc1, *fc2;
  CUtensorMap tm_qkv, tm_o, tm_fc1, tm_fc2;
};
struct MimiBlockW {
  bf16 *upw, *r1w, *r2w;
  float *upb, *r1b, *r2b;
  CUtensorMap tm_up, tm_r1, tm_r2;
  int r2k;  // K of the k1 conv padded to 64
};

struct VoxMimi {
  int device = 0;
  VoxMimiCfg cfg{};
  std::string err;
  cudaStream_t st = nullptr;
  // weights
  float* tabs = nullptr;  // [n_q][cb][D]
  float* up = nullptr;    // [D][4]
  float* inv_freq = nullptr;
  std::vector<MimiLayerW> layers;
  bf16* c0w = nullptr;
  float* c0b = nullptr;
  CUtensorMap tm_c0;
  std::vector<MimiBlockW> blocks;
  float* outw = nullptr;
  float outb = 0.f;
  // state
  float* state = nullptr;
  int64_t half = 0, off_up = 0, off_c0 = 0, off_ct[4] = {}, off_r1[4] = {}, off_out = 0;
  float* kv = nullptr;
  int ring = 0, max_chunk = 0;  // K/V ring positions; max new frames per stream per call
  std::vector<int> used, parity, pos;
  // workspaces
  float *h = nullptr, *qkv = nullptr, *q = nullptr, *tmp = nullptr, *xa = nullptr, *xb = nullptr, *pcm = nullptr;
  bf16 *xbf = nullptr, *col = nullptr;
  int32_t* d_stage = nullptr;  // reqs | frame_req | codes
  int32_t* h_stage = nullptr;
  float* h_pcm = nullptr;
  size_t stage_ints = 0;
  int64_t launches = 0;
  std::vector<int> chans;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr;  // device time of the last decode's kernels
  double last_ms = 0.0;
};

namespace {
std::mutex g_mimi_err_mu;
std::string g_mimi_err;

int mfail(VoxMimi* m, int code, const std::string& msg) {
  if (m) m->err = msg;
  std::lock_guard<std::mutex> g(g_mimi_err_mu);
  g_mimi_err = msg;
  return code;
}

#define MCK(x)                                                                              \
  do {                                                                                      \
    cudaError_t e_ = (x);                                                                   \
    if (e_ != cudaSuccess) return mfail(m, VOX_ERR_CUDA, std::string(#x ": ") + cudaGetErrorString(e_)); \
  } while (0)
#define MRET(x)                      \
  do {                               \
    int r_ = (x);                    \
    if (r_ != VOX_OK) return r_;     \
  } while (0)

template <typename T>
cudaError_t dal(T** p, size_t n) {
  return cudaMalloc(reinterpret_cast<void**>(p), sizeof(T) * (n > 0 ? n : 1));
}

uint64_t key(const VoxMimi* m, uint64_t seed, uint64_t tid, uint64_t l) { return tensor_key(seed, tid, l); }

int gemm(VoxMimi* m, const CUtensorMap& tw, int M, const bf16* x, int K, int64_t rows, float* out, int64_t ldo,
         const float* bias, const float* resid, int64_t ldr) {
  const cudaError_t e = codec_gemm(tw, M, x, K, rows, out, ldo, bias, resid, ldr, m->st, &m->launches);
  if (e != cudaSuccess) return mfail(m, VOX_ERR_CUDA, std::string("mimi gemm: ") + cudaGetErrorString(e));
  return VOX_OK;
}

int wmap(VoxMimi* m, CUtensorMap* t, const bf16* w, int M, int K) {
  if (!codec_wmap(t, w, M, K)) return mfail(m, VOX_ERR_CUDA, "mimi: weight map");
  return VOX_OK;
}

int create_weights(VoxMimi* m, uint64_t seed) {
  const VoxMimiCfg& g = m->cfg;
  const int D = g.hidden, cd = g.cb_dim, cb = g.cb_size, F = g.ffn;
  cudaStream_t st = m->st;
  auto bf = [&](bf16** p, int64_t n, uint64_t tid, uint64_t l, float scale) -> int {
    MCK(dal(p, n));
    launch_init_bf16(*p, n, key(m, seed, tid, l), scale, st);
    MCK(cudaGetLastError());
    return VOX_OK;
  };
  auto fl = [&](float** p, int64_t n, uint64_t tid, uint64_t l, float scale, float off) -> int {
    MCK(dal(p, n));
    launch_init_f32(*p, n, key(m, seed, tid, l), scale, off, st);
    MCK(cudaGetLastError());
    return VOX_OK;
  };
  // projected codebook tables
  MCK(dal(&m->tabs, static_cast<size_t>(g.n_q) * cb * D));
  {
    bf16 *psem, *pac;
    MRET(bf(&psem, static_cast<int64_t>(D) * cd, T_MI_PSEM, 0, std::sqrt(3.0f / cd)));
    MRET(bf(&pac, static_cast<int64_t>(D) * cd, T_MI_PAC, 0, std::sqrt(3.0f / cd)));
    float* emb;
    MCK(dal(&emb, static_cast<size_t>(cb) * cd));
    for (int qq = 0; qq < g.n_q; ++qq) {
      launch_init_f32(emb, static_cast<int64_t>(cb) * cd, key(m, seed, T_MI_EMB, qq), std::sqrt(3.0f / g.n_q), 0.f, st);
      mimi_tables_kernel<<<cb, 256, 0, st>>>(emb, qq < g.n_semantic ? psem : pac, cd, D,
                                             m->tabs + static_cast<int64_t>(qq) * cb * D);
      MCK(cudaGetLastError());
    }
    MCK(cudaStreamSynchronize(st));
    cudaFree(emb);
    cudaFree(psem);
    cudaFree(pac);
  }
  MRET(fl(&m->up, 4LL * D, T_MI_UP, 0, 0.5f, 0.f));
  {
    std::vector<float> inv(g.hidden / g.n_heads / 2);
    const int hd = g.hidden / g.n_heads;
    for (size_t i = 0; i < inv.size(); ++i)
      inv[i] = 1.0f / std::pow(g.rope_theta, static_cast<float>(2 * i) / static_cast<float>(hd));
    MCK(dal(&m->inv_freq, inv.size()));
    MCK(cudaMemcpy(m->inv_freq, inv.data(), inv.size() * 4, cudaMemcpyHostToDevice));
  }
  m->layers.resize(g.n_layers);
  for (int l = 0; l < g.n_layers; ++l) {
    MimiLayerW& w = m->layers[l];
    MRET(fl(&w.ln1w, D, T_MI_LN1W, l, 0.25f, 1.f));
    MRET(fl(&w.ln1b, D, T_MI_LN1B, l, 0.05f, 0.f));
    MRET(fl(&w.ln2w, D, T_MI_LN2W, l, 0.25f, 1.f));
    MRET(fl(&w.ln2b, D, T_MI_LN2B, l, 0.05f, 0.f));
    MRET(bf(&w.qkv, 3LL * D * D, T_MI_QKV, l, std::sqrt(3.0f / D)));
    MRET(bf(&w.o, static_cast<int64_t>(D) * D, T_MI_O, l, std::sqrt(3.0f / D)));
    MRET(bf(&w.fc1, static_cast<int64_t>(F) * D, T_MI_FC1, l, std::sqrt(3.0f / D)));
    MRET(bf(&w.fc2, static_cast<int64_t>(D) * F, T_MI_FC2, l, std::sqrt(3.0f / F)));
    MRET(fl(&w.ls1, D, T_MI_LS1, l, 0.05f, 0.1f));
    MRET(fl(&w.ls2, D, T_MI_LS2, l, 0.05f, 0.1f));
    MRET(wmap(m, &w.tm_qkv, w.qkv, 3 * D, D));
    MRET(wmap(m, &w.tm_o, w.o, D, D));
    MRET(wmap(m, &w.tm_fc1, w.fc1, F, D));
    MRET(wmap(m, &w.tm_fc2, w.fc2, D, F));
  }
  const std::vector<int>& ch = m->chans;
  MRET(bf(&m->c0w, static_cast<int64_t>(ch[0]) * g.kernel * D, T_MI_C0W, 0, std::sqrt(3.0f / (g.kernel * D))));
  MRET(fl(&m->c0b, ch[0], T_MI_C0B, 0, 0.05f, 0.f));
  MRET(wmap(m, &m->tm_c0, m->c0w, ch[0], g.kernel * D));
  m->blocks.resize(g.n_ratios);
  for (int b = 0; b < g.n_ratios; ++b) {
    MimiBlockW& w = m->blocks[b];
    const int Ci = ch[b], Co = ch[b + 1], s = g.ratios[b], hh = Co / g.compress;
    MRET(bf(&w.upw, static_cast<int64_t>(s) * Co * 2 * Ci, T_MI_UPW, b, std::sqrt(3.0f / (2.0f * Ci))));
    float* small;
    MRET(fl(&small, Co, T_MI_UPB, b, 0.05f, 0.f));
    MCK(dal(&w.upb, static_cast<size_t>(s) * Co));
    for (int j = 0; j < s; ++j)
      MCK(cudaMemcpyAsync(w.upb + static_cast<int64_t>(j) * Co, small, Co * 4, cudaMemcpyDeviceToDevice, st));
    MRET(bf(&w.r1w, static_cast<int64_t>(hh) * g.res_kernel * Co, T_MI_R1W, b, std::sqrt(3.0f / (g.res_kernel * Co))));
    MRET(fl(&w.r1b, hh, T_MI_R1B, b, 0.05f, 0.f));
    w.r2k = (hh + 63) / 64 * 64;
    bf16* r2;
    MRET(bf(&r2, static_cast<int64_t>(Co) * hh, T_MI_R2W, b, 0.5f * std::sqrt(3.0f / hh)));
    MCK(dal(&w.r2w, static_cast<size_t>(Co) * w.r2k));
    MCK(cudaMemsetAsync(w.r2w, 0, static_cast<size_t>(Co) * w.r2k * 2, st));
    MCK(cudaMemcpy2DAsync(w.r2w, w.r2k * 2, r2, hh * 2, hh * 2, Co, cudaMemcpyDeviceToDevice, st));
    MRET(fl(&w.r2b, Co, T_MI_R2B, b, 0.05f, 0.f));
    MCK(cudaStreamSynchronize(st));
    cudaFree(small);
    cudaFree(r2);
    MRET(wmap(m, &w.tm_up, w.upw, s * Co, 2 * Ci));
    MRET(wmap(m, &w.tm_r1, w.r1w, hh, g.res_kernel * Co));
    MRET(wmap(m, &w.tm_r2, w.r2w, Co, w.r2k));
  }
  const int C4 = ch[g.n_ratios];
  MRET(fl(&m->outw, static_cast<int64_t>(g.last_kernel) * C4, T_MI_OUTW, 0, std::sqrt(3.0f / (g.last_kernel * C4)), 0.f));
  {
    float* tb;
    MRET(fl(&tb, 1, T_MI_OUTB, 0, 0.05f, 0.f));
    MCK(cudaStreamSynchronize(st));
    MCK(cudaMemcpy(&m->outb, tb, 4, cudaMemcpyDeviceToHost));
    cudaFree(tb);
  }
  return VOX_OK;
}

int create_state(VoxMimi* m) {
  const VoxMimiCfg& g = m->cfg;
  const std::vector<int>& ch = m->chans;
  int64_t off = 0;
  m->off_up = off;
  off += g.hidden;
  m->off_c0 = off;
  off += static_cast<int64_t>(g.kernel - 1) * g.hidden;
  for (int b = 0; b < g.n_ratios; ++b) {
    m->off_ct[b] = off;
    off += ch[b];
    m->off_r1[b] = off;
    off += static_cast<int64_t>(g.res_kernel - 1) * ch[b + 1];
  }
  m->off_out = off;
  off += static_cast<int64_t>(g.last_kernel - 1) * ch[g.n_ratios];
  m->half = (off + 63) / 64 * 64;
  MCK(dal(&m->state, static_cast<size_t>(g.max_slots) * 2 * m->half));
  MCK(cudaMemset(m->state, 0, static_cast<size_t>(g.max_slots) * 2 * m->half * 4));
  m->max_chunk = std::min(g.max_frames, 64);
  m->ring = g.window + 2 * m->max_chunk;
  MCK(dal(&m->kv, static_cast<size_t>(g.max_slots) * g.n_layers * m->ring * 2 * g.hidden));
  m->used.assign(g.max_slots, 0);
  m->parity.assign(g.max_slots, 0);
  m->pos.assign(g.max_slots, 0);
  // workspaces sized by max_frames
  const int64_t F = g.max_frames, R0 = 2 * F, D = g.hidden;
  int64_t mx = R0 * ch[0], mcol = R0 * std::max<int64_t>(g.kernel * D, g.ffn);
  int64_t u = 2;
  for (int b = 0; b < g.n_ratios; ++b) {
    mcol = std::max<int64_t>(mcol, F * u * 2 * ch[b]);
    u *= g.ratios[b];
    mx = std::max<int64_t>(mx, F * u * ch[b + 1]);
    mcol = std::max<int64_t>(mcol, F * u * std::max(g.res_kernel * ch[b + 1], (ch[b + 1] / g.compress + 63) / 64 * 64));
  }
  MCK(dal(&m->h, R0 * D));
  MCK(dal(&m->qkv, R0 * 3 * D));
  MCK(dal(&m->q, R0 * D));
  MCK(dal(&m->tmp, R0 * std::max<int64_t>(g.ffn, D)));
  MCK(dal(&m->xa, mx));
  MCK(dal(&m->xb, mx));
  MCK(dal(&m->xbf, R0 * std::max<int64_t>(g.ffn, D)));
  MCK(dal(&m->col, mcol));
  MCK(dal(&m->pcm, F * u));
  m->stage_ints = 8 * static_cast<size_t>(g.max_slots) + F + F * g.n_q;
  MCK(dal(&m->d_stage, m->stage_ints));
  MCK(cudaHostAlloc(&m->h_stage, m->stage_ints * 4, cudaHostAllocDefault));
  MCK(cudaHostAlloc(&m->h_pcm, F * u * 4, cudaHostAllocDefault));
  return VOX_OK;
}

#define LK(...)                                   \
  do {                                            \
    __VA_ARGS__;                                  \
    m->launches++;                                \
    MCK(cudaGetLastError());                      \
  } while (0)

int enqueue(VoxMimi* m, int n, int Ftot) {
  const VoxMimiCfg& g = m->cfg;
  const int D = g.hidden, hd = g.hidden / g.n_heads;
  const std::vector<int>& ch = m->chans;
  cudaStream_t st = m->st;
  const SegDev* reqs = reinterpret_cast<const SegDev*>(m->d_stage);
  const int32_t* frame_req = m->d_stage + 8 * g.max_slots;
  const int32_t* codes = frame_req + g.max_frames;
  StateView sv{m->state, 2 * m->half, m->half};
  const int64_t R0 = 2LL * Ftot;
  LK(mimi_embed_up_kernel<<<Ftot, 128, 0, st>>>(codes, frame_req, reqs, g.n_q, g.cb_size, D, m->tabs,
                                                reinterpret_cast<const float4*>(m->up), sv, m->off_up, m->h));
  // transformer
  for (int l = 0; l < g.n_layers; ++l) {
    const MimiLayerW& w = m->layers[l];
    const bool first = l == 0;
    const MimiLayerW* prev = first ? nullptr : &m->layers[l - 1];
    LK(launch_codec_ln(m->h, first ? nullptr : m->tmp, first ? nullptr : prev->ls2, w.ln1w,
                                          w.ln1b, m->xbf, D, g.eps, R0, st));
    MRET(gemm(m, w.tm_qkv, 3 * D, m->xbf, D, R0, m->qkv, 3 * D, nullptr, nullptr, 0));
    LK(mimi_rope_kv_kernel<<<R0, 128, 0, st>>>(m->qkv, frame_req, reqs, D, hd, m->ring, g.n_layers, l,
                                               m->inv_freq, m->kv, m->q));
    LK(mimi_attn_kernel<<<dim3(n, g.n_heads), 128, 0, st>>>(m->q, reqs, m->kv, D, hd, g.window, m->ring, g.n_layers, l,
                                                            m->xbf));
    MRET(gemm(m, w.tm_o, D, m->xbf, D, R0, m->tmp, D, nullptr, nullptr, 0));
    LK(launch_codec_ln(m->h, m->tmp, w.ls1, w.ln2w, w.ln2b, m->xbf, D, g.eps, R0, st));
    MRET(gemm(m, w.tm_fc1, g.ffn, m->xbf, D, R0, m->tmp, g.ffn, nullptr, nullptr, 0));
    const int64_t ne = R0 * g.ffn;
    LK(codec_gelu_kernel<<<static_cast<unsigned>((ne + 255) / 256), 256, 0, st>>>(m->tmp, m->xbf, ne));
    MRET(gemm(m, w.tm_fc2, D, m->xbf, g.ffn, R0, m->tmp, D, nullptr, nullptr, 0));
  }
  // h += ls2 * fc2 of the last layer (residual into the conv stack's input rows)
  {
    // reuse mimi_ln's residual update: LN output discarded into xbf (cheap, R0 rows)
    const MimiLayerW& w = m->layers[g.n_layers - 1];
    LK(launch_codec_ln(m->h, m->tmp, w.ls2, w.ln1w, w.ln1b, m->xbf, D, g.eps, R0, st));
  }
  auto im2col = [&](const float* x, int C, int k, int elu_on, int Kp, int u, int64_t off, int64_t rows) -> int {
    const int64_t tot = rows * (Kp / 8);
    LK(codec_im2col_kernel<<<static_cast<unsigned>((tot + 255) / 256), 256, 0, st>>>(x, C, k, elu_on ? kActElu : kActNone, 0.f, Kp, u, frame_req,
                                                                                    reqs, sv, off, rows, m->col));
    if (k > 1) LK(codec_hist_kernel<<<n, 256, 0, st>>>(x, C, k, u, reqs, sv, off));
    return VOX_OK;
  };
  // SEANet: k7 conv 512 -> ch0 (no activation before it)
  int u = 2;
  MRET(im2col(m->h, D, g.kernel, 0, g.kernel * D, u, m->off_c0, R0));
  MRET(gemm(m, m->tm_c0, ch[0], m->col, g.kernel * D, R0, m->xa, ch[0], m->c0b, nullptr, 0));
  float* x = m->xa;
  for (int b = 0; b < g.n_ratios; ++b) {
    const MimiBlockW& w = m->blocks[b];
    const int Ci = ch[b], Co = ch[b + 1], s = g.ratios[b], hh = Co / g.compress;
    const int64_t rows = static_cast<int64_t>(Ftot) * u;
    MRET(im2col(x, Ci, 2, 1, 2 * Ci, u, m->off_ct[b], rows));
    float* y = x == m->xa ? m->xb : m->xa;
    MRET(gemm(m, w.tm_up, s * Co, m->col, 2 * Ci, rows, y, static_cast<int64_t>(s) * Co, w.upb, nullptr, 0));
    x = y;
    u *= s;
    const int64_t rows2 = static_cast<int64_t>(Ftot) * u;
    // residual block: ELU -> k3 conv Co -> hh -> ELU -> k1 conv hh -> Co, + x
    MRET(im2col(x, Co, g.res_kernel, 1, g.res_kernel * Co, u, m->off_r1[b], rows2));
    float* t = x == m->xa ? m->xb : m->xa;
    MRET(gemm(m, w.tm_r1, hh, m->col, g.res_kernel * Co, rows2, t, hh, w.r1b, nullptr, 0));
    MRET(im2col(t, hh, 1, 1, w.r2k, u, 0, rows2));
    MRET(gemm(m, w.tm_r2, Co, m->col, w.r2k, rows2, x, Co, w.r2b, x, Co));
  }
  {
    const int C4 = ch[g.n_ratios];
    const int64_t rows = static_cast<int64_t>(Ftot) * u;
    LK(mimi_out_kernel<<<static_cast<unsigned>((rows + 255) / 256), 256, 0, st>>>(
        x, C4, g.last_kernel, u, frame_req, reqs, sv, m->off_out, m->outw, m->outb, rows, m->pcm));
    LK(codec_hist_kernel<<<n, 256, 0, st>>>(x, C4, g.last_kernel, u, reqs, sv, m->off_out));
  }
  return VOX_OK;
}

}  // namespace

extern "C" {

const char* vox_mimi_last_error(const VoxMimi* m) {
  if (m) return m->err.c_str();
  return g_mimi_err.c_str();
}

int vox_mimi_create(int device, const VoxMimiCfg* cfg, uint64_t seed, VoxMimi** out) {
  VoxMimi* m = nullptr;
  if (!cfg || !out) return mfail(m, VOX_ERR_INVALID, "null argument");
  *out = nullptr;
  const VoxMimiCfg& g = *cfg;
  if ((g.hidden != 256 && g.hidden != 512 && g.hidden != 768 && g.hidden != 1024) || g.n_heads < 1 || g.hidden % g.n_heads || (g.hidden / g.n_heads) % 4 ||
      g.hidden / g.n_heads > 128 || g.window < 1 || g.window > kMaxWin || g.n_ratios < 1 || g.n_ratios > 4 ||
      g.n_q < 2 || g.n_semantic < 1 || g.n_semantic >= g.n_q || g.cb_dim < 1 || g.ffn % 64 || g.kernel < 1 ||
      g.last_kernel < 1 || g.res_kernel < 1 || g.compress < 1 || g.max_slots < 1 || g.max_frames < 1 ||
      g.filters % 32)
    return mfail(m, VOX_ERR_INVALID, "unsupported Mimi configuration");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev)
    return mfail(m, VOX_ERR_NO_DEVICE, "no CUDA device");
  cudaDeviceProp prop{};
  cudaGetDeviceProperties(&prop, device);
  if (prop.major != 10) return mfail(m, VOX_ERR_NO_DEVICE, "requires an sm_100 (B200) device");
  m = new VoxMimi();
  m->device = device;
  m->cfg = g;
  m->chans.push_back(g.filters << g.n_ratios);
  for (int b = 0; b < g.n_ratios; ++b) m->chans.push_back(m->chans.back() / 2);
  for (int b = 0; b <= g.n_ratios; ++b)
    if (m->chans[b] % 64 || (b > 0 && m->chans[b] / g.compress < 8)) {
      delete m;
      return mfail(nullptr, VOX_ERR_INVALID, "SEANet channels must be multiples of 64");
    }
  cudaSetDevice(device);
  int lo = 0, hi = 0;
  cudaDeviceGetStreamPriorityRange(&lo, &hi);
  int rc = cudaStreamCreateWithPriority(&m->st, cudaStreamNonBlocking, lo) == cudaSuccess ? VOX_OK : VOX_ERR_CUDA;
  if (rc == VOX_OK && (cudaEventCreate(&m->ev0) != cudaSuccess || cudaEventCreate(&m->ev1) != cudaSuccess))
    rc = mfail(m, VOX_ERR_CUDA, "event create");
  if (rc == VOX_OK) rc = create_weights(m, seed);
  if (rc == VOX_OK) rc = create_state(m);
  if (rc == VOX_OK && cudaStreamSynchronize(m->st) != cudaSuccess) rc = mfail(m, VOX_ERR_CUDA, "init sync");
  if (rc != VOX_OK) {
    g_mimi_err = m->err;
    vox_mimi_destroy(m);
    return rc;
  }
  *out = m;
  return VOX_OK;
}

void vox_mimi_destroy(VoxMimi* m) {
  if (!m) return;
  cudaSetDevice(m->device);
  if (m->st) cudaStreamSynchronize(m->st);
  for (auto& w : m->layers)
    for (void* p : {static_cast<void*>(w.ln1w), static_cast<void*>(w.ln1b), static_cast<void*>(w.ln2w),
                    static_cast<void*>(w.ln2b), static_cast<void*>(w.ls1), static_cast<void*>(w.ls2),
                    static_cast<void*>(w.qkv), static_cast<void*>(w.o), static_cast<void*>(w.fc1),
                    static_cast<void*>(w.fc2)})
      cudaFree(p);
  for (auto& w : m->blocks)
    for (void* p : {static_cast<void*>(w.upw), static_cast<void*>(w.r1w), static_cast<void*>(w.r2w),
                    static_cast<void*>(w.upb), static_cast<void*>(w.r1b), static_cast<void*>(w.r2b)})
      cudaFree(p);
  for (void* p : {static_cast<void*>(m->tabs), static_cast<void*>(m->up), static_cast<void*>(m->inv_freq),
                  static_cast<void*>(m->c0w), static_cast<void*>(m->c0b), static_cast<void*>(m->outw),
                  static_cast<void*>(m->state), static_cast<void*>(m->kv), static_cast<void*>(m->h),
                  static_cast<void*>(m->qkv), static_cast<void*>(m->q), static_cast<void*>(m->tmp),
                  static_cast<void*>(m->xa), static_cast<void*>(m->xb), static_cast<void*>(m->xbf),
                  static_cast<void*>(m->col), static_cast<void*>(m->pcm), static_cast<void*>(m->d_stage)})
    cudaFree(p);
  if (m->h_stage) cudaFreeHost(m->h_stage);
  if (m->h_pcm) cudaFreeHost(m->h_pcm);
  if (m->ev0) cudaEventDestroy(m->ev0);
  if (m->ev1) cudaEventDestroy(m->ev1);
  if (m->st) cudaStreamDestroy(m->st);
  delete m;
}

int vox_mimi_open(VoxMimi* m, int32_t* slot) {
  if (!m || !slot) return mfail(m, VOX_ERR_INVALID, "null argument");
  cudaSetDevice(m->device);
  for (int s = 0; s < m->cfg.max_slots; ++s)
    if (!m->used[s]) {
      // fresh stream: zero conv histories (both parities); the K/V ring needs no reset
      // (a query at position p reads ring entries of positions max(0, p-W+1)..p only)
      MCK(cudaMemsetAsync(m->state + static_cast<int64_t>(s) * 2 * m->half, 0, 2 * m->half * 4, m->st));
      m->used[s] = 1;
      m->parity[s] = 0;
      m->pos[s] = 0;
      *slot = s;
      return VOX_OK;
    }
  return mfail(m, VOX_ERR_OUT_OF_MEMORY, "no free Mimi stream slot");
}

int vox_mimi_close(VoxMimi* m, int32_t slot) {
  if (!m || slot < 0 || slot >= m->cfg.max_slots || !m->used[slot])
    return mfail(m, VOX_ERR_CACHE_MISSING, "close of an unknown Mimi stream");
  m->used[slot] = 0;
  return VOX_OK;
}

int vox_mimi_decode(VoxMimi* m, const VoxMimiReq* reqs, int32_t n, const int32_t* codes, float* pcm_out,
                    int64_t* n_samples) {
  if (!m || (!reqs && n > 0) || !codes) return mfail(m, VOX_ERR_INVALID, "null argument");
  if (n <= 0) return mfail(m, VOX_ERR_EMPTY_BATCH, "empty Mimi batch");
  const VoxMimiCfg& g = m->cfg;
  cudaSetDevice(m->device);
  SegDev* hr = reinterpret_cast<SegDev*>(m->h_stage);
  int32_t* frame_req = m->h_stage + 8 * g.max_slots;
  int32_t* hcodes = frame_req + g.max_frames;
  if (n > g.max_slots) return mfail(m, VOX_ERR_BATCH_TOO_LARGE, "more streams than Mimi slots");
  int F = 0;
  std::vector<int> seen;
  for (int i = 0; i < n; ++i) {
    const VoxMimiReq& r = reqs[i];
    if (r.slot < 0 || r.slot >= g.max_slots || !m->used[r.slot])
      return mfail(m, VOX_ERR_CACHE_MISSING, "decode of an unopened Mimi stream");
    if (std::find(seen.begin(), seen.end(), r.slot) != seen.end())
      return mfail(m, VOX_ERR_INVALID, "a stream appears twice in one Mimi batch");
    seen.push_back(r.slot);
    if (r.n_frames < 1) return mfail(m, VOX_ERR_INVALID, "Mimi request without frames");
    if (r.n_frames > m->max_chunk)
      return mfail(m, VOX_ERR_BATCH_TOO_LARGE, "Mimi request exceeds 64 frames (or max_frames) per call");
    if (F + r.n_frames > g.max_frames) return mfail(m, VOX_ERR_BATCH_TOO_LARGE, "Mimi batch exceeds max_frames");
    hr[i] = SegDev{r.slot, F, r.n_frames, m->parity[r.slot], m->pos[r.slot], 0, {0, 0}};
    for (int f = 0; f < r.n_frames; ++f) frame_req[F + f] = i;
    F += r.n_frames;
  }
  for (int64_t e = 0; e < static_cast<int64_t>(F) * g.n_q; ++e) {
    if (codes[e] < 0 || codes[e] >= g.cb_size) return mfail(m, VOX_ERR_INVALID, "Mimi code outside the codebook");
    hcodes[e] = codes[e];
  }
  MCK(cudaMemcpyAsync(m->d_stage, m->h_stage, m->stage_ints * 4, cudaMemcpyHostToDevice, m->st));
  MCK(cudaEventRecord(m->ev0, m->st));
  MRET(enqueue(m, n, F));
  MCK(cudaEventRecord(m->ev1, m->st));
  int64_t hop = 2;
  for (int b = 0; b < g.n_ratios; ++b) hop *= g.ratios[b];
  const int64_t total = F * hop;
  MCK(cudaMemcpyAsync(m->h_pcm, m->pcm, total * 4, cudaMemcpyDeviceToHost, m->st));
  MCK(cudaStreamSynchronize(m->st));
  {
    float ms = 0.f;
    MCK(cudaEventElapsedTime(&ms, m->ev0, m->ev1));
    m->last_ms = ms;
  }
  if (pcm_out) std::copy(m->h_pcm, m->h_pcm + total, pcm_out);
  if (n_samples) *n_samples = total;
  for (int i = 0; i < n; ++i) {
    m->parity[reqs[i].slot] ^= 1;
    m->pos[reqs[i].slot] += 2 * reqs[i].n_frames;
  }
  return VOX_OK;
}

int vox_mimi_last_ms(VoxMimi* m, double* ms) {
  if (!m || !ms) return mfail(m, VOX_ERR_INVALID, "null argument");
  *ms = m->last_ms;
  return VOX_OK;
}

int vox_mimi_launch_count(VoxMimi* m, int64_t* launches) {
  if (!m || !launches) return mfail(m, VOX_ERR_INVALID, "null argument");
  *launches = m->launches;
  return VOX_OK;
}

}  // extern "C"
