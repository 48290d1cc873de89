// sampler.cu — K1: fused logits processing + token draw, one CTA per row.
//
// Restates sample() / apply_repetition_penalty() / _truncate_and_sample()
// (/root/reference/pkg/src/speechserve/model_api.py:311-381) on device:
//   1. NaN / +inf rejection (model_api.py:370-371) -> err flag VOX_ERR_NONFINITE
//   2. windowed repetition penalty over the DISTINCT ids of the recent window
//      (counts>0 mask, model_api.py:131,149-150,342-352): x>0 -> x/p else x*p
//   3. T == 0 (or top_k == 1): argmax, ties -> lowest id (np.argmax).  Window
//      tokens are compared in fp64 exactly like the reference; all other
//      candidates are exact fp32 values, so the greedy id is bit-exact.
//   4. T > 0: y = x'/T; top-k then top-p keep the stable-descending prefix
//      (ties broken by lowest id, model_api.py:317) found WITHOUT sorting by
//      radix select on order-preserving 32-bit keys (count radix for top-k,
//      probability-mass radix for top-p: the boundary element is the first
//      whose inclusive cumulative mass reaches p, model_api.py:332-334); the
//      draw is Gumbel-max over the kept set with a counter-based RNG keyed by
//      (request seed, step) — an exact sample from the renormalised softmax
//      (distributional parity; the reference's PCG64 stream is host-side).
// Candidates are restricted to [lo, hi) (Orpheus frame-slot codebook-offset
// mask; entries outside are -inf in the reference-visible logits).
#include <float.h>

#include "common.cuh"
#include "kernels.h"

namespace vox {
VOX_TRACE_TU(trace_set_sampler)


constexpr int kST = 512;      // threads per row
constexpr int kBins = 2048;   // radix histogram bins (11 bits)
constexpr int kMaxWin = 256;

constexpr int kFastE = 8;     // register-resident elements per thread (span <= 4096)

struct SampSmem {
  float part[2][kST / 32][8];  // fast path: per-warp partial sums of the 7 probes
  float hmass[kBins];
  uint32_t hcnt[kBins];
  int win[kMaxWin];
  float redf[kST / 32];
  int redi[kST / 32];
  uint32_t redu[kST / 32];
  double redd[kST / 32];
  // broadcast scalars
  uint32_t sel_prefix, sel_mask;
  float f_a, f_b;
  int i_a, i_b;
  uint32_t u_a, u_b;
  double d_a;
  int errv;
};

VOX_DEV uint32_t f2key(float f) {
  const uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
VOX_DEV float key2f(uint32_t k) {
  const uint32_t u = (k & 0x80000000u) ? (k & 0x7fffffffu) : ~k;
  return __uint_as_float(u);
}

// (value desc, index asc) argmax combine
VOX_DEV void better(float& v, int& i, float v2, int i2) {
  if (i2 < 0) return;
  if (i < 0 || v2 > v || (v2 == v && i2 < i)) {
    v = v2;
    i = i2;
  }
}

template <typename T>
VOX_DEV T block_reduce_sum(T v, T* red, T* out_slot) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0) red[w] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    T t = 0;
    for (int k = 0; k < kST / 32; ++k) t += red[k];
    *out_slot = t;
  }
  __syncthreads();
  return *out_slot;
}

// Descending-bin scan by one warp (replaces a serial loop over the bins):
// visits bins nb-1 .. 0, skipping empty ones (cnt == 0), and stops at the
// first bin whose inclusive cumulative weight reaches `target`.  Returns that
// bin (or the lowest non-empty bin if the target is never reached) and, in
// *before, the cumulative weight of the bins strictly above it (or the full
// total when the target is never reached, matching the serial loop).
// weight(b) is the bin's mass (top-p) or count (top-k) as float/int.
template <typename T, typename WF, typename CF>
VOX_DEV int warp_scan_desc(int nb, T target, WF weight, CF nonempty, T* before) {
  const int lane = threadIdx.x & 31;
  T acc = 0;
  int last_nz = -1;
  for (int base = nb - 1; base >= 0; base -= 32) {
    const int b = base - lane;
    const bool ne = b >= 0 && nonempty(b);
    const T m = ne ? weight(b) : T(0);
    T incl = m;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const T t = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += t;
    }
    const T tot = __shfl_sync(0xffffffffu, incl, 31);
    const uint32_t hit = __ballot_sync(0xffffffffu, ne && acc + incl >= target);
    if (hit) {
      const int l = __ffs(hit) - 1;
      *before = acc + __shfl_sync(0xffffffffu, incl - m, l);
      return base - l;
    }
    const uint32_t nz = __ballot_sync(0xffffffffu, ne);
    if (nz) last_nz = base - (31 - __clz(nz));
    acc += tot;
  }
  *before = acc;
  return last_nz;
}

struct RowCtx {
  const float* row;  // row[id - col_base]
  int col_base, lo, hi;
  const uint32_t* bm;  // window bitmap over [lo, hi)
  bool pen_on;
  float pen_f;
  float inv_t;  // 1 / T (stochastic path)
  float temp;
};

VOX_DEV bool in_win(const RowCtx& c, int id) {
  const int o = id - c.lo;
  return c.pen_on && ((c.bm[o >> 5] >> (o & 31)) & 1u);
}

// penalised, temperature-scaled fp32 value (stochastic path)
VOX_DEV float yval(const RowCtx& c, int id) {
  float x = c.row[id - c.col_base];
  if (in_win(c, id)) x = x > 0.f ? __fdiv_rn(x, c.pen_f) : __fmul_rn(x, c.pen_f);
  return __fdiv_rn(x, c.temp);
}

// Histogram pass: elements whose key matches (prefix under mask) and that are
// admissible under the current top-k boundary contribute count (and mass).
// shift/nbits select the digit.
template <bool MASS>
VOX_DEV void hist_pass(const RowCtx& c, SampSmem& S, uint32_t prefix, uint32_t mask, int shift,
                       int nbits, float ymax, uint32_t kb_key, int kb_tie_idx) {
  for (int b = threadIdx.x; b < kBins; b += kST) {
    S.hcnt[b] = 0;
    S.hmass[b] = 0.f;
  }
  __syncthreads();
  const uint32_t dmask = (1u << nbits) - 1u;
  for (int id = c.lo + threadIdx.x; id < c.hi; id += kST) {
    const float y = yval(c, id);
    const uint32_t k = f2key(y);
    if ((k & mask) != prefix) continue;
    if (k < kb_key || (k == kb_key && id > kb_tie_idx)) continue;  // outside top-k set
    const uint32_t bin = (k >> shift) & dmask;
    if (MASS) {
      if (y > -INFINITY) atomicAdd(&S.hmass[bin], expf(y - ymax));
    } else {
      atomicAdd(&S.hcnt[bin], 1u);
    }
  }
  __syncthreads();
}

// Select the (1-based) rank-th smallest index among elements with key == kk
// and admissible; returns that index.  Two 9-bit levels over an 18-bit index.
VOX_DEV int select_tie_index(const RowCtx& c, SampSmem& S, uint32_t kk, int rank) {
  uint32_t prefix = 0, mask = 0;
  int shifts[3] = {18, 9, 0};
  int bits[3] = {9, 9, 9};
  for (int lv = 0; lv < 3; ++lv) {
    for (int b = threadIdx.x; b < 512; b += kST) S.hcnt[b] = 0;
    __syncthreads();
    for (int id = c.lo + threadIdx.x; id < c.hi; id += kST) {
      if (f2key(yval(c, id)) != kk) continue;
      const uint32_t o = static_cast<uint32_t>(id - c.lo);
      if ((o & mask) != prefix) continue;
      atomicAdd(&S.hcnt[(o >> shifts[lv]) & 511u], 1u);
    }
    __syncthreads();
    if (threadIdx.x == 0) {
      int acc = 0;
      for (int b = 0; b < 512; ++b) {  // ascending index order
        const int cnt = static_cast<int>(S.hcnt[b]);
        if (acc + cnt >= rank) {
          S.u_a = static_cast<uint32_t>(b);
          S.i_a = rank - acc;
          break;
        }
        acc += cnt;
      }
    }
    __syncthreads();
    prefix |= S.u_a << shifts[lv];
    mask |= 511u << shifts[lv];
    rank = S.i_a;
    __syncthreads();
  }
  return c.lo + static_cast<int>(prefix);
}

// ---------------------------------------------------------------------------
// Stochastic path for spans of <= kST * kFastE candidates (the Orpheus 4096-id
// frame slot): every thread keeps its 8 penalised/tempered values, keys and
// softmax weights in registers, and the top-k / top-p boundaries are found by
// an 8-ary search over the 32-bit key space with deterministic block
// reductions (fixed-order warp shuffles + per-warp partials) -- no shared-
// memory atomics (the radix histogram's hot bins serialise) and no re-reads
// of the logits.  Same boundary semantics as the histogram path below.
// ---------------------------------------------------------------------------
VOX_DEV int sample_row_fast(SampSmem& S, const RowCtx& c, float ymax, int nfin, uint64_t seed,
                            uint64_t step, const VoxSampling& prm, int* err_flag) {
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  float y[kFastE], w[kFastE];
  uint32_t key[kFastE];
  bool valid[kFastE];
#pragma unroll
  for (int e = 0; e < kFastE; ++e) {
    const int id = c.lo + tid + e * kST;
    y[e] = id < c.hi ? yval(c, id) : -INFINITY;
    valid[e] = y[e] > -INFINITY;
    key[e] = f2key(y[e]);
    w[e] = valid[e] ? expf(y[e] - ymax) : 0.f;
  }
  int rnd = 0;
  // F(b) = sum of wt over masked elements with key >= b, for 7 probes at once
  auto probe_sums = [&](const uint32_t (&b)[7], const bool (&m)[kFastE], bool counts, float (&out)[7]) {
    float acc[7];
#pragma unroll
    for (int j = 0; j < 7; ++j) {
      float a = 0.f;
#pragma unroll
      for (int e = 0; e < kFastE; ++e)
        if (m[e] && key[e] >= b[j]) a += counts ? 1.f : w[e];
      acc[j] = warp_sum(a);
    }
    float (*P)[8] = S.part[rnd & 1];
    if (lane == 0)
#pragma unroll
      for (int j = 0; j < 7; ++j) P[wid][j] = acc[j];
    __syncthreads();
    // every warp reduces the kST/32 partials lane-parallel (fixed shuffle
    // tree: deterministic, identical in all warps) instead of each thread
    // summing them serially
#pragma unroll
    for (int j = 0; j < 7; ++j) {
      float t = lane < kST / 32 ? P[lane][j] : 0.f;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
      out[j] = t;
    }
    ++rnd;  // next round writes the other buffer (no WAR barrier needed)
  };
  // largest key b with F(b) >= target (F non-increasing; F(0) >= target)
  auto search = [&](const bool (&m)[kFastE], bool counts, float target) -> uint32_t {
    uint32_t lo = 0u, hi = 0xFFFFFFFFu;
    while (lo < hi) {
      const uint64_t len = static_cast<uint64_t>(hi) - lo + 1;
      uint32_t b[7];
#pragma unroll
      for (int j = 0; j < 7; ++j) b[j] = lo + static_cast<uint32_t>((len * (j + 1)) / 8);
      float f[7];
      probe_sums(b, m, counts, f);
      uint32_t nlo = lo, nhi = hi;
#pragma unroll
      for (int j = 0; j < 7; ++j) {
        if (b[j] <= nlo) continue;
        if (f[j] >= target) {
          nlo = b[j];
        } else {
          nhi = b[j] - 1;
          break;
        }
      }
      lo = nlo;
      hi = nhi;
    }
    return lo;
  };
  // F at a single key, plus the count of masked elements equal to it
  auto mass_gt_and_ties = [&](const bool (&m)[kFastE], bool counts, uint32_t tau, float& gt,
                              float& ties) {
    uint32_t b[7];
    for (int j = 0; j < 7; ++j) b[j] = tau;
    if (tau != 0xFFFFFFFFu) b[0] = tau + 1;
    float f[7];
    probe_sums(b, m, counts, f);
    gt = tau != 0xFFFFFFFFu ? f[0] : 0.f;
    bool eqm[kFastE];
#pragma unroll
    for (int e = 0; e < kFastE; ++e) eqm[e] = m[e] && key[e] == tau;
    uint32_t z[7] = {0u, 0u, 0u, 0u, 0u, 0u, 0u};
    probe_sums(z, eqm, true, f);
    ties = f[0];
  };

  // ---- top-k: keep keys > kb_key, and ties at kb_key with id <= kb_tie_idx
  bool kset = false;
  uint32_t kb_key = 0u;
  int kb_tie_idx = INT32_MAX;
  int kb_ties_kept = 0;
  bool in_k[kFastE];
#pragma unroll
  for (int e = 0; e < kFastE; ++e) in_k[e] = valid[e];
  if (prm.top_k > 0 && prm.top_k < nfin) {
    const uint32_t tau = search(valid, true, static_cast<float>(prm.top_k));
    float gt, ties;
    mass_gt_and_ties(valid, true, tau, gt, ties);
    kset = true;
    kb_key = tau;
    kb_ties_kept = prm.top_k - static_cast<int>(gt);
    if (kb_ties_kept < static_cast<int>(ties)) kb_tie_idx = select_tie_index(c, S, tau, kb_ties_kept);
#pragma unroll
    for (int e = 0; e < kFastE; ++e) {
      const int id = c.lo + tid + e * kST;
      in_k[e] = valid[e] && (key[e] > kb_key || (key[e] == kb_key && id <= kb_tie_idx));
    }
  }
  uint32_t fb_key = kset ? kb_key : 0u;
  int fb_tie_idx = kb_tie_idx;
  bool kept[kFastE];
#pragma unroll
  for (int e = 0; e < kFastE; ++e) kept[e] = in_k[e];
  if (prm.top_p < 1.0) {
    // ---- top-p inside the top-k set: minimal prefix whose mass reaches p * Z
    uint32_t z[7] = {0u, 0u, 0u, 0u, 0u, 0u, 0u};
    float f[7];
    probe_sums(z, in_k, false, f);
    const float target = static_cast<float>(prm.top_p) * f[0];
    const uint32_t tau = search(in_k, false, target);
    float gt, ties;
    mass_gt_and_ties(in_k, false, tau, gt, ties);
    const float w_tau = expf(key2f(tau) - ymax);
    const int n_ties = static_cast<int>(ties);
    int keep = (w_tau > 0.f) ? static_cast<int>(ceilf((target - gt) / w_tau)) : n_ties;
    if (keep < 1) keep = 1;
    if (keep > n_ties) keep = n_ties;
    fb_key = tau;
    if (keep < n_ties)
      fb_tie_idx = select_tie_index(c, S, tau, keep);  // lowest ids first (<= kb_tie_idx)
    else
      fb_tie_idx = (kset && tau == kb_key) ? kb_tie_idx : INT32_MAX;
#pragma unroll
    for (int e = 0; e < kFastE; ++e) {
      const int id = c.lo + tid + e * kST;
      kept[e] = in_k[e] && (key[e] > fb_key || (key[e] == fb_key && id <= fb_tie_idx));
    }
  }
  // ---- Gumbel-max draw over the kept set (counter RNG keyed by seed, step, id)
  const uint64_t rkey = mix64(seed ^ (step * 0xD1B54A32D192ED03ull));
  float gv = -INFINITY;
  int gi = -1;
#pragma unroll
  for (int e = 0; e < kFastE; ++e) {
    if (!kept[e]) continue;
    const int id = c.lo + tid + e * kST;
    const float u = unit_open01(mix64(rkey + static_cast<uint64_t>(id)));
    better(gv, gi, y[e] - logf(-logf(u)), id);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float v2 = __shfl_xor_sync(0xffffffffu, gv, o);
    const int i2 = __shfl_xor_sync(0xffffffffu, gi, o);
    better(gv, gi, v2, i2);
  }
  __syncthreads();
  if (lane == 0) {
    S.redf[wid] = gv;
    S.redi[wid] = gi;
  }
  __syncthreads();
  if (tid == 0) {
    float v = S.redf[0];
    int i = S.redi[0];
    for (int k = 1; k < kST / 32; ++k) better(v, i, S.redf[k], S.redi[k]);
    if (i < 0) atomicMax(err_flag, static_cast<int>(VOX_ERR_DEGENERATE));
    S.i_b = i;
  }
  __syncthreads();
  return S.i_b;
}

// Whole-CTA sampling of one row.  Returns the token id (same in all threads).
VOX_DEV int sample_row(SampSmem& S, uint32_t* bm, const float* row, int col_base, int lo, int hi,
                       const int* win, int wlen, uint64_t seed, uint64_t step,
                       const VoxSampling& prm, int* err_flag) {
  const int tid = threadIdx.x;
  const int n = hi - lo;
  const int nwords = (n + 31) >> 5;
  if (wlen > kMaxWin) wlen = kMaxWin;
  const bool pen_on = prm.repetition_penalty != 1.0 && wlen > 0;
  for (int i = tid; i < nwords; i += kST) bm[i] = 0u;
  if (tid == 0) S.errv = 0;
  __syncthreads();
  if (pen_on) {
    for (int j = tid; j < wlen; j += kST) {
      const int t = win[j];
      S.win[j] = t;
      if (t >= lo && t < hi) atomicOr(&bm[(t - lo) >> 5], 1u << ((t - lo) & 31));
    }
  }
  __syncthreads();

  RowCtx c;
  c.row = row;
  c.col_base = col_base;
  c.lo = lo;
  c.hi = hi;
  c.bm = bm;
  c.pen_on = pen_on;
  c.pen_f = static_cast<float>(prm.repetition_penalty);
  c.temp = static_cast<float>(prm.temperature);
  c.inv_t = 0.f;

  const bool greedy = prm.temperature == 0.0 || prm.top_k == 1;

  // ---------------- pass 1: validation + (greedy argmax | max of y) ----------------
  float bv = -INFINITY;
  int bi = -1;
  int nfin = 0;
  bool bad = false;
  for (int id = lo + tid; id < hi; id += kST) {
    const float x = row[id - col_base];
    if (isnan(x) || x == INFINITY) bad = true;
    if (greedy) {
      if (!in_win(c, id)) better(bv, bi, x, id);
    } else {
      const float y = yval(c, id);
      if (y > -INFINITY) ++nfin;
      better(bv, bi, y, id);
    }
  }
  if (bad) atomicOr(&S.errv, 1);
  // block argmax (value desc, index asc)
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float v2 = __shfl_xor_sync(0xffffffffu, bv, o);
    const int i2 = __shfl_xor_sync(0xffffffffu, bi, o);
    better(bv, bi, v2, i2);
  }
  if ((tid & 31) == 0) {
    S.redf[tid >> 5] = bv;
    S.redi[tid >> 5] = bi;
  }
  nfin = static_cast<int>(block_reduce_sum<uint32_t>(static_cast<uint32_t>(nfin), S.redu, &S.u_b));
  if (tid == 0) {
    float v = S.redf[0];
    int i = S.redi[0];
    for (int k = 1; k < kST / 32; ++k) better(v, i, S.redf[k], S.redi[k]);
    S.f_a = v;
    S.i_a = i;
  }
  __syncthreads();
  if (S.errv) {
    if (tid == 0) atomicMax(err_flag, static_cast<int>(VOX_ERR_NONFINITE));
    return -1;
  }

  if (greedy) {
    // window tokens in fp64 (reference applies the penalty to fp64 values)
    if (tid == 0) {
      double best = (S.i_a >= 0) ? static_cast<double>(S.f_a) : -INFINITY;
      int besti = S.i_a;
      if (pen_on) {
        for (int j = 0; j < wlen; ++j) {
          const int t = S.win[j];
          if (t < lo || t >= hi) continue;
          const double xd = static_cast<double>(row[t - col_base]);
          const double pd = xd > 0.0 ? xd / prm.repetition_penalty : xd * prm.repetition_penalty;
          if (pd > best || (pd == best && (besti < 0 || t < besti))) {
            best = pd;
            besti = t;
          }
        }
      }
      if (best == -INFINITY) {  // all -inf (np.isfinite(arr).any() false)
        atomicMax(err_flag, static_cast<int>(VOX_ERR_DEGENERATE));
        besti = -1;
      }
      S.i_b = besti;
    }
    __syncthreads();
    return S.i_b;
  }

  // ---------------- stochastic ----------------
  const float ymax = S.f_a;
  if (nfin == 0) {
    if (tid == 0) atomicMax(err_flag, static_cast<int>(VOX_ERR_DEGENERATE));
    return -1;
  }
  if (n <= kST * kFastE) return sample_row_fast(S, c, ymax, nfin, seed, step, prm, err_flag);
  // boundary of the admissible (top-k) set: keys > kb_key, plus ties at
  // kb_key with index <= kb_tie_idx.  Default: everything finite.
  uint32_t kb_key = f2key(-INFINITY) + 1u;
  int kb_tie_idx = INT32_MAX;
  int kb_ties_kept = 0;  // ties at kb_key inside the set (for mass bookkeeping)
  const int shifts[3] = {21, 10, 0};
  const int nbits[3] = {11, 11, 10};

  if (prm.top_k > 0 && prm.top_k < nfin) {
    uint32_t prefix = 0, mask = 0;
    int rank = prm.top_k;  // rank-th largest
    for (int lv = 0; lv < 3; ++lv) {
      hist_pass<false>(c, S, prefix, mask, shifts[lv], nbits[lv], ymax, 0u, INT32_MAX);
      if (tid < 32) {
        int before = 0;
        const int r0 = rank;
        const int b = warp_scan_desc<int>(
            1 << nbits[lv], r0, [&](int x) { return static_cast<int>(S.hcnt[x]); },
            [&](int) { return true; }, &before);
        if (tid == 0) {
          S.u_a = static_cast<uint32_t>(b < 0 ? 0 : b);
          S.i_a = rank - before;
          S.i_b = b < 0 ? 0 : static_cast<int>(S.hcnt[b]);
        }
      }
      __syncthreads();
      prefix |= S.u_a << shifts[lv];
      mask |= ((1u << nbits[lv]) - 1u) << shifts[lv];
      rank = S.i_a;
      __syncthreads();
    }
    // prefix = exact key of the k-th largest; rank = how many of its ties are kept
    const int ties_total = S.i_b;
    kb_key = prefix;
    kb_ties_kept = rank;
    if (rank < ties_total) kb_tie_idx = select_tie_index(c, S, prefix, rank);
  }

  // final kept-set boundary (key, tie-index cut)
  uint32_t fb_key = kb_key;
  int fb_tie_idx = kb_tie_idx;
  if (prm.top_p < 1.0) {
    // total admissible mass Z with the first digit histogram
    uint32_t prefix = 0, mask = 0;
    float target = 0.f;
    int ties_at = 0;
    float w_tau = 0.f, s_gt = 0.f;
    for (int lv = 0; lv < 3; ++lv) {
      // levels 0,1: mass per bin; level 2 fixes the full key, so counts suffice
      if (lv < 2)
        hist_pass<true>(c, S, prefix, mask, shifts[lv], nbits[lv], ymax, kb_key, kb_tie_idx);
      else
        hist_pass<false>(c, S, prefix, mask, shifts[lv], nbits[lv], ymax, kb_key, kb_tie_idx);
      if (lv == 0) {
        float z = 0.f;
        for (int b = tid; b < kBins; b += kST) z += S.hmass[b];
        z = block_reduce_sum<float>(z, S.redf, &S.f_b);
        if (tid == 0) S.f_b = static_cast<float>(prm.top_p) * z;
      }
      __syncthreads();
      if (lv == 0) target = S.f_b;
      if (lv < 2) {
        if (tid < 32) {
          float before = 0.f;
          const int sel = warp_scan_desc<float>(
              1 << nbits[lv], target, [&](int x) { return S.hmass[x]; },
              [&](int x) { return S.hmass[x] > 0.f; }, &before);
          if (tid == 0) {
            S.u_a = static_cast<uint32_t>(sel < 0 ? 0 : sel);
            S.f_a = before;
          }
        }
        __syncthreads();
        prefix |= S.u_a << shifts[lv];
        mask |= ((1u << nbits[lv]) - 1u) << shifts[lv];
        target -= S.f_a;
        s_gt += S.f_a;
        __syncthreads();
      } else {
        // last digit: per-bin element value is exact (full key known)
        if (tid < 32) {
          // ties at the top-k boundary key count only up to the kept number
          auto cnt_of = [&](int x) {
            int cnt = static_cast<int>(S.hcnt[x]);
            const uint32_t kk = prefix | static_cast<uint32_t>(x);
            if (kk == kb_key && kb_ties_kept > 0 && cnt > kb_ties_kept) cnt = kb_ties_kept;
            return cnt;
          };
          float before = 0.f;
          const int sel = warp_scan_desc<float>(
              1 << nbits[lv], target,
              [&](int x) { return expf(key2f(prefix | static_cast<uint32_t>(x)) - ymax) * cnt_of(x); },
              [&](int x) { return S.hcnt[x] != 0u; }, &before);
          if (tid == 0) {
            S.u_a = static_cast<uint32_t>(sel < 0 ? 0 : sel);
            S.f_a = before;
            S.i_a = sel < 0 ? 0 : cnt_of(sel);
          }
        }
        __syncthreads();
        prefix |= S.u_a;
        target -= S.f_a;
        ties_at = S.i_a;
        __syncthreads();
      }
    }
    w_tau = expf(key2f(prefix) - ymax);
    int keep = (w_tau > 0.f) ? static_cast<int>(ceilf(target / w_tau)) : ties_at;
    if (keep < 1) keep = 1;
    if (keep > ties_at) keep = ties_at;
    (void)s_gt;
    fb_key = prefix;
    if (keep < ties_at || (prefix == kb_key && kb_tie_idx != INT32_MAX)) {
      // keep the `keep` lowest ids among admissible ties
      if (keep < ties_at) {
        fb_tie_idx = select_tie_index(c, S, prefix, keep);
      } else {
        fb_tie_idx = kb_tie_idx;
      }
    } else {
      fb_tie_idx = INT32_MAX;
    }
  }

  // ---------------- Gumbel-max draw over the kept set ----------------
  const uint64_t rkey = mix64(seed ^ (step * 0xD1B54A32D192ED03ull));
  float gv = -INFINITY;
  int gi = -1;
  for (int id = lo + tid; id < hi; id += kST) {
    const float y = yval(c, id);
    if (!(y > -INFINITY)) continue;
    const uint32_t k = f2key(y);
    if (k < fb_key || (k == fb_key && id > fb_tie_idx)) continue;
    const float u = unit_open01(mix64(rkey + static_cast<uint64_t>(id)));
    const float g = -logf(-logf(u));
    better(gv, gi, y + g, id);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const float v2 = __shfl_xor_sync(0xffffffffu, gv, o);
    const int i2 = __shfl_xor_sync(0xffffffffu, gi, o);
    better(gv, gi, v2, i2);
  }
  __syncthreads();
  if ((tid & 31) == 0) {
    S.redf[tid >> 5] = gv;
    S.redi[tid >> 5] = gi;
  }
  __syncthreads();
  if (tid == 0) {
    float v = S.redf[0];
    int i = S.redi[0];
    for (int k = 1; k < kST / 32; ++k) better(v, i, S.redf[k], S.redi[k]);
    if (i < 0) atomicMax(err_flag, static_cast<int>(VOX_ERR_DEGENERATE));
    S.i_b = i;
  }
  __syncthreads();
  return S.i_b;
}

// ---------------------------------------------------------------------------
// kernels
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kST)
    sample_desc_kernel(const float* __restrict__ logits, const SampRowDesc* __restrict__ rows,
                       const int* __restrict__ window_ids, int* __restrict__ out,
                       int* __restrict__ err_flag) {
  VOX_TRACE(kTrSampler);
  griddep_wait();
  griddep_launch();
  extern __shared__ uint32_t dyn_bm[];
  __shared__ SampSmem S;
  const SampRowDesc d = rows[blockIdx.x];
  const int tok = sample_row(S, dyn_bm, logits + d.logit_off, d.col_base, d.lo, d.hi,
                             window_ids + d.woff, d.wlen, d.seed, d.step, d.params, err_flag);
  if (threadIdx.x == 0) out[d.out_index] = tok;
}

__global__ void __launch_bounds__(kST) sample_fused_kernel(SampFusedArgs a) {
  VOX_TRACE(kTrSampler);
  // everything but the logits was written by the host or >= 2 launches upstream
  // (every kernel launches its dependents only after its own griddep_wait), so the
  // row, slot parameters and penalty window load before waiting for the LM head
  extern __shared__ uint32_t dyn_bm[];
  __shared__ SampSmem S;
  __shared__ int wbuf[kMaxWin];
  const int i = blockIdx.x;
  const int ri = a.sample_rows[i];
  if (ri < 0) {  // padding of the sample bucket
    griddep_wait();
    griddep_launch();
    if (threadIdx.x == 0) a.tokens_out[i] = -1;
    return;
  }
  const RowDev rw = a.rows[ri];
  if (rw.slot < 0) {
    griddep_wait();
    griddep_launch();
    return;
  }
  const int slot = rw.slot;
  const int P = a.slot_prompt_len[slot];
  const VoxSampling prm = a.slot_params[slot];
  const int step = rw.pos + 1 - P;  // generated-token index being produced
  int lo = 0, hi = a.vocab;
  if (a.audio_base >= 0) {
    const int k = step % a.frame_tokens;
    lo = a.audio_base + k * a.codebook_size;
    hi = lo + a.codebook_size;
  }
  // recent window = last W generated tokens (store positions P .. pos)
  int W = prm.penalty_window < kMaxWin ? prm.penalty_window : kMaxWin;
  const int ngen = step;  // tokens generated so far
  const int wlen = ngen < W ? ngen : W;
  const int* ts = a.token_store + static_cast<int64_t>(slot) * a.max_ctx;
  for (int j = threadIdx.x; j < wlen; j += kST) wbuf[j] = ts[P + ngen - wlen + j];
  griddep_wait();  // the LM head's logits
  griddep_launch();
  __syncthreads();
  const int tok = sample_row(S, dyn_bm, a.logits + static_cast<int64_t>(i) * a.ld, a.col_base, lo,
                             hi, wbuf, wlen, a.slot_seed[slot], static_cast<uint64_t>(step), prm,
                             a.err_flag);
  if (threadIdx.x == 0) {
    a.tokens_out[i] = tok;
    if (tok >= 0 && rw.pos + 1 < a.max_ctx)
      a.token_store[static_cast<int64_t>(slot) * a.max_ctx + rw.pos + 1] = tok;
  }
}

void launch_sample_fused(const SampFusedArgs& a, cudaStream_t st) {
  if (a.n_sample <= 0) return;
  const int span = a.audio_base >= 0 ? a.codebook_size : a.vocab;
  const size_t bm_bytes = static_cast<size_t>((span + 31) / 32) * 4;
  launch_k(sample_fused_kernel, dim3(a.n_sample), dim3(kST), bm_bytes, st, a);
}

void launch_sample_desc(const float* logits, const SampRowDesc* rows, int n,
                        const int* window_ids, int* tokens_out, int* err_flag, int max_span,
                        cudaStream_t st) {
  if (n <= 0) return;
  const size_t bm_bytes = static_cast<size_t>((max_span + 31) / 32) * 4;
  launch_k(sample_desc_kernel, dim3(n), dim3(kST), bm_bytes, st, logits, rows, window_ids, tokens_out, err_flag);
}

}  // namespace vox
