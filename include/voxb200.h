/*
 * voxb200.h — C-ABI of the B200-native streaming-TTS serving hot path.
 *
 * This is the drop-in boundary behind the reference's Python model-execution
 * interface (/root/reference/pkg/src/speechserve/model_api.py).  Every entry
 * point takes plain pointers and sizes; no torch or C++ types cross it.  The
 * reference is pure Python, so the "reference-side binding" is a ctypes stub
 * (see INTEGRATION.md); the Python mirror of the reference Executor Protocol
 * lives in paper_2602_00269_b200/executor.py.
 *
 * Which reference interface each entry point replaces (file:line in
 * /root/reference/pkg/src/speechserve/):
 *   vox_admit         preprocess()                      model_api.py:238-275
 *   vox_forward       Executor.forward / lm_forward     model_api.py:209-211, 278-294
 *                     + sample()/sample_batch() fused   model_api.py:355-395
 *                     + next_input()                    model_api.py:297-308
 *   vox_sample_logits sample_batch() on given logits    model_api.py:384-395
 *   vox_detok         Executor.detokenize_windows       model_api.py:213-220, 398-435
 *                                                       profiles.py:333-356
 *   vox_release       (no reference hook; called on the final window,
 *                      profiles.py:279-290 / engine.py:346-353)
 *
 * Status codes map 1:1 onto the reference exception tree (errors.py:4-77);
 * see paper_2602_00269_b200/_lib.py:_STATUS_TO_EXC.
 *
 * Ownership: a VoxCtx owns ALL device memory (weights, paged KV pool, token
 * store, detokenizer state pool, workspaces, CUDA graphs).  One ctx per GPU
 * per process; calls on one ctx must be serialised by the caller (one engine
 * loop per ctx, as the reference requires: model_api.py:199-205).
 */
#ifndef VOXB200_H_
#define VOXB200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define VOX_ABI_VERSION 1

typedef enum VoxStatus {
  VOX_OK = 0,
  VOX_ERR_INVALID = 1,             /* ValueError                                  */
  VOX_ERR_BATCH_TOO_LARGE = 2,     /* errors.BatchTooLarge       errors.py:28     */
  VOX_ERR_DEGENERATE = 3,          /* errors.DegenerateDistribution errors.py:36  */
  VOX_ERR_CODEBOOK_MISMATCH = 4,   /* errors.CodebookMismatch    errors.py:40     */
  VOX_ERR_WINDOW_RULE = 5,         /* errors.WindowRuleViolation errors.py:44     */
  VOX_ERR_CACHE_MISSING = 6,       /* errors.CacheMissing        errors.py:48     */
  VOX_ERR_PROMPT_TOO_LONG = 7,     /* errors.PromptTooLong       errors.py:24     */
  VOX_ERR_INVALID_TOKEN_COUNT = 8, /* errors.InvalidTokenCount   errors.py:16     */
  VOX_ERR_NONFINITE = 9,           /* ValueError: NaN/+inf logits model_api.py:370 */
  VOX_ERR_OUT_OF_MEMORY = 10,      /* KV page pool / slot pool exhausted          */
  VOX_ERR_CUDA = 11,               /* CUDA runtime error (message in last_error)  */
  VOX_ERR_NO_DEVICE = 12,          /* no sm_100 device                            */
  VOX_ERR_EMPTY_BATCH = 13         /* errors.EmptyBatch          errors.py:32     */
} VoxStatus;

/* Model + capacity configuration.  Shapes follow a Llama-style backbone
 * (Orpheus-3B = Llama-3.2-3B dims) and a causal SNAC-24kHz-style decoder. */
typedef struct VoxModelCfg {
  /* backbone */
  int32_t n_layers, d_model, n_heads, n_kv_heads, head_dim, d_ff, vocab;
  float rope_theta, rms_eps;
  float embed_scale;        /* uniform init half-width of the (tied) embedding */
  int32_t text_vocab;       /* synthetic prompt ids are drawn from [0, text_vocab) */
  /* Orpheus audio-token layout: frame slot k of 7 may only emit ids in
   * [audio_base + k*codebook_size, audio_base + (k+1)*codebook_size).
   * audio_base < 0 disables the mask (generic LM). */
  int32_t audio_base, codebook_size, frame_tokens;
  /* capacity */
  int32_t page_size, n_pages, max_slots, max_ctx, max_rows;
  /* detokenizer (SNAC-24k-style, causal); detok_enabled = 0 skips it */
  int32_t detok_enabled;
  int32_t latent_dim, decoder_dim, n_rates;
  int32_t rates[4];
  int32_t max_detok_frames; /* max latent frames per detok call (all requests) */
  /* Qwen2-style bias on the fused q|k|v projection (CosyVoice2's LM); 0 = Llama */
  int32_t qkv_bias;
  /* CSM-style multi-codebook frames: n_codebooks > 1 adds a frame store of the
   * codebook-1..n-1 ids of every position; the input embedding of a position is
   * the sum of the embedding rows of all its ids (codebook 0 in the token store) */
  int32_t n_codebooks;
  /* ext_dim > 0: rows with token == -2 take their input from an external hidden
   * state of width ext_dim projected by this ctx's input projector (CSM depth
   * decoder position 0 = projected backbone state), see vox_project_ext */
  int32_t ext_dim;
} VoxModelCfg;

/* Per-request sampling parameters (SamplingParams, model_api.py:105-121). */
typedef struct VoxSampling {
  double temperature;        /* 0 = greedy (Python float, fp64 like the reference) */
  double top_p;              /* (0, 1]                                             */
  double repetition_penalty; /* >= 1                                               */
  int32_t top_k;             /* 0 = disabled                                       */
  int32_t penalty_window;    /* ring-window length (<= 256)                        */
} VoxSampling;

/* One row of a mixed prefill/decode batch.  A row feeds token_store[slot][pos]
 * (or `token` when >= 0, which is also written to the store) at position pos.
 * Rows with sample != 0 produce the next token into token_store[slot][pos+1]. */
typedef struct VoxRow {
  int32_t slot;
  int32_t pos;
  int32_t token;
  int32_t sample;
} VoxRow;

/* One detokenizer window (WindowSpec, profiles.py:115-124) bound to a slot. */
typedef struct VoxWindow {
  int32_t slot;
  int32_t index;      /* 1-based chunk ordinal */
  int32_t start;      /* first token (generated-token index) of the window */
  int32_t length;
  int32_t new_tokens; /* the last new_tokens of the window are new audio */
  int32_t final;
} VoxWindow;

typedef struct VoxCtx VoxCtx;

/* forward flags */
#define VOX_FWD_SAMPLE 1u       /* run K1 on rows with sample != 0 (clear: logits only) */
#define VOX_FWD_FULL_LOGITS 2u  /* LM head over the full vocab (parity path)        */
#define VOX_FWD_SYNC 4u         /* block until done (implied by host outputs)       */
#define VOX_FWD_NO_GRAPH 8u     /* eager launches (timing / debugging)              */

int vox_abi_version(void);
const char* vox_last_error(const VoxCtx* ctx); /* ctx may be NULL (global error) */

int vox_create(int device, const VoxModelCfg* cfg, uint64_t weight_seed, VoxCtx** out);
void vox_destroy(VoxCtx* ctx);

/* preprocess(): allocate a slot, reserve KV pages for prompt_len+target_len
 * tokens, write the synthetic prompt ids, reset detok state. */
int vox_admit(VoxCtx* ctx, uint64_t req_seed, int32_t prompt_len, int32_t target_len,
              const VoxSampling* params, int32_t* slot_out);
int vox_release(VoxCtx* ctx, int32_t slot);
int vox_page_table(VoxCtx* ctx, int32_t slot, int32_t* out, int32_t cap, int32_t* n_out);
int vox_read_tokens(VoxCtx* ctx, int32_t slot, int32_t pos, int32_t n, int32_t* out);
/* write host-chosen token ids into the device token store (drop-in path,
 * where the reference engine samples on the host: engine.py:294-303) */
int vox_write_tokens(VoxCtx* ctx, int32_t slot, int32_t pos, int32_t n, const int32_t* ids);
int vox_slot_info(VoxCtx* ctx, int32_t slot, int32_t* prompt_len, int32_t* target_len);

/* Mixed prefill/decode forward over n rows.  logits_out (host, may be NULL):
 * [n_sample, vocab] fp32 masked logits of the sampling rows, in row order
 * (requires VOX_FWD_FULL_LOGITS).  tokens_out (host, may be NULL): the sampled
 * ids of the sampling rows.  With both NULL and without VOX_FWD_SYNC the call
 * is asynchronous on the LM stream. */
int vox_forward(VoxCtx* ctx, const VoxRow* rows, int32_t n, uint32_t flags,
                float* logits_out, int32_t* tokens_out);

/* `steps` consecutive decode steps over the same rows in one call (no host round
 * trip between them): step k runs `rows` with every pos advanced by k, each
 * sampled row feeding the next step from the token store (CSM depth loop).
 * No host outputs; flags as vox_forward (VOX_FWD_SAMPLE required). */
int vox_forward_steps(VoxCtx* ctx, const VoxRow* rows, int32_t n, int32_t steps, uint32_t flags);

/* test/diagnostic readback of the logits the last vox_forward computed, exactly
 * as the LM head left them for K1 (graph path included): [n_rows][ld] fp32, column
 * j = vocabulary id col_base + j (the packed audio head covers the frame slots'
 * codebook rows only).  out == NULL only reports the layout; otherwise rows <=
 * n_rows and cols == ld.  Synchronises the LM stream. */
int vox_read_logits(VoxCtx* ctx, float* out, int32_t rows, int32_t cols, int32_t* n_rows,
                    int32_t* ld, int32_t* col_base);

/* sequence number of the last issued vox_forward (1-based), and a host wait
 * for forward `seq` to complete on the device (bounds host run-ahead) */
int vox_forward_seq(VoxCtx* ctx, int64_t* seq);
int vox_forward_wait(VoxCtx* ctx, int64_t seq);

/* K1 alone over caller logits (host, [n, vocab] fp32): window_ids [n, wcap]
 * (window_len[i] valid entries, oldest first), seeds/steps drive the
 * counter-based RNG, lo/hi restrict the candidate range ([0,vocab) = none). */
int vox_sample_logits(VoxCtx* ctx, const float* logits, int32_t n, int32_t vocab,
                      const VoxSampling* params, const int32_t* window_ids, int32_t wcap,
                      const int32_t* window_len, const uint64_t* seeds, const uint64_t* steps,
                      const int32_t* lo, const int32_t* hi, int32_t* tokens_out);

/* Detokenize n windows on the detok stream (after the LM stream's last
 * forward).  pcm_out (host, may be NULL): concatenated float PCM, request i
 * at offset sum(n_samples[:i]).  Returns a ticket usable with
 * vox_ticket_* when async (pcm_out == NULL). */
#define VOX_TICKET_RING 32 /* a ticket stays valid for the next 31 vox_detok calls */
int vox_detok(VoxCtx* ctx, const VoxWindow* w, int32_t n, float* pcm_out,
              int32_t* n_samples, int64_t* ticket);
int vox_ticket_query(VoxCtx* ctx, int64_t ticket, int32_t* done, double* t_ms);
int vox_ticket_pcm(VoxCtx* ctx, int64_t ticket, const float** pcm, int32_t* total);
int vox_clock_reset(VoxCtx* ctx); /* epoch event for vox_ticket_query t_ms */
int vox_synchronize(VoxCtx* ctx);

/* streams (cudaStream_t as void*) for external event timing */
int vox_streams(VoxCtx* ctx, void** lm_stream, void** detok_stream);

/* kernel-class timing with CUDA events on the launching stream (eager mode only) */
int vox_timing_enable(VoxCtx* ctx, int32_t on);
int vox_timing_read(VoxCtx* ctx, const char* name, double* total_ms, int64_t* launches,
                    double* bytes);
int vox_launch_count(VoxCtx* ctx, int64_t* launches); /* our kernels launched so far */
/* SMs of the LM stream's and the detok stream's partitions (detok 0: no split,
   both streams share every SM); VOX_DETOK_SMS at vox_create sets the split */
int vox_sm_partition(VoxCtx* ctx, int32_t* lm_sms, int32_t* detok_sms);

/* in-graph kernel tracer (diagnostics): vox_trace_arm allocates room for
 * `capacity` records and arms every instrumented kernel; vox_trace_read
 * synchronizes, copies up to `max_records` records {u32 tag, u32 smid,
 * u64 t_start_ns, u64 t_end_ns} (one per CTA, %globaltimer) and disarms. */
int vox_trace_arm(VoxCtx* ctx, int64_t capacity);
int vox_trace_read(VoxCtx* ctx, void* records, int64_t max_records, int64_t* n_records);

/* K3 alone (parity tests / roofline): out[n, m] = sum_k W[m, k] X[n, k] (+bias[m])
 * with W [M, K], X [N, K] bf16 (raw uint16 bits), fp32 out [N, M]; K % 64 == 0.
 * splits > 1 returns the split-K partial sum reduced on the host side of the
 * call.  iters > 1 repeats the launch and reports the mean kernel time. */
int vox_gemm_test(VoxCtx* ctx, const uint16_t* w, const uint16_t* x, const float* bias,
                  int32_t M, int32_t N, int32_t K, int32_t splits, int32_t iters, float* out,
                  double* mean_ms);

/* test-only: copy the last detok stage output (fp32) and the bf16 GEMM operand
 * buffer to the host, then make the next vox_detok stop after `stop_after`
 * pipeline stages (<= 0: run to completion). */
int vox_debug_detok(VoxCtx* ctx, int32_t stop_after, float* out, size_t n_floats,
                    uint16_t* bf_out, size_t n_bf);

/* multi-codebook frames (n_codebooks > 1): ids of codebooks 1..n-1 at positions
 * [pos, pos + n_pos) of a slot, [n_pos][n_codebooks - 1], -1 = none */
int vox_write_frame(VoxCtx* ctx, int32_t slot, int32_t pos, int32_t n_pos, const int32_t* ids);
int vox_read_frame(VoxCtx* ctx, int32_t slot, int32_t pos, int32_t n_pos, int32_t* out);
/* ext rows (ext_dim > 0): ext[0..n) = src.final_hidden[0..n) * P^T on the device,
 * where src.final_hidden are the sampled rows of src's last vox_forward (in row
 * order) and P [d_model, ext_dim] is this ctx's input projector.  Ordered after
 * src's LM stream; the next vox_forward of ctx reads ext row r for its row r
 * when that row has token == -2. */
int vox_project_ext(VoxCtx* ctx, VoxCtx* src, int32_t n);
/* device-side token hand-over between two ctxs on one device (no host sync):
 * links[i] = {dst_slot, dst_pos, src_slot, src_pos}.
 * mode 0: dst.tokens[dst_slot][dst_pos] = src.tokens[src_slot][src_pos] + offset
 * mode 1: dst.frame[dst_slot][dst_pos][k] = src.tokens[src_slot][src_pos + k] + offset,
 *         k = 0 .. dst.n_codebooks - 2 */
int vox_link_tokens(VoxCtx* dst, VoxCtx* src, const int32_t* links, int32_t n, int32_t offset,
                    int32_t mode);

/* Disaggregated LM -> detok (reference engine.py:119-123,150-156): copy
 * token-store spans spans[n][5] = {dst_slot, dst_pos, src_slot, src_pos, len} from the LM
 * context `src` into the detokenizer context `dst` (same GPU or an NVLink peer), ordered
 * after src's enqueued forwards and before dst's next detok work. */
int vox_copy_tokens(VoxCtx* dst, VoxCtx* src, const int32_t* spans, int32_t n);

/* weights / state introspection for parity tests (host copies) */
int vox_read_weight(VoxCtx* ctx, const char* name, int32_t layer, void* out, size_t bytes);
int vox_read_kv(VoxCtx* ctx, int32_t layer, int32_t slot, int32_t pos, float* k_out,
                float* v_out);

/* ------------------------------------------------------------------------
 * K7: Mimi-style 12.5 Hz streaming detokenizer (BASELINE config 3, CSM-1B-style;
 * [3P] transformers MimiModel.decode, modeling_mimi.py:1613-1680).  Replaces
 * Executor.detokenize_windows (model_api.py:213-220) for a depth-stage profile
 * (profiles.py:214-231: token_rate 12.5, stateful_detok) -- the reference's own
 * detokenizer is a stub (profiles.py:333-356).  A stream (vox_mimi_open) keeps its
 * conv padding caches and a sliding-window K/V ring on the device, so consecutive
 * vox_mimi_decode calls over its frames reproduce the full-sequence decode.
 * ------------------------------------------------------------------------ */
typedef struct VoxMimiCfg {
  int32_t n_q, n_semantic, cb_size, cb_dim;   /* split RVQ: codebooks x codes x dim  */
  int32_t hidden, n_layers, n_heads, ffn, window;
  float rope_theta, eps;
  int32_t filters, n_ratios, ratios[4];       /* SEANet: channels filters << n_ratios */
  int32_t kernel, last_kernel, res_kernel, compress;
  int32_t max_slots;                          /* concurrent streams                   */
  int32_t max_frames;                         /* 12.5 Hz frames per decode call       */
} VoxMimiCfg;

typedef struct VoxMimiReq {
  int32_t slot;     /* stream from vox_mimi_open                                  */
  int32_t n_frames; /* new frames, in order; 1 <= n_frames <= min(64, max_frames) */
} VoxMimiReq;

typedef struct VoxMimi VoxMimi;

int vox_mimi_create(int device, const VoxMimiCfg* cfg, uint64_t weight_seed, VoxMimi** out);
void vox_mimi_destroy(VoxMimi* m);
const char* vox_mimi_last_error(const VoxMimi* m); /* m may be NULL */
int vox_mimi_open(VoxMimi* m, int32_t* slot);      /* new stream, zero history     */
int vox_mimi_close(VoxMimi* m, int32_t slot);
/* codes: host [sum n_frames][n_q] int32 (request order); pcm_out: host
 * [sum n_frames * frame_samples] float (request order), blocking. */
int vox_mimi_decode(VoxMimi* m, const VoxMimiReq* reqs, int32_t n, const int32_t* codes,
                    float* pcm_out, int64_t* n_samples);
int vox_mimi_launch_count(VoxMimi* m, int64_t* launches);
/* CUDA-event time of the last decode's kernels (H2D of codes / D2H of PCM excluded) */
int vox_mimi_last_ms(VoxMimi* m, double* ms);

/* ------------------------------------------------------------------------
 * K8: CosyVoice2-style chunked detokenizer (BASELINE config 4): token-to-mel flow
 * matching (transformer encoder, CFG Euler ODE over a transformer estimator) + a
 * causal HiFT-style vocoder with an iSTFT head.  Replaces
 * Executor.detokenize_windows (model_api.py:213-220) for cosy_like
 * (profiles.py:163-179; its stub is profiles.py:333-356).  Every call consumes
 * the request's ref_tokens reference tokens plus the chunk's new tokens
 * (profiles.py:135 ref_window_tokens); the vocoder keeps per-request
 * conv histories + the iSTFT overlap tail across calls.
 * ------------------------------------------------------------------------ */
typedef struct VoxCosyCfg {
  int32_t vocab, ref_tokens;
  int32_t d_enc, enc_layers, enc_heads, enc_ffn, mel;
  int32_t d_est, est_layers, est_heads, est_ffn, n_steps;
  float cfg_rate, rope_theta, eps;
  int32_t voc_ch, n_ratios, ratios[4], voc_kernel, res_kernel, post_kernel, n_fft, hop;
  float slope;
  int32_t max_slots, max_tokens, max_chunk;
} VoxCosyCfg;

typedef struct VoxCosyReq {
  int32_t slot;     /* stream from vox_cosy_open                         */
  int32_t n_tokens; /* new speech tokens of this chunk (<= max_chunk)    */
} VoxCosyReq;

typedef struct VoxCosy VoxCosy;

int vox_cosy_create(int device, const VoxCosyCfg* cfg, uint64_t weight_seed, VoxCosy** out);
void vox_cosy_destroy(VoxCosy* m);
const char* vox_cosy_last_error(const VoxCosy* m); /* m may be NULL */
/* new request: reference tokens / speaker embedding / reference mel derived from
 * req_seed, zero vocoder history */
int vox_cosy_open(VoxCosy* m, uint64_t req_seed, int32_t* slot);
int vox_cosy_close(VoxCosy* m, int32_t slot);
/* tokens: host [sum n_tokens] int32 (request order); pcm_out: host
 * [sum n_tokens * samples_per_token] float, blocking */
int vox_cosy_decode(VoxCosy* m, const VoxCosyReq* reqs, int32_t n, const int32_t* tokens, float* pcm_out,
                    int64_t* n_samples);
int vox_cosy_last_ms(VoxCosy* m, double* ms);
int vox_cosy_launch_count(VoxCosy* m, int64_t* launches);

#ifdef __cplusplus
}
#endif
#endif /* VOXB200_H_ */
