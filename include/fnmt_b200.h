/*
 * fnmt_b200.h — C ABI of the B200-native translation engine.
 *
 * The reference (`fastnmt`, /root/reference/pkg/src/fastnmt) is pure Python
 * with no FFI; its hot path is reached through a duck-typed protocol
 * (TranslationModel.encode / init_cache / step, model.py:370-389) and the
 * per-GEMM operator Projection.apply (model.py:84-90).  This header is the
 * drop-in boundary a reference-side binding (ctypes)
 * calls instead.  Every entry point:
 *   - takes plain pointers and sizes (no torch types);
 *   - returns 0 on success or a negative FNMT_E* status; fnmt_last_error()
 *     returns a thread-local message for the last failure on this thread;
 *   - per-op kernels (fnmt_linear ... fnmt_gather_rows) take DEVICE pointers
 *     and a cudaStream_t passed as void*, are stream-ordered, non-blocking,
 *     allocation-free and CUDA-graph capturable;
 *   - engine calls own their device memory and stream.
 * dtype codes: 0 = f32, 1 = f16, 2 = bf16; engines also take 3 = int8
 * (f32 activations, per-column int8 GEMM weights: the reference's int8
 * precision, store.py:29-36 / quant8.py).
 */
#ifndef FNMT_B200_H
#define FNMT_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

enum {
  FNMT_OK = 0,
  FNMT_E_INVALID = -1,  /* bad argument / shape (reference: ShapeError, ValueError) */
  FNMT_E_CUDA = -2,     /* CUDA runtime / driver failure */
  FNMT_E_LENGTH = -3,   /* exceeds max_positions (reference: LengthError, model.py:41) */
  FNMT_E_STATE = -4,    /* call order violated (e.g. translate before finalize) */
};

enum { FNMT_F32 = 0, FNMT_F16 = 1, FNMT_BF16 = 2 };

/* Mirrors ModelConfig (model.py:45-70). */
typedef struct fnmt_arch {
  int32_t n_enc_layers, n_dec_layers, d_model, n_heads_enc, n_heads_dec;
  int32_t ffn_dim_enc, ffn_dim_dec, vocab_size, max_positions;
  int32_t norm_l1;            /* 0 = "l2", 1 = "l1" */
  int32_t shared_embeddings;  /* 1 = src/tgt/out_proj share one table */
} fnmt_arch;

/* Mirrors RunConfig batching/search fields (cli.py:34-45) and SearchConfig
 * (search.py:28-39). */
typedef struct fnmt_run {
  int32_t sbatch, wbatch;     /* DecodeLimits (batching.py:35-42) */
  double max_len_ratio;       /* 1.5; binary64 like the reference's Python float */
  int32_t max_len_offset;     /* 5 */
  int32_t beam_size;          /* 1 = greedy */
  int32_t bos_id, eos_id, pad_id;
} fnmt_run;

typedef struct fnmt_stats {
  int64_t sentences, source_tokens, target_tokens, batches, decode_steps;
  int64_t gpu_launches;       /* kernel launches issued (graph nodes counted per replay) */
  double encode_ms, decode_ms, total_ms;
  int64_t device_bytes;       /* engine-owned device memory */
} fnmt_stats;

const char* fnmt_last_error(void);
const char* fnmt_version(void);

/* ---- per-op kernels (device pointers, stream-ordered) -------------------- */

/* C[M,N] = act(A[M,K] . W[N,K]^T + bias (+ resid)).  Replaces Projection.apply
 * (model.py:84-90) -> tensor.matmul (tensor.py:46-57).  a_dtype f16/bf16 runs
 * the tcgen05 kernel (W same dtype); f32 runs the fp32 SIMT kernel. */
int fnmt_linear(const void* A, int lda, int a_dtype, const void* W, int ldw, const float* bias,
                void* C, int ldc, int c_dtype, int M, int N, int K, int relu, const float* resid,
                int ld_resid, void* stream);

/* x = norm(x + A . W^T + bias) * gain + beta in place (f32 x [M, N]), plus
 * its copy in the A dtype (x_act, may be NULL) — Projection.apply followed by
 * the post-norm residual block of encode / decode_step (model.py:279-286,
 * :327-343, tensor.py:98-129): the GEMM adds into x in its epilogue, then one
 * row kernel normalises. */
int fnmt_linear_add_norm(const void* A, int lda, int a_dtype, const void* W, int ldw,
                         const float* bias, float* x, void* x_act, const float* gain,
                         const float* beta, int l1, int M, int N, int K, void* stream);

/* out_idx[m] = argmax_n (A[m,:] . W[n,:] + bias[n]), lowest n on ties — the
 * vocab projection (model.py:344) fused with np.argmax (search.py:71).
 * keys_scratch: M uint64 device words. */
int fnmt_linear_argmax(const void* A, int lda, int a_dtype, const void* W, int ldw,
                       const float* bias, int M, int N, int K, uint64_t* keys_scratch,
                       int32_t* out_idx, void* stream);

/* int8 projection: C = f32(qgemm(quantize_activations(A), W)) + bias — the
 * packed-int8 branch of Projection.apply (model.py:84-90 -> quant8.py:171-195,
 * :246-278) on tcgen05 kind::i8.  A: f32 [M, K] (lda).  Wq: s8 W^T [N, Kp]
 * K-major, Kp = K rounded up to 16, zero padded; scale / zp: per-column f32
 * (quant8.QuantizedMatrix.col_scale / col_zeropoint); colsum: s32 per-column
 * sum of the K real levels.  workspace: fnmt_qgemm_workspace(M, K) device
 * bytes.  Bit-identical to the reference's qgemm + bias in f32. */
int64_t fnmt_qgemm_workspace(int64_t M, int K);
int fnmt_qgemm(const float* A, int lda, const int8_t* Wq, const float* scale, const float* zp,
               const int32_t* colsum, const float* bias, float* C, int ldc, int M, int N, int K,
               int relu, void* workspace, int64_t workspace_bytes, void* stream);

/* x = table[ids] * scale + pos_table[pos_ids]  (model.py:276-277) */
int fnmt_embed(const int32_t* ids, const int32_t* pos_ids, const float* table,
               const float* pos_table, float scale, float* out32, void* out_act, int act_dtype,
               int n, int d, void* stream);

/* out = norm(x + y) * gain + bias; l1 = 0 -> layer_norm_l2, 1 -> layer_norm_l1
 * (model.py:193-196, tensor.py:98-129).  y may be NULL. */
int fnmt_add_norm(const float* x, const float* y, const float* gain, const float* bias, int l1,
                  float* out32, void* out_act, int act_dtype, int rows, int d, void* stream);

/* Varlen masked attention (model.py:199-245).  Sequence b: queries rows
 * q_start[b] .. +q_len[b], keys rows k_start[b] .. +k_len[b] (k_len 0 =>
 * all k_pad keys masked with -1e9, as the reference does). */
int fnmt_attention(const void* q, int ldq, const void* k, const void* v, int ldkv, void* out,
                   int ldo, int dtype, int heads, int dk, const int32_t* q_start,
                   const int32_t* q_len, const int32_t* k_start, const int32_t* k_len,
                   int k_pad, int n_seq, int max_q, int max_k, void* stream);

int fnmt_argmax_rows(const float* logits, int ld, int rows, int n, int32_t* out_idx,
                     void* stream);

/* dst row r = src row idx[r] (DecodeCache.select, model.py:170-181). */
int fnmt_gather_rows(const void* src, void* dst, const int32_t* idx, int rows,
                     int64_t row_bytes, int64_t src_stride, int64_t dst_stride, void* stream);

/* ---- engine (owns device weights, workspace, stream, CUDA graphs) -------- */

typedef struct fnmt_engine fnmt_engine;

/* dtype: FNMT_F16 / FNMT_BF16 (tensor cores, fp32 residual/LN/logits) or
 * FNMT_F32 (parity mode, TF32 off). */
int fnmt_engine_create(const fnmt_arch* arch, int device, int dtype, fnmt_engine** out);
void fnmt_engine_destroy(fnmt_engine* e);

/* Host float32 tensors by the reference manifest names (store.py:88-115) in
 * the reference orientation: gemm weights [k, n] (x @ W), out_proj [vocab, d]
 * (aliases src_embed when shared; may be omitted then). */
int fnmt_engine_set_tensor(fnmt_engine* e, const char* name, const float* host, int64_t numel);

/* int8 engines (dtype 3): a quantized GEMM weight by manifest name (or
 * "out_proj" as the [d, vocab] projection) in the reference orientation —
 * q s8 [k, n] row-major with per-column scale / zeropoint, exactly
 * quant8.QuantizedMatrix (quant8.py:74-82, store.py:337-361). */
int fnmt_engine_set_qtensor(fnmt_engine* e, const char* name, const int8_t* q, const float* scale,
                            const float* zp, int64_t k, int64_t n);

/* Validate, pre-transpose to K-major, cast, upload ("extract the transpose
 * operations to the beginning of decoding"). */
int fnmt_engine_finalize(fnmt_engine* e);

/* Size the workspace for batches under these caps (GPU defaults 3072/64000,
 * PAPER.md:179). */
int fnmt_engine_reserve(fnmt_engine* e, const fnmt_run* run);

/* Output budget per sentence: max(1, min(maxpos, ceil(ratio*len)+offset))
 * (search.py:49-51); writes budgets[n] and returns their sum (or <0). */
int64_t fnmt_budgets(const int32_t* lengths, int n, double ratio, int offset, int max_positions,
                     int32_t* budgets);

/* The scheduler's batch plan, host only (no GPU needed): plan_batches
 * (batching.py:100-109) — stable length-descending order, greedy maximal
 * batches under count <= sbatch and count * longest <= wbatch.  Writes the
 * sorted sentence order perm[n] (batching.py:68-70's permutation) and, per
 * batch, sizes[] / max_len[] / oversize[] (arrays of capacity n; max_len and
 * oversize may be NULL).  Returns the batch count (or <0).  This is the
 * planner fnmt_engine_translate runs internally. */
int fnmt_plan_batches(const int32_t* lengths, int n, int sbatch, int wbatch, int32_t* perm,
                      int32_t* sizes, int32_t* max_len, uint8_t* oversize);

/* Corpus-level greedy translation (greedy_translate over plan_batches,
 * batching.py:100-122 + search.py:58-86), HOST buffers:
 *   src ids for sentence i at ids[offsets[i] .. offsets[i+1]) (offsets n+1);
 *   output ids of sentence i written at out_ids[out_off[i] ..], out_len[i]
 *   tokens (out_off = exclusive prefix sum of fnmt_budgets). */
int fnmt_engine_translate(fnmt_engine* e, const int32_t* ids, const int64_t* offsets, int n,
                          const fnmt_run* run, int32_t* out_ids, const int64_t* out_off,
                          int32_t* out_len, fnmt_stats* stats);

/* Same, all buffers DEVICE-resident except `lengths` and `out_off` (host
 * copies of the metadata the scheduler plans with). */
int fnmt_engine_translate_device(fnmt_engine* e, const int32_t* d_ids, const int64_t* d_offsets,
                                 const int32_t* lengths, int n, const fnmt_run* run,
                                 int32_t* d_out_ids, const int64_t* out_off,
                                 const int64_t* d_out_off, int32_t* d_out_len,
                                 fnmt_stats* stats);

/* Protocol level (TranslationModel.encode / init_cache / step, model.py:370-389).
 * encode_padded: tokens int32 [b*s] row-major, lengths [b]; pad positions are
 * computed as queries (masked as keys) like the reference; writes f32 states
 * [b*s, d] and the compute-dtype copy [b*s, d]. */
int fnmt_engine_encode_padded(fnmt_engine* e, const int32_t* d_tokens, const int32_t* d_lengths,
                              int b, int s, float* d_states32, void* d_states_act);

/* Cross K/V of decoder layer `layer` from the compute-dtype encoder states:
 * out [rows, 2d] (k | v) in the compute dtype (model.py:290-305). */
int fnmt_engine_cross_kv(fnmt_engine* e, const void* d_states_act, int rows, int layer,
                         void* d_out);

/* One incremental decoder step (model.py:308-344) for `rows` rows at position
 * t.  self_k/self_v: per-layer device pointers to [rows, cap, d] caches;
 * cross_kv: per-layer [*, 2d]; row r attends to cross rows
 * k_start[r] .. +k_len[r] (k_len 0 => all k_pad masked).  Writes f32 logits
 * [rows, vocab]. */
int fnmt_engine_decode_step(fnmt_engine* e, const int32_t* d_prev, int t, int rows, int cap,
                            void* const* self_k, void* const* self_v,
                            const void* const* cross_kv, const int32_t* d_k_start,
                            const int32_t* d_k_len, int k_pad, int max_k, float* d_logits);

int64_t fnmt_engine_device_bytes(const fnmt_engine* e);

/* Concurrent decode lanes: extra workspaces/streams/graphs sharing the
 * weights; batches are dealt longest-first / shortest-first across lanes so
 * latency-bound decode steps overlap.  Default 3 (env FNMT_LANES). */
int fnmt_engine_set_lanes(fnmt_engine* e, int lanes);
void* fnmt_engine_stream(fnmt_engine* e);

/* Kernel classes for the per-launch profiler. */
enum {
  FNMT_K_EMBED = 0, FNMT_K_GEMM_ENC, FNMT_K_ATTN_ENC, FNMT_K_NORM, FNMT_K_GEMM_DEC,
  FNMT_K_ATTN_DEC, FNMT_K_VOCAB, FNMT_K_SEARCH, FNMT_K_OTHER, FNMT_K_COUNT
};
/* enable != 0: bracket every engine launch with CUDA events on the engine
 * stream (decode steps run un-captured) and reset the counters. */
int fnmt_engine_profile(fnmt_engine* e, int enable);
/* Per-class totals (arrays of FNMT_K_COUNT): device ms, launches, algorithmic
 * FLOPs, algorithmic bytes. */
int fnmt_engine_profile_read(fnmt_engine* e, double* ms, int64_t* launches, double* flops,
                             double* bytes);

/* Every launch of the profiled runs in launch order: kernel class, event
 * time (ms) and the algorithmic FLOPs / bytes counted for it.
 * Writes min(cap, count) entries (any pointer may be NULL) and returns the
 * count; lets a per-launch ncu DRAM-bytes list be matched launch by launch. */
int64_t fnmt_engine_profile_log(fnmt_engine* e, int32_t* cls, float* ms, double* flops,
                                double* bytes, int64_t cap);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif

#ifdef __cplusplus
}
#endif

#endif /* FNMT_B200_H */
