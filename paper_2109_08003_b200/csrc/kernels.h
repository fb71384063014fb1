// Internal launcher declarations shared by the engine and the C-ABI layer.
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <mutex>
#include <set>
#include <string>
#include <utility>

namespace fnmt {

// Opt a kernel into the full 227 KB of dynamic shared memory once (thread
// safe: decode lanes launch the same kernels from several host threads, and a
// per-launch attribute would race with another thread's launch).
inline cudaError_t set_max_smem(const void* func) {
  static std::mutex mu;
  static std::set<const void*> done;
  std::lock_guard<std::mutex> g(mu);
  if (done.count(func)) return cudaSuccess;
  cudaError_t e =
      cudaFuncSetAttribute(func, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
  if (e == cudaSuccess) done.insert(func);
  return e;
}

// Launch with the programmatic-stream-serialization attribute (PDL) unless
// FNMT_PDL=0.  Kernels launched this way call pdl_wait() before touching
// their predecessor's data (common.cuh).
bool pdl_enabled();
bool dual_cta_enabled();   // FNMT_GEMM_DUAL=0 disables 2-CTA/SM decoder GEMMs
template <typename... KArgs, typename... Args>
cudaError_t launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t s,
                     Args&&... args) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// GEMM epilogues: what happens to acc = A[m,:] . W[n,:] (fp32) for each (m, n).
enum Epilogue : int {
  kEpiStore = 0,   // C[m,n] = act(acc + bias[n] (+ resid[m,n]))   in c_dtype
  kEpiArgmax = 1,  // keys[m] = max over n < valid_n of key(acc + bias[n], n)
  kEpiTopK = 2,    // per (row, 256-column tile): max, sum exp(x - max), top-K (value, index)
  kEpiQKV = 3,     // decoder self q|k|v: q -> C, k / v -> KV cache slot (row*cap + *t_ptr)
  kEpiSlot = 4,    // C[(m*cap + *t_ptr), n] = acc + bias[n]: a whole row into its cache slot
};

// Per-(row, N-tile) partials of the beam epilogue; tile = n / kTopKTile.
constexpr int kTopKTile = 256;   // one partial per (row, 256-column GEMM tile)
constexpr int kTopKMax = 8;
struct TopKPartials {
  float* pmax;     // [rows][tiles]
  double* psum;    // [rows][tiles]
  float* pval;     // [rows][tiles][K]
  int32_t* pidx;   // [rows][tiles][K]
  int tiles;
  int K;           // 4 or 8 entries kept per tile
};

// Per-call scratch of the int8 GEMM: quantized activations [M, Kp] u8,
// their row sums, and the min / max keys of the f32 input.
struct QScratch {
  uint8_t* qa = nullptr;
  int32_t* rowsum = nullptr;
  unsigned int* stats = nullptr;   // [0] = key(max), [1] = ~key(min)  (zeroed per call)
  int64_t qa_bytes = 0;
  int64_t rows = 0;
};
inline int round_up16(int k) { return (k + 15) & ~15; }
int64_t qgemm_scratch_bytes(int64_t M, int K);   // qa + rowsum + stats, 256-B aligned parts
QScratch qgemm_scratch(void* base, int64_t M, int K);

// Encode the TMA descriptor of an s8 / u8 row-major [rows, Kp] matrix (box
// = [box_rows, 128 bytes], 128-B swizzle) for the int8 tcgen05 GEMM.
bool make_tmap_8(CUtensorMap* out, const void* base, int64_t rows, int64_t kp, int box_rows,
                 std::string* err);


struct GemmArgs {
  const void* A = nullptr;  // [M, K] row-major, leading dim lda (elements)
  int lda = 0;
  const void* W = nullptr;  // [N, K] row-major (K-major), leading dim ldw
  int ldw = 0;
  int in_dtype = 1;         // kF32 -> SIMT fp32 path; kF16 / kBF16 -> tcgen05 path
  const float* bias = nullptr;
  int M = 0, N = 0, K = 0;
  int epi = kEpiStore;
  void* C = nullptr;
  int ldc = 0;
  int c_dtype = 0;
  int relu = 0;
  const float* resid = nullptr;  // optional fp32 residual added before store
  int ld_resid = 0;
  unsigned long long* keys = nullptr;  // argmax keys per row (must be pre-zeroed)
  TopKPartials topk{};                 // kEpiTopK outputs
  void* kc = nullptr;                  // kEpiQKV: self K / V caches [rows*cap, seg]
  void* vc = nullptr;
  int cap = 0, seg = 0;
  const int32_t* t_ptr = nullptr;
  // greedy decode steps: rows [m_tab[*t_ptr], M) are past their budgets this
  // step (batch rows are in non-increasing budget order), so the GEMM stops
  // there (null: all M rows)
  const int32_t* m_tab = nullptr;
  // Pre-encoded TMA descriptors (tcgen05 path).  If null the launcher encodes
  // them on the fly (host cost ~ microseconds).
  const CUtensorMap* tmap_a = nullptr;
  const CUtensorMap* tmap_w = nullptr;
  // int8 path (quant8.py): A is f32 [M, K] activations, quantized per call to
  // u8 with one scale / zeropoint over the whole matrix; W is s8 W^T [N, Kp]
  // (Kp = K rounded up to 16, zero padded) with per-column scale / zeropoint
  // and column sums.  Set qw to select it (in_dtype must be kF32).
  const int8_t* qw = nullptr;
  const float* qscale = nullptr;
  const float* qzp = nullptr;
  const int32_t* qcolsum = nullptr;
  int Kp = 0;
  const CUtensorMap* qtmap_w = nullptr;
  QScratch qs{};
};

// Encode a 2-D TMA descriptor for a row-major [rows, cols] 16-bit matrix with
// leading dimension ld (elements), box = [box_rows, 64 cols], 128 B swizzle.
bool make_tmap_16(CUtensorMap* out, const void* base, int dtype, int64_t rows, int64_t cols,
                  int64_t ld, int box_rows, std::string* err);

int gemm_tile_n();  // N tile of the tcgen05 kernel (for W descriptors)

cudaError_t launch_gemm(const GemmArgs& g, cudaStream_t s);
// int8: quantize A (min / max, u8 + row sums) then the s8 tcgen05 GEMM (qgemm.cu)
cudaError_t launch_qgemm(const GemmArgs& g, cudaStream_t s);
cudaError_t launch_tc_i8(const CUtensorMap& ta, const GemmArgs& g, cudaStream_t s);

// ---------------------------------------------------------------------------
// row kernels

// x32[i,:] = table[ids[i],:] * scale + pos_table[pos(i),:]
// pos(i) = pos_ids ? pos_ids[i] : (*pos_scalar)  (device step counter)
cudaError_t launch_embed(const int32_t* ids, const int32_t* pos_ids, const int32_t* pos_scalar,
                         const float* table, const float* pos_table, float scale, float* x32,
                         void* xact, int act_dtype, int n, int d, cudaStream_t s);

// out = norm(x + y) with gain/bias; variant 0 = l2, 1 = l1 (tensor.py:98-129)
cudaError_t launch_add_norm(const float* x, const float* y, const float* gain,
                            const float* bias, int l1, float* out32, void* out_act,
                            int act_dtype, int rows, int d, cudaStream_t s,
                            const int32_t* rows_tab = nullptr, const int32_t* t_ptr = nullptr);
// same, the residual branch given as ny partial sums y + k * ystride (k < ny),
// added in order ((y0 + y1) + y2) + ... (split-K GEMM outputs)

// ---------------------------------------------------------------------------
// attention (model.py:199-240)

struct AttnArgs {
  const void* q; int ldq;         // query rows
  const void* k; const void* v; int ldkv;  // key / value rows
  void* out; int ldo;
  int dtype;                      // storage dtype of q/k/v/out
  int heads, dk;
  // varlen description: sequence b has queries rows [q_start[b], q_start[b]+q_len[b])
  // and keys rows [k_start[b], k_start[b] + k_len[b]); k_len[b]==0 means "all
  // k_pad keys masked" (reference's -1e9 everywhere case).
  const int32_t* q_start; const int32_t* q_len;
  const int32_t* k_start; const int32_t* k_len;
  int k_pad;                      // padded key count for the all-masked case
  int n_seq, max_q, max_k;
};
cudaError_t launch_attention_varlen(const AttnArgs& a, cudaStream_t s);
// tensor-core (mma.sync) variant for fp16 / bf16, dk % 16 == 0, <= 256 keys (attn_mma.cu)
bool attention_mma_ok(const AttnArgs& a);
cudaError_t launch_attention_varlen_mma(const AttnArgs& a, cudaStream_t s);

// Single-query attention for the incremental decoder.
// Self mode: keys of row r live at kv + (r*cap + j)*ldkv, j in [0, len) where
//   len = *len_scalar + 1 (device step counter), and this step's k/v (from
//   new_k/new_v rows) is first written to slot j = *len_scalar.
//   anc (optional, beam): key j of row r is taken from cache row anc[r*cap + j].
// Cross mode: row r attends to sequence seq = r / rows_per_seq, keys
//   kv + (k_start[seq] + j)*ldkv for j < k_len[seq] (k_len 0 -> all k_pad masked).
struct DecAttnArgs {
  const void* q; int ldq;
  const void* k; const void* v; int ldkv;
  void* k_w; void* v_w;                 // self mode: caches written at slot t
  const void* new_k; const void* new_v; int ld_new;
  void* out; int ldo;
  int dtype, heads, dk, rows;
  int self_mode;
  int cap;                              // self: slots per row
  const int32_t* t_ptr;                 // self: device step counter
  const int32_t* anc;                   // self beam: ancestor tables, 2 x [rows, cap] or null
  int64_t anc_buf_stride;               // elements between the two tables (step parity t & 1)
  const int32_t* k_start; const int32_t* k_len; int k_pad; int rows_per_seq;
  int max_k;
  // folded cross attention (engine.cu, fused_cross): each key row also carries
  // a per-key score offset at column kc_off (added as qscale * c_j; -1 = none),
  // and the output is written in fp32 with out_bias added (the o-projection's
  // bias: the values are already o-projected).
  int kc_off = -1;
  const float* out_bias = nullptr;
  int out_f32 = 0;
  // greedy corpus decode: rows whose sentence has finished (search.py:72 feeds
  // them PAD and discards their output) skip the attention entirely
  const uint8_t* row_done = nullptr;
};
cudaError_t launch_attention_decode(const DecAttnArgs& a, cudaStream_t s);

// Fused decoder attention block, single-head folded decoders (dec_layer.cu):
// self attention over the folded self cache -> + residual -> norm1 -> cross
// attention over the folded cross cache -> + residual -> norm2, one CTA per row.
struct DecLayerArgs {
  const void* q; int ldq;               // layer input (activation copy of x32)
  float* x32;                           // [rows, d] residual stream, updated in place
  void* xa;                             // [rows, d] activation copy of the output
  const void* kself; int ld_self;       // folded self cache rows r*cap + j
  int cap; const int32_t* t_ptr;
  const void* kcross; int ld_cross;     // folded cross cache rows k_start[seq] + j
  const int32_t* k_start; const int32_t* k_len; int k_pad; int rows_per_seq;
  int voff, kc_off;                     // V~ and c columns inside a cached row
  const float* bo_self; const float* g1; const float* b1;
  const float* bo_cross; const float* g2; const float* b2;
  int l1, dtype, d, rows;
  const uint8_t* row_done;
  // this step's self key row [rows, ld_self] written contiguously by the GEMM
  // (null: already in the cache slot); the kernel reads key t from here and
  // appends it to cache slot r*cap + t
  const void* knew;
};
bool dec_layer_fused_ok(int dtype, int d, int heads);
cudaError_t launch_dec_layer_fused(const DecLayerArgs& a, cudaStream_t s);

// ---------------------------------------------------------------------------
// search bookkeeping (search.py:58-86)

struct GreedyState {
  unsigned long long* keys;   // [rows] argmax keys of this step (reset to 0 here)
  int32_t* prev;              // [rows] next decoder input
  uint8_t* finished;          // [rows]
  const int32_t* budget;      // [rows]
  int32_t* out_ids;           // [rows, out_cap]
  int32_t* out_len;           // [rows]
  int32_t* t;                 // device step counter (incremented here)
  int32_t* alive;             // [1] rows still running after this step
  int rows, out_cap, eos, pad;
};
cudaError_t launch_greedy_update(const GreedyState& g, cudaStream_t s);
// next-step decoder input written by the greedy update (greedy_embed_kernel)
// Layer-0 folded self key row of a decoder input (engine.h DecL::tok_tab):
// knew[r] = act(tok_tab[tok] + pos_tab[pos]), [rows, w] (w = 2d + 8)
struct StepKey {
  const float* tok_tab;
  const float* pos_tab;
  void* knew;   // null: not used
  int w;
  // multi-head q | k | v rows (kc set): columns [0, seg) -> knew[r, seg],
  // [seg, 2 seg) -> kc[r cap + pos], [2 seg, 3 seg) -> vc[r cap + pos]
  void* kc;
  void* vc;
  int seg, cap;
};
cudaError_t launch_step_key(const StepKey& k, const int32_t* tok, const int32_t* t_ptr, int rows,
                            int act_dtype, cudaStream_t s);

struct GreedyEmbed {
  const float* table;   // [V, d] fp32 target embedding
  const float* pos;     // [n_pos, d] sinusoid table
  float scale;          // f32(sqrt(d))
  float* x32;           // [rows, d]
  void* xa;             // [rows, d] activation copy (fp16 / bf16) or null
  int act_dtype, d, n_pos;
  int32_t* done;        // CTA-completion counter (zero between launches)
  int32_t* alive_acc;   // alive accumulator (zero between launches)
  StepKey key;          // also write the next step's layer-0 self key row (key.knew set)
};
cudaError_t launch_greedy_embed(const GreedyState& g, const GreedyEmbed& e, cudaStream_t s);

cudaError_t launch_keys_to_index(const unsigned long long* keys, int rows, int32_t* out,
                                 cudaStream_t s);

// ---------------------------------------------------------------------------
// beam search (search.py:105-147), batched: row = sentence * k + slot

struct BeamState {
  int nS, k, cap, rows;
  int eos, pad;
  TopKPartials part;            // from the vocab GEMM epilogue (or logits_topk_partials)
  float* rval;                  // [rows][k] row top-k logits
  int32_t* ridx;                // [rows][k]
  double* rlogz;                // [rows] log-sum-exp of the row's logits
  int32_t* prev;                // [rows] next decoder input
  double* score;                // [rows]
  uint8_t* active;              // [rows]
  int32_t* anc;                 // 2 x [rows][cap] ancestor tables (parity t & 1)
  int32_t* tok_hist;            // [cap][rows] token appended at step t to slot
  int32_t* par_hist;            // [cap][rows] parent slot at step t
  const int32_t* budget;        // [nS]
  uint8_t* finished;            // [nS]
  int32_t* n_done;              // [nS]
  double* done_score;           // [nS][2k]
  int32_t* done_t;              // [nS][2k]
  int32_t* done_slot;           // [nS][2k]
  int32_t* fin_t;               // [nS] step of the final active set
  int32_t* fin_n;               // [nS] size of the final active set
  int32_t* t;                   // device step counter
  int32_t* alive;               // sentences still running
  uint32_t* ticket;             // grid-completion counter (last CTA bumps t)
  int32_t* out_ids;             // [nS][cap] final tokens
  int32_t* out_len;             // [nS]
  int32_t* scratch;             // [nS][2k][cap] backtracking buffer
};
cudaError_t launch_beam_init(const BeamState& b, int bos, cudaStream_t s);
cudaError_t launch_logits_topk_partials(const float* logits, int rows, int n,
                                        const TopKPartials& p, cudaStream_t s);
cudaError_t launch_beam_row_reduce(const BeamState& b, cudaStream_t s);
cudaError_t launch_beam_select(const BeamState& b, cudaStream_t s);
cudaError_t launch_beam_final(const BeamState& b, cudaStream_t s);
cudaError_t launch_argmax_rows(const float* logits, int ld, int rows, int n,
                               int32_t* out_idx, cudaStream_t s);
cudaError_t launch_gather_rows(const void* src, void* dst, const int32_t* idx, int rows,
                               int64_t row_bytes, int64_t src_stride, int64_t dst_stride,
                               cudaStream_t s);

}  // namespace fnmt
