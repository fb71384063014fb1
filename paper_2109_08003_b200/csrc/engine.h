// Engine object behind the fnmt_engine_* C ABI (see engine.cu).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>

#include <functional>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <unordered_map>
#include <vector>

#include "../../include/fnmt_b200.h"
#include "kernels.h"

namespace fnmt {

struct EngineError {
  int code;
  std::string msg;
  EngineError(int c, std::string m) : code(c), msg(std::move(m)) {}
};

extern thread_local std::string g_last_error;
void set_error(const std::string& m);

struct Lin {
  void* w = nullptr;   // W^T [N, K] in the compute dtype
  float* b = nullptr;  // [N]
  int N = 0, K = 0;
  CUtensorMap tm;      // TMA descriptor of W^T (tensor-core path)
  // int8 engines: s8 W^T [N, Kp] + per-column scale / zeropoint / level sums
  int8_t* qw = nullptr;
  float* qscale = nullptr;
  float* qzp = nullptr;
  int32_t* qcolsum = nullptr;
  int Kp = 0;
  CUtensorMap qtm;
};
struct HostQ {
  std::vector<int8_t> q;   // [k, n] row-major (reference orientation)
  std::vector<float> scale, zp;
  int64_t k = 0, n = 0;
};
struct Norm {
  float* g = nullptr;
  float* b = nullptr;
};
struct EncL {
  Lin qkv, o, f1, f2;
  Norm n1, n2;
};
struct DecL {
  Lin sqkv, so, cq, ckv, co, f1, f2;
  Lin fck;   // folded cross K|V|c (fused_cross): [K Wq^T | V Wo | bq.k] per encoder row
  Lin fsk;   // folded self K|V|c (fused_self): the same per decoder input row
  // layer 0 of a folded decoder: the layer input is the embedding E[tok] s + P[t],
  // so its folded self row is tok_tab[tok] + pos_tab[t] (fp32, [V, 2d + 8] and
  // [max_positions, 2d + 8], bias in pos_tab) -- a gather instead of a GEMM
  float* tok_tab = nullptr;
  float* pos_tab = nullptr;
  Norm n1, n2, n3;
  bool ffn = false;
};

struct Batch {
  std::vector<int32_t> rows;  // indices into the planned length list
  int32_t max_len = 0;
  bool oversize = false;
};
std::vector<Batch> plan_batches(const std::vector<int32_t>& lengths, int sbatch, int wbatch);
int budget_of(int32_t len, double ratio, int offset, int max_positions);

struct Workspace {
  int tok_cap = 0, row_cap = 0;
  int64_t pool_cap = 0;
  int64_t bytes = 0;
  std::vector<void*> owned;
  int32_t *ids = nullptr, *pos = nullptr, *cu = nullptr, *len = nullptr;
  int32_t *qstart = nullptr, *qlen = nullptr;
  float *x32 = nullptr, *y32 = nullptr;
  void *xa = nullptr, *qkv = nullptr, *att = nullptr, *h = nullptr;
  std::vector<void*> ckv, kc, vc;
  float *dx32 = nullptr, *dy32 = nullptr;
  void *dxa = nullptr, *dqkv = nullptr, *datt = nullptr, *dq = nullptr, *dh = nullptr;
  unsigned long long* keys = nullptr;
  int32_t *prev = nullptr, *budget = nullptr, *out_len = nullptr, *out_ids = nullptr;
  int32_t *t = nullptr, *alive = nullptr;
  uint8_t* finished = nullptr;
  CUtensorMap tm_xa, tm_att, tm_h, tm_dxa, tm_datt, tm_dh;
  QScratch qs{};   // int8 engines: quantized activations of the current GEMM
};

struct StepView {
  int rows = 0, cap = 0;
  const int32_t* prev = nullptr;
  const int32_t* t_ptr = nullptr;
  void* const* kc = nullptr;
  void* const* vc = nullptr;
  const void* const* ckv = nullptr;
  const int32_t* k_start = nullptr;
  const int32_t* k_len = nullptr;
  int k_pad = 0, rows_per_seq = 1, max_k = 0;
  const int32_t* anc = nullptr;        // beam: 2 ancestor tables (parity of t)
  int64_t anc_stride = 0;
  int host_t = 0;                      // host copy of the step (profiling byte counts only)
  // profiling (SURVEY §8(d) algorithmic counts): live rows at step t and the
  // sum of their unpadded source lengths; null = count every row / max_k keys
  const std::vector<int>* prof_live = nullptr;
  const std::vector<double>* prof_src = nullptr;
  const uint8_t* row_done = nullptr;   // greedy: finished flags (attention skips those rows)
  bool ws_caches = false;              // kc/vc/ckv are the workspace buffers (TMA maps valid)
  unsigned long long* keys = nullptr;  // argmax output (greedy)
  float* logits = nullptr;             // or full logits (protocol path / fp32 beam)
  const TopKPartials* topk = nullptr;  // beam: per-tile top-K partials
  const int32_t* m_tab = nullptr;      // greedy: rows inside their budget at step t (GemmArgs::m_tab)
  bool embed_done = false;             // the decoder input was written by the previous
                                       // step's greedy update (greedy_embed_kernel)
};

// Host + device metadata of one translate call, shared by all lanes.
struct PlanCtx {
  const std::vector<Batch>& plan;
  const std::vector<int32_t>& live_len;
  const std::vector<int32_t>& budget_all;
  const std::vector<int64_t>& batch_row0;
  const std::vector<int64_t>& batch_cu0;
  const int32_t* meta_perm;
  const int32_t* meta_cu;
  const int32_t* meta_budget;
  const int32_t* d_ids;
  const int64_t* d_off;
  int32_t* d_out_ids;
  const int64_t* d_out_off;
  int32_t* d_out_len;
  const fnmt_run& run;
};

struct BeamWs {
  std::vector<void*> owned;
  int64_t bytes = 0;
  int sent_cap = 0, k = 0;
  int64_t pool_cap = 0;
  TopKPartials part{};
  float* rval = nullptr;
  int32_t* ridx = nullptr;
  double* rlogz = nullptr;
  double* score = nullptr;
  uint8_t* active = nullptr;
  int32_t *anc = nullptr, *tok_hist = nullptr, *par_hist = nullptr;
  uint8_t* finished = nullptr;
  int32_t *n_done = nullptr, *fin_t = nullptr, *fin_n = nullptr;
  double* done_score = nullptr;
  int32_t *done_t = nullptr, *done_slot = nullptr;
  uint32_t* ticket = nullptr;
  int32_t *out_ids = nullptr, *out_len = nullptr, *scratch = nullptr;
  float* logits = nullptr;
};

class Engine {
 public:
  Engine(const fnmt_arch& a, int device, int dtype);
  ~Engine();

  void set_tensor(const std::string& name, const float* host, int64_t numel);
  void set_qtensor(const std::string& name, const int8_t* q, const float* scale, const float* zp,
                   int64_t k, int64_t n);
  bool q8 = false;   // int8 GEMM weights (dtype code 3): activations stay f32
  // Folded cross attention for single-head decoders (fp16 / bf16): the cross
  // query and output projections are multiplied into the per-batch cross K/V
  // (K~ = K Wq^T, V~ = V Wo, c = bq.k), removing two GEMMs from every step.
  bool fused_cross = false;
  // ... and the self attention folded the same way (greedy corpus decode): the
  // per-step q and self-o GEMMs disappear, the cache holds [K~ | V~ | c] rows.
  bool fused_self = false;
  int ckv_ld = 0;    // row stride (elements) of the workspace cross K/V
  void finalize();
  void reserve(int tok_cap, int row_cap, int64_t pool_cap);
  void reserve_for(const fnmt_run& run);

  void translate_device(const int32_t* d_ids, const int64_t* d_off,
                        const std::vector<int32_t>& lengths, const fnmt_run& run,
                        int32_t* d_out_ids, const int64_t* d_out_off, int32_t* d_out_len,
                        fnmt_stats* st);

  void encode_padded(const int32_t* d_tokens, const int32_t* d_lengths, int b, int s,
                     float* d_states32, void* d_states_act);
  void cross_kv(const void* d_states_act, int rows, int layer, void* d_out);
  void decode_step(const int32_t* d_prev, int t, int rows, int cap, void* const* self_k,
                   void* const* self_v, const void* const* cross_kv, const int32_t* d_k_start,
                   const int32_t* d_k_len, int k_pad, int max_k, float* d_logits);

  fnmt_arch arch;
  int device;
  int dt;
  cudaStream_t stream = nullptr;
  int64_t device_bytes = 0;
  int64_t launches = 0;

  // Concurrent decode lanes (engines sharing these weights); 4 by default
  // (r01: 1 / 2 / 3 lanes = 5.10 / 5.82 / 6.00 M target words/s on the early kernels;
  // final kernels 2 / 3 / 4 lanes = 6.71 / 6.98 / 7.04 M; each lane holds its own
  // ~1.3 GB workspace at the 3072 / 64000 caps).
  int n_lanes = 4;
  int64_t total_device_bytes() const {
    int64_t b = device_bytes;
    for (const auto& L : lanes) b += L->device_bytes;
    return b;
  }
  std::vector<std::unique_ptr<Engine>> lanes;
  std::unique_ptr<Engine> make_lane();
  int64_t run_batch(const PlanCtx& P, size_t bi);
  cudaEvent_t ev_done = nullptr;

  // Per-kernel-class profiling (CUDA events around every launch; disables
  // graph capture while on).  Totals are folded in after each translate call.
  void set_profiling(bool on);
  bool profiling = false;
  double prof_ms[FNMT_K_COUNT] = {};
  int64_t prof_n[FNMT_K_COUNT] = {};
  double prof_flops[FNMT_K_COUNT] = {};
  double prof_bytes[FNMT_K_COUNT] = {};
  // every profiled launch in launch order (class, event ms, algorithmic counts):
  // matched launch by launch against an ncu DRAM-bytes list of the same run
  struct ProfLog {
    int cls;
    float ms;
    double flops, bytes;
  };
  std::vector<ProfLog> prof_log;

 private:
  int prof_begin(cudaStream_t s);
  void prof_end(cudaStream_t s, int ev, int cls, double flops, double bytes);
  void prof_collect();
  struct ProfRec {
    int ev, cls;
    double flops, bytes;
  };
  std::vector<cudaEvent_t> prof_events;
  std::vector<ProfRec> prof_recs;
  size_t prof_used = 0;
  int gemm_cls = FNMT_K_GEMM_ENC;
  double prof_m = -1.0;   // >= 0: rows the profiler counts for GEMM / norm launches (live rows)
  // decode-step GEMMs / norms stop at the rows inside their budget (run_step)
  const int32_t* step_m_tab = nullptr;
  const int32_t* step_t_ptr = nullptr;
  int32_t* d_live_tab = nullptr;   // [max_positions + 2] live rows per step of the current batch
  int32_t* h_live_tab = nullptr;   // pinned staging of d_live_tab
  cudaEvent_t ev_live = nullptr;   // its copy has been issued / completed

  void* dalloc(size_t bytes);
  const std::vector<float>& need(const std::string& name, int64_t numel) const;
  float* upload_f32(const std::vector<float>& v);
  void* upload_act(const std::vector<float>& v);
  Lin make_lin(const std::vector<std::string>& wnames, const std::vector<std::string>& bnames,
               int k, const std::vector<int>& ns);
  Lin make_folded(const std::string& prefix, const std::string& blk,
                  std::vector<float>* wt_out = nullptr, std::vector<float>* bias_out = nullptr);
  void make_step_tables(DecL& L, const std::vector<float>& wt, const std::vector<float>& bias);
  StepKey step_keys_of(const StepView& v) const;
  void finish_lin(Lin& L);
  void make_qlin(Lin& L, const std::vector<std::string>& wnames, int k, const std::vector<int>& ns);
  void attach_q(GemmArgs& g, const Lin& L) const;
  Norm make_norm(const std::string& prefix);
  float emb_scale() const;

  void gemm(const void* A, const CUtensorMap* tmA, int lda, const Lin& L, int M, void* C, int ldc,
            int c_dtype, int relu, cudaStream_t s, const float* resid = nullptr);
  void gemm_argmax(const void* A, const CUtensorMap* tmA, int lda, int M,
                   unsigned long long* keys, cudaStream_t s);
  void norm(const float* x, const float* y, const Norm& n, float* o32, void* oa, int rows,
            cudaStream_t s);
  // x32 = norm(x32 + A.W + b) (and its storage-dtype copy xa): GEMM + add_norm.
  void gemm_norm(const void* A, const CUtensorMap* tmA, int lda, const Lin& L, int M, float* x32,
                 void* xa, float* y32, const Norm& n, cudaStream_t s, bool keep32 = true);
  void encoder_layers(int n_tok, int n_seq, int max_q, int max_k, const int32_t* qstart,
                      const int32_t* qlen, const int32_t* kstart, const int32_t* klen, int k_pad,
                      cudaStream_t s);
  void cross_kv_all(int n_tok, cudaStream_t s);
  void run_step(const StepView& v, cudaStream_t s);
  int64_t capture_step(const std::function<void()>& body);
  int drive_steps(int cap, int64_t nodes, const std::function<void(int)>& direct);
  StepView step_view(int rows, int cap, int max_len, int rows_per_seq);
  int decode_greedy(int R, int cap, int max_len, const fnmt_run& run,
                    const std::vector<int32_t>& src_len, const std::vector<int32_t>& budgets);
  int decode_beam(int R, int cap, int max_len, const fnmt_run& run,
                  const std::vector<int32_t>& budgets);
  const int32_t* live_table(const std::vector<int32_t>& budgets, int cap, int mult);
  void reserve_beam(int sent_cap, int k, int64_t pool_cap);
  BeamWs beam;
  void lens_from_cu(int R);
  void ensure_meta(size_t rows, size_t cus);

  std::unordered_map<std::string, std::vector<float>> host_tensors;
  std::unordered_map<std::string, HostQ> host_q;
  bool finalized = false;
  std::vector<void*> allocations;
  float* src_emb32 = nullptr;
  float* tgt_emb32 = nullptr;
  float* pos32 = nullptr;
  Lin out;
  std::vector<EncL> enc;
  std::vector<DecL> dec;
  Workspace ws;
  cudaGraphExec_t graph_exec = nullptr;
  std::vector<void*> graph_funcs;   // kernel functions of graph_exec's nodes, in node order
  cudaEvent_t ev_poll[2] = {nullptr, nullptr};
  cudaEvent_t ev_t0 = nullptr, ev_t1 = nullptr;
  int32_t* h_alive = nullptr;
  int32_t* d_bad = nullptr;   // source-id validation flag
  int32_t* meta_perm = nullptr;
  int32_t* meta_cu = nullptr;
  int32_t* meta_budget = nullptr;
  size_t meta_rows_cap = 0, meta_cu_cap = 0;
};

}  // namespace fnmt
