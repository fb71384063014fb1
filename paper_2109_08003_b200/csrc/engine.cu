// The translation engine: device-resident weights, a capacity-sized
// workspace, the packed-varlen encoder, the CUDA-graph-captured incremental
// decoder and the corpus-level scheduler.
//
// Reference path it replaces (pkg/src/fastnmt):
//   store.random_model / assemble_weights (store.py:191-253, :539-572)
//     -> fnmt_engine_set_tensor + finalize (pre-transposed, cast, uploaded once)
//   model.encode (model.py:261-287)            -> Engine::encode
//   model.init_cross_cache (model.py:290-305)  -> Engine::cross_kv
//   model.decode_step (model.py:308-344)       -> Engine::run_step (graph node list)
//   search.greedy_translate (search.py:58-86)  -> fused argmax epilogue + greedy_update kernel
//   batching.plan_batches / restore_order (batching.py:68-122)
//                                              -> plan_batches (host) + scatter kernel
//
// Layout in HBM (compute dtype T = f16/bf16, or f32 in parity mode):
//   weights: every projection W^T [N, K] (K-major), encoder/decoder q|k|v
//   fused to [3d, d], cross k|v fused to [2d, d]; the vocab projection is the
//   [V, d] embedding table itself (out_proj = src_embed^T => W^T = src_embed);
//   fp32 copies of the lookup tables and the sinusoid table.
//   encoder activations: packed varlen rows [tokens, *] (no padding rows).
//   self K/V cache: per layer [rows * cap, d], row r's step j at r*cap + j.
//   cross K/V: per layer packed [tokens, 2d].
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstring>
#include <map>
#include <numeric>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/fnmt_b200.h"
#include "common.cuh"
#include "engine.h"
#include "kernels.h"

namespace fnmt {

namespace {

__global__ void gather_batch_kernel(const int32_t* __restrict__ ids, const int64_t* __restrict__ off,
                                    const int32_t* __restrict__ perm, const int32_t* __restrict__ cu,
                                    int rows, int32_t* __restrict__ out_ids,
                                    int32_t* __restrict__ out_pos) {
  const int r = blockIdx.x;
  if (r >= rows) return;
  const int i = perm[r];
  const int64_t src = off[i];
  const int beg = cu[r], len = cu[r + 1] - cu[r];
  for (int j = threadIdx.x; j < len; j += blockDim.x) {
    out_ids[beg + j] = ids[src + j];
    out_pos[beg + j] = j;
  }
}

__global__ void scatter_out_kernel(const int32_t* __restrict__ out_ids, const int32_t* __restrict__ out_len,
                                   int cap, const int32_t* __restrict__ perm, int rows,
                                   const int64_t* __restrict__ dst_off, int32_t* __restrict__ dst_ids,
                                   int32_t* __restrict__ dst_len) {
  const int r = blockIdx.x;
  if (r >= rows) return;
  const int i = perm[r];
  const int n = out_len[r];
  const int64_t o = dst_off[i];
  for (int j = threadIdx.x; j < n; j += blockDim.x) dst_ids[o + j] = out_ids[(size_t)r * cap + j];
  if (threadIdx.x == 0) dst_len[i] = n;
}

__global__ void init_decode_kernel(int32_t* prev, uint8_t* finished, int32_t* out_len,
                                   unsigned long long* keys, int32_t* t, int32_t* alive, int rows,
                                   int bos) {
  for (int r = blockIdx.x * blockDim.x + threadIdx.x; r < rows; r += gridDim.x * blockDim.x) {
    prev[r] = bos;
    finished[r] = 0;
    out_len[r] = 0;
    keys[r] = 0ull;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    *t = 0;
    *alive = rows;
    t[2] = 0;   // greedy_embed_kernel: CTA-completion counter
    t[3] = 0;   // and alive accumulator
  }
}

// Reference _check_tokens (model.py:254-258): every source id in [0, V).
__global__ void check_ids_kernel(const int32_t* __restrict__ ids, const int64_t* __restrict__ off0,
                                 int64_t total, int V, int32_t* bad) {
  const int64_t base = *off0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t v = ids[base + i];
    if (v < 0 || v >= V) *bad = 1;
  }
}

__global__ void fill_i32_kernel(int32_t* p, int n, int v) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) p[i] = v;
}

__global__ void lens_from_cu_kernel(const int32_t* cu, int32_t* len, int R) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < R) len[r] = cu[r + 1] - cu[r];
}

__global__ void iota_pos_kernel(int32_t* pos, int b, int s) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < b * s) pos[i] = i % s;
}

__global__ void seq_table_kernel(int32_t* start, int32_t* qlen, int b, int s) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < b) {
    start[i] = i * s;
    qlen[i] = s;
  }
}

}  // namespace

thread_local std::string g_last_error;

void set_error(const std::string& m) { g_last_error = m; }

#define CK(expr)                                                                     \
  do {                                                                               \
    cudaError_t _e = (expr);                                                         \
    if (_e != cudaSuccess) {                                                         \
      throw EngineError(FNMT_E_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e)); \
    }                                                                                \
  } while (0)

// ---------------------------------------------------------------------------

std::vector<Batch> plan_batches(const std::vector<int32_t>& lengths, int sbatch, int wbatch) {
  // batching.py:68-109: stable length-descending order, then greedy maximal
  // batches under (count <= sbatch) and (count * longest <= wbatch).
  std::vector<int32_t> order(lengths.size());
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(),
                   [&](int32_t a, int32_t b) { return lengths[a] > lengths[b]; });
  std::vector<Batch> out;
  Batch cur;
  for (int32_t idx : order) {
    const int32_t L = lengths[idx];
    if (!cur.rows.empty()) {
      const int64_t n1 = (int64_t)cur.rows.size() + 1;
      if (n1 <= sbatch && n1 * cur.max_len <= wbatch) {
        cur.rows.push_back(idx);
        continue;
      }
      cur.oversize = cur.max_len > wbatch;
      out.push_back(std::move(cur));
      cur = Batch();
    }
    cur.rows.push_back(idx);
    cur.max_len = L;
  }
  if (!cur.rows.empty()) {
    cur.oversize = cur.max_len > wbatch;
    out.push_back(std::move(cur));
  }
  return out;
}

int budget_of(int32_t len, double ratio, int offset, int max_positions) {
  // search.py:49-51 (python float math: ceil(ratio * len) in binary64; the ratio
  // crosses the C ABI as a double so e.g. 1.2 is the same value Python multiplies)
  const double v = std::ceil(ratio * (double)len) + offset;
  int64_t b = (int64_t)v;
  b = std::min<int64_t>(b, max_positions);
  return (int)std::max<int64_t>(1, b);
}

// ---------------------------------------------------------------------------

Engine::Engine(const fnmt_arch& a, int device, int dtype) : arch(a), device(device), dt(dtype) {
  if (a.n_enc_layers < 1 || a.n_dec_layers < 1 || a.d_model < 1 || a.n_heads_enc < 1 ||
      a.n_heads_dec < 1 || a.ffn_dim_enc < 1 || a.vocab_size < 1 || a.max_positions < 1 ||
      a.ffn_dim_dec < 0)
    throw EngineError(FNMT_E_INVALID, "all sizes except ffn_dim_dec must be >= 1");
  if (a.d_model % a.n_heads_enc || a.d_model % a.n_heads_dec)
    throw EngineError(FNMT_E_INVALID, "d_model must be divisible by both head counts");
  if (a.d_model % 8 || a.ffn_dim_enc % 8 || a.ffn_dim_dec % 8)
    throw EngineError(FNMT_E_INVALID,
                      "the B200 engine needs d_model and FFN widths divisible by 8 (TMA strides)");
  if (dtype != kF32 && dtype != kF16 && dtype != kBF16 && dtype != 3)
    throw EngineError(FNMT_E_INVALID, "dtype must be 0 (f32), 1 (f16), 2 (bf16) or 3 (int8)");
  if (dtype == 3) {   // int8: f32 activations everywhere, int8 GEMM weights
    q8 = true;
    dt = kF32;
  }
  CK(cudaSetDevice(device));
  CK(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
  // blocking-sync poll events: a lane thread waiting on its alive count sleeps
  // instead of spinning a host core (8 ranks x 4 lanes share one host at N = 8)
  CK(cudaEventCreateWithFlags(&ev_poll[0], cudaEventDisableTiming | cudaEventBlockingSync));
  CK(cudaEventCreateWithFlags(&ev_poll[1], cudaEventDisableTiming | cudaEventBlockingSync));
  CK(cudaEventCreate(&ev_t0));
  CK(cudaEventCreate(&ev_t1));
  CK(cudaEventCreateWithFlags(&ev_done, cudaEventDisableTiming));
  if (const char* e = getenv("FNMT_LANES")) n_lanes = std::max(1, atoi(e));
  CK(cudaHostAlloc(&h_alive, 4 * sizeof(int32_t), cudaHostAllocDefault));
}

void Engine::set_profiling(bool on) {
  CK(cudaStreamSynchronize(stream));
  profiling = on;
  prof_used = 0;
  prof_recs.clear();
  prof_log.clear();
  for (int i = 0; i < FNMT_K_COUNT; ++i) {
    prof_ms[i] = prof_flops[i] = prof_bytes[i] = 0.0;
    prof_n[i] = 0;
  }
}

int Engine::prof_begin(cudaStream_t s) {
  if (!profiling) return -1;
  if (prof_used + 2 > prof_events.size()) {
    for (int i = 0; i < 256; ++i) {
      cudaEvent_t e;
      CK(cudaEventCreate(&e));
      prof_events.push_back(e);
    }
  }
  const int ev = (int)prof_used;
  prof_used += 2;
  CK(cudaEventRecord(prof_events[ev], s));
  return ev;
}

void Engine::prof_end(cudaStream_t s, int ev, int cls, double flops, double bytes) {
  if (ev < 0) return;
  CK(cudaEventRecord(prof_events[ev + 1], s));
  prof_recs.push_back(ProfRec{ev, cls, flops, bytes});
}

void Engine::prof_collect() {
  for (const ProfRec& r : prof_recs) {
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, prof_events[r.ev], prof_events[r.ev + 1]));
    prof_ms[r.cls] += ms;
    prof_n[r.cls] += 1;
    prof_flops[r.cls] += r.flops;
    prof_bytes[r.cls] += r.bytes;
    prof_log.push_back(ProfLog{r.cls, ms, r.flops, r.bytes});
  }
  prof_recs.clear();
  prof_used = 0;
}

Engine::~Engine() {
  lanes.clear();   // lanes share this engine's weights
  if (ev_done) cudaEventDestroy(ev_done);
  for (cudaEvent_t e : prof_events) cudaEventDestroy(e);
  cudaSetDevice(device);
  if (graph_exec) cudaGraphExecDestroy(graph_exec);
  if (stream) cudaStreamSynchronize(stream);
  for (void* p : allocations) cudaFree(p);
  if (h_alive) cudaFreeHost(h_alive);
  if (h_live_tab) {
    cudaEventDestroy(ev_live);
    cudaFreeHost(h_live_tab);
  }
  cudaEventDestroy(ev_poll[0]);
  cudaEventDestroy(ev_poll[1]);
  cudaEventDestroy(ev_t0);
  cudaEventDestroy(ev_t1);
  if (stream) cudaStreamDestroy(stream);
}

void* Engine::dalloc(size_t bytes) {
  void* p = nullptr;
  if (bytes == 0) bytes = 16;
  CK(cudaMalloc(&p, bytes));
  allocations.push_back(p);
  device_bytes += (int64_t)bytes;
  return p;
}

void Engine::set_tensor(const std::string& name, const float* host, int64_t numel) {
  host_tensors[name].assign(host, host + numel);
}

void Engine::set_qtensor(const std::string& name, const int8_t* q, const float* scale,
                         const float* zp, int64_t k, int64_t n) {
  if (!q8) throw EngineError(FNMT_E_INVALID, "set_qtensor needs an int8 engine (dtype 3)");
  HostQ& h = host_q[name];
  h.q.assign(q, q + k * n);
  h.scale.assign(scale, scale + n);
  h.zp.assign(zp, zp + n);
  h.k = k;
  h.n = n;
}

// int8 W^T [sum(n_i), Kp] from quantized [k, n_i] weights; the per-column
// statistics concatenate with the columns (fused q|k|v share one activation
// quantization because they project the same input, model.py:248-251).
void Engine::make_qlin(Lin& L, const std::vector<std::string>& wnames, int k,
                       const std::vector<int>& ns) {
  const int Kp = round_up16(k);
  int N = 0;
  for (int n : ns) N += n;
  std::vector<int8_t> wt((size_t)N * Kp, 0);
  std::vector<float> sc(N), zp(N);
  std::vector<int32_t> cs(N, 0);
  int row0 = 0;
  for (size_t p = 0; p < wnames.size(); ++p) {
    auto it = host_q.find(wnames[p]);
    if (it == host_q.end()) throw EngineError(FNMT_E_INVALID, "missing int8 tensor " + wnames[p]);
    const HostQ& h = it->second;
    if (h.k != k || h.n != ns[p])
      throw EngineError(FNMT_E_INVALID, "int8 tensor " + wnames[p] + " has the wrong shape");
    for (int i = 0; i < k; ++i)
      for (int j = 0; j < ns[p]; ++j) {
        const int8_t v = h.q[(size_t)i * ns[p] + j];
        wt[(size_t)(row0 + j) * Kp + i] = v;
        cs[row0 + j] += v;
      }
    std::copy(h.scale.begin(), h.scale.end(), sc.begin() + row0);
    std::copy(h.zp.begin(), h.zp.end(), zp.begin() + row0);
    row0 += ns[p];
  }
  L.Kp = Kp;
  L.qw = (int8_t*)dalloc(wt.size());
  CK(cudaMemcpy(L.qw, wt.data(), wt.size(), cudaMemcpyHostToDevice));
  L.qscale = upload_f32(sc);
  L.qzp = upload_f32(zp);
  L.qcolsum = (int32_t*)dalloc(sizeof(int32_t) * N);
  CK(cudaMemcpy(L.qcolsum, cs.data(), sizeof(int32_t) * N, cudaMemcpyHostToDevice));
  std::string err;
  if (!make_tmap_8(&L.qtm, L.qw, N, Kp, 64, &err))
    throw EngineError(FNMT_E_CUDA, "int8 weight TMA descriptor: " + err);
}

void Engine::attach_q(GemmArgs& g, const Lin& L) const {
  if (!L.qw) return;
  g.qw = L.qw;
  g.qscale = L.qscale;
  g.qzp = L.qzp;
  g.qcolsum = L.qcolsum;
  g.Kp = L.Kp;
  g.qtmap_w = &L.qtm;
  g.qs = ws.qs;
}

const std::vector<float>& Engine::need(const std::string& name, int64_t numel) const {
  auto it = host_tensors.find(name);
  if (it == host_tensors.end()) throw EngineError(FNMT_E_INVALID, "missing tensor " + name);
  if ((int64_t)it->second.size() != numel)
    throw EngineError(FNMT_E_INVALID, "tensor " + name + " has " +
                                          std::to_string(it->second.size()) + " values, expected " +
                                          std::to_string(numel));
  return it->second;
}

float* Engine::upload_f32(const std::vector<float>& v) {
  float* p = (float*)dalloc(v.size() * sizeof(float));
  CK(cudaMemcpy(p, v.data(), v.size() * sizeof(float), cudaMemcpyHostToDevice));
  return p;
}

void* Engine::upload_act(const std::vector<float>& v) {
  const size_t n = v.size();
  if (dt == kF32) return upload_f32(v);
  std::vector<uint16_t> h(n);
  for (size_t i = 0; i < n; ++i) {
    if (dt == kF16) {
      __half x = __float2half_rn(v[i]);
      std::memcpy(&h[i], &x, 2);
    } else {
      __nv_bfloat16 x = __float2bfloat16_rn(v[i]);
      std::memcpy(&h[i], &x, 2);
    }
  }
  void* p = dalloc(n * 2);
  CK(cudaMemcpy(p, h.data(), n * 2, cudaMemcpyHostToDevice));
  return p;
}

// Build W^T [sum(n_i), k] from reference-orientation weights [k, n_i] (x @ W).
Lin Engine::make_lin(const std::vector<std::string>& wnames, const std::vector<std::string>& bnames,
                     int k, const std::vector<int>& ns) {
  int N = 0;
  for (int n : ns) N += n;
  std::vector<float> wt(q8 ? 0 : (size_t)N * k), bias(N);
  int row0 = 0;
  for (size_t p = 0; p < wnames.size(); ++p) {
    const int n = ns[p];
    const auto& b = need(bnames[p], n);
    if (!q8) {
      const auto& w = need(wnames[p], (int64_t)k * n);
      for (int i = 0; i < k; ++i)
        for (int j = 0; j < n; ++j) wt[(size_t)(row0 + j) * k + i] = w[(size_t)i * n + j];
    }
    std::copy(b.begin(), b.end(), bias.begin() + row0);
    row0 += n;
  }
  Lin L;
  L.N = N;
  L.K = k;
  L.b = upload_f32(bias);
  if (q8) {
    make_qlin(L, wnames, k, ns);
    return L;
  }
  L.w = upload_act(wt);
  finish_lin(L);
  return L;
}

void Engine::finish_lin(Lin& L) {
  if (dt == kF32) return;
  std::string err;
  if (!make_tmap_16(&L.tm, L.w, dt, L.N, L.K, L.K, gemm_tile_n(), &err))
    throw EngineError(FNMT_E_CUDA, "weight TMA descriptor: " + err);
}

Norm Engine::make_norm(const std::string& prefix) {
  const int d = arch.d_model;
  return Norm{upload_f32(need(prefix + ".gain", d)), upload_f32(need(prefix + ".bias", d))};
}

// Folded attention weights of decoder layer `p`, block `blk` ("cross" or
// "self"; reference orientation x @ W, all [d, d]): rows of W^T [2d + 8, d]
//   a < d      : (Wk Wq^T)^T  -> K~ = E (Wk Wq^T) + bk Wq^T          (K Wq^T)
//   d + c      : (Wv Wo)^T    -> V~ = E (Wv Wo) + bv Wo              (V Wo)
//   2d         : Wk bq        -> c  = E (Wk bq) + bk . bq            (bq . k)
//   2d+1..2d+7 : 0 (16-byte row alignment)
// so q.k = x.K~ + c and (sum_j p_j v_j) Wo + bo = sum_j p_j V~_j + bo: the
// block's q and o GEMMs disappear from every decode step (model.py:316-336
// reassociated; computed in double, rounded once to the compute dtype).  E is
// the encoder output (cross, once per batch) or the decoder layer input of
// step j (self, appended to the cache at slot j).
Lin Engine::make_folded(const std::string& p, const std::string& blk, std::vector<float>* wt_out,
                        std::vector<float>* bias_out) {
  const int d = arch.d_model, N = 2 * d + 8;
  const auto& Wq = need(p + "." + blk + ".q_w", (int64_t)d * d);
  const auto& Wk = need(p + "." + blk + ".k_w", (int64_t)d * d);
  const auto& Wv = need(p + "." + blk + ".v_w", (int64_t)d * d);
  const auto& Wo = need(p + "." + blk + ".o_w", (int64_t)d * d);
  const auto& bq = need(p + "." + blk + ".q_b", d);
  const auto& bk = need(p + "." + blk + ".k_b", d);
  const auto& bv = need(p + "." + blk + ".v_b", d);
  std::vector<double> woT((size_t)d * d);   // woT[c][n] = Wo[n][c]
  for (int n = 0; n < d; ++n)
    for (int c = 0; c < d; ++c) woT[(size_t)c * d + n] = Wo[(size_t)n * d + c];
  std::vector<float> wt((size_t)N * d, 0.f), bias(N, 0.f);
  for (int a = 0; a < d; ++a) {
    const float* q = &Wq[(size_t)a * d];
    for (int b = 0; b < d; ++b) {
      const float* k = &Wk[(size_t)b * d];
      double acc = 0.0;
      for (int n = 0; n < d; ++n) acc += (double)k[n] * q[n];
      wt[(size_t)a * d + b] = (float)acc;
    }
    double bb = 0.0;
    for (int n = 0; n < d; ++n) bb += (double)bk[n] * q[n];
    bias[a] = (float)bb;
  }
  for (int c = 0; c < d; ++c) {
    const double* o = &woT[(size_t)c * d];
    for (int b = 0; b < d; ++b) {
      const float* v = &Wv[(size_t)b * d];
      double acc = 0.0;
      for (int n = 0; n < d; ++n) acc += (double)v[n] * o[n];
      wt[(size_t)(d + c) * d + b] = (float)acc;
    }
    double bb = 0.0;
    for (int n = 0; n < d; ++n) bb += (double)bv[n] * o[n];
    bias[d + c] = (float)bb;
  }
  for (int b = 0; b < d; ++b) {
    double acc = 0.0;
    for (int n = 0; n < d; ++n) acc += (double)Wk[(size_t)b * d + n] * bq[n];
    wt[(size_t)(2 * d) * d + b] = (float)acc;
  }
  double bc = 0.0;
  for (int n = 0; n < d; ++n) bc += (double)bk[n] * bq[n];
  bias[2 * d] = (float)bc;
  Lin L;
  L.N = N;
  L.K = d;
  L.w = upload_act(wt);
  L.b = upload_f32(bias);
  finish_lin(L);
  if (wt_out) *wt_out = std::move(wt);
  if (bias_out) *bias_out = std::move(bias);
  return L;
}

// Step tables of a layer-0 folded self block (see DecL::tok_tab): true-fp32
// GEMMs at load (gemm_simt_kernel, ascending-k FMA) of the scaled embedding
// table E s (fp32, as embed computes it) and of the sinusoid table P with the
// folded weights; the bias goes into the position table.  decode_step's layer-0
// input is x = tgt_embed[prev] sqrt(d) + positions[t] (model.py:327-328) and its
// self k / v projections (model.py:330-334, folded) are linear in x, so the
// step's key row is tok_tab[prev] + pos_tab[t] (distributivity; one rounding).
void Engine::make_step_tables(DecL& L, const std::vector<float>& wt,
                              const std::vector<float>& bias) {
  const int d = arch.d_model, N = (int)bias.size(), V = arch.vocab_size, np = arch.max_positions;
  const auto& E = arch.shared_embeddings ? need("src_embed", (int64_t)V * d)
                                         : need("tgt_embed", (int64_t)V * d);
  const float s = emb_scale();
  std::vector<float> es(E.size());
  for (size_t i = 0; i < E.size(); ++i) es[i] = E[i] * s;
  auto tmp = [](const std::vector<float>& v) {   // load-time temporaries (freed below)
    float* p = nullptr;
    CK(cudaMalloc(&p, v.size() * sizeof(float)));
    CK(cudaMemcpy(p, v.data(), v.size() * sizeof(float), cudaMemcpyHostToDevice));
    return p;
  };
  float* es_d = tmp(es);
  float* w_d = tmp(wt);
  float* b_d = tmp(bias);
  L.tok_tab = (float*)dalloc(sizeof(float) * (size_t)V * N);
  L.pos_tab = (float*)dalloc(sizeof(float) * (size_t)np * N);
  auto run = [&](const float* A, int M, const float* b, float* C) {
    GemmArgs g;
    g.A = A;
    g.lda = d;
    g.W = w_d;
    g.ldw = d;
    g.in_dtype = kF32;
    g.bias = b;
    g.M = M;
    g.N = N;
    g.K = d;
    g.epi = kEpiStore;
    g.C = C;
    g.ldc = N;
    g.c_dtype = kF32;
    CK(launch_gemm(g, stream));
  };
  run(es_d, V, nullptr, L.tok_tab);
  run(pos32, np, b_d, L.pos_tab);
  CK(cudaStreamSynchronize(stream));
  CK(cudaFree(es_d));
  CK(cudaFree(w_d));
  CK(cudaFree(b_d));
}

// multi-head decoders (opt-in, FNMT_STEP_TABLES_MH=1): 6-1-8 bench 7.49 vs 7.31 M
// words/s, but the s618 corpus fixture drops to 504 / 512 identical (all
// near-ties, vs 509 / 512 with the QKV GEMM) -- under the 99% bar
bool step_tables_mh_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("FNMT_STEP_TABLES_MH");
    on = e && e[0] == '1';
  }
  return on != 0;
}

bool step_tables_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("FNMT_STEP_TABLES");
    on = !(e && e[0] == '0');
  }
  return on != 0;
}

bool live_rows_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("FNMT_LIVE_ROWS");
    on = !(e && e[0] == '0');
  }
  return on != 0;
}

bool greedy_embed_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("FNMT_GREEDY_EMBED");
    on = !(e && e[0] == '0');
  }
  return on != 0;
}

bool knew_staging_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("FNMT_KNEW_STAGE");
    on = !(e && e[0] == '0');
  }
  return on != 0;
}

bool fused_self_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("FNMT_FUSED_SELF");
    on = !(e && e[0] == '0');
  }
  return on != 0;
}

bool fused_cross_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("FNMT_FUSED_CROSS");
    on = !(e && e[0] == '0');
  }
  return on != 0;
}

void Engine::finalize() {
  CK(cudaSetDevice(device));
  const int d = arch.d_model, V = arch.vocab_size;
  const auto& src = need("src_embed", (int64_t)V * d);
  src_emb32 = upload_f32(src);
  if (arch.shared_embeddings) {
    tgt_emb32 = src_emb32;
  } else {
    tgt_emb32 = upload_f32(need("tgt_embed", (int64_t)V * d));
  }
  // positions: prefer the caller's table (bit-identical to numpy's sinusoid);
  // otherwise compute it (model.py:184-190).
  if (host_tensors.count("positions")) {
    pos32 = upload_f32(need("positions", (int64_t)arch.max_positions * d));
  } else {
    std::vector<float> p((size_t)arch.max_positions * d);
    for (int r = 0; r < arch.max_positions; ++r)
      for (int i = 0; i < d; ++i) {
        const double ang = (double)r / std::pow(10000.0, (2.0 * std::floor(i / 2.0)) / d);
        p[(size_t)r * d + i] = (float)((i % 2 == 0) ? std::sin(ang) : std::cos(ang));
      }
    pos32 = upload_f32(p);
  }
  // vocab projection W^T == out_proj table [V, d]
  {
    out.N = V;
    out.K = d;
    out.b = upload_f32(need("out_bias", V));
    if (q8) {
      make_qlin(out, {"out_proj"}, d, {V});   // quantized [d, vocab] projection
    } else {
      const std::vector<float>* table = &src;
      if (!arch.shared_embeddings) table = &need("out_proj", (int64_t)V * d);
      out.w = upload_act(*table);
      finish_lin(out);
    }
  }
  enc.clear();
  for (int i = 0; i < arch.n_enc_layers; ++i) {
    const std::string p = "enc." + std::to_string(i);
    EncL L;
    L.qkv = make_lin({p + ".attn.q_w", p + ".attn.k_w", p + ".attn.v_w"},
                     {p + ".attn.q_b", p + ".attn.k_b", p + ".attn.v_b"}, d, {d, d, d});
    L.o = make_lin({p + ".attn.o_w"}, {p + ".attn.o_b"}, d, {d});
    L.f1 = make_lin({p + ".ffn.w1"}, {p + ".ffn.b1"}, d, {arch.ffn_dim_enc});
    L.f2 = make_lin({p + ".ffn.w2"}, {p + ".ffn.b2"}, arch.ffn_dim_enc, {d});
    L.n1 = make_norm(p + ".norm1");
    L.n2 = make_norm(p + ".norm2");
    enc.push_back(L);
  }
  fused_cross = dt != kF32 && !q8 && arch.n_heads_dec == 1 && d % 256 == 0 &&
                fused_cross_enabled();
  ckv_ld = fused_cross ? 2 * d + 8 : 2 * d;
  fused_self = fused_cross && fused_self_enabled();
  dec.clear();
  for (int i = 0; i < arch.n_dec_layers; ++i) {
    const std::string p = "dec." + std::to_string(i);
    DecL L;
    L.sqkv = make_lin({p + ".self.q_w", p + ".self.k_w", p + ".self.v_w"},
                      {p + ".self.q_b", p + ".self.k_b", p + ".self.v_b"}, d, {d, d, d});
    L.so = make_lin({p + ".self.o_w"}, {p + ".self.o_b"}, d, {d});
    L.cq = make_lin({p + ".cross.q_w"}, {p + ".cross.q_b"}, d, {d});
    L.ckv = make_lin({p + ".cross.k_w", p + ".cross.v_w"}, {p + ".cross.k_b", p + ".cross.v_b"},
                     d, {d, d});
    L.co = make_lin({p + ".cross.o_w"}, {p + ".cross.o_b"}, d, {d});
    if (fused_cross) L.fck = make_folded(p, "cross");
    if (fused_self) {
      std::vector<float> wt, bias;
      const bool tables = i == 0 && step_tables_enabled();
      L.fsk = make_folded(p, "self", tables ? &wt : nullptr, tables ? &bias : nullptr);
      if (tables) make_step_tables(L, wt, bias);
    } else if (i == 0 && dt != kF32 && !q8 && step_tables_mh_enabled()) {
      // layer-0 q | k | v of a multi-head (unfolded) decoder: W^T [3d, d] in fp32
      std::vector<float> wt((size_t)3 * d * d), bias((size_t)3 * d);
      const char* part[3] = {"q", "k", "v"};
      for (int s3 = 0; s3 < 3; ++s3) {
        const auto& w = need(p + ".self." + part[s3] + "_w", (int64_t)d * d);
        const auto& b = need(p + ".self." + part[s3] + "_b", d);
        for (int k = 0; k < d; ++k)
          for (int n = 0; n < d; ++n) wt[((size_t)s3 * d + n) * d + k] = w[(size_t)k * d + n];
        std::copy(b.begin(), b.end(), bias.begin() + (size_t)s3 * d);
      }
      make_step_tables(L, wt, bias);
    }
    L.n1 = make_norm(p + ".norm1");
    L.n2 = make_norm(p + ".norm2");
    L.ffn = arch.ffn_dim_dec > 0;
    if (L.ffn) {
      L.f1 = make_lin({p + ".ffn.w1"}, {p + ".ffn.b1"}, d, {arch.ffn_dim_dec});
      L.f2 = make_lin({p + ".ffn.w2"}, {p + ".ffn.b2"}, arch.ffn_dim_dec, {d});
      L.n3 = make_norm(p + ".norm3");
    }
    dec.push_back(L);
  }
  host_tensors.clear();
  host_tensors.rehash(0);
  host_q.clear();
  finalized = true;
  CK(cudaDeviceSynchronize());
}

// ---------------------------------------------------------------------------
// workspace

void Engine::reserve(int tok_cap, int row_cap, int64_t pool_cap) {
  if (!finalized) throw EngineError(FNMT_E_STATE, "finalize() before reserve()");
  if (tok_cap <= ws.tok_cap && row_cap <= ws.row_cap && pool_cap <= ws.pool_cap) return;
  tok_cap = std::max(tok_cap, ws.tok_cap);
  row_cap = std::max(row_cap, ws.row_cap);
  pool_cap = std::max(pool_cap, ws.pool_cap);
  CK(cudaStreamSynchronize(stream));
  for (void* p : ws.owned) {
    cudaFree(p);
    allocations.erase(std::find(allocations.begin(), allocations.end(), p));
  }
  device_bytes -= ws.bytes;
  ws = Workspace();
  const int64_t before = device_bytes;
  auto alloc = [&](size_t bytes) {
    void* p = dalloc(bytes);
    ws.owned.push_back(p);
    return p;
  };
  const int d = arch.d_model, es = dtype_size(dt);
  const int fe = arch.ffn_dim_enc, fd = std::max(arch.ffn_dim_dec, 8);
  ws.tok_cap = tok_cap;
  ws.row_cap = row_cap;
  ws.pool_cap = pool_cap;
  ws.ids = (int32_t*)alloc(sizeof(int32_t) * tok_cap);
  ws.pos = (int32_t*)alloc(sizeof(int32_t) * tok_cap);
  ws.cu = (int32_t*)alloc(sizeof(int32_t) * (row_cap + 1));
  ws.len = (int32_t*)alloc(sizeof(int32_t) * row_cap);
  ws.qstart = (int32_t*)alloc(sizeof(int32_t) * row_cap);
  ws.qlen = (int32_t*)alloc(sizeof(int32_t) * row_cap);
  ws.x32 = (float*)alloc(sizeof(float) * (size_t)tok_cap * d);
  ws.y32 = (float*)alloc(sizeof(float) * (size_t)tok_cap * d);
  ws.xa = dt == kF32 ? (void*)ws.x32 : alloc((size_t)es * tok_cap * d);
  ws.qkv = alloc((size_t)es * tok_cap * 3 * d);
  ws.att = alloc((size_t)es * tok_cap * d);
  ws.h = alloc((size_t)es * tok_cap * fe);
  ws.ckv.assign(arch.n_dec_layers, nullptr);
  ws.kc.assign(arch.n_dec_layers, nullptr);
  ws.vc.assign(arch.n_dec_layers, nullptr);
  for (int l = 0; l < arch.n_dec_layers; ++l) {
    ws.ckv[l] = alloc((size_t)es * tok_cap * ckv_ld);
    // self K / V caches [pool_cap, d] each; with folded self attention the same
    // allocation also holds the interleaved [K~ | V~ | c | 0] rows [pool_cap, 2d + 8]
    ws.kc[l] = alloc((size_t)es * pool_cap * (fused_self ? 2 * d + 8 : 2 * d));
    ws.vc[l] = (char*)ws.kc[l] + (size_t)es * pool_cap * d;
  }
  ws.dx32 = (float*)alloc(sizeof(float) * (size_t)row_cap * d);
  ws.dy32 = (float*)alloc(sizeof(float) * (size_t)row_cap * d);
  ws.dxa = dt == kF32 ? (void*)ws.dx32 : alloc((size_t)es * row_cap * d);
  ws.dqkv = alloc((size_t)es * row_cap * 3 * d);
  ws.datt = alloc((size_t)es * row_cap * d);
  ws.dq = alloc((size_t)es * row_cap * d);
  ws.dh = alloc((size_t)es * row_cap * fd);
  ws.keys = (unsigned long long*)alloc(sizeof(unsigned long long) * row_cap);
  ws.prev = (int32_t*)alloc(sizeof(int32_t) * row_cap);
  ws.budget = (int32_t*)alloc(sizeof(int32_t) * row_cap);
  ws.out_len = (int32_t*)alloc(sizeof(int32_t) * row_cap);
  ws.finished = (uint8_t*)alloc(row_cap);
  ws.out_ids = (int32_t*)alloc(sizeof(int32_t) * pool_cap);
  ws.t = (int32_t*)alloc(sizeof(int32_t) * 4);
  ws.alive = ws.t + 1;
  if (q8) {
    const int kmax = std::max(d, std::max(fe, fd));
    const int64_t rows = std::max<int64_t>(tok_cap, row_cap);
    ws.qs = qgemm_scratch(alloc(qgemm_scratch_bytes(rows, kmax)), rows, kmax);
  }
  if (dt != kF32) {
    std::string err;
    bool ok = make_tmap_16(&ws.tm_xa, ws.xa, dt, tok_cap, d, d, 128, &err) &&
              make_tmap_16(&ws.tm_att, ws.att, dt, tok_cap, d, d, 128, &err) &&
              make_tmap_16(&ws.tm_h, ws.h, dt, tok_cap, fe, fe, 128, &err) &&
              make_tmap_16(&ws.tm_dxa, ws.dxa, dt, row_cap, d, d, 128, &err) &&
              make_tmap_16(&ws.tm_datt, ws.datt, dt, row_cap, d, d, 128, &err) &&
              make_tmap_16(&ws.tm_dh, ws.dh, dt, row_cap, fd, fd, 128, &err);
    if (!ok) throw EngineError(FNMT_E_CUDA, "workspace TMA descriptor: " + err);
  }
  ws.bytes = device_bytes - before;
}

void Engine::reserve_for(const fnmt_run& run) {
  const int tok = std::max(run.wbatch, arch.max_positions);
  const int rows = std::max(run.sbatch, 1) * std::max(run.beam_size, 1);
  const int64_t pool = std::max<int64_t>(
      (int64_t)std::ceil(run.max_len_ratio * (double)run.wbatch) +
          (int64_t)(run.max_len_offset + 1) * run.sbatch,
      arch.max_positions) * std::max(run.beam_size, 1);
  reserve(tok, rows, pool);
}

// ---------------------------------------------------------------------------
// building blocks

void Engine::gemm(const void* A, const CUtensorMap* tmA, int lda, const Lin& L, int M, void* C,
                  int ldc, int c_dtype, int relu, cudaStream_t s, const float* resid) {
  GemmArgs g;
  g.A = A;
  g.lda = lda;
  g.W = L.w;
  g.ldw = L.K;
  g.in_dtype = dt;
  g.bias = L.b;
  g.M = M;
  g.N = L.N;
  g.K = L.K;
  g.C = C;
  g.ldc = ldc;
  g.c_dtype = c_dtype;
  g.relu = relu;
  g.resid = resid;
  g.ld_resid = ldc;
  g.tmap_a = tmA;
  g.tmap_w = dt == kF32 ? nullptr : &L.tm;
  if (step_m_tab && !q8) {
    g.m_tab = step_m_tab;
    g.t_ptr = step_t_ptr;
  }
  attach_q(g, L);
  const int ev = prof_begin(s);
  CK(launch_gemm(g, s));
  const double Mc = prof_m >= 0 ? prof_m : (double)M;
  prof_end(s, ev, gemm_cls, 2.0 * Mc * L.N * L.K,
           Mc * L.K * dtype_size(dt) + (double)L.N * L.K * dtype_size(dt) +
               Mc * L.N * (dtype_size(c_dtype) + (resid ? 4.0 : 0.0)));
  ++launches;
}

void Engine::gemm_argmax(const void* A, const CUtensorMap* tmA, int lda, int M,
                         unsigned long long* keys, cudaStream_t s) {
  GemmArgs g;
  g.A = A;
  g.lda = lda;
  g.W = out.w;
  g.ldw = out.K;
  g.in_dtype = dt;
  g.bias = out.b;
  g.M = M;
  g.N = out.N;
  g.K = out.K;
  g.epi = kEpiArgmax;
  g.keys = keys;
  g.tmap_a = tmA;
  g.tmap_w = dt == kF32 ? nullptr : &out.tm;
  if (step_m_tab && !q8) {
    g.m_tab = step_m_tab;
    g.t_ptr = step_t_ptr;
  }
  attach_q(g, out);
  const int ev = prof_begin(s);
  CK(launch_gemm(g, s));
  const double Mc = prof_m >= 0 ? prof_m : (double)M;
  prof_end(s, ev, FNMT_K_VOCAB, 2.0 * Mc * out.N * out.K,
           Mc * out.K * dtype_size(dt) + (double)out.N * out.K * dtype_size(dt));
  ++launches;
}

void Engine::norm(const float* x, const float* y, const Norm& n, float* o32, void* oa, int rows,
                  cudaStream_t s) {
  const int ev = prof_begin(s);
  CK(launch_add_norm(x, y, n.g, n.b, arch.norm_l1, o32, dt == kF32 ? nullptr : oa,
                     dt, rows, arch.d_model, s, step_m_tab, step_t_ptr));
  prof_end(s, ev, FNMT_K_NORM, 0.0,
           (prof_m >= 0 ? prof_m : (double)rows) * arch.d_model *
               ((y ? 8.0 : 4.0) + (o32 ? 4.0 : 0.0) + (dt == kF32 ? 0 : dtype_size(dt))));
  ++launches;
}

// x32 = norm(x32 + A.W + b): GEMM into y32 (fp32), then add_norm.  (r01: the residual
// add in the GEMM epilogue measured slower, 6.30M vs 6.78M words/s, and a clustered
// GEMM + LayerNorm epilogue exchanging row statistics over DSMEM 4.23M vs 6.81M: the
// row-local epilogue serialises behind the 1-deep TMEM double buffer.)
void Engine::gemm_norm(const void* A, const CUtensorMap* tmA, int lda, const Lin& L, int M,
                       float* x32, void* xa, float* y32, const Norm& n, cudaStream_t s,
                       bool keep32) {
  gemm(A, tmA, lda, L, M, y32, L.N, kF32, 0, s);
  norm(x32, y32, n, keep32 ? x32 : nullptr, xa, M, s);
}

// Encoder over rows already embedded in ws.x32 / ws.xa (model.py:279-286).
void Engine::encoder_layers(int n_tok, int n_seq, int max_q, int max_k, const int32_t* qstart,
                            const int32_t* qlen, const int32_t* kstart, const int32_t* klen,
                            int k_pad, cudaStream_t s) {
  const int d = arch.d_model;
  const bool tc = dt != kF32;
  gemm_cls = FNMT_K_GEMM_ENC;
  for (const EncL& L : enc) {
    gemm(ws.xa, tc ? &ws.tm_xa : nullptr, d, L.qkv, n_tok, ws.qkv, 3 * d, dt, 0, s);
    AttnArgs a{};
    a.q = ws.qkv;
    a.ldq = 3 * d;
    a.k = (const char*)ws.qkv + (size_t)d * dtype_size(dt);
    a.v = (const char*)ws.qkv + (size_t)2 * d * dtype_size(dt);
    a.ldkv = 3 * d;
    a.out = ws.att;
    a.ldo = d;
    a.dtype = dt;
    a.heads = arch.n_heads_enc;
    a.dk = d / arch.n_heads_enc;
    a.q_start = qstart;
    a.q_len = qlen;
    a.k_start = kstart;
    a.k_len = klen;
    a.k_pad = k_pad;
    a.n_seq = n_seq;
    a.max_q = max_q;
    a.max_k = std::max(max_k, k_pad);
    {
      const int ev = prof_begin(s);
      CK(launch_attention_varlen(a, s));
      prof_end(s, ev, FNMT_K_ATTN_ENC, 0.0, (double)n_tok * 4 * d * dtype_size(dt));
    }
    ++launches;
    gemm_norm(ws.att, tc ? &ws.tm_att : nullptr, d, L.o, n_tok, ws.x32, ws.xa, ws.y32, L.n1, s);
    gemm(ws.xa, tc ? &ws.tm_xa : nullptr, d, L.f1, n_tok, ws.h, arch.ffn_dim_enc, dt, 1, s);
    gemm_norm(ws.h, tc ? &ws.tm_h : nullptr, arch.ffn_dim_enc, L.f2, n_tok, ws.x32, ws.xa, ws.y32,
              L.n2, s);
  }
}

void Engine::cross_kv_all(int n_tok, cudaStream_t s) {
  const int d = arch.d_model;
  gemm_cls = FNMT_K_GEMM_ENC;
  for (int l = 0; l < arch.n_dec_layers; ++l)
    gemm(ws.xa, dt != kF32 ? &ws.tm_xa : nullptr, d, fused_cross ? dec[l].fck : dec[l].ckv, n_tok,
         ws.ckv[l], ckv_ld, dt, 0, s);
}

// Layer-0 step tables in use for this step view: the greedy workspace path of
// a folded single-head decoder whose fused layer kernel runs (the key row goes
// through the dqkv staging buffer); knew null otherwise.
StepKey Engine::step_keys_of(const StepView& v) const {
  StepKey k{};
  if (dec.empty() || !dec[0].tok_tab || !v.ws_caches || v.anc) return k;
  k.tok_tab = dec[0].tok_tab;
  k.pos_tab = dec[0].pos_tab;
  if (fused_self) {
    if (!fused_cross || !dec_layer_fused_ok(dt, arch.d_model, arch.n_heads_dec)) return StepKey{};
    k.knew = ws.dqkv;
    k.w = 2 * arch.d_model + 8;
    return k;
  }
  // multi-head: q -> dq, k / v -> this step's self-cache slots (the QKV GEMM's epilogue)
  k.knew = ws.dq;
  k.w = 3 * arch.d_model;
  k.seg = arch.d_model;
  k.kc = v.kc[0];
  k.vc = v.vc[0];
  k.cap = v.cap;
  return k;
}

// One decoder step for v.rows rows (model.py:308-344).  All sizes that vary
// per step live in device memory (step counter), so the launch sequence is
// graph-capturable and replayable.
void Engine::run_step(const StepView& v, cudaStream_t s) {
  const int d = arch.d_model, es = dtype_size(dt);
  const bool tc = dt != kF32;
  const int R = v.rows;
  gemm_cls = FNMT_K_GEMM_DEC;
  // profiler counts: live rows only, unpadded source keys
  const double Rl = (profiling && v.prof_live) ? (double)(*v.prof_live)[v.host_t] : (double)R;
  const double Sl = (profiling && v.prof_src) ? (*v.prof_src)[v.host_t] : (double)R * v.max_k;
  prof_m = profiling ? Rl : -1.0;
  step_m_tab = v.m_tab;
  step_t_ptr = v.t_ptr;
  if (!v.embed_done) {
    const int ev = prof_begin(s);
    CK(launch_embed(v.prev, nullptr, v.t_ptr, tgt_emb32, pos32, emb_scale(), ws.dx32,
                    tc ? ws.dxa : nullptr, dt, R, d, s));
    prof_end(s, ev, FNMT_K_EMBED, 0.0, Rl * d * (8.0 + dtype_size(dt)));
    ++launches;
    const StepKey k = step_keys_of(v);
    if (k.knew) {
      const int ev2 = prof_begin(s);
      CK(launch_step_key(k, v.prev, v.t_ptr, R, dt, s));
      prof_end(s, ev2, FNMT_K_EMBED, 0.0, Rl * k.w * (8.0 + es));
      ++launches;
    }
  }
  for (int l = 0; l < arch.n_dec_layers; ++l) {
    const DecL& L = dec[l];
    bool layer_fused = false;
    if (fused_self && v.ws_caches && !v.anc) {
      // folded self attention: this step's [K~ | V~ | c] row straight into cache
      // slot t; the query is the layer input itself and the attention writes the
      // o-projected output (+ bo, fp32) into the residual branch
      const int fl = 2 * d + 8;
      GemmArgs g;
      g.A = ws.dxa;
      g.lda = d;
      g.W = L.fsk.w;
      g.ldw = L.fsk.K;
      g.in_dtype = dt;
      g.bias = L.fsk.b;
      g.M = R;
      g.N = fl;
      g.K = d;
      // with the fused layer kernel the GEMM writes contiguous rows into the
      // staging buffer (dqkv, [rows, 3d] >= [rows, 2d + 8]) and the layer
      // kernel appends them to the cache slots (the per-row slot scatter from
      // the GEMM epilogue measured 23 vs 8 us per step at 3072 rows)
      const bool layer_ok = fused_cross && dec_layer_fused_ok(dt, d, arch.n_heads_dec);
      const bool tabled = layer_ok && l == 0 && step_keys_of(v).knew;   // no GEMM: step tables
      const bool staged = layer_ok && !tabled && knew_staging_enabled();
      g.epi = staged ? kEpiStore : kEpiSlot;
      g.C = staged ? ws.dqkv : v.kc[l];
      g.ldc = fl;
      g.c_dtype = dt;
      g.cap = v.cap;
      g.t_ptr = v.t_ptr;
      g.tmap_a = &ws.tm_dxa;
      g.tmap_w = &L.fsk.tm;
      if (!tabled) {
        const int ev = prof_begin(s);
        CK(launch_gemm(g, s));
        prof_end(s, ev, gemm_cls, 2.0 * Rl * fl * d, Rl * d * es + (double)fl * d * es + Rl * fl * es);
        ++launches;
      }
      if (layer_ok) {
        // one kernel: self attention, + residual, norm1, cross attention, + residual, norm2
        DecLayerArgs f{};
        f.q = ws.dxa;
        f.ldq = d;
        f.x32 = ws.dx32;
        f.xa = ws.dxa;
        f.kself = v.kc[l];
        f.ld_self = fl;
        f.cap = v.cap;
        f.t_ptr = v.t_ptr;
        f.kcross = v.ckv[l];
        f.ld_cross = ckv_ld;
        f.k_start = v.k_start;
        f.k_len = v.k_len;
        f.k_pad = v.k_pad;
        f.rows_per_seq = v.rows_per_seq;
        f.voff = d;
        f.kc_off = 2 * d;
        f.bo_self = L.so.b;
        f.g1 = L.n1.g;
        f.b1 = L.n1.b;
        f.bo_cross = L.co.b;
        f.g2 = L.n2.g;
        f.b2 = L.n2.b;
        f.l1 = arch.norm_l1;
        f.dtype = dt;
        f.d = d;
        f.rows = R;
        f.row_done = v.row_done;
        // tables: the previous kernel (greedy_embed / step_key) wrote key t into dqkv
        f.knew = (staged || tabled) ? ws.dqkv : nullptr;
        const int ev2 = prof_begin(s);
        CK(launch_dec_layer_fused(f, s));
        // SURVEY §8(d) attention bytes (self t+1 keys + cross S keys, 2 d each,
        // live rows) plus the row's residual in / out and query reads
        prof_end(s, ev2, FNMT_K_ATTN_DEC, 0.0,
                 (Rl * (v.host_t + 1) + Sl) * 2 * d * es + Rl * d * (8.0 + 2 * es));
        ++launches;
        layer_fused = true;
      } else {
      DecAttnArgs a{};
      a.q = ws.dxa;
      a.ldq = d;
      a.k = v.kc[l];
      a.v = (const char*)v.kc[l] + (size_t)d * es;
      a.ldkv = fl;
      a.kc_off = 2 * d;
      a.out = ws.dy32;
      a.ldo = d;
      a.out_f32 = 1;
      a.out_bias = L.so.b;
      a.dtype = dt;
      a.heads = 1;
      a.dk = d;
      a.rows = R;
      a.self_mode = 1;
      a.cap = v.cap;
      a.t_ptr = v.t_ptr;
      a.max_k = v.cap;
      a.row_done = v.row_done;
      {
        const int ev2 = prof_begin(s);
        CK(launch_attention_decode(a, s));
        prof_end(s, ev2, FNMT_K_ATTN_DEC, 0.0, Rl * (v.host_t + 1) * 2 * d * es);
      }
      ++launches;
      norm(ws.dx32, ws.dy32, L.n1, ws.dx32, ws.dxa, R, s);
      }
    } else {
    if (!(l == 0 && step_keys_of(v).kc)) {   // else: written by greedy_embed / step_key
      // q -> ws.dq, this step's k / v straight into the self cache slot t (fused append)
      GemmArgs g;
      g.A = ws.dxa;
      g.lda = d;
      g.W = L.sqkv.w;
      g.ldw = L.sqkv.K;
      g.in_dtype = dt;
      g.bias = L.sqkv.b;
      g.M = R;
      g.N = L.sqkv.N;
      g.K = L.sqkv.K;
      g.epi = kEpiQKV;
      g.C = ws.dq;
      g.ldc = d;
      g.c_dtype = dt;
      g.kc = v.kc[l];
      g.vc = v.vc[l];
      g.cap = v.cap;
      g.seg = d;
      g.t_ptr = v.t_ptr;
      g.tmap_a = tc ? &ws.tm_dxa : nullptr;
      g.tmap_w = tc ? &L.sqkv.tm : nullptr;
      attach_q(g, L.sqkv);
      const int ev = prof_begin(s);
      CK(launch_gemm(g, s));
      prof_end(s, ev, gemm_cls, 2.0 * Rl * L.sqkv.N * L.sqkv.K,
               Rl * d * es + (double)L.sqkv.N * L.sqkv.K * es + 3.0 * Rl * d * es);
      ++launches;
    }
    DecAttnArgs a{};
    a.q = ws.dq;
    a.ldq = d;
    a.k = v.kc[l];
    a.v = v.vc[l];
    a.ldkv = d;
    a.k_w = nullptr;   // appended by the QKV epilogue
    a.v_w = nullptr;
    a.new_k = nullptr;
    a.new_v = nullptr;
    a.ld_new = 0;
    a.out = ws.datt;
    a.ldo = d;
    a.dtype = dt;
    a.heads = arch.n_heads_dec;
    a.dk = d / arch.n_heads_dec;
    a.rows = R;
    a.self_mode = 1;
    a.cap = v.cap;
    a.t_ptr = v.t_ptr;
    a.anc = v.anc;
    a.anc_buf_stride = v.anc_stride;
    a.max_k = v.cap;
    a.row_done = v.row_done;
    {
      const int ev = prof_begin(s);
      CK(launch_attention_decode(a, s));
      prof_end(s, ev, FNMT_K_ATTN_DEC, 0.0, Rl * (v.host_t + 1) * 2 * d * es);
    }
    ++launches;
    gemm_norm(ws.datt, tc ? &ws.tm_datt : nullptr, d, L.so, R, ws.dx32, ws.dxa, ws.dy32, L.n1, s);
    }
    if (!layer_fused) {
    // folded cross attention (workspace caches only): q is the norm1 output itself,
    // the attention writes the o-projection output (fp32, + bias) straight into dy32
    const bool folded = fused_cross && v.ws_caches;
    if (!folded) gemm(ws.dxa, tc ? &ws.tm_dxa : nullptr, d, L.cq, R, ws.dq, d, dt, 0, s);
    DecAttnArgs c{};
    c.q = folded ? ws.dxa : ws.dq;
    c.ldq = d;
    c.k = v.ckv[l];
    c.v = (const char*)v.ckv[l] + (size_t)d * es;
    c.ldkv = v.ws_caches ? ckv_ld : 2 * d;
    c.out = folded ? (void*)ws.dy32 : ws.datt;
    c.ldo = d;
    if (folded) {
      c.kc_off = 2 * d;
      c.out_f32 = 1;
      c.out_bias = L.co.b;
    }
    c.dtype = dt;
    c.heads = arch.n_heads_dec;
    c.dk = d / arch.n_heads_dec;
    c.rows = R;
    c.self_mode = 0;
    c.k_start = v.k_start;
    c.k_len = v.k_len;
    c.k_pad = v.k_pad;
    c.rows_per_seq = v.rows_per_seq;
    c.max_k = v.max_k;
    c.row_done = v.row_done;
    {
      const int ev = prof_begin(s);
      CK(launch_attention_decode(c, s));
      prof_end(s, ev, FNMT_K_ATTN_DEC, 0.0, Sl * 2 * d * es);
    }
    ++launches;
    if (folded)
      norm(ws.dx32, ws.dy32, L.n2, ws.dx32, ws.dxa, R, s);
    else
      gemm_norm(ws.datt, tc ? &ws.tm_datt : nullptr, d, L.co, R, ws.dx32, ws.dxa, ws.dy32, L.n2, s);
    }
    if (L.ffn) {
      gemm(ws.dxa, tc ? &ws.tm_dxa : nullptr, d, L.f1, R, ws.dh, arch.ffn_dim_dec, dt, 1, s);
      // the last layer's fp32 residual stream has no reader (the vocabulary
      // projection takes the activation copy; the next step re-embeds)
      gemm_norm(ws.dh, tc ? &ws.tm_dh : nullptr, arch.ffn_dim_dec, L.f2, R, ws.dx32, ws.dxa,
                ws.dy32, L.n3, s, dt == kF32 || l + 1 < arch.n_dec_layers);
    }
  }
  if (v.topk && tc) {
    // beam: vocab projection fused with per-tile max / sum-exp / top-K
    GemmArgs g;
    g.A = ws.dxa;
    g.lda = d;
    g.W = out.w;
    g.ldw = out.K;
    g.in_dtype = dt;
    g.bias = out.b;
    g.M = R;
    g.N = out.N;
    g.K = out.K;
    g.epi = kEpiTopK;
    g.topk = *v.topk;
    g.tmap_a = &ws.tm_dxa;
    g.tmap_w = &out.tm;
    const int ev = prof_begin(s);
    CK(launch_gemm(g, s));
    prof_end(s, ev, FNMT_K_VOCAB, 2.0 * Rl * out.N * out.K,
             Rl * out.K * dtype_size(dt) + (double)out.N * out.K * dtype_size(dt));
    ++launches;
  } else if (v.logits) {
    gemm_cls = FNMT_K_VOCAB;
    gemm(ws.dxa, tc ? &ws.tm_dxa : nullptr, d, out, R, v.logits, arch.vocab_size, kF32, 0, s);
    if (v.topk) {
      CK(launch_logits_topk_partials(v.logits, R, arch.vocab_size, *v.topk, s));
      ++launches;
    }
  } else {
    gemm_argmax(ws.dxa, tc ? &ws.tm_dxa : nullptr, d, R, v.keys, s);
  }
  prof_m = -1.0;
  step_m_tab = nullptr;
  step_t_ptr = nullptr;
}

float Engine::emb_scale() const { return (float)std::sqrt((double)arch.d_model); }

// ---------------------------------------------------------------------------
// corpus translation

void Engine::translate_device(const int32_t* d_ids, const int64_t* d_off,
                              const std::vector<int32_t>& lengths, const fnmt_run& run,
                              int32_t* d_out_ids, const int64_t* d_out_off, int32_t* d_out_len,
                              fnmt_stats* st) {
  if (!finalized) throw EngineError(FNMT_E_STATE, "engine not finalized");
  if (run.beam_size < 1 || run.beam_size > kTopKMax)
    throw EngineError(FNMT_E_INVALID, "beam_size must be in [1, 8]");
  if (run.sbatch < 1 || run.wbatch < 1) throw EngineError(FNMT_E_INVALID, "sbatch/wbatch must be >= 1");
  const int kb = run.beam_size;
  CK(cudaSetDevice(device));
  const int n = (int)lengths.size();
  for (int32_t L : lengths) {
    if (L < 0) throw EngineError(FNMT_E_INVALID, "negative sentence length");
    if (L > arch.max_positions)
      throw EngineError(FNMT_E_LENGTH, "source length " + std::to_string(L) +
                                           " exceeds max_positions " +
                                           std::to_string(arch.max_positions));
  }
  {
    int64_t total = 0;
    for (int32_t L : lengths) total += L;
    if (total > 0) {
      if (!d_bad) d_bad = (int32_t*)dalloc(sizeof(int32_t));
      CK(cudaMemsetAsync(d_bad, 0, sizeof(int32_t), stream));
      const int blocks = (int)std::min<int64_t>((total + 255) / 256, 148 * 8);
      check_ids_kernel<<<blocks, 256, 0, stream>>>(d_ids, d_off, total, arch.vocab_size, d_bad);
      CK(cudaGetLastError());
      CK(cudaMemcpyAsync(h_alive + 2, d_bad, sizeof(int32_t), cudaMemcpyDeviceToHost, stream));
      CK(cudaStreamSynchronize(stream));
      if (h_alive[2]) throw EngineError(FNMT_E_INVALID, "token id out of range");
    }
  }
  const int64_t launches0 = launches;
  CK(cudaEventRecord(ev_t0, stream));
  // Empty sentences produce empty output without touching the GPU pipeline
  // (the reference's Translator maps empty lines to empty lines).
  std::vector<int32_t> live_len;
  std::vector<int32_t> live_idx;
  live_len.reserve(n);
  live_idx.reserve(n);
  for (int i = 0; i < n; ++i)
    if (lengths[i] > 0) {
      live_len.push_back(lengths[i]);
      live_idx.push_back(i);
    }
  std::vector<Batch> plan = plan_batches(live_len, run.sbatch, run.wbatch);
  // Host metadata for the whole plan: permutation (original sentence index
  // per batch row), per-batch cu / budgets; uploaded once.
  std::vector<int32_t> perm, cu_all, budget_all;
  std::vector<int64_t> batch_row0, batch_cu0;
  perm.reserve(live_idx.size());
  for (const Batch& b : plan) {
    batch_row0.push_back((int64_t)perm.size());
    batch_cu0.push_back((int64_t)cu_all.size());
    int32_t acc = 0;
    for (int32_t li : b.rows) {
      perm.push_back(live_idx[li]);
      cu_all.push_back(acc);
      acc += live_len[li];
      budget_all.push_back(budget_of(live_len[li], run.max_len_ratio, run.max_len_offset,
                                     arch.max_positions));
    }
    cu_all.push_back(acc);
  }
  // size the workspace for the largest batch of this plan (grows, never shrinks)
  {
    int tok_need = 1, rows_need = 1;
    int64_t pool_need = 1;
    for (size_t bi = 0; bi < plan.size(); ++bi) {
      const int R = (int)plan[bi].rows.size();
      const int n_tok = cu_all[batch_cu0[bi] + R];
      int cap = 0;
      for (int r = 0; r < R; ++r) cap = std::max(cap, budget_all[batch_row0[bi] + r]);
      tok_need = std::max(tok_need, n_tok);
      rows_need = std::max(rows_need, R);
      pool_need = std::max<int64_t>(pool_need, (int64_t)R * cap);
    }
    reserve(tok_need, rows_need * kb, pool_need * kb);
    if (kb > 1) reserve_beam(rows_need, kb, pool_need * kb);
  }
  ensure_meta(perm.size(), cu_all.size());
  if (!perm.empty()) {
    CK(cudaMemcpyAsync(meta_perm, perm.data(), perm.size() * 4, cudaMemcpyHostToDevice, stream));
    CK(cudaMemcpyAsync(meta_cu, cu_all.data(), cu_all.size() * 4, cudaMemcpyHostToDevice, stream));
    CK(cudaMemcpyAsync(meta_budget, budget_all.data(), budget_all.size() * 4,
                       cudaMemcpyHostToDevice, stream));
  }
  // zero lengths for empty sentences
  for (int i = 0; i < n; ++i)
    if (lengths[i] == 0) {
      // tiny synchronous-order write via the stream
      CK(cudaMemsetAsync(d_out_len + i, 0, sizeof(int32_t), stream));
    }
  PlanCtx P{plan, live_len, budget_all, batch_row0, batch_cu0, meta_perm, meta_cu, meta_budget,
            d_ids, d_off, d_out_ids, d_out_off, d_out_len, run};
  int64_t steps_total = 0;
  // Lanes: extra engines sharing these weights, each with its own workspace,
  // stream and decode graph.  Batches are dealt longest-first to this engine
  // and shortest-first to the others, so a latency-bound long-sentence decode
  // (few rows, many steps) overlaps with short-sentence batches.
  const int want_lanes = profiling ? 1 : std::min<int>(n_lanes, (int)plan.size());
  if (want_lanes <= 1) {
    for (size_t bi = 0; bi < plan.size(); ++bi) steps_total += run_batch(P, bi);
  } else {
    while ((int)lanes.size() < want_lanes - 1) lanes.push_back(make_lane());
    std::vector<Engine*> eng{this};
    for (int i = 0; i < want_lanes - 1; ++i) {
      Engine* L = lanes[i].get();
      L->reserve(ws.tok_cap, ws.row_cap, ws.pool_cap);
      if (kb > 1) L->reserve_beam(beam.sent_cap, beam.k, beam.pool_cap);
      eng.push_back(L);
    }
    cudaEvent_t ready;
    CK(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming));
    CK(cudaEventRecord(ready, stream));
    for (size_t i = 1; i < eng.size(); ++i) CK(cudaStreamWaitEvent(eng[i]->stream, ready, 0));
    std::mutex mu;
    int front = 0, back = (int)plan.size() - 1;
    std::vector<int64_t> steps(eng.size(), 0), l0(eng.size());
    std::vector<std::exception_ptr> errs(eng.size());
    for (size_t i = 0; i < eng.size(); ++i) l0[i] = eng[i]->launches;
    std::vector<std::thread> th;
    for (size_t i = 0; i < eng.size(); ++i) {
      th.emplace_back([&, i] {
        try {
          CK(cudaSetDevice(device));
          for (;;) {
            int bi;
            {
              std::lock_guard<std::mutex> g(mu);
              if (front > back) break;
              bi = i == 0 ? front++ : back--;
            }
            steps[i] += eng[i]->run_batch(P, (size_t)bi);
          }
        } catch (...) {
          errs[i] = std::current_exception();
        }
      });
    }
    for (auto& t : th) t.join();
    for (size_t i = 1; i < eng.size(); ++i) {
      CK(cudaEventRecord(eng[i]->ev_done, eng[i]->stream));
      CK(cudaStreamWaitEvent(stream, eng[i]->ev_done, 0));
      launches += eng[i]->launches - l0[i];
    }
    cudaEventDestroy(ready);
    for (auto& e : errs)
      if (e) std::rethrow_exception(e);
    for (int64_t s : steps) steps_total += s;
  }
  CK(cudaEventRecord(ev_t1, stream));
  CK(cudaStreamSynchronize(stream));
  if (profiling) prof_collect();
  if (st) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, ev_t0, ev_t1);
    st->sentences += n;
    int64_t src = 0;
    for (int32_t L : lengths) src += L;
    st->source_tokens += src;
    st->batches += (int64_t)plan.size();
    st->decode_steps += steps_total;
    st->gpu_launches += launches - launches0;
    st->total_ms += ms;
    st->device_bytes = device_bytes;
    for (auto& L : lanes) st->device_bytes += L->device_bytes;
  }
}

std::unique_ptr<Engine> Engine::make_lane() {
  std::unique_ptr<Engine> L(new Engine(arch, device, q8 ? 3 : dt));
  L->src_emb32 = src_emb32;
  L->tgt_emb32 = tgt_emb32;
  L->pos32 = pos32;
  L->out = out;
  L->enc = enc;
  L->dec = dec;
  L->finalized = true;   // weights are shared (owned by this engine)
  L->fused_cross = fused_cross;
  L->fused_self = fused_self;
  L->ckv_ld = ckv_ld;
  L->n_lanes = 1;
  return L;
}

// One planned batch on this engine's workspace / stream: gather -> encode ->
// decode (greedy or beam) -> scatter to the sentence slots.
int64_t Engine::run_batch(const PlanCtx& P, size_t bi) {
  const Batch& b = P.plan[bi];
  const fnmt_run& run = P.run;
  const int32_t* d_ids = P.d_ids;
  const int64_t* d_off = P.d_off;
  int32_t* d_out_ids = P.d_out_ids;
  const int64_t* d_out_off = P.d_out_off;
  int32_t* d_out_len = P.d_out_len;
  int64_t steps_total = 0;
  {
    const int R = (int)b.rows.size();
    const int32_t* perm_b = P.meta_perm + P.batch_row0[bi];
    const int32_t* cu_b = P.meta_cu + P.batch_cu0[bi];
    int n_tok = 0, cap = 0;
    for (int r = 0; r < R; ++r) {
      n_tok += P.live_len[b.rows[r]];
      cap = std::max(cap, P.budget_all[P.batch_row0[bi] + r]);
    }
    // 1) gather this batch's source ids into the packed workspace
    int ev = prof_begin(stream);
    gather_batch_kernel<<<R, 128, 0, stream>>>(d_ids, d_off, perm_b, cu_b, R, ws.ids, ws.pos);
    CK(cudaGetLastError());
    prof_end(stream, ev, FNMT_K_OTHER, 0.0, (double)n_tok * 12);
    ++launches;
    // per-sequence tables: q/k start = cu, len = cu diff
    CK(cudaMemcpyAsync(ws.cu, cu_b, sizeof(int32_t) * (R + 1), cudaMemcpyDeviceToDevice, stream));
    CK(cudaMemcpyAsync(ws.budget, P.meta_budget + P.batch_row0[bi], sizeof(int32_t) * R,
                       cudaMemcpyDeviceToDevice, stream));
    lens_from_cu(R);
    // 2) encoder (packed varlen: only real tokens are rows)
    ev = prof_begin(stream);
    CK(launch_embed(ws.ids, ws.pos, nullptr, src_emb32, pos32, emb_scale(), ws.x32,
                    dt != kF32 ? ws.xa : nullptr, dt, n_tok, arch.d_model, stream));
    prof_end(stream, ev, FNMT_K_EMBED, 0.0, (double)n_tok * arch.d_model * (12.0 + dtype_size(dt)));
    ++launches;
    encoder_layers(n_tok, R, b.max_len, b.max_len, ws.cu, ws.len, ws.cu, ws.len, 0, stream);
    cross_kv_all(n_tok, stream);
    // 3) decode: one CUDA graph per step (greedy, or batched beam)
    const int32_t* res_ids = ws.out_ids;
    const int32_t* res_len = ws.out_len;
    if (run.beam_size <= 1) {
      std::vector<int32_t> src(R), bud(R);
      for (int r = 0; r < R; ++r) {
        src[r] = P.live_len[b.rows[r]];
        bud[r] = P.budget_all[P.batch_row0[bi] + r];
      }
      steps_total += decode_greedy(R, cap, b.max_len, run, src, bud);
    } else {
      std::vector<int32_t> bud(R);
      for (int r = 0; r < R; ++r) bud[r] = P.budget_all[P.batch_row0[bi] + r];
      steps_total += decode_beam(R, cap, b.max_len, run, bud);
      res_ids = beam.out_ids;
      res_len = beam.out_len;
    }
    // 4) restore order: scatter rows to their sentence slots
    ev = prof_begin(stream);
    scatter_out_kernel<<<R, 64, 0, stream>>>(res_ids, res_len, cap, perm_b, R, d_out_off,
                                            d_out_ids, d_out_len);
    CK(cudaGetLastError());
    prof_end(stream, ev, FNMT_K_OTHER, 0.0, (double)R * cap * 8);
    ++launches;
  }
  return steps_total;
}

// Replay the captured step (or, when profiling, launch `direct(t)`) for up to
// `cap` steps; every 8 steps the device `alive` count is copied back and the
// loop stops once it reads zero (checked two chunks behind, so the host
// never waits on the chunk it just queued).
int Engine::drive_steps(int cap, int64_t nodes, const std::function<void(int)>& direct) {
  const int chunk = 8;
  int steps = 0, inflight = 0;
  bool stop = false;
  for (int c0 = 0; c0 < cap && !stop; c0 += chunk) {
    const int c1 = std::min(cap, c0 + chunk);
    if (profiling) {
      for (int t = c0; t < c1; ++t) direct(t);
    } else {
      for (int t = c0; t < c1; ++t) CK(cudaGraphLaunch(graph_exec, stream));
      launches += nodes * (c1 - c0);
    }
    steps += c1 - c0;
    const int slot = (c0 / chunk) & 1;
    if (inflight == 2) {
      CK(cudaEventSynchronize(ev_poll[slot]));
      if (h_alive[slot] == 0) stop = true;
      --inflight;
    }
    CK(cudaMemcpyAsync(h_alive + slot, ws.alive, sizeof(int32_t), cudaMemcpyDeviceToHost, stream));
    CK(cudaEventRecord(ev_poll[slot], stream));
    ++inflight;
  }
  return steps;
}

StepView Engine::step_view(int rows, int cap, int max_len, int rows_per_seq) {
  StepView v;
  v.rows = rows;
  v.cap = cap;
  v.prev = ws.prev;
  v.t_ptr = ws.t;
  v.kc = ws.kc.data();
  v.vc = ws.vc.data();
  v.ckv = (const void* const*)ws.ckv.data();
  v.k_start = ws.cu;
  v.k_len = ws.len;
  v.k_pad = 0;
  v.rows_per_seq = rows_per_seq;
  v.max_k = max_len;
  v.ws_caches = true;
  return v;
}

// Rows inside their budget at each step t of a batch, uploaded for the
// decode-step GEMMs / norm (GemmArgs::m_tab).  The batch's sentences come
// length-descending (plan_batches), so budgets are non-increasing and the live
// rows at step t are the prefix [0, mult * #{budget > t}) (mult = beam rows
// per sentence).  Null when the order does not hold or the bound is off.
const int32_t* Engine::live_table(const std::vector<int32_t>& budgets, int cap, int mult) {
  if (dt == kF32 || q8 || !live_rows_enabled() || cap <= 0 || budgets.empty() ||
      !std::is_sorted(budgets.rbegin(), budgets.rend()))
    return nullptr;
  const size_t n_tab = (size_t)arch.max_positions + 2;
  if (!d_live_tab) {
    d_live_tab = (int32_t*)dalloc(sizeof(int32_t) * n_tab);
    CK(cudaMallocHost(&h_live_tab, sizeof(int32_t) * n_tab));
    CK(cudaEventCreateWithFlags(&ev_live, cudaEventDisableTiming | cudaEventBlockingSync));
  } else {
    CK(cudaEventSynchronize(ev_live));   // the previous batch's copy has read the buffer
  }
  for (int t = 0, r = (int)budgets.size(); t <= cap; ++t) {
    while (r > 0 && budgets[r - 1] <= t) --r;
    h_live_tab[t] = r * mult;
  }
  CK(cudaMemcpyAsync(d_live_tab, h_live_tab, sizeof(int32_t) * (cap + 1), cudaMemcpyHostToDevice,
                     stream));
  CK(cudaEventRecord(ev_live, stream));
  return d_live_tab;
}

int Engine::decode_greedy(int R, int cap, int max_len, const fnmt_run& run,
                          const std::vector<int32_t>& src_len, const std::vector<int32_t>& budgets) {
  init_decode_kernel<<<(R + 255) / 256, 256, 0, stream>>>(ws.prev, ws.finished, ws.out_len,
                                                         ws.keys, ws.t, ws.alive, R, run.bos_id);
  CK(cudaGetLastError());
  ++launches;
  StepView v = step_view(R, cap, max_len, 1);
  v.keys = ws.keys;
  v.row_done = ws.finished;
  // rows inside their budget at step t (decode-step GEMMs / norm stop there)
  v.m_tab = live_table(budgets, cap, 1);
  // profiler: rows still inside their budget at step t (random weights never
  // emit EOS; an EOS-finished row would still be counted, an upper bound)
  std::vector<int> live;
  std::vector<double> live_src;
  if (profiling) {
    live.assign(cap, 0);
    live_src.assign(cap, 0.0);
    for (int r = 0; r < R; ++r)
      for (int t = 0; t < std::min(cap, budgets[r]); ++t) {
        live[t] += 1;
        live_src[t] += src_len[r];
      }
    v.prof_live = &live;
    v.prof_src = &live_src;
  }
  GreedyState gs;
  gs.keys = ws.keys;
  gs.prev = ws.prev;
  gs.finished = ws.finished;
  gs.budget = ws.budget;
  gs.out_ids = ws.out_ids;
  gs.out_len = ws.out_len;
  gs.t = ws.t;
  gs.alive = ws.alive;
  gs.rows = R;
  gs.out_cap = cap;
  gs.eos = run.eos_id;
  gs.pad = run.pad_id;
  // greedy update fused with the next step's embedding (the step graph then
  // starts at the first decoder GEMM); the first input is embedded here
  const bool fuse_embed = greedy_embed_enabled();
  GreedyEmbed ge{};
  if (fuse_embed) {
    ge.table = tgt_emb32;
    ge.pos = pos32;
    ge.scale = emb_scale();
    ge.x32 = ws.dx32;
    ge.xa = dt == kF32 ? nullptr : ws.dxa;
    ge.act_dtype = dt;
    ge.d = arch.d_model;
    ge.n_pos = arch.max_positions;
    ge.done = ws.t + 2;
    ge.alive_acc = ws.t + 3;
    const int ev = prof_begin(stream);
    CK(launch_embed(ws.prev, nullptr, ws.t, tgt_emb32, pos32, emb_scale(), ws.dx32,
                    dt == kF32 ? nullptr : ws.dxa, dt, R, arch.d_model, stream));
    prof_end(stream, ev, FNMT_K_EMBED, 0.0, (double)R * arch.d_model * (8.0 + dtype_size(dt)));
    ++launches;
    ge.key = step_keys_of(v);
    if (ge.key.knew) {
      const int ev2 = prof_begin(stream);
      CK(launch_step_key(ge.key, ws.prev, ws.t, R, dt, stream));
      prof_end(stream, ev2, FNMT_K_EMBED, 0.0, (double)R * ge.key.w * (8.0 + dtype_size(dt)));
      ++launches;
    }
    v.embed_done = true;
  }
  auto body = [&](int t) {
    v.host_t = t;
    run_step(v, stream);
    const int ev = prof_begin(stream);
    const double rl = profiling ? (double)live[t] : (double)R;
    if (fuse_embed) {
      CK(launch_greedy_embed(gs, ge, stream));
      prof_end(stream, ev, FNMT_K_SEARCH, 0.0,
               rl * 24 + rl * arch.d_model * (8.0 + dtype_size(dt)) +
                   (ge.key.knew ? rl * ge.key.w * (8.0 + dtype_size(dt)) : 0.0));
    } else {
      CK(launch_greedy_update(gs, stream));
      prof_end(stream, ev, FNMT_K_SEARCH, 0.0, rl * 24);
    }
    ++launches;
  };
  const int64_t nodes = profiling ? 0 : capture_step([&] { body(0); });
  return drive_steps(cap, nodes, body);
}

void Engine::reserve_beam(int sent_cap, int k, int64_t pool_cap) {
  const int rows = sent_cap * k;
  const int tiles = (arch.vocab_size + kTopKTile - 1) / kTopKTile;
  const int K = k <= 4 ? 4 : 8;
  if (beam.owned.size() && sent_cap <= beam.sent_cap && k <= beam.k && pool_cap <= beam.pool_cap &&
      K <= beam.part.K)
    return;
  CK(cudaStreamSynchronize(stream));
  for (void* p : beam.owned) {
    cudaFree(p);
    allocations.erase(std::find(allocations.begin(), allocations.end(), p));
  }
  device_bytes -= beam.bytes;
  beam = BeamWs();
  const int64_t before = device_bytes;
  auto alloc = [&](size_t bytes) {
    void* p = dalloc(bytes);
    beam.owned.push_back(p);
    return p;
  };
  beam.sent_cap = sent_cap;
  beam.k = k;
  beam.pool_cap = pool_cap;
  const int64_t cap_per_row = pool_cap / rows + 1;
  beam.part.tiles = tiles;
  beam.part.K = K;
  beam.part.pmax = (float*)alloc(sizeof(float) * (size_t)rows * tiles);
  beam.part.psum = (double*)alloc(sizeof(double) * (size_t)rows * tiles);
  beam.part.pval = (float*)alloc(sizeof(float) * (size_t)rows * tiles * K);
  beam.part.pidx = (int32_t*)alloc(sizeof(int32_t) * (size_t)rows * tiles * K);
  beam.rval = (float*)alloc(sizeof(float) * (size_t)rows * k);
  beam.ridx = (int32_t*)alloc(sizeof(int32_t) * (size_t)rows * k);
  beam.rlogz = (double*)alloc(sizeof(double) * rows);
  beam.score = (double*)alloc(sizeof(double) * rows);
  beam.active = (uint8_t*)alloc(rows);
  beam.anc = (int32_t*)alloc(sizeof(int32_t) * 2 * (size_t)pool_cap);
  beam.tok_hist = (int32_t*)alloc(sizeof(int32_t) * (size_t)pool_cap);
  beam.par_hist = (int32_t*)alloc(sizeof(int32_t) * (size_t)pool_cap);
  beam.finished = (uint8_t*)alloc(sent_cap);
  beam.n_done = (int32_t*)alloc(sizeof(int32_t) * sent_cap);
  beam.fin_t = (int32_t*)alloc(sizeof(int32_t) * sent_cap);
  beam.fin_n = (int32_t*)alloc(sizeof(int32_t) * sent_cap);
  beam.done_score = (double*)alloc(sizeof(double) * sent_cap * 2 * k);
  beam.done_t = (int32_t*)alloc(sizeof(int32_t) * sent_cap * 2 * k);
  beam.done_slot = (int32_t*)alloc(sizeof(int32_t) * sent_cap * 2 * k);
  beam.ticket = (uint32_t*)alloc(sizeof(uint32_t) * 2);
  // per batch: R sentences x cap steps <= pool_cap / k (the plan's max R * cap)
  (void)cap_per_row;
  beam.out_ids = (int32_t*)alloc(sizeof(int32_t) * (size_t)(pool_cap / k + 1));
  beam.out_len = (int32_t*)alloc(sizeof(int32_t) * sent_cap);
  beam.scratch = (int32_t*)alloc(sizeof(int32_t) * (size_t)(2 * pool_cap + 1));
  if (dt == kF32) beam.logits = (float*)alloc(sizeof(float) * (size_t)rows * arch.vocab_size);
  beam.bytes = device_bytes - before;
}

int Engine::decode_beam(int R, int cap, int max_len, const fnmt_run& run,
                        const std::vector<int32_t>& budgets) {
  const int k = run.beam_size;
  const int rows = R * k;
  BeamState bs;
  bs.nS = R;
  bs.k = k;
  bs.cap = cap;
  bs.rows = rows;
  bs.eos = run.eos_id;
  bs.pad = run.pad_id;
  bs.part = beam.part;
  bs.rval = beam.rval;
  bs.ridx = beam.ridx;
  bs.rlogz = beam.rlogz;
  bs.prev = ws.prev;
  bs.score = beam.score;
  bs.active = beam.active;
  bs.anc = beam.anc;
  bs.tok_hist = beam.tok_hist;
  bs.par_hist = beam.par_hist;
  bs.budget = ws.budget;
  bs.finished = beam.finished;
  bs.n_done = beam.n_done;
  bs.done_score = beam.done_score;
  bs.done_t = beam.done_t;
  bs.done_slot = beam.done_slot;
  bs.fin_t = beam.fin_t;
  bs.fin_n = beam.fin_n;
  bs.t = ws.t;
  bs.alive = ws.alive;
  bs.ticket = beam.ticket;
  bs.out_ids = beam.out_ids;
  bs.out_len = beam.out_len;
  bs.scratch = beam.scratch;
  CK(cudaMemsetAsync(beam.anc, 0, sizeof(int32_t) * 2 * (size_t)rows * cap, stream));
  CK(launch_beam_init(bs, run.bos_id, stream));
  ++launches;
  StepView v = step_view(rows, cap, max_len, k);
  v.anc = beam.anc;
  v.anc_stride = (int64_t)rows * cap;
  v.topk = &beam.part;
  v.m_tab = live_table(budgets, cap, k);   // the top-K vocab GEMM keeps all rows
  v.logits = dt == kF32 ? beam.logits : nullptr;
  auto body = [&](int t) {
    v.host_t = t;
    run_step(v, stream);
    int ev = prof_begin(stream);
    CK(launch_beam_row_reduce(bs, stream));
    CK(launch_beam_select(bs, stream));
    prof_end(stream, ev, FNMT_K_SEARCH, 0.0, (double)rows * beam.part.tiles * 8 * (4 + beam.part.K));
    launches += 2;
  };
  const int64_t nodes = profiling ? 0 : capture_step([&] { body(0); });
  const int steps = drive_steps(cap, nodes, body);
  CK(launch_beam_final(bs, stream));
  ++launches;
  return steps;
}

void Engine::lens_from_cu(int R) {
  lens_from_cu_kernel<<<(R + 255) / 256, 256, 0, stream>>>(ws.cu, ws.len, R);
  CK(cudaGetLastError());
  ++launches;
}

void Engine::ensure_meta(size_t rows, size_t cus) {
  if (rows > meta_rows_cap) {
    meta_perm = (int32_t*)dalloc(std::max<size_t>(rows, 1) * 4);
    meta_budget = (int32_t*)dalloc(std::max<size_t>(rows, 1) * 4);
    meta_rows_cap = rows;
  }
  if (cus > meta_cu_cap) {
    meta_cu = (int32_t*)dalloc(std::max<size_t>(cus, 1) * 4);
    meta_cu_cap = cus;
  }
}

// Capture one decode step (+ greedy bookkeeping) into a graph; reuse the
// executable graph through cudaGraphExecUpdate when the topology matches.
int64_t Engine::capture_step(const std::function<void()>& body) {
  const int64_t l0 = launches;
  cudaGraph_t g = nullptr;
  CK(cudaStreamBeginCapture(stream, cudaStreamCaptureModeRelaxed));
  try {
    body();
  } catch (...) {
    cudaStreamEndCapture(stream, &g);
    if (g) cudaGraphDestroy(g);
    throw;
  }
  CK(cudaStreamEndCapture(stream, &g));
  const int64_t nodes = launches - l0;
  launches = l0;  // counted per replay by the caller
  // In-place update only when the new graph has the same kernels in the same
  // order (a batch with another tile choice or launch sequence gets a fresh
  // instantiation instead of a failed cudaGraphExecUpdate)
  std::vector<void*> funcs;
  {
    size_t n = 0;
    CK(cudaGraphGetNodes(g, nullptr, &n));
    std::vector<cudaGraphNode_t> nodes_v(n);
    if (n) CK(cudaGraphGetNodes(g, nodes_v.data(), &n));
    funcs.reserve(n);
    for (cudaGraphNode_t nd : nodes_v) {
      cudaGraphNodeType t;
      CK(cudaGraphNodeGetType(nd, &t));
      void* f = nullptr;
      if (t == cudaGraphNodeTypeKernel) {
        cudaKernelNodeParams kp;
        CK(cudaGraphKernelNodeGetParams(nd, &kp));
        f = kp.func;
      }
      funcs.push_back(f);
    }
  }
  bool updated = false;
  if (graph_exec && funcs == graph_funcs) {
    cudaGraphExecUpdateResultInfo info;
    if (cudaGraphExecUpdate(graph_exec, g, &info) == cudaSuccess) updated = true;
    else cudaGetLastError();
  }
  if (!updated) {
    if (graph_exec) cudaGraphExecDestroy(graph_exec);
    graph_exec = nullptr;
    CK(cudaGraphInstantiate(&graph_exec, g, 0));
    graph_funcs = std::move(funcs);
  }
  CK(cudaGraphDestroy(g));
  return nodes;
}

// ---------------------------------------------------------------------------
// protocol-level entry points (used by the Python drop-in TranslationModel)

void Engine::encode_padded(const int32_t* d_tokens, const int32_t* d_lengths, int b, int s,
                           float* d_states32, void* d_states_act) {
  if (s > arch.max_positions)
    throw EngineError(FNMT_E_LENGTH, "source length " + std::to_string(s) +
                                         " exceeds max_positions " +
                                         std::to_string(arch.max_positions));
  const int n_tok = b * s;
  if (n_tok == 0) return;
  reserve(std::max(n_tok, ws.tok_cap), std::max(b, ws.row_cap), ws.pool_cap);
  CK(cudaMemcpyAsync(ws.ids, d_tokens, sizeof(int32_t) * n_tok, cudaMemcpyDeviceToDevice, stream));
  iota_pos_kernel<<<(n_tok + 255) / 256, 256, 0, stream>>>(ws.pos, b, s);
  seq_table_kernel<<<(b + 255) / 256, 256, 0, stream>>>(ws.qstart, ws.qlen, b, s);
  CK(cudaMemcpyAsync(ws.len, d_lengths, sizeof(int32_t) * b, cudaMemcpyDeviceToDevice, stream));
  CK(launch_embed(ws.ids, ws.pos, nullptr, src_emb32, pos32, emb_scale(), ws.x32,
                  dt != kF32 ? ws.xa : nullptr, dt, n_tok, arch.d_model, stream));
  // queries: every padded position; keys: the real prefix (k_len 0 => all s masked)
  encoder_layers(n_tok, b, s, s, ws.qstart, ws.qlen, ws.qstart, ws.len, s, stream);
  if (d_states32)
    CK(cudaMemcpyAsync(d_states32, ws.x32, sizeof(float) * n_tok * arch.d_model,
                       cudaMemcpyDeviceToDevice, stream));
  if (d_states_act)
    CK(cudaMemcpyAsync(d_states_act, ws.xa, (size_t)dtype_size(dt) * n_tok * arch.d_model,
                       cudaMemcpyDeviceToDevice, stream));
  CK(cudaStreamSynchronize(stream));
}

void Engine::cross_kv(const void* d_states_act, int rows, int layer, void* d_out) {
  if (layer < 0 || layer >= arch.n_dec_layers) throw EngineError(FNMT_E_INVALID, "bad layer");
  GemmArgs g;
  g.A = d_states_act;
  g.lda = arch.d_model;
  g.W = dec[layer].ckv.w;
  g.ldw = dec[layer].ckv.K;
  g.in_dtype = dt;
  g.bias = dec[layer].ckv.b;
  g.M = rows;
  g.N = dec[layer].ckv.N;
  g.K = dec[layer].ckv.K;
  g.C = d_out;
  g.ldc = 2 * arch.d_model;
  g.c_dtype = dt;
  g.tmap_w = dt == kF32 ? nullptr : &dec[layer].ckv.tm;
  attach_q(g, dec[layer].ckv);
  CK(launch_gemm(g, stream));
  CK(cudaStreamSynchronize(stream));
}

void Engine::decode_step(const int32_t* d_prev, int t, int rows, int cap, void* const* self_k,
                         void* const* self_v, const void* const* cross_kv,
                         const int32_t* d_k_start, const int32_t* d_k_len, int k_pad, int max_k,
                         float* d_logits) {
  if (t >= arch.max_positions)
    throw EngineError(FNMT_E_LENGTH, "decode position " + std::to_string(t) +
                                         " exceeds max_positions " +
                                         std::to_string(arch.max_positions));
  if (t >= cap) throw EngineError(FNMT_E_INVALID, "self-attention cache capacity exceeded");
  if (rows == 0) return;
  reserve(ws.tok_cap, std::max(rows, ws.row_cap), ws.pool_cap);
  fill_i32_kernel<<<1, 32, 0, stream>>>(ws.t, 1, t);
  CK(cudaMemcpyAsync(ws.prev, d_prev, sizeof(int32_t) * rows, cudaMemcpyDeviceToDevice, stream));
  StepView v;
  v.rows = rows;
  v.cap = cap;
  v.prev = ws.prev;
  v.t_ptr = ws.t;
  std::vector<void*> kc(self_k, self_k + arch.n_dec_layers), vc(self_v, self_v + arch.n_dec_layers);
  std::vector<const void*> ckv(cross_kv, cross_kv + arch.n_dec_layers);
  v.kc = kc.data();
  v.vc = vc.data();
  v.ckv = ckv.data();
  v.k_start = d_k_start;
  v.k_len = d_k_len;
  v.k_pad = k_pad;
  v.rows_per_seq = 1;
  v.max_k = std::max(max_k, k_pad);
  v.logits = d_logits;
  run_step(v, stream);
  CK(cudaStreamSynchronize(stream));
}

}  // namespace fnmt
