// extern "C" boundary (include/fnmt_b200.h).  Every entry point converts C++
// exceptions / CUDA errors into a negative status and a thread-local message.
#include <cuda_runtime.h>

#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/fnmt_b200.h"
#include "common.cuh"
#include "engine.h"
#include "kernels.h"

using fnmt::EngineError;

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  void ensure(size_t need) {
    if (need <= bytes) return;
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
    if (cudaMalloc(&p, need) != cudaSuccess) throw EngineError(FNMT_E_CUDA, "cudaMalloc failed");
    bytes = need;
  }
  ~DevBuf() {
    if (p) cudaFree(p);
  }
};

struct fnmt_engine {
  fnmt::Engine* eng = nullptr;
  DevBuf ids, off, out_ids, out_off, out_len;
};

namespace {

int fail(int code, const std::string& msg) {
  fnmt::set_error(msg);
  return code;
}

int cuda_status(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return FNMT_OK;
  return fail(FNMT_E_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}

template <typename F>
int guarded(F&& f) {
  try {
    return f();
  } catch (const EngineError& e) {
    return fail(e.code, e.msg);
  } catch (const std::exception& e) {
    return fail(FNMT_E_INVALID, e.what());
  } catch (...) {
    return fail(FNMT_E_INVALID, "unknown C++ exception");
  }
}

bool valid_dtype(int dt) { return dt == FNMT_F32 || dt == FNMT_F16 || dt == FNMT_BF16; }

}  // namespace

extern "C" {

const char* fnmt_last_error(void) { return fnmt::g_last_error.c_str(); }

const char* fnmt_version(void) { return "fnmt_b200 0.1.0 (sm_100a tcgen05)"; }

int fnmt_linear(const void* A, int lda, int a_dtype, const void* W, int ldw, const float* bias,
                void* C, int ldc, int c_dtype, int M, int N, int K, int relu, const float* resid,
                int ld_resid, void* stream) {
  if (!valid_dtype(a_dtype) || !valid_dtype(c_dtype) || M < 0 || N < 0 || K < 1 || !A || !W || !C)
    return fail(FNMT_E_INVALID, "fnmt_linear: bad arguments");
  if (lda < K || ldw < K || ldc < N) return fail(FNMT_E_INVALID, "fnmt_linear: leading dims");
  fnmt::GemmArgs g;
  g.A = A;
  g.lda = lda;
  g.W = W;
  g.ldw = ldw;
  g.in_dtype = a_dtype;
  g.bias = bias;
  g.M = M;
  g.N = N;
  g.K = K;
  g.C = C;
  g.ldc = ldc;
  g.c_dtype = c_dtype;
  g.relu = relu;
  g.resid = resid;
  g.ld_resid = ld_resid;
  return cuda_status(fnmt::launch_gemm(g, (cudaStream_t)stream), "fnmt_linear");
}

int fnmt_linear_add_norm(const void* A, int lda, int a_dtype, const void* W, int ldw,
                         const float* bias, float* x, void* x_act, const float* gain,
                         const float* beta, int l1, int M, int N, int K, void* stream) {
  if (!valid_dtype(a_dtype) || !A || !W || !x || !gain || !beta || M < 0 || N < 4 || N % 4 ||
      K < 1 || lda < K || ldw < K)
    return fail(FNMT_E_INVALID, "fnmt_linear_add_norm: bad arguments");
  if (M == 0) return FNMT_OK;
  cudaStream_t s = (cudaStream_t)stream;
  fnmt::GemmArgs g;
  g.A = A;
  g.lda = lda;
  g.W = W;
  g.ldw = ldw;
  g.in_dtype = a_dtype;
  g.bias = bias;
  g.M = M;
  g.N = N;
  g.K = K;
  // x += A.W + b in place (the epilogue reads and writes each element from the
  // same thread), then the post-norm over the full rows (tensor.py:98-129)
  g.C = x;
  g.ldc = N;
  g.c_dtype = fnmt::kF32;
  g.resid = x;
  g.ld_resid = N;
  cudaError_t e = fnmt::launch_gemm(g, s);
  if (e == cudaSuccess)
    e = fnmt::launch_add_norm(x, nullptr, gain, beta, l1, x, x_act, a_dtype, M, N, s);
  return cuda_status(e, "fnmt_linear_add_norm");
}

int64_t fnmt_qgemm_workspace(int64_t M, int K) {
  if (M < 0 || K < 1) return fail(FNMT_E_INVALID, "fnmt_qgemm_workspace: bad arguments");
  return fnmt::qgemm_scratch_bytes(std::max<int64_t>(M, 1), K);
}

int fnmt_qgemm(const float* A, int lda, const int8_t* Wq, const float* scale, const float* zp,
               const int32_t* colsum, const float* bias, float* C, int ldc, int M, int N, int K,
               int relu, void* workspace, int64_t workspace_bytes, void* stream) {
  if (!A || !Wq || !scale || !zp || !colsum || !C || !workspace || M < 0 || N < 1 || K < 1 ||
      lda < K || ldc < N)
    return fail(FNMT_E_INVALID, "fnmt_qgemm: bad arguments");
  if (M == 0) return FNMT_OK;
  if (workspace_bytes < fnmt::qgemm_scratch_bytes(M, K))
    return fail(FNMT_E_INVALID, "fnmt_qgemm: workspace smaller than fnmt_qgemm_workspace(M, K)");
  const int Kp = fnmt::round_up16(K);
  CUtensorMap tw;
  std::string err;
  if (!fnmt::make_tmap_8(&tw, Wq, N, Kp, 64, &err))
    return fail(FNMT_E_INVALID, "fnmt_qgemm: " + err);
  fnmt::GemmArgs g;
  g.A = A;
  g.lda = lda;
  g.in_dtype = fnmt::kF32;
  g.bias = bias;
  g.M = M;
  g.N = N;
  g.K = K;
  g.C = C;
  g.ldc = ldc;
  g.c_dtype = fnmt::kF32;
  g.relu = relu;
  g.qw = Wq;
  g.qscale = scale;
  g.qzp = zp;
  g.qcolsum = colsum;
  g.Kp = Kp;
  g.qtmap_w = &tw;
  g.qs = fnmt::qgemm_scratch(workspace, M, K);
  return cuda_status(fnmt::launch_gemm(g, (cudaStream_t)stream), "fnmt_qgemm");
}

int fnmt_linear_argmax(const void* A, int lda, int a_dtype, const void* W, int ldw,
                       const float* bias, int M, int N, int K, uint64_t* keys_scratch,
                       int32_t* out_idx, void* stream) {
  if (!valid_dtype(a_dtype) || !bias || !keys_scratch || !out_idx || M < 0 || N < 1 || K < 1)
    return fail(FNMT_E_INVALID, "fnmt_linear_argmax: bad arguments");
  cudaStream_t s = (cudaStream_t)stream;
  cudaError_t e = cudaMemsetAsync(keys_scratch, 0, sizeof(uint64_t) * (size_t)M, s);
  if (e != cudaSuccess) return cuda_status(e, "memset");
  fnmt::GemmArgs g;
  g.A = A;
  g.lda = lda;
  g.W = W;
  g.ldw = ldw;
  g.in_dtype = a_dtype;
  g.bias = bias;
  g.M = M;
  g.N = N;
  g.K = K;
  g.epi = fnmt::kEpiArgmax;
  g.keys = (unsigned long long*)keys_scratch;
  e = fnmt::launch_gemm(g, s);
  if (e != cudaSuccess) return cuda_status(e, "fnmt_linear_argmax");
  return cuda_status(fnmt::launch_keys_to_index((const unsigned long long*)keys_scratch, M,
                                                out_idx, s),
                     "keys_to_index");
}

int fnmt_embed(const int32_t* ids, const int32_t* pos_ids, const float* table,
               const float* pos_table, float scale, float* out32, void* out_act, int act_dtype,
               int n, int d, void* stream) {
  if (!ids || !pos_ids || !table || !pos_table || n < 0 || d < 4 || d % 4)
    return fail(FNMT_E_INVALID, "fnmt_embed: bad arguments (d must be a multiple of 4)");
  return cuda_status(fnmt::launch_embed(ids, pos_ids, nullptr, table, pos_table, scale, out32,
                                        out_act, act_dtype, n, d, (cudaStream_t)stream),
                     "fnmt_embed");
}

int fnmt_add_norm(const float* x, const float* y, const float* gain, const float* bias, int l1,
                  float* out32, void* out_act, int act_dtype, int rows, int d, void* stream) {
  if (!x || !gain || !bias || rows < 0 || d < 4 || d % 4 || d > 2048)
    return fail(FNMT_E_INVALID, "fnmt_add_norm: bad arguments (d multiple of 4, <= 2048)");
  return cuda_status(fnmt::launch_add_norm(x, y, gain, bias, l1, out32, out_act, act_dtype, rows,
                                           d, (cudaStream_t)stream),
                     "fnmt_add_norm");
}

int fnmt_attention(const void* q, int ldq, const void* k, const void* v, int ldkv, void* out,
                   int ldo, int dtype, int heads, int dk, const int32_t* q_start,
                   const int32_t* q_len, const int32_t* k_start, const int32_t* k_len,
                   int k_pad, int n_seq, int max_q, int max_k, void* stream) {
  if (!valid_dtype(dtype) || heads < 1 || dk < 1 || n_seq < 0 || max_q < 0 || max_k < 0 ||
      max_k > 4096)
    return fail(FNMT_E_INVALID, "fnmt_attention: bad arguments");
  fnmt::AttnArgs a{};
  a.q = q;
  a.ldq = ldq;
  a.k = k;
  a.v = v;
  a.ldkv = ldkv;
  a.out = out;
  a.ldo = ldo;
  a.dtype = dtype;
  a.heads = heads;
  a.dk = dk;
  a.q_start = q_start;
  a.q_len = q_len;
  a.k_start = k_start;
  a.k_len = k_len;
  a.k_pad = k_pad;
  a.n_seq = n_seq;
  a.max_q = max_q;
  a.max_k = max_k > k_pad ? max_k : k_pad;
  return cuda_status(fnmt::launch_attention_varlen(a, (cudaStream_t)stream), "fnmt_attention");
}

int fnmt_argmax_rows(const float* logits, int ld, int rows, int n, int32_t* out_idx,
                     void* stream) {
  if (!logits || !out_idx || rows < 0 || n < 1 || ld < n)
    return fail(FNMT_E_INVALID, "fnmt_argmax_rows: bad arguments");
  return cuda_status(fnmt::launch_argmax_rows(logits, ld, rows, n, out_idx, (cudaStream_t)stream),
                     "fnmt_argmax_rows");
}

int fnmt_gather_rows(const void* src, void* dst, const int32_t* idx, int rows,
                     int64_t row_bytes, int64_t src_stride, int64_t dst_stride, void* stream) {
  if (!src || !dst || !idx || rows < 0 || rows > 65535 || row_bytes < 0)
    return fail(FNMT_E_INVALID, "fnmt_gather_rows: bad arguments");
  return cuda_status(fnmt::launch_gather_rows(src, dst, idx, rows, row_bytes, src_stride,
                                              dst_stride, (cudaStream_t)stream),
                     "fnmt_gather_rows");
}

// ---------------------------------------------------------------------------

int fnmt_engine_create(const fnmt_arch* arch, int device, int dtype, fnmt_engine** out) {
  if (!arch || !out) return fail(FNMT_E_INVALID, "fnmt_engine_create: null argument");
  return guarded([&] {
    fnmt_engine* h = new fnmt_engine();
    try {
      h->eng = new fnmt::Engine(*arch, device, dtype);
    } catch (...) {
      delete h;
      throw;
    }
    *out = h;
    return FNMT_OK;
  });
}

void fnmt_engine_destroy(fnmt_engine* e) {
  if (!e) return;
  int dev = e->eng ? e->eng->device : 0;
  cudaSetDevice(dev);
  delete e->eng;
  delete e;
}

int fnmt_engine_set_tensor(fnmt_engine* e, const char* name, const float* host, int64_t numel) {
  if (!e || !name || !host || numel < 0) return fail(FNMT_E_INVALID, "set_tensor: bad arguments");
  return guarded([&] {
    e->eng->set_tensor(name, host, numel);
    return FNMT_OK;
  });
}

int fnmt_engine_set_qtensor(fnmt_engine* e, const char* name, const int8_t* q, const float* scale,
                            const float* zp, int64_t k, int64_t n) {
  if (!e || !name || !q || !scale || !zp || k < 1 || n < 1)
    return fail(FNMT_E_INVALID, "set_qtensor: bad arguments");
  return guarded([&] {
    e->eng->set_qtensor(name, q, scale, zp, k, n);
    return FNMT_OK;
  });
}

int fnmt_engine_finalize(fnmt_engine* e) {
  if (!e) return fail(FNMT_E_INVALID, "null engine");
  return guarded([&] {
    e->eng->finalize();
    return FNMT_OK;
  });
}

int fnmt_engine_reserve(fnmt_engine* e, const fnmt_run* run) {
  if (!e || !run) return fail(FNMT_E_INVALID, "null argument");
  return guarded([&] {
    cudaSetDevice(e->eng->device);
    e->eng->reserve_for(*run);
    return FNMT_OK;
  });
}

int64_t fnmt_budgets(const int32_t* lengths, int n, double ratio, int offset, int max_positions,
                     int32_t* budgets) {
  if ((!lengths && n) || n < 0 || max_positions < 1) {
    fnmt::set_error("fnmt_budgets: bad arguments");
    return FNMT_E_INVALID;
  }
  int64_t total = 0;
  for (int i = 0; i < n; ++i) {
    const int b = lengths[i] > 0 ? fnmt::budget_of(lengths[i], ratio, offset, max_positions) : 0;
    if (budgets) budgets[i] = b;
    total += b;
  }
  return total;
}

int fnmt_plan_batches(const int32_t* lengths, int n, int sbatch, int wbatch, int32_t* perm,
                      int32_t* sizes, int32_t* max_len, uint8_t* oversize) {
  if ((!lengths && n) || n < 0 || sbatch < 1 || wbatch < 1 || (n && (!perm || !sizes))) {
    fnmt::set_error("fnmt_plan_batches: bad arguments");
    return FNMT_E_INVALID;
  }
  std::vector<int32_t> L(lengths, lengths + n);
  const auto plan = fnmt::plan_batches(L, sbatch, wbatch);
  int k = 0, j = 0;
  for (const auto& b : plan) {
    for (int32_t r : b.rows) perm[j++] = r;
    sizes[k] = (int32_t)b.rows.size();
    if (max_len) max_len[k] = b.max_len;
    if (oversize) oversize[k] = b.oversize ? 1 : 0;
    ++k;
  }
  return k;
}

int fnmt_engine_translate_device(fnmt_engine* e, const int32_t* d_ids, const int64_t* d_offsets,
                                 const int32_t* lengths, int n, const fnmt_run* run,
                                 int32_t* d_out_ids, const int64_t* out_off,
                                 const int64_t* d_out_off, int32_t* d_out_len,
                                 fnmt_stats* stats) {
  (void)out_off;
  if (!e || !run || n < 0 || (n && (!lengths || !d_ids || !d_offsets || !d_out_ids ||
                                    !d_out_off || !d_out_len)))
    return fail(FNMT_E_INVALID, "translate_device: bad arguments");
  return guarded([&] {
    std::vector<int32_t> L(lengths, lengths + n);
    e->eng->translate_device(d_ids, d_offsets, L, *run, d_out_ids, d_out_off, d_out_len, stats);
    return FNMT_OK;
  });
}

int fnmt_engine_translate(fnmt_engine* e, const int32_t* ids, const int64_t* offsets, int n,
                          const fnmt_run* run, int32_t* out_ids, const int64_t* out_off,
                          int32_t* out_len, fnmt_stats* stats) {
  if (!e || !run || n < 0 || (n && (!ids || !offsets || !out_ids || !out_off || !out_len)))
    return fail(FNMT_E_INVALID, "translate: bad arguments");
  return guarded([&] {
    fnmt::Engine* g = e->eng;
    cudaSetDevice(g->device);
    cudaStream_t s = g->stream;
    std::vector<int32_t> L(n);
    int64_t out_total = 0;
    for (int i = 0; i < n; ++i) {
      const int64_t len = offsets[i + 1] - offsets[i];
      if (len < 0 || len > (1 << 30)) throw EngineError(FNMT_E_INVALID, "bad offsets");
      L[i] = (int32_t)len;
      const int b = len > 0 ? fnmt::budget_of((int32_t)len, run->max_len_ratio,
                                              run->max_len_offset, g->arch.max_positions)
                            : 0;
      out_total = std::max<int64_t>(out_total, out_off[i] + b);
    }
    const int64_t n_ids = n ? offsets[n] - offsets[0] : 0;
    e->ids.ensure(sizeof(int32_t) * std::max<int64_t>(n_ids, 1));
    e->off.ensure(sizeof(int64_t) * (n + 1));
    e->out_ids.ensure(sizeof(int32_t) * std::max<int64_t>(out_total, 1));
    e->out_off.ensure(sizeof(int64_t) * std::max(n, 1));
    e->out_len.ensure(sizeof(int32_t) * std::max(n, 1));
    // rebase offsets so ids[offsets[0]] is element 0 on the device
    std::vector<int64_t> off(n + 1);
    for (int i = 0; i <= n; ++i) off[i] = offsets[i] - (n ? offsets[0] : 0);
    auto ck = [](cudaError_t err, const char* what) {
      if (err != cudaSuccess) throw EngineError(FNMT_E_CUDA, std::string(what) + ": " + cudaGetErrorString(err));
    };
    ck(cudaMemcpyAsync(e->ids.p, ids + (n ? offsets[0] : 0), sizeof(int32_t) * n_ids,
                       cudaMemcpyHostToDevice, s), "H2D ids");
    ck(cudaMemcpyAsync(e->off.p, off.data(), sizeof(int64_t) * (n + 1), cudaMemcpyHostToDevice, s),
       "H2D offsets");
    ck(cudaMemcpyAsync(e->out_off.p, out_off, sizeof(int64_t) * n, cudaMemcpyHostToDevice, s),
       "H2D out offsets");
    g->translate_device((const int32_t*)e->ids.p, (const int64_t*)e->off.p, L, *run,
                        (int32_t*)e->out_ids.p, (const int64_t*)e->out_off.p,
                        (int32_t*)e->out_len.p, stats);
    ck(cudaMemcpyAsync(out_ids, e->out_ids.p, sizeof(int32_t) * out_total, cudaMemcpyDeviceToHost, s),
       "D2H ids");
    ck(cudaMemcpyAsync(out_len, e->out_len.p, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, s),
       "D2H lens");
    ck(cudaStreamSynchronize(s), "sync");
    return FNMT_OK;
  });
}

int fnmt_engine_encode_padded(fnmt_engine* e, const int32_t* d_tokens, const int32_t* d_lengths,
                              int b, int s, float* d_states32, void* d_states_act) {
  if (!e || b < 0 || s < 0 || (b > 0 && s > 0 && (!d_tokens || !d_lengths)))
    return fail(FNMT_E_INVALID, "encode_padded: bad arguments");
  return guarded([&] {
    cudaSetDevice(e->eng->device);
    e->eng->encode_padded(d_tokens, d_lengths, b, s, d_states32, d_states_act);
    return FNMT_OK;
  });
}

int fnmt_engine_cross_kv(fnmt_engine* e, const void* d_states_act, int rows, int layer,
                         void* d_out) {
  if (!e || rows < 0 || (rows && (!d_states_act || !d_out)))
    return fail(FNMT_E_INVALID, "cross_kv: bad arguments");
  return guarded([&] {
    cudaSetDevice(e->eng->device);
    e->eng->cross_kv(d_states_act, rows, layer, d_out);
    return FNMT_OK;
  });
}

int fnmt_engine_decode_step(fnmt_engine* e, const int32_t* d_prev, int t, int rows, int cap,
                            void* const* self_k, void* const* self_v,
                            const void* const* cross_kv, const int32_t* d_k_start,
                            const int32_t* d_k_len, int k_pad, int max_k, float* d_logits) {
  if (!e || rows < 0 || t < 0 || cap < 1 || !self_k || !self_v || !cross_kv || !d_logits)
    return fail(FNMT_E_INVALID, "decode_step: bad arguments");
  return guarded([&] {
    cudaSetDevice(e->eng->device);
    e->eng->decode_step(d_prev, t, rows, cap, self_k, self_v, cross_kv, d_k_start, d_k_len, k_pad,
                        max_k, d_logits);
    return FNMT_OK;
  });
}

int fnmt_engine_profile(fnmt_engine* e, int enable) {
  if (!e) return fail(FNMT_E_INVALID, "null engine");
  return guarded([&] {
    cudaSetDevice(e->eng->device);
    e->eng->set_profiling(enable != 0);
    return FNMT_OK;
  });
}

int fnmt_engine_profile_read(fnmt_engine* e, double* ms, int64_t* launches, double* flops,
                             double* bytes) {
  if (!e) return fail(FNMT_E_INVALID, "null engine");
  for (int i = 0; i < FNMT_K_COUNT; ++i) {
    if (ms) ms[i] = e->eng->prof_ms[i];
    if (launches) launches[i] = e->eng->prof_n[i];
    if (flops) flops[i] = e->eng->prof_flops[i];
    if (bytes) bytes[i] = e->eng->prof_bytes[i];
  }
  return FNMT_OK;
}

int64_t fnmt_engine_profile_log(fnmt_engine* e, int32_t* cls, float* ms, double* flops,
                                double* bytes, int64_t cap) {
  if (!e || cap < 0) return fail(FNMT_E_INVALID, "profile_log: bad arguments");
  const auto& log = e->eng->prof_log;
  const int64_t n = std::min<int64_t>(cap, (int64_t)log.size());
  for (int64_t i = 0; i < n; ++i) {
    if (cls) cls[i] = log[i].cls;
    if (ms) ms[i] = log[i].ms;
    if (flops) flops[i] = log[i].flops;
    if (bytes) bytes[i] = log[i].bytes;
  }
  return (int64_t)log.size();
}

int64_t fnmt_engine_device_bytes(const fnmt_engine* e) {
  return e ? e->eng->total_device_bytes() : 0;
}

int fnmt_engine_set_lanes(fnmt_engine* e, int lanes) {
  if (!e || lanes < 1 || lanes > 16) return fail(FNMT_E_INVALID, "set_lanes: 1..16");
  e->eng->n_lanes = lanes;
  return FNMT_OK;
}

void* fnmt_engine_stream(fnmt_engine* e) { return e ? (void*)e->eng->stream : nullptr; }

}  // extern "C"
