// Memory-bound row kernels: embedding + sinusoid position, residual add +
// LayerNorm (l2 / l1), and the search bookkeeping kernels.
//
// Numerics follow the reference exactly where fp32 allows:
//  * embed: x = E[id] * f32(sqrt(d)) + P[pos]            (model.py:276-277, :327-328)
//  * norm:  mu = f64 mean -> f32; dev = x - mu; scale = sqrt(mean(dev^2)) (l2)
//           or mean(|dev|) (l1); y = (g * dev) / (scale + 1e-6) + b   (tensor.py:84-129)
//  * greedy: argmax lowest-id ties, EOS finishes without emitting, budget
//           token is emitted, finished rows are fed PAD  (search.py:58-86)
#include <algorithm>

#include <type_traits>

#include "common.cuh"
#include "kernels.h"

namespace fnmt {

namespace {

template <typename T>
__device__ __forceinline__ void store4(T* dst, float4 v);
template <>
__device__ __forceinline__ void store4<float>(float* dst, float4 v) {
  *reinterpret_cast<float4*>(dst) = v;
}
template <>
__device__ __forceinline__ void store4<__half>(__half* dst, float4 v) {
  __half2 a = __floats2half2_rn(v.x, v.y), b = __floats2half2_rn(v.z, v.w);
  uint2 u = make_uint2(*reinterpret_cast<uint32_t*>(&a), *reinterpret_cast<uint32_t*>(&b));
  *reinterpret_cast<uint2*>(dst) = u;
}
template <>
__device__ __forceinline__ void store4<__nv_bfloat16>(__nv_bfloat16* dst, float4 v) {
  __nv_bfloat162 a = __floats2bfloat162_rn(v.x, v.y), b = __floats2bfloat162_rn(v.z, v.w);
  uint2 u = make_uint2(*reinterpret_cast<uint32_t*>(&a), *reinterpret_cast<uint32_t*>(&b));
  *reinterpret_cast<uint2*>(dst) = u;
}

template <typename TA>
__global__ void embed_kernel(const int32_t* __restrict__ ids, const int32_t* __restrict__ pos_ids,
                             const int32_t* __restrict__ pos_scalar,
                             const float* __restrict__ table, const float* __restrict__ ptab,
                             float scale, float* __restrict__ x32, TA* __restrict__ xact, int n,
                             int d) {
  pdl_trigger();
  pdl_wait();
  const int d4 = d >> 2;
  const int64_t total = (int64_t)n * d4;
  const int pscalar = pos_scalar ? *pos_scalar : 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total;
       i += (int64_t)gridDim.x * blockDim.x) {
    const int row = (int)(i / d4);
    const int c = (int)(i - (int64_t)row * d4) * 4;
    const int tok = ids[row];
    const int p = pos_ids ? pos_ids[row] : pscalar;
    float4 e = *reinterpret_cast<const float4*>(table + (size_t)tok * d + c);
    float4 q = *reinterpret_cast<const float4*>(ptab + (size_t)p * d + c);
    float4 o;
    o.x = __fadd_rn(__fmul_rn(e.x, scale), q.x);
    o.y = __fadd_rn(__fmul_rn(e.y, scale), q.y);
    o.z = __fadd_rn(__fmul_rn(e.z, scale), q.z);
    o.w = __fadd_rn(__fmul_rn(e.w, scale), q.w);
    if (x32) store4(x32 + (size_t)row * d + c, o);
    if (xact) store4(xact + (size_t)row * d + c, o);
  }
}

// One warp per row; each lane holds up to NV float4 chunks of the row.  The
// row, gain and bias loads are all issued before the live-row bound is read
// (rows past the bound are in the buffer, their values are just not used),
// so a row costs one memory round trip before the two reductions.
template <typename TA, int NV>
__global__ void add_norm_kernel(const float* __restrict__ x, const float* __restrict__ y,
                                const float* __restrict__ gain, const float* __restrict__ bias,
                                int l1, float* __restrict__ out32, TA* __restrict__ out_act,
                                int rows, int d, const int32_t* rows_tab, const int32_t* t_ptr) {
  pdl_trigger();
  pdl_wait();
  const int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp >= rows) return;
  const int d4 = d >> 2;
  const float* xr = x + (size_t)warp * d;
  const float* yr = y ? y + (size_t)warp * d : nullptr;
  float4 v[NV], gv[NV], bv[NV];
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int c = lane + 32 * i;
    if (c < d4) {
      v[i] = reinterpret_cast<const float4*>(xr)[c];
      if (yr) gv[i] = reinterpret_cast<const float4*>(yr)[c];
    }
  }
  if (rows_tab && warp >= rows_tab[*t_ptr]) return;   // rows past their budgets: skipped
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int c = lane + 32 * i;
    if (c < d4) {
      float4 a = v[i];
      if (yr) {
        const float4 b = gv[i];
        a.x = a.x + b.x;
        a.y = a.y + b.y;
        a.z = a.z + b.z;
        a.w = a.w + b.w;
      }
      v[i] = a;
      gv[i] = reinterpret_cast<const float4*>(gain)[c];
      bv[i] = reinterpret_cast<const float4*>(bias)[c];
      s += (double)a.x + (double)a.y + (double)a.z + (double)a.w;
    }
  }
  s = warp_sum_d(s);
  const float mu = (float)(s / (double)d);
  double q = 0.0;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int c = lane + 32 * i;
    if (c < d4) {
      v[i].x -= mu;
      v[i].y -= mu;
      v[i].z -= mu;
      v[i].w -= mu;
      if (l1)
        q += (double)fabsf(v[i].x) + (double)fabsf(v[i].y) + (double)fabsf(v[i].z) +
             (double)fabsf(v[i].w);
      else
        q += (double)(v[i].x * v[i].x) + (double)(v[i].y * v[i].y) + (double)(v[i].z * v[i].z) +
             (double)(v[i].w * v[i].w);
    }
  }
  q = warp_sum_d(q);
  float sc = (float)(q / (double)d);
  if (!l1) sc = sqrtf(sc);
  const float den = sc + 1e-6f;
#pragma unroll
  for (int i = 0; i < NV; ++i) {
    const int c = lane + 32 * i;
    if (c < d4) {
      const float4 g = gv[i];
      const float4 b = bv[i];
      float4 o;
      o.x = g.x * v[i].x / den + b.x;
      o.y = g.y * v[i].y / den + b.y;
      o.z = g.z * v[i].z / den + b.z;
      o.w = g.w * v[i].w / den + b.w;
      if (out32) store4(out32 + (size_t)warp * d + 4 * c, o);
      if (out_act) store4(out_act + (size_t)warp * d + 4 * c, o);
    }
  }
}

template <typename TA>
cudaError_t add_norm_dispatch(const float* x, const float* y, const float* g, const float* b,
                              int l1, float* o32, TA* oa, int rows, int d, cudaStream_t s,
                              const int32_t* rows_tab = nullptr, const int32_t* t_ptr = nullptr) {
  const int threads = 256;
  const int blocks = (int)(((int64_t)rows * 32 + threads - 1) / threads);
  const int nv = (d / 4 + 31) / 32;
  void (*k)(const float*, const float*, const float*, const float*, int, float*, TA*, int, int,
            const int32_t*, const int32_t*) = nullptr;
  if (nv <= 1)
    k = add_norm_kernel<TA, 1>;
  else if (nv <= 2)
    k = add_norm_kernel<TA, 2>;
  else if (nv <= 4)
    k = add_norm_kernel<TA, 4>;
  else if (nv <= 6)
    k = add_norm_kernel<TA, 6>;
  else if (nv <= 8)
    k = add_norm_kernel<TA, 8>;
  else if (nv <= 16)
    k = add_norm_kernel<TA, 16>;
  else
    return cudaErrorInvalidValue;
  return launch_k(k, dim3(blocks), dim3(threads), 0, s, x, y, g, b, l1, o32, oa, rows, d,
                  rows_tab, t_ptr);
}

// Single CTA: every row reads the same step counter, then thread 0 bumps it.
__global__ void __launch_bounds__(1024) greedy_update_kernel(GreedyState g) {
  pdl_trigger();
  pdl_wait();
  __shared__ int alive_s;
  const int t = *g.t;
  if (threadIdx.x == 0) alive_s = 0;
  __syncthreads();
  int alive = 0;
  for (int r = threadIdx.x; r < g.rows; r += blockDim.x) {
    const unsigned long long key = g.keys[r];
    g.keys[r] = 0ull;
    if (g.finished[r]) {
      g.prev[r] = g.pad;
      continue;
    }
    const int tok = (int)argmax_key_index(key);
    if (tok == g.eos) {
      g.finished[r] = 1;
      g.prev[r] = g.pad;
      continue;
    }
    if (t < g.out_cap) g.out_ids[(size_t)r * g.out_cap + t] = tok;
    g.out_len[r] = t + 1;
    g.prev[r] = tok;
    if (t + 1 >= g.budget[r])
      g.finished[r] = 1;
    else
      ++alive;
  }
  alive = __reduce_add_sync(0xffffffffu, alive);
  if ((threadIdx.x & 31) == 0 && alive) atomicAdd(&alive_s, alive);
  __syncthreads();
  if (threadIdx.x == 0) {
    *g.alive = alive_s;
    *g.t = t + 1;
  }
}

__global__ void argmax_rows_kernel(const float* __restrict__ logits, int ld, int n,
                                   int32_t* __restrict__ out) {
  const float* row = logits + (size_t)blockIdx.x * ld;
  unsigned long long best = 0ull;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    unsigned long long k = argmax_key(row[i], (uint32_t)i);
    best = k > best ? k : best;
  }
  __shared__ unsigned long long red[32];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    unsigned long long other = __shfl_xor_sync(0xffffffffu, best, o);
    best = other > best ? other : best;
  }
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = best;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) best = red[w] > best ? red[w] : best;
    best = red[0] > best ? red[0] : best;
    out[blockIdx.x] = (int32_t)argmax_key_index(best);
  }
}

__global__ void gather_rows_kernel(const uint8_t* __restrict__ src, uint8_t* __restrict__ dst,
                                   const int32_t* __restrict__ idx, int rows, int64_t row_bytes,
                                   int64_t sstride, int64_t dstride) {
  const int r = blockIdx.y;
  if (r >= rows) return;
  const uint8_t* s = src + (int64_t)idx[r] * sstride;
  uint8_t* d = dst + (int64_t)r * dstride;
  const bool vec = ((reinterpret_cast<uintptr_t>(s) | reinterpret_cast<uintptr_t>(d) | row_bytes) & 15) == 0;
  if (vec) {
    const int64_t n16 = row_bytes >> 4;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n16;
         i += (int64_t)gridDim.x * blockDim.x)
      reinterpret_cast<uint4*>(d)[i] = reinterpret_cast<const uint4*>(s)[i];
  } else {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < row_bytes;
         i += (int64_t)gridDim.x * blockDim.x)
      d[i] = s[i];
  }
}

__global__ void keys_to_index_kernel(const unsigned long long* keys, int rows, int32_t* out) {
  const int r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r < rows) out[r] = (int32_t)argmax_key_index(keys[r]);
}

}  // namespace

cudaError_t launch_keys_to_index(const unsigned long long* keys, int rows, int32_t* out,
                                 cudaStream_t s) {
  if (rows <= 0) return cudaSuccess;
  keys_to_index_kernel<<<(rows + 255) / 256, 256, 0, s>>>(keys, rows, out);
  return cudaGetLastError();
}

cudaError_t launch_embed(const int32_t* ids, const int32_t* pos_ids, const int32_t* pos_scalar,
                         const float* table, const float* pos_table, float scale, float* x32,
                         void* xact, int act_dtype, int n, int d, cudaStream_t s) {
  if (n <= 0) return cudaSuccess;
  if (d % 4) return cudaErrorInvalidValue;
  const int64_t total = (int64_t)n * (d / 4);
  const int threads = 256;
  const int blocks = (int)std::min<int64_t>((total + threads - 1) / threads, 148 * 32);
  if (act_dtype == kF16 || !xact)
    return launch_k(embed_kernel<__half>, dim3(blocks), dim3(threads), 0, s, ids, pos_ids,
                    pos_scalar, table, pos_table, scale, x32, (__half*)xact, n, d);
  if (act_dtype == kBF16)
    return launch_k(embed_kernel<__nv_bfloat16>, dim3(blocks), dim3(threads), 0, s, ids, pos_ids,
                    pos_scalar, table, pos_table, scale, x32, (__nv_bfloat16*)xact, n, d);
  return launch_k(embed_kernel<float>, dim3(blocks), dim3(threads), 0, s, ids, pos_ids,
                  pos_scalar, table, pos_table, scale, x32, (float*)xact, n, d);
}


cudaError_t launch_add_norm(const float* x, const float* y, const float* gain, const float* bias,
                            int l1, float* out32, void* out_act, int act_dtype, int rows, int d,
                            cudaStream_t s, const int32_t* rows_tab, const int32_t* t_ptr) {
  if (rows <= 0) return cudaSuccess;
  if (d % 4 || (rows_tab && !t_ptr)) return cudaErrorInvalidValue;
  if (act_dtype == kF16 || !out_act)
    return add_norm_dispatch<__half>(x, y, gain, bias, l1, out32, (__half*)out_act, rows, d, s,
                                     rows_tab, t_ptr);
  if (act_dtype == kBF16)
    return add_norm_dispatch<__nv_bfloat16>(x, y, gain, bias, l1, out32,
                                            (__nv_bfloat16*)out_act, rows, d, s, rows_tab, t_ptr);
  return add_norm_dispatch<float>(x, y, gain, bias, l1, out32, (float*)out_act, rows, d, s,
                                  rows_tab, t_ptr);
}

// Row map of the step kernels: out[c] = f(a[c], b[c]) over n4 float4 columns
// of two read-only table rows, one warp per row.  Each lane issues all U of
// its loads (both rows) before its first store, so a row costs one L2 round
// trip per 32 U columns instead of one per 32 (the stores may alias nothing
// the loads read, but the compiler cannot know that through plain pointers).
template <int U, typename F>
__device__ __forceinline__ void row_map4(const float* a, const float* b, int n4, int lane,
                                         F&& put) {
  const float4* a4 = reinterpret_cast<const float4*>(a);
  const float4* b4 = reinterpret_cast<const float4*>(b);
  for (int base = 0; base < n4; base += 32 * U) {
    float4 va[U], vb[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int c = base + lane + 32 * u;
      if (c < n4) {
        va[u] = __ldg(a4 + c);
        vb[u] = __ldg(b4 + c);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int c = base + lane + 32 * u;
      if (c < n4) put(4 * c, va[u], vb[u]);
    }
  }
}

constexpr int kKeyU = 9;   // w = 2 d + 8 = 1032 (d = 512): 258 float4 -> one pass
constexpr int kEmbU = 4;   // d = 512: 128 float4 -> one pass

// One warp writes row r's layer-0 self key: act(tok_tab[tok] + pos_tab[pos])
// (fp32 sum, one rounding).
template <typename TA>
__device__ __forceinline__ void step_key_row(const StepKey& k, int r, int tok, int pos, int lane) {
  if (k.kc && pos >= k.cap) return;   // no further step for this batch (cache slots end at cap)
  row_map4<kKeyU>(k.tok_tab + (size_t)tok * k.w, k.pos_tab + (size_t)pos * k.w, k.w >> 2, lane,
                  [&](int c, float4 a, float4 b) {
                    const float4 o = make_float4(a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w);
                    TA* dst;
                    if (!k.kc) {
                      dst = reinterpret_cast<TA*>(k.knew) + (size_t)r * k.w + c;
                    } else {
                      const int sec = c / k.seg;
                      c -= sec * k.seg;
                      dst = sec == 0 ? reinterpret_cast<TA*>(k.knew) + (size_t)r * k.seg + c
                                     : reinterpret_cast<TA*>(sec == 1 ? k.kc : k.vc) +
                                           ((size_t)r * k.cap + pos) * k.seg + c;
                    }
                    store4(dst, o);
                  });
}

constexpr int kStepRows = 4;   // rows (warps) per CTA of the step kernels

template <typename TA>
__global__ void __launch_bounds__(32 * kStepRows) step_key_kernel(StepKey k, const int32_t* tok,
                                                                  const int32_t* t_ptr, int rows) {
  pdl_trigger();
  pdl_wait();
  const int r = blockIdx.x * kStepRows + (threadIdx.x >> 5);
  if (r < rows) step_key_row<TA>(k, r, tok[r], *t_ptr, threadIdx.x & 31);
}

cudaError_t launch_step_key(const StepKey& k, const int32_t* tok, const int32_t* t_ptr, int rows,
                            int act_dtype, cudaStream_t s) {
  if (rows <= 0) return cudaSuccess;
  if (k.w % 4 || (k.kc && k.seg % 4)) return cudaErrorInvalidValue;
  const dim3 grid((rows + kStepRows - 1) / kStepRows), block(32 * kStepRows);
  if (act_dtype == kF16) return launch_k(step_key_kernel<__half>, grid, block, 0, s, k, tok, t_ptr, rows);
  if (act_dtype == kBF16)
    return launch_k(step_key_kernel<__nv_bfloat16>, grid, block, 0, s, k, tok, t_ptr, rows);
  return cudaErrorInvalidValue;
}

// Greedy bookkeeping fused with the next step's decoder-input embedding
// (search.py:64-85 + decode_step's embed, model.py:327-328): warp per row.
// Lane 0 applies the greedy rules of greedy_update_kernel; the warp then
// writes E[prev] * sqrt(d) + P[t + 1] (prev = the emitted token, or PAD for a
// finished row) as the next step's residual stream and activation copy.  The
// step counter is bumped by the last CTA to finish (every CTA has read t by
// then), which also publishes the alive count.  Lane 0's row state is read
// together with the step counter (it does not depend on t).
template <typename TA>
__global__ void __launch_bounds__(32 * kStepRows) greedy_embed_kernel(GreedyState g, GreedyEmbed e) {
  pdl_trigger();
  pdl_wait();
  __shared__ int alive_s;
  const int lane = threadIdx.x & 31;
  const int r = blockIdx.x * kStepRows + (threadIdx.x >> 5);
  const bool lead = r < g.rows && lane == 0;
  unsigned long long key = 0ull;
  int fin = 1, budget = 0;
  if (lead) {
    key = g.keys[r];
    fin = g.finished[r];
    budget = g.budget[r];
  }
  const int t = *g.t;
  if (threadIdx.x == 0) alive_s = 0;
  __syncthreads();
  int tok = g.pad, alive = 0;
  if (lead) {
    g.keys[r] = 0ull;
    if (!fin) {
      const int w = (int)argmax_key_index(key);
      if (w == g.eos) {
        g.finished[r] = 1;
      } else {
        if (t < g.out_cap) g.out_ids[(size_t)r * g.out_cap + t] = w;
        g.out_len[r] = t + 1;
        tok = w;
        if (t + 1 >= budget)
          g.finished[r] = 1;
        else
          alive = 1;
      }
    }
    g.prev[r] = tok;
  }
  tok = __shfl_sync(0xffffffffu, tok, 0);
  if (r < g.rows && t + 1 < e.n_pos) {
    float* x32 = e.x32 + (size_t)r * e.d;
    TA* xa = e.xa ? reinterpret_cast<TA*>(e.xa) + (size_t)r * e.d : nullptr;
    const float scale = e.scale;
    row_map4<kEmbU>(e.table + (size_t)tok * e.d, e.pos + (size_t)(t + 1) * e.d, e.d >> 2, lane,
                    [&](int c, float4 a, float4 q) {
                      float4 o;
                      o.x = __fadd_rn(__fmul_rn(a.x, scale), q.x);
                      o.y = __fadd_rn(__fmul_rn(a.y, scale), q.y);
                      o.z = __fadd_rn(__fmul_rn(a.z, scale), q.z);
                      o.w = __fadd_rn(__fmul_rn(a.w, scale), q.w);
                      store4(x32 + c, o);
                      if (xa) store4(xa + c, o);
                    });
    if constexpr (!std::is_same<TA, float>::value) {
      if (e.key.knew) step_key_row<TA>(e.key, r, tok, t + 1, lane);
    }
  }
  if (lane == 0 && alive) atomicAdd(&alive_s, 1);
  __syncthreads();
  if (threadIdx.x == 0) {
    if (alive_s) atomicAdd(e.alive_acc, alive_s);
    __threadfence();
    if (atomicAdd(e.done, 1) == (int)gridDim.x - 1) {
      __threadfence();
      *g.alive = atomicExch(e.alive_acc, 0);
      *e.done = 0;
      *g.t = t + 1;
    }
  }
}

cudaError_t launch_greedy_embed(const GreedyState& g, const GreedyEmbed& e, cudaStream_t s) {
  const dim3 grid((g.rows + kStepRows - 1) / kStepRows), block(32 * kStepRows);
  if (e.act_dtype == kF16) return launch_k(greedy_embed_kernel<__half>, grid, block, 0, s, g, e);
  if (e.act_dtype == kBF16)
    return launch_k(greedy_embed_kernel<__nv_bfloat16>, grid, block, 0, s, g, e);
  GreedyEmbed f = e;
  f.xa = nullptr;
  return launch_k(greedy_embed_kernel<float>, grid, block, 0, s, g, f);
}

cudaError_t launch_greedy_update(const GreedyState& g, cudaStream_t s) {
  return launch_k(greedy_update_kernel, dim3(1), dim3(1024), 0, s, g);
}

cudaError_t launch_argmax_rows(const float* logits, int ld, int rows, int n, int32_t* out_idx,
                               cudaStream_t s) {
  if (rows <= 0) return cudaSuccess;
  argmax_rows_kernel<<<rows, 256, 0, s>>>(logits, ld, n, out_idx);
  return cudaGetLastError();
}

cudaError_t launch_gather_rows(const void* src, void* dst, const int32_t* idx, int rows,
                               int64_t row_bytes, int64_t src_stride, int64_t dst_stride,
                               cudaStream_t s) {
  if (rows <= 0 || row_bytes <= 0) return cudaSuccess;
  const int64_t n16 = (row_bytes + 15) / 16;
  dim3 grid((unsigned)std::min<int64_t>((n16 + 255) / 256, 64), rows);
  gather_rows_kernel<<<grid, 256, 0, s>>>((const uint8_t*)src, (uint8_t*)dst, idx, rows,
                                          row_bytes, src_stride, dst_stride);
  return cudaGetLastError();
}

}  // namespace fnmt
