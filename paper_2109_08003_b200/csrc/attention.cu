// Scaled dot-product attention with padding masks (model.py:199-245).
//
// Semantics kept from the reference:
//  * the query is scaled by f32(1/sqrt(dk)) before the score product
//    (model.py:223, "exact reorder" of score scaling);
//  * softmax subtracts the row max, exponentiates, divides by the row sum
//    (tensor.py:70-81); weights are normalised before the value product;
//  * masked keys carry an additive -1e9 (model.py:37-38, :243-245).  For a
//    row with at least one real key the masked keys get exactly zero weight,
//    so they are skipped (bit-identical to adding them); a row whose keys are
//    ALL masked attends over every padded key with the -1e9 offset applied,
//    exactly like the reference.
//
// Two kernels:
//  * attention_varlen_kernel — encoder self-attention over packed varlen
//    sequences.  CTA = (16-query tile, sequence, head).  Q tile, a 32-key K/V
//    tile, the score rows and the output accumulator are staged in shared
//    memory (padded rows, conflict-free); fp32 math throughout.
//  * attention_decode_kernel — one query per row against the self-KV cache
//    (appending this step's k/v first) or the cached cross K/V.  CTA =
//    (row, head); warps stride over keys, lanes over head dims.
#include <math.h>

#include "common.cuh"
#include "kernels.h"

namespace fnmt {

namespace {

constexpr int kQT = 16;   // queries per CTA
constexpr int kKT = 32;   // keys per smem tile
constexpr int kThreads = 128;
constexpr float kMaskValue = -1e9f;

template <typename T>
__global__ void __launch_bounds__(kThreads)
    attention_varlen_kernel(AttnArgs a, float qscale, int kcap) {
  extern __shared__ float sm[];
  const int dk = a.dk;
  const int ldp = dk + 1;
  float* Qs = sm;                    // [kQT][dk+1]
  float* KV = Qs + kQT * ldp;        // [kKT][dk+1]
  float* O = KV + kKT * ldp;         // [kQT][dk]
  float* P = O + kQT * dk;           // [kQT][kcap]

  const int b = blockIdx.y, h = blockIdx.z;
  const int q0 = blockIdx.x * kQT;
  const int nq = a.q_len[b];
  if (q0 >= nq) return;
  const int kl = a.k_len[b];
  const bool all_masked = kl == 0;
  const int nk = all_masked ? a.k_pad : kl;
  const int qrow0 = a.q_start[b] + q0;
  const int krow0 = a.k_start[b];
  const int qn = min(kQT, nq - q0);
  const T* q = reinterpret_cast<const T*>(a.q);
  const T* k = reinterpret_cast<const T*>(a.k);
  const T* v = reinterpret_cast<const T*>(a.v);
  const int tid = threadIdx.x;
  const int warp = tid >> 5, lane = tid & 31;

  for (int i = tid; i < kQT * dk; i += kThreads) {
    const int qi = i / dk, e = i - qi * dk;
    float val = 0.f;
    if (qi < qn) val = to_f32(q[(size_t)(qrow0 + qi) * a.ldq + h * dk + e]) * qscale;
    Qs[qi * ldp + e] = val;
    O[i] = 0.f;
  }

  // pass 1: scores
  for (int kt = 0; kt < nk; kt += kKT) {
    const int kn = min(kKT, nk - kt);
    __syncthreads();
    for (int i = tid; i < kKT * dk; i += kThreads) {
      const int j = i / dk, e = i - j * dk;
      KV[j * ldp + e] = j < kn ? to_f32(k[(size_t)(krow0 + kt + j) * a.ldkv + h * dk + e]) : 0.f;
    }
    __syncthreads();
    for (int p = tid; p < kQT * kKT; p += kThreads) {
      const int qi = p / kKT, j = p - qi * kKT;
      if (qi < qn && j < kn) {
        const float* qr = Qs + qi * ldp;
        const float* kr = KV + j * ldp;
        float s = 0.f;
        for (int e = 0; e < dk; ++e) s = fmaf(qr[e], kr[e], s);
        if (all_masked) s = s + kMaskValue;
        P[qi * kcap + kt + j] = s;
      }
    }
  }
  __syncthreads();
  // softmax per query row (warp per row)
  for (int qi = warp; qi < qn; qi += kThreads / 32) {
    float* pr = P + qi * kcap;
    float mx = -INFINITY;
    for (int j = lane; j < nk; j += 32) mx = fmaxf(mx, pr[j]);
    mx = warp_max(mx);
    float sum = 0.f;
    for (int j = lane; j < nk; j += 32) {
      const float e = expf(pr[j] - mx);
      pr[j] = e;
      sum += e;
    }
    sum = warp_sum(sum);
    for (int j = lane; j < nk; j += 32) pr[j] = pr[j] / sum;
  }
  // pass 2: weights . V
  for (int kt = 0; kt < nk; kt += kKT) {
    const int kn = min(kKT, nk - kt);
    __syncthreads();
    for (int i = tid; i < kKT * dk; i += kThreads) {
      const int j = i / dk, e = i - j * dk;
      KV[j * ldp + e] = j < kn ? to_f32(v[(size_t)(krow0 + kt + j) * a.ldkv + h * dk + e]) : 0.f;
    }
    __syncthreads();
    for (int i = tid; i < qn * dk; i += kThreads) {
      const int qi = i / dk, e = i - qi * dk;
      const float* pr = P + qi * kcap + kt;
      float acc = O[i];
      for (int j = 0; j < kn; ++j) acc = fmaf(pr[j], KV[j * ldp + e], acc);
      O[i] = acc;
    }
  }
  __syncthreads();
  T* out = reinterpret_cast<T*>(a.out);
  for (int i = tid; i < qn * dk; i += kThreads) {
    const int qi = i / dk, e = i - qi * dk;
    out[(size_t)(qrow0 + qi) * a.ldo + h * dk + e] = from_f32<T>(O[i]);
  }
}

template <typename T>
__global__ void __launch_bounds__(kThreads)
    attention_decode_kernel(DecAttnArgs a, float qscale) {
  extern __shared__ float sm[];
  const int dk = a.dk;
  float* qs = sm;          // [dk]
  float* S = sm + dk;      // [max_k]
  const int r = blockIdx.x, h = blockIdx.y;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const T* kbase = reinterpret_cast<const T*>(a.k);
  const T* vbase = reinterpret_cast<const T*>(a.v);

  int nk;
  bool all_masked = false;
  int t = 0;
  int64_t seq_row0 = 0;
  if (a.self_mode) {
    t = *a.t_ptr;
    nk = t + 1;
    // append this step's key/value (this head's slice) at slot t
    T* kw = reinterpret_cast<T*>(a.k_w);
    T* vw = reinterpret_cast<T*>(a.v_w);
    const T* nkp = reinterpret_cast<const T*>(a.new_k) + (size_t)r * a.ld_new + h * dk;
    const T* nvp = reinterpret_cast<const T*>(a.new_v) + (size_t)r * a.ld_new + h * dk;
    const size_t slot = ((size_t)r * a.cap + t) * a.ldkv + h * dk;
    for (int e = tid; e < dk; e += kThreads) {
      kw[slot + e] = nkp[e];
      vw[slot + e] = nvp[e];
    }
  } else {
    const int seq = r / a.rows_per_seq;
    const int kl = a.k_len[seq];
    all_masked = kl == 0;
    nk = all_masked ? a.k_pad : kl;
    seq_row0 = a.k_start[seq];
  }
  const T* q = reinterpret_cast<const T*>(a.q) + (size_t)r * a.ldq + h * dk;
  for (int e = tid; e < dk; e += kThreads) qs[e] = to_f32(q[e]) * qscale;
  __syncthreads();

  auto key_row = [&](int j) -> int64_t {
    if (a.self_mode) {
      const int src = (a.anc && j < t) ? a.anc[(size_t)r * a.cap + j] : r;
      return (int64_t)src * a.cap + j;
    }
    return seq_row0 + j;
  };

  for (int j = warp; j < nk; j += kThreads / 32) {
    const T* kr = kbase + key_row(j) * a.ldkv + h * dk;
    float s = 0.f;
    for (int e = lane; e < dk; e += 32) s = fmaf(qs[e], to_f32(kr[e]), s);
    s = warp_sum(s);
    if (lane == 0) S[j] = all_masked ? s + kMaskValue : s;
  }
  __syncthreads();
  if (warp == 0) {
    float mx = -INFINITY;
    for (int j = lane; j < nk; j += 32) mx = fmaxf(mx, S[j]);
    mx = warp_max(mx);
    float sum = 0.f;
    for (int j = lane; j < nk; j += 32) {
      const float e = expf(S[j] - mx);
      S[j] = e;
      sum += e;
    }
    sum = warp_sum(sum);
    for (int j = lane; j < nk; j += 32) S[j] = S[j] / sum;
  }
  __syncthreads();
  T* out = reinterpret_cast<T*>(a.out) + (size_t)r * a.ldo + h * dk;
  for (int e = tid; e < dk; e += kThreads) {
    float acc = 0.f;
    for (int j = 0; j < nk; ++j) acc = fmaf(S[j], to_f32(vbase[key_row(j) * a.ldkv + h * dk + e]), acc);
    out[e] = from_f32<T>(acc);
  }
}

template <typename T>
cudaError_t varlen_dispatch(const AttnArgs& a, cudaStream_t s) {
  const int kcap = ((a.max_k + 31) / 32) * 32;
  const size_t smem = sizeof(float) * ((size_t)kQT * (a.dk + 1) + (size_t)kKT * (a.dk + 1) +
                                       (size_t)kQT * a.dk + (size_t)kQT * kcap);
  if (smem > 227 * 1024) return cudaErrorInvalidValue;
  cudaError_t e = cudaFuncSetAttribute(attention_varlen_kernel<T>,
                                       cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  if (e != cudaSuccess) return e;
  dim3 grid((a.max_q + kQT - 1) / kQT, a.n_seq, a.heads);
  const float qscale = (float)(1.0 / sqrt((double)a.dk));
  attention_varlen_kernel<T><<<grid, kThreads, smem, s>>>(a, qscale, kcap);
  return cudaGetLastError();
}

template <typename T>
cudaError_t decode_dispatch(const DecAttnArgs& a, cudaStream_t s) {
  const size_t smem = sizeof(float) * ((size_t)a.dk + (size_t)a.max_k + 32);
  if (smem > 227 * 1024) return cudaErrorInvalidValue;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(attention_decode_kernel<T>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return e;
  }
  dim3 grid(a.rows, a.heads);
  const float qscale = (float)(1.0 / sqrt((double)a.dk));
  attention_decode_kernel<T><<<grid, kThreads, smem, s>>>(a, qscale);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_attention_varlen(const AttnArgs& a, cudaStream_t s) {
  if (a.n_seq <= 0 || a.max_q <= 0) return cudaSuccess;
  switch (a.dtype) {
    case kF32: return varlen_dispatch<float>(a, s);
    case kF16: return varlen_dispatch<__half>(a, s);
    case kBF16: return varlen_dispatch<__nv_bfloat16>(a, s);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_attention_decode(const DecAttnArgs& a, cudaStream_t s) {
  if (a.rows <= 0) return cudaSuccess;
  switch (a.dtype) {
    case kF32: return decode_dispatch<float>(a, s);
    case kF16: return decode_dispatch<__half>(a, s);
    case kBF16: return decode_dispatch<__nv_bfloat16>(a, s);
  }
  return cudaErrorInvalidValue;
}

}  // namespace fnmt
