// Scaled dot-product attention with padding masks (model.py:199-245).
//
// Semantics kept from the reference:
//  * the query is scaled by f32(1/sqrt(dk)) before the score product
//    (model.py:223, the "exact reorder" of score scaling);
//  * softmax subtracts the row max, exponentiates, divides by the row sum
//    (tensor.py:70-81); weights are normalised before the value product;
//  * masked keys carry an additive -1e9 (model.py:37-38, :243-245).  For a
//    row with at least one real key the masked keys get exactly zero weight,
//    so they are skipped (bit-identical to adding them); a row whose keys are
//    ALL masked attends over every padded key with the -1e9 offset applied,
//    exactly like the reference.
//
// Kernels (fp32 math everywhere, storage T = f32 / f16 / bf16):
//  * attn_varlen_kernel — encoder self-attention over packed varlen
//    sequences.  CTA = (32-query tile, sequence, head), 256 threads.  Both
//    contractions are register-tiled mini-GEMMs through shared memory:
//    scores = Q K^T in (32 q x 64 k) tiles over 32-dim chunks (2x4 outputs
//    per thread), the full score rows stay in shared memory for the
//    softmax, then O = P V in (32 q x 64 d) tiles over 32-key chunks.
//  * attn_decode_kernel — one query per row against the self-KV cache
//    (appending this step's k/v first) or the cached cross K/V.  CTA =
//    (row, head), 128 threads; G lanes per key with 16-byte vector loads,
//    32/G keys per warp in flight; value product split over key groups and
//    reduced in a fixed order (deterministic).
//  * attn_decode_generic — scalar fallback for head sizes that are not a
//    multiple of one 16-byte vector (tiny test models).
#include <math.h>

#include <type_traits>

#include "common.cuh"
#include "kernels.h"

namespace fnmt {

namespace {

constexpr float kMaskValue = -1e9f;

template <typename T>
struct Vec16 {
  static constexpr int N = 16 / sizeof(T);
};

__device__ __forceinline__ void load16(const float* p, float (&f)[4]) {
  const float4 v = *reinterpret_cast<const float4*>(p);
  f[0] = v.x; f[1] = v.y; f[2] = v.z; f[3] = v.w;
}
__device__ __forceinline__ void load16(const __half* p, float (&f)[8]) {
  const uint4 u = *reinterpret_cast<const uint4*>(p);
  const __half2* h = reinterpret_cast<const __half2*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 x = __half22float2(h[i]);
    f[2 * i] = x.x;
    f[2 * i + 1] = x.y;
  }
}
__device__ __forceinline__ void load16(const __nv_bfloat16* p, float (&f)[8]) {
  const uint4 u = *reinterpret_cast<const uint4*>(p);
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 x = __bfloat1622float2(h[i]);
    f[2 * i] = x.x;
    f[2 * i + 1] = x.y;
  }
}

// ---------------------------------------------------------------------------
// encoder varlen attention

constexpr int kQT = 32;   // queries per CTA
constexpr int kKT = 64;   // keys per score tile
constexpr int kDC = 32;   // head dims per score-chunk
constexpr int kPK = 32;   // keys per value-chunk
constexpr int kPD = 64;   // head dims per output tile
constexpr int kVThreads = 256;

template <typename T>
__global__ void __launch_bounds__(kVThreads)
    attn_varlen_kernel(AttnArgs a, float qscale, int kcap) {
  extern __shared__ float sm[];
  float* S = sm;                               // [kQT][kcap]
  float* Qs = S + kQT * kcap;                  // [kDC][kQT + 4]   dim-major
  float* Ks = Qs + kDC * (kQT + 4);            // [kDC][kKT + 4]   dim-major  (also V tile)
  const int dk = a.dk;
  const int b = blockIdx.y, h = blockIdx.z;
  const int q0 = blockIdx.x * kQT;
  const int nq = a.q_len[b];
  if (q0 >= nq) return;
  const int kl = a.k_len[b];
  const bool all_masked = kl == 0;
  const int nk = all_masked ? a.k_pad : kl;
  const int qn = min(kQT, nq - q0);
  const int64_t qrow0 = a.q_start[b] + q0;
  const int64_t krow0 = a.k_start[b];
  const T* q = reinterpret_cast<const T*>(a.q) + h * dk;
  const T* k = reinterpret_cast<const T*>(a.k) + h * dk;
  const T* v = reinterpret_cast<const T*>(a.v) + h * dk;
  const int tid = threadIdx.x;
  const int tq = tid >> 4;   // 0..15 -> query rows 2*tq, 2*tq+1
  const int tc = tid & 15;   // 0..15 -> columns 4*tc .. 4*tc+3

  // ---- scores S = (q * scale) K^T --------------------------------------------
  for (int k0 = 0; k0 < nk; k0 += kKT) {
    float acc[2][4] = {};
    for (int d0 = 0; d0 < dk; d0 += kDC) {
      __syncthreads();
      for (int i = tid; i < kQT * kDC; i += kVThreads) {
        const int qi = i / kDC, dd = i % kDC;
        float val = 0.f;
        if (qi < qn && d0 + dd < dk) val = to_f32(q[(qrow0 + qi) * a.ldq + d0 + dd]) * qscale;
        Qs[dd * (kQT + 4) + qi] = val;
      }
      for (int i = tid; i < kKT * kDC; i += kVThreads) {
        const int kj = i / kDC, dd = i % kDC;
        float val = 0.f;
        if (k0 + kj < nk && d0 + dd < dk) val = to_f32(k[(krow0 + k0 + kj) * a.ldkv + d0 + dd]);
        Ks[dd * (kKT + 4) + kj] = val;
      }
      __syncthreads();
#pragma unroll 8
      for (int dd = 0; dd < kDC; ++dd) {
        const float2 qv = *reinterpret_cast<const float2*>(Qs + dd * (kQT + 4) + 2 * tq);
        const float4 kv = *reinterpret_cast<const float4*>(Ks + dd * (kKT + 4) + 4 * tc);
        acc[0][0] = fmaf(qv.x, kv.x, acc[0][0]);
        acc[0][1] = fmaf(qv.x, kv.y, acc[0][1]);
        acc[0][2] = fmaf(qv.x, kv.z, acc[0][2]);
        acc[0][3] = fmaf(qv.x, kv.w, acc[0][3]);
        acc[1][0] = fmaf(qv.y, kv.x, acc[1][0]);
        acc[1][1] = fmaf(qv.y, kv.y, acc[1][1]);
        acc[1][2] = fmaf(qv.y, kv.z, acc[1][2]);
        acc[1][3] = fmaf(qv.y, kv.w, acc[1][3]);
      }
    }
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int qi = 2 * tq + i, kj = k0 + 4 * tc + j;
        if (qi < qn && kj < nk) S[qi * kcap + kj] = all_masked ? acc[i][j] + kMaskValue : acc[i][j];
      }
  }
  __syncthreads();

  // ---- softmax per query row (warp per row) ----------------------------------
  const int warp = tid >> 5, lane = tid & 31;
  for (int qi = warp; qi < qn; qi += kVThreads / 32) {
    float* pr = S + qi * kcap;
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

  // ---- O = P V ------------------------------------------------------------------
  float* Vs = Ks;   // [kPK][kPD + 4]  key-major
  T* out = reinterpret_cast<T*>(a.out) + h * dk;
  for (int d0 = 0; d0 < dk; d0 += kPD) {
    float acc[2][4] = {};
    for (int j0 = 0; j0 < nk; j0 += kPK) {
      const int jn = min(kPK, nk - j0);
      __syncthreads();
      for (int i = tid; i < kPK * kPD; i += kVThreads) {
        const int kj = i / kPD, dd = i % kPD;
        float val = 0.f;
        if (kj < jn && d0 + dd < dk) val = to_f32(v[(krow0 + j0 + kj) * a.ldkv + d0 + dd]);
        Vs[kj * (kPD + 4) + dd] = val;
      }
      __syncthreads();
      const float* p0 = S + (2 * tq) * kcap + j0;
      const float* p1 = p0 + kcap;
      for (int kj = 0; kj < jn; ++kj) {
        const float w0 = p0[kj], w1 = p1[kj];
        const float4 vv = *reinterpret_cast<const float4*>(Vs + kj * (kPD + 4) + 4 * tc);
        acc[0][0] = fmaf(w0, vv.x, acc[0][0]);
        acc[0][1] = fmaf(w0, vv.y, acc[0][1]);
        acc[0][2] = fmaf(w0, vv.z, acc[0][2]);
        acc[0][3] = fmaf(w0, vv.w, acc[0][3]);
        acc[1][0] = fmaf(w1, vv.x, acc[1][0]);
        acc[1][1] = fmaf(w1, vv.y, acc[1][1]);
        acc[1][2] = fmaf(w1, vv.z, acc[1][2]);
        acc[1][3] = fmaf(w1, vv.w, acc[1][3]);
      }
    }
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int qi = 2 * tq + i, dd = d0 + 4 * tc + j;
        if (qi < qn && dd < dk) out[(qrow0 + qi) * a.ldo + dd] = from_f32<T>(acc[i][j]);
      }
  }
}

// ---------------------------------------------------------------------------
// decode attention (one query per row)

constexpr int kDThreads = 128;

struct DecCtx {
  int nk;
  bool all_masked;
  int t;
  int64_t seq_row0;
};

template <typename T>
__device__ __forceinline__ DecCtx decode_setup(const DecAttnArgs& a, int r, int h) {
  DecCtx c{};
  if (a.self_mode) {
    c.t = *a.t_ptr;
    c.nk = c.t + 1;
    if (a.new_k) {   // append this step's k/v (unless the QKV GEMM epilogue already did)
      T* kw = reinterpret_cast<T*>(a.k_w);
      T* vw = reinterpret_cast<T*>(a.v_w);
      const T* nkp = reinterpret_cast<const T*>(a.new_k) + (size_t)r * a.ld_new + h * a.dk;
      const T* nvp = reinterpret_cast<const T*>(a.new_v) + (size_t)r * a.ld_new + h * a.dk;
      const size_t slot = ((size_t)r * a.cap + c.t) * a.ldkv + h * a.dk;
      for (int e = threadIdx.x; e < a.dk; e += blockDim.x) {
        kw[slot + e] = nkp[e];
        vw[slot + e] = nvp[e];
      }
    }
  } else {
    const int seq = r / a.rows_per_seq;
    const int kl = a.k_len[seq];
    c.all_masked = kl == 0;
    c.nk = c.all_masked ? a.k_pad : kl;
    c.seq_row0 = a.k_start[seq];
  }
  return c;
}

__device__ __forceinline__ int64_t decode_key_row(const DecAttnArgs& a, const DecCtx& c, int r,
                                                  int j) {
  if (a.self_mode) {
    // beam: key j of row r was written by cache row anc_t[r][j] (table for step parity t & 1)
    const int src = (a.anc && j < c.t)
                        ? a.anc[(size_t)(c.t & 1) * a.anc_buf_stride + (size_t)r * a.cap + j]
                        : r;
    return (int64_t)src * a.cap + j;
  }
  return c.seq_row0 + j;
}

__device__ __forceinline__ void softmax_inplace(float* S, int nk) {
  const int lane = threadIdx.x & 31;
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

// G lanes cooperate on one key (CH 16-byte chunks each); 32/G keys per warp.
// NT threads per (row, head): 128 normally, 512 when there are too few rows
// to fill the machine (long-sentence batches).
template <typename T>
__device__ __forceinline__ void cvt16(const uint4& u, float (&f)[Vec16<T>::N]);
template <>
__device__ __forceinline__ void cvt16<float>(const uint4& u, float (&f)[4]) {
  f[0] = __uint_as_float(u.x); f[1] = __uint_as_float(u.y);
  f[2] = __uint_as_float(u.z); f[3] = __uint_as_float(u.w);
}
template <>
__device__ __forceinline__ void cvt16<__half>(const uint4& u, float (&f)[8]) {
  const __half2* h = reinterpret_cast<const __half2*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 x = __half22float2(h[i]);
    f[2 * i] = x.x;
    f[2 * i + 1] = x.y;
  }
}
template <>
__device__ __forceinline__ void cvt16<__nv_bfloat16>(const uint4& u, float (&f)[8]) {
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 x = __bfloat1622float2(h[i]);
    f[2 * i] = x.x;
    f[2 * i + 1] = x.y;
  }
}

// U: score rounds in flight per warp (U * KPW keys, U * CH raw 16-byte
// vectors per lane); UV: value rows in flight per thread.  Loads land in raw
// uint4 registers and are widened to fp32 only at the FMA, so deeper unrolls
// cost 4 registers per vector instead of 8 floats.
template <typename T, int G, int CH, int NT, int U = 1, int UV = 1>
__global__ void __launch_bounds__(NT) attn_decode_kernel(DecAttnArgs a, float qscale) {
  pdl_trigger();
  pdl_wait();
  if (a.row_done && a.row_done[blockIdx.x]) return;   // finished sentence (search.py:72)
  constexpr int VEC = Vec16<T>::N;
  extern __shared__ float sm[];
  const int dk = a.dk;
  float* qs = sm;                  // [dk]
  float* S = qs + dk;              // [max_k]
  float* red = S + a.max_k + 4;    // [groups][dk]
  const int r = blockIdx.x, h = blockIdx.y;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const DecCtx c = decode_setup<T>(a, r, h);
  const T* q = reinterpret_cast<const T*>(a.q) + (size_t)r * a.ldq + h * dk;
  for (int e = tid; e < dk; e += NT) qs[e] = to_f32(q[e]) * qscale;
  __syncthreads();

  const T* kb = reinterpret_cast<const T*>(a.k) + h * dk;
  constexpr int KPW = 32 / G;            // keys per warp per round (lane groups)
  const int g = lane / G, li = lane % G;
  const int stride = (NT / 32) * KPW;
  for (int j0 = warp * KPW; j0 < c.nk; j0 += stride * U) {
    uint4 raw[U][CH];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int j = j0 + u * stride + g;
      if (j < c.nk) {
        const T* kr = kb + decode_key_row(a, c, r, j) * a.ldkv;
#pragma unroll
        for (int ch = 0; ch < CH; ++ch) {
          const int e0 = (li + ch * G) * VEC;
          if (e0 < dk) raw[u][ch] = *reinterpret_cast<const uint4*>(kr + e0);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int j = j0 + u * stride + g;
      float s = 0.f;
      if (j < c.nk) {
#pragma unroll
        for (int ch = 0; ch < CH; ++ch) {
          const int e0 = (li + ch * G) * VEC;
          if (e0 < dk) {
            float f[VEC];
            cvt16<T>(raw[u][ch], f);
#pragma unroll
            for (int i = 0; i < VEC; ++i) s = fmaf(qs[e0 + i], f[i], s);
          }
        }
      }
#pragma unroll
      for (int o = G / 2; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (li == 0 && j < c.nk) {
        if (a.kc_off >= 0)   // folded cross attention: + qscale * (b_q . k_j)
          s += qscale * to_f32(kb[decode_key_row(a, c, r, j) * a.ldkv + a.kc_off - h * dk]);
        S[j] = c.all_masked ? s + kMaskValue : s;
      }
    }
  }
  __syncthreads();
  if (warp == 0) softmax_inplace(S, c.nk);
  __syncthreads();

  // value product: thread = (chunk, key group); keys in a fixed order per group
  const int nch = dk / VEC;
  const int groups = NT / nch;
  const int ch = tid % nch, grp = tid / nch;
  const T* vb = reinterpret_cast<const T*>(a.v) + h * dk + ch * VEC;
  float acc[VEC];
#pragma unroll
  for (int i = 0; i < VEC; ++i) acc[i] = 0.f;
  if (grp < groups) {
    for (int j0 = grp; j0 < c.nk; j0 += groups * UV) {
      uint4 rv[UV];
#pragma unroll
      for (int u = 0; u < UV; ++u) {
        const int j = j0 + u * groups;
        if (j < c.nk) rv[u] = *reinterpret_cast<const uint4*>(vb + decode_key_row(a, c, r, j) * a.ldkv);
      }
#pragma unroll
      for (int u = 0; u < UV; ++u) {
        const int j = j0 + u * groups;
        if (j < c.nk) {
          const float w = S[j];
          float f[VEC];
          cvt16<T>(rv[u], f);
#pragma unroll
          for (int i = 0; i < VEC; ++i) acc[i] = fmaf(w, f[i], acc[i]);
        }
      }
    }
#pragma unroll
    for (int i = 0; i < VEC; ++i) red[grp * dk + ch * VEC + i] = acc[i];
  }
  __syncthreads();
  if (a.out_f32) {   // folded cross attention: o-projection output in fp32 (+ its bias)
    float* out = reinterpret_cast<float*>(a.out) + (size_t)r * a.ldo + h * dk;
    for (int e = tid; e < dk; e += NT) {
      float sum = red[e];
      for (int gg = 1; gg < groups; ++gg) sum += red[gg * dk + e];
      out[e] = a.out_bias ? sum + a.out_bias[h * dk + e] : sum;
    }
    return;
  }
  T* out = reinterpret_cast<T*>(a.out) + (size_t)r * a.ldo + h * dk;
  for (int e = tid; e < dk; e += NT) {
    float sum = red[e];
    for (int gg = 1; gg < groups; ++gg) sum += red[gg * dk + e];
    out[e] = from_f32<T>(sum);
  }
}


// Multi-head decode attention, one CTA per ROW covering all H heads.  A key
// row of all heads is d contiguous elements (H x dk), so a warp streams it
// exactly like the single-head dk = d case (G = 32 lanes, CH 16-byte chunks per
// lane); lane li's chunk ch belongs to head (li + 32 ch) / LPH, LPH = dk / VEC
// lanes per head, and the score of each head is a shuffle reduction inside its
// LPH-lane group.  The value pass weights chunk c with its own head's softmax
// row.  Versus a CTA per (row, head) this loads 8x fewer, 8x larger key
// vectors per CTA and runs 8x fewer CTAs.  Same two-pass numerics as
// attn_decode_kernel.
template <typename T, int CH, int NT, int LPH, int U = 2, int UV = 4>
__global__ void __launch_bounds__(NT) attn_decode_rows_kernel(DecAttnArgs a, float qscale) {
  pdl_trigger();
  pdl_wait();
  if (a.row_done && a.row_done[blockIdx.x]) return;   // finished sentence (search.py:72)
  constexpr int VEC = Vec16<T>::N;
  // LPH 8 / 16 / 32: head score = shuffle reduction inside the head's lane
  // group.  LPH 0 (head sizes that do not map to a power-of-two lane group,
  // e.g. dk 96): per-chunk partials go through shared memory and lane h sums
  // head h's chunks in order.
  static_assert(LPH == 0 || LPH == 8 || LPH == 16 || LPH == 32, "lanes per head");
  constexpr int NW = NT / 32;
  extern __shared__ float sm[];
  const int H = a.heads, dk = a.dk, d = H * dk;
  float* qs = sm;                  // [d]
  float* S = qs + d;               // [H][max_k]
  float* red = S + (size_t)H * a.max_k + 4;   // [groups][d]
  const int groups_v = NT / (d / VEC);
  float* part = red + (size_t)groups_v * d;    // LPH 0: [NW][U][32 CH]
  const int r = blockIdx.x;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  DecCtx c = decode_setup<T>(a, r, 0);
  for (int hh = 1; hh < H && a.self_mode && a.new_k; ++hh) c = decode_setup<T>(a, r, hh);  // append all heads
  const T* q = reinterpret_cast<const T*>(a.q) + (size_t)r * a.ldq;
  for (int e = tid; e < d; e += NT) qs[e] = to_f32(q[e]) * qscale;
  __syncthreads();

  const T* kb = reinterpret_cast<const T*>(a.k);
  for (int j0 = warp; j0 < c.nk; j0 += NW * U) {
    uint4 raw[U][CH];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int j = j0 + u * NW;
      if (j < c.nk) {
        const T* kr = kb + decode_key_row(a, c, r, j) * a.ldkv;
#pragma unroll
        for (int ch = 0; ch < CH; ++ch) {
          const int e0 = (lane + ch * 32) * VEC;
          if (e0 < d) raw[u][ch] = *reinterpret_cast<const uint4*>(kr + e0);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int j = j0 + u * NW;
#pragma unroll
      for (int ch = 0; ch < CH; ++ch) {
        const int e0 = (lane + ch * 32) * VEC;
        float sacc = 0.f;
        if (j < c.nk && e0 < d) {
          float f[VEC];
          cvt16<T>(raw[u][ch], f);
#pragma unroll
          for (int i = 0; i < VEC; ++i) sacc = fmaf(qs[e0 + i], f[i], sacc);
        }
        if constexpr (LPH > 0) {
#pragma unroll
          for (int o = LPH / 2; o > 0; o >>= 1) sacc += __shfl_xor_sync(0xffffffffu, sacc, o);
          if ((lane % LPH) == 0 && j < c.nk && e0 < d) {
            const int hh = e0 / dk;
            S[(size_t)hh * a.max_k + j] = c.all_masked ? sacc + kMaskValue : sacc;
          }
        } else {
          part[(warp * U + u) * 32 * CH + lane + ch * 32] = sacc;
        }
      }
    }
    if constexpr (LPH == 0) {
      __syncwarp();
      const int lpc = dk / VEC;   // chunks per head
      if (lane < H) {
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int j = j0 + u * NW;
          if (j < c.nk) {
            const float* pp = part + (warp * U + u) * 32 * CH + lane * lpc;
            float sacc = 0.f;
            for (int i = 0; i < lpc; ++i) sacc += pp[i];
            S[(size_t)lane * a.max_k + j] = c.all_masked ? sacc + kMaskValue : sacc;
          }
        }
      }
      __syncwarp();
    }
  }
  __syncthreads();
  for (int hh = warp; hh < H; hh += NW) softmax_inplace(S + (size_t)hh * a.max_k, c.nk);
  __syncthreads();

  const int nch = d / VEC;
  const int groups = NT / nch;
  const int chn = tid % nch, grp = tid / nch;
  const T* vb = reinterpret_cast<const T*>(a.v) + chn * VEC;
  const float* Sh = S + (size_t)((chn * VEC) / dk) * a.max_k;
  float acc[VEC];
#pragma unroll
  for (int i = 0; i < VEC; ++i) acc[i] = 0.f;
  if (grp < groups) {
    for (int j0 = grp; j0 < c.nk; j0 += groups * UV) {
      uint4 rv[UV];
#pragma unroll
      for (int u = 0; u < UV; ++u) {
        const int j = j0 + u * groups;
        if (j < c.nk) rv[u] = *reinterpret_cast<const uint4*>(vb + decode_key_row(a, c, r, j) * a.ldkv);
      }
#pragma unroll
      for (int u = 0; u < UV; ++u) {
        const int j = j0 + u * groups;
        if (j < c.nk) {
          const float w = Sh[j];
          float f[VEC];
          cvt16<T>(rv[u], f);
#pragma unroll
          for (int i = 0; i < VEC; ++i) acc[i] = fmaf(w, f[i], acc[i]);
        }
      }
    }
#pragma unroll
    for (int i = 0; i < VEC; ++i) red[grp * d + chn * VEC + i] = acc[i];
  }
  __syncthreads();
  T* out = reinterpret_cast<T*>(a.out) + (size_t)r * a.ldo;
  for (int e = tid; e < d; e += NT) {
    float sum = red[e];
    for (int gg = 1; gg < groups; ++gg) sum += red[gg * d + e];
    out[e] = from_f32<T>(sum);
  }
}

__device__ __forceinline__ void cp_async16(void* smem_dst, const void* gmem_src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(smem_dst)),
               "l"(gmem_src)
               : "memory");
}
__device__ __forceinline__ void cp_async_wait_all() {
  asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
}
template <typename T>
__device__ __forceinline__ void smem16(const T* p, float (&f)[Vec16<T>::N]) {
  load16(p, f);
}

// Same contract as attn_decode_kernel, latency-hiding version: every lane
// stages its 16-byte chunks of U keys with cp.async into a private smem slot
// (no register cost, U x more bytes in flight), waits once, then computes.
// Both passes (q.K scores, then weights.V) walk keys warp-cooperatively:
// G lanes per key, 32/G keys per warp round.
template <typename T, int G, int CH, int NT>
__global__ void __launch_bounds__(NT) attn_decode_async_kernel(DecAttnArgs a, float qscale) {
  pdl_trigger();
  pdl_wait();
  constexpr int VEC = Vec16<T>::N;
  constexpr int U = 8;                       // warp rounds staged per batch
  constexpr int KPW = 32 / G;
  constexpr int NW = NT / 32;
  extern __shared__ __align__(16) uint8_t smem_a[];
  const int dk = a.dk;
  // per-lane staging: [warp][U][lane][CH] x 16 B
  uint8_t* stage = smem_a;
  float* qs = reinterpret_cast<float*>(smem_a + (size_t)NW * U * 32 * CH * 16);
  float* S = qs + dk;
  float* red = S + a.max_k + 4;              // [NW][dk]
  const int r = blockIdx.x, h = blockIdx.y;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const DecCtx c = decode_setup<T>(a, r, h);
  const T* q = reinterpret_cast<const T*>(a.q) + (size_t)r * a.ldq + h * dk;
  for (int e = tid; e < dk; e += NT) qs[e] = to_f32(q[e]) * qscale;
  __syncthreads();

  const int g = lane / G, li = lane % G;
  uint8_t* my = stage + (((size_t)warp * U) * 32 + lane) * CH * 16;   // + u * 32 * CH * 16
  const T* kb = reinterpret_cast<const T*>(a.k) + h * dk;
  const T* vb = reinterpret_cast<const T*>(a.v) + h * dk;
  const int round = NW * KPW;                // keys per CTA round
  // ---- pass 1: scores ----------------------------------------------------------
  for (int j0 = warp * KPW; j0 < c.nk; j0 += round * U) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int j = j0 + u * round + g;
      if (j < c.nk) {
        const T* kr = kb + decode_key_row(a, c, r, j) * a.ldkv;
#pragma unroll
        for (int ch = 0; ch < CH; ++ch) {
          const int e0 = (li + ch * G) * VEC;
          if (e0 < dk) cp_async16(my + ((size_t)u * 32 * CH + ch) * 16, kr + e0);
        }
      }
    }
    cp_async_wait_all();
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int j = j0 + u * round + g;
      float s = 0.f;
      if (j < c.nk) {
#pragma unroll
        for (int ch = 0; ch < CH; ++ch) {
          const int e0 = (li + ch * G) * VEC;
          if (e0 < dk) {
            float f[VEC];
            smem16(reinterpret_cast<const T*>(my + ((size_t)u * 32 * CH + ch) * 16), f);
#pragma unroll
            for (int i = 0; i < VEC; ++i) s = fmaf(qs[e0 + i], f[i], s);
          }
        }
      }
#pragma unroll
      for (int o = G / 2; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
      if (li == 0 && j < c.nk) S[j] = c.all_masked ? s + kMaskValue : s;
    }
  }
  __syncthreads();
  if (warp == 0) softmax_inplace(S, c.nk);
  __syncthreads();
  // ---- pass 2: weights . V (lane owns chunks li + ch*G of its key group) ----------
  float acc[CH][VEC];
#pragma unroll
  for (int ch = 0; ch < CH; ++ch)
#pragma unroll
    for (int i = 0; i < VEC; ++i) acc[ch][i] = 0.f;
  for (int j0 = warp * KPW; j0 < c.nk; j0 += round * U) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int j = j0 + u * round + g;
      if (j < c.nk) {
        const T* vr = vb + decode_key_row(a, c, r, j) * a.ldkv;
#pragma unroll
        for (int ch = 0; ch < CH; ++ch) {
          const int e0 = (li + ch * G) * VEC;
          if (e0 < dk) cp_async16(my + ((size_t)u * 32 * CH + ch) * 16, vr + e0);
        }
      }
    }
    cp_async_wait_all();
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int j = j0 + u * round + g;
      if (j < c.nk) {
        const float w = S[j];
#pragma unroll
        for (int ch = 0; ch < CH; ++ch) {
          const int e0 = (li + ch * G) * VEC;
          if (e0 < dk) {
            float f[VEC];
            smem16(reinterpret_cast<const T*>(my + ((size_t)u * 32 * CH + ch) * 16), f);
#pragma unroll
            for (int i = 0; i < VEC; ++i) acc[ch][i] = fmaf(w, f[i], acc[ch][i]);
          }
        }
      }
    }
  }
  // reduce over the KPW key groups of the warp (fixed xor order), then over warps
#pragma unroll
  for (int ch = 0; ch < CH; ++ch)
#pragma unroll
    for (int i = 0; i < VEC; ++i)
#pragma unroll
      for (int o = G; o < 32; o <<= 1) acc[ch][i] += __shfl_xor_sync(0xffffffffu, acc[ch][i], o);
  if (g == 0) {
#pragma unroll
    for (int ch = 0; ch < CH; ++ch) {
      const int e0 = (li + ch * G) * VEC;
      if (e0 < dk)
#pragma unroll
        for (int i = 0; i < VEC; ++i) red[warp * dk + e0 + i] = acc[ch][i];
    }
  }
  __syncthreads();
  T* out = reinterpret_cast<T*>(a.out) + (size_t)r * a.ldo + h * dk;
  for (int e = tid; e < dk; e += NT) {
    float sum = red[e];
    for (int w = 1; w < NW; ++w) sum += red[w * dk + e];
    out[e] = from_f32<T>(sum);
  }
}

template <typename T>
__global__ void __launch_bounds__(kDThreads) attn_decode_generic(DecAttnArgs a, float qscale) {
  extern __shared__ float sm[];
  const int dk = a.dk;
  float* qs = sm;
  float* S = sm + dk;
  const int r = blockIdx.x, h = blockIdx.y;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const DecCtx c = decode_setup<T>(a, r, h);
  const T* q = reinterpret_cast<const T*>(a.q) + (size_t)r * a.ldq + h * dk;
  for (int e = tid; e < dk; e += kDThreads) qs[e] = to_f32(q[e]) * qscale;
  __syncthreads();
  const T* kb = reinterpret_cast<const T*>(a.k) + h * dk;
  const T* vb = reinterpret_cast<const T*>(a.v) + h * dk;
  for (int j = warp; j < c.nk; j += kDThreads / 32) {
    const T* kr = kb + decode_key_row(a, c, r, j) * a.ldkv;
    float s = 0.f;
    for (int e = lane; e < dk; e += 32) s = fmaf(qs[e], to_f32(kr[e]), s);
    s = warp_sum(s);
    if (lane == 0) S[j] = c.all_masked ? s + kMaskValue : s;
  }
  __syncthreads();
  if (warp == 0) softmax_inplace(S, c.nk);
  __syncthreads();
  T* out = reinterpret_cast<T*>(a.out) + (size_t)r * a.ldo + h * dk;
  for (int e = tid; e < dk; e += kDThreads) {
    float acc = 0.f;
    for (int j = 0; j < c.nk; ++j) acc = fmaf(S[j], to_f32(vb[decode_key_row(a, c, r, j) * a.ldkv + e]), acc);
    out[e] = from_f32<T>(acc);
  }
}

// ---------------------------------------------------------------------------
// Bulk-copy decode attention (single head, 16-bit K/V, no ancestor table).
//
// One CTA per query row.  A row's keys are contiguous in HBM — self K / V at
// cache rows r*cap + j (d elements each), cross keys at k_start[seq] + j in
// the interleaved [K | V (| c)] rows of the cross cache — so thread 0 moves a
// chunk of CH keys with one or two cp.async.bulk copies (TMA engine, no
// registers, no per-lane address math) into a double-buffered smem ring and
// the next chunk is already in flight while this one is consumed.  Per chunk:
// warp-per-key scores from shared memory (each lane holds its 16-byte slices
// of the scaled query in registers), then every thread accumulates its CPT
// output columns over the chunk's keys with an online softmax (running max m,
// running sum l; a row that fits in one chunk is exactly
// sum_j exp(s_j - max) v_j / sum_j exp(s_j - max), the reference's
// max-shifted softmax, tensor.py:70-81).  Rows of finished sentences exit at
// once (search.py:72: their outputs are discarded).
template <typename T, int NT, int CPT>
__global__ void __launch_bounds__(NT) attn_dec_bulk_kernel(DecAttnArgs a, float qscale, int CH,
                                                           int voff, uint32_t buf_bytes) {
  pdl_trigger();
  pdl_wait();
  const int r = blockIdx.x;
  if (a.row_done && a.row_done[r]) return;
  constexpr int VEC = 8;                      // 16-bit elements per 16-byte vector
  constexpr int NW = NT / 32;
  constexpr int D = NT * CPT;                 // row width (single head: dk == d)
  constexpr int NVL = (D / VEC + 31) / 32;    // 16-byte vectors per lane in a key row
  extern __shared__ __align__(128) uint8_t smem_b[];
  uint8_t* buf0 = smem_b;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem_b + 2 * (size_t)buf_bytes);
  float* S = reinterpret_cast<float*>(bar + 2);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const bool self = a.self_mode != 0;
  const bool interleaved = voff > 0;
  int nk, t = 0;
  bool all_masked = false;
  int64_t row0;
  if (self) {
    t = *a.t_ptr;
    nk = t + 1;
    row0 = (int64_t)r * a.cap;
  } else {
    const int seq = r / a.rows_per_seq;
    const int kl = a.k_len[seq];
    all_masked = kl == 0;
    nk = all_masked ? a.k_pad : kl;
    row0 = a.k_start[seq];
  }
  const T* kb = reinterpret_cast<const T*>(a.k);
  const T* vb = reinterpret_cast<const T*>(a.v);
  const size_t row_bytes = (size_t)a.ldkv * sizeof(T);
  const int nchunks = (nk + CH - 1) / CH;
  auto issue = [&](int c) {
    const int j0 = c * CH;
    const int n = min(CH, nk - j0);
    uint8_t* dst = buf0 + (size_t)(c & 1) * buf_bytes;
    const uint32_t bytes = (uint32_t)(n * row_bytes);
    mbar_expect_tx(bar + (c & 1), interleaved ? bytes : 2 * bytes);
    bulk_g2s(dst, kb + (row0 + j0) * a.ldkv, bytes, bar + (c & 1));
    if (!interleaved)
      bulk_g2s(dst + (size_t)CH * row_bytes, vb + (row0 + j0) * a.ldkv, bytes, bar + (c & 1));
  };
  if (tid == 0) {
    mbar_init(bar, 1);
    mbar_init(bar + 1, 1);
    fence_mbar_init();
    issue(0);
    if (nchunks > 1) issue(1);
  }
  // scaled query slices in registers (lane holds vectors lane, lane + 32, ...)
  float qr[NVL][VEC];
  const T* q = reinterpret_cast<const T*>(a.q) + (size_t)r * a.ldq;
#pragma unroll
  for (int i = 0; i < NVL; ++i) {
    const int e0 = (lane + 32 * i) * VEC;
    if (e0 < D) {
      float f[VEC];
      cvt16<T>(*reinterpret_cast<const uint4*>(q + e0), f);
#pragma unroll
      for (int k = 0; k < VEC; ++k) qr[i][k] = f[k] * qscale;
    }
  }
  __syncthreads();   // barrier init visible to all waiters
  float acc[CPT];
#pragma unroll
  for (int i = 0; i < CPT; ++i) acc[i] = 0.f;
  float m_run = -INFINITY, l_run = 0.f;
  for (int c = 0; c < nchunks; ++c) {
    const int n = min(CH, nk - c * CH);
    const uint8_t* kbuf = buf0 + (size_t)(c & 1) * buf_bytes;
    const T* vrow0 = reinterpret_cast<const T*>(interleaved ? kbuf : kbuf + (size_t)CH * row_bytes) +
                     (interleaved ? voff : 0);
    mbar_wait(bar + (c & 1), (uint32_t)(c >> 1) & 1u);
    // scores: warp w takes keys w, w + NW, ...
    for (int j = warp; j < n; j += NW) {
      const T* kr = reinterpret_cast<const T*>(kbuf + (size_t)j * row_bytes);
      float sacc = 0.f;
#pragma unroll
      for (int i = 0; i < NVL; ++i) {
        const int e0 = (lane + 32 * i) * VEC;
        if (e0 < D) {
          float f[VEC];
          cvt16<T>(*reinterpret_cast<const uint4*>(kr + e0), f);
#pragma unroll
          for (int k = 0; k < VEC; ++k) sacc = fmaf(qr[i][k], f[k], sacc);
        }
      }
      sacc = warp_sum(sacc);
      if (lane == 0) {
        if (a.kc_off >= 0) sacc += qscale * to_f32(kr[a.kc_off]);
        S[j] = all_masked ? sacc + kMaskValue : sacc;
      }
    }
    __syncthreads();
    // online softmax over this chunk (every thread walks the same S in order,
    // so m / l are identical across the CTA)
    float cmax = -INFINITY;
    for (int j = 0; j < n; ++j) cmax = fmaxf(cmax, S[j]);
    const float m_new = fmaxf(m_run, cmax);
    const float alpha = expf(m_run - m_new);
    l_run *= alpha;
#pragma unroll
    for (int i = 0; i < CPT; ++i) acc[i] *= alpha;
    const int col = tid * CPT;
    for (int j = 0; j < n; ++j) {
      const float pj = expf(S[j] - m_new);
      l_run += pj;
      const T* vr = vrow0 + (size_t)j * a.ldkv + col;
      if constexpr (CPT == 2) {
        float2 v2;
        if constexpr (sizeof(T) == 2 && std::is_same<T, __half>::value)
          v2 = __half22float2(*reinterpret_cast<const __half2*>(vr));
        else
          v2 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(vr));
        acc[0] = fmaf(pj, v2.x, acc[0]);
        acc[1] = fmaf(pj, v2.y, acc[1]);
      } else if constexpr (CPT == 8) {
        float f[8];
        cvt16<T>(*reinterpret_cast<const uint4*>(vr), f);
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i] = fmaf(pj, f[i], acc[i]);
      } else {
#pragma unroll
        for (int i = 0; i < CPT; ++i) acc[i] = fmaf(pj, to_f32(vr[i]), acc[i]);
      }
    }
    m_run = m_new;
    __syncthreads();   // buffer (c & 1) and S fully consumed
    if (tid == 0 && c + 2 < nchunks) {
      fence_proxy_async_smem();
      issue(c + 2);
    }
  }
  const int col = tid * CPT;
  const float inv = 1.f / l_run;
  if (a.out_f32) {
    float* o = reinterpret_cast<float*>(a.out) + (size_t)r * a.ldo + col;
#pragma unroll
    for (int i = 0; i < CPT; ++i) {
      const float v = acc[i] * inv;
      o[i] = a.out_bias ? v + a.out_bias[col + i] : v;
    }
  } else {
    T* o = reinterpret_cast<T*>(a.out) + (size_t)r * a.ldo + col;
#pragma unroll
    for (int i = 0; i < CPT; ++i) o[i] = from_f32<T>(acc[i] * inv);
  }
}

// Bulk-copy kernel applicability and launch (returns cudaErrorNotSupported to
// fall through to the register-staged kernels).
// Ring slot size (FNMT_BULK_KB, default 16 KB) and block width (FNMT_BULK_NT, default 128).
uint32_t bulk_buf_bytes() {
  static uint32_t b = 0;
  if (!b) {
    const char* e = getenv("FNMT_BULK_KB");
    const int kb = e ? atoi(e) : 16;
    b = (uint32_t)std::max(4, std::min(100, kb)) * 1024u;
  }
  return b;
}
int bulk_nt() {
  static int n = -1;
  if (n < 0) {
    const char* e = getenv("FNMT_BULK_NT");
    n = e ? atoi(e) : 128;   // r02 A/B (6-1-1 bench): 128 threads x 16 KB slots best
    if (n != 64 && n != 128 && n != 256) n = 128;
  }
  return n;
}

bool dec_bulk_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("FNMT_DEC_BULK");
    on = !(e && e[0] == '0');
  }
  return on != 0;
}

template <typename T>
cudaError_t try_dec_bulk(const DecAttnArgs& a, float qscale, cudaStream_t s) {
  if (!dec_bulk_enabled() || a.heads != 1 || a.anc || a.new_k || a.dk % 8) return cudaErrorNotSupported;
  const int d = a.dk;
  const size_t row_bytes = (size_t)a.ldkv * sizeof(T);
  if (row_bytes % 16 || (reinterpret_cast<uintptr_t>(a.k) & 15) ||
      (reinterpret_cast<uintptr_t>(a.v) & 15) || (reinterpret_cast<uintptr_t>(a.q) & 15) ||
      a.ldq % 8)
    return cudaErrorNotSupported;
  // interleaved rows (cross caches, folded self cache): V at element offset
  // voff of the K row, one copy per chunk; else separate K / V caches of d
  int voff = 0;
  const ptrdiff_t off = reinterpret_cast<const T*>(a.v) - reinterpret_cast<const T*>(a.k);
  if (off > 0 && off + d <= a.ldkv)
    voff = (int)off;
  else if (!a.self_mode || a.ldkv != d)
    return cudaErrorNotSupported;
  const size_t per_key = voff ? row_bytes : 2 * row_bytes;
  const int CH = (int)std::min<size_t>(64, bulk_buf_bytes() / per_key);
  if (CH < 4) return cudaErrorNotSupported;
  const uint32_t buf = (uint32_t)(((size_t)CH * per_key + 127) & ~(size_t)127);
  const size_t smem = 2 * (size_t)buf + 16 + sizeof(float) * CH;
  auto pick = [&](auto kern, int nt) -> cudaError_t {
    cudaError_t e = set_max_smem((const void*)kern);
    if (e != cudaSuccess) return e;
    return launch_k(kern, dim3(a.rows), dim3(nt), smem, s, a, qscale, CH, voff, buf);
  };
  if (d == 512) {
    if (bulk_nt() == 64) return pick(attn_dec_bulk_kernel<T, 64, 8>, 64);
    return bulk_nt() == 128 ? pick(attn_dec_bulk_kernel<T, 128, 4>, 128)
                            : pick(attn_dec_bulk_kernel<T, 256, 2>, 256);
  }
  if (d == 256) return pick(attn_dec_bulk_kernel<T, 128, 2>, 128);
  if (d == 1024) return pick(attn_dec_bulk_kernel<T, 256, 4>, 256);
  return cudaErrorNotSupported;
}

// ---------------------------------------------------------------------------
// dispatch

template <typename T>
cudaError_t varlen_dispatch(const AttnArgs& a, cudaStream_t s) {
  const int kcap = ((a.max_k + kKT - 1) / kKT) * kKT;
  const size_t smem =
      sizeof(float) * ((size_t)kQT * kcap + (size_t)kDC * (kQT + 4) + (size_t)kDC * (kKT + 4));
  static_assert(kDC * (kKT + 4) >= kPK * (kPD + 4), "V tile must fit in the K tile region");
  if (smem > 227 * 1024) return cudaErrorInvalidValue;
  cudaError_t e = set_max_smem((const void*)attn_varlen_kernel<T>);
  if (e != cudaSuccess) return e;
  dim3 grid((a.max_q + kQT - 1) / kQT, a.n_seq, a.heads);
  const float qscale = (float)(1.0 / sqrt((double)a.dk));
  attn_varlen_kernel<T><<<grid, kVThreads, smem, s>>>(a, qscale, kcap);
  return cudaGetLastError();
}

// Two-pass kernel unroll: 2 score rounds / 4 value rows in flight per warp /
// thread (r01 A/B of (U, UV) = (1,1) (1,4) (1,8) (2,4) (2,8): 6.82 / 6.86 / 6.47 /
// 6.87 / 6.70 M words/s).
template <typename T, int G, int CH, int NT, int U, int UV>
cudaError_t launch_dec_nt_u(const DecAttnArgs& a, float qscale, cudaStream_t s) {
  const int groups = NT / (a.dk / Vec16<T>::N);
  const size_t smem = sizeof(float) * ((size_t)a.dk + a.max_k + 4 + (size_t)groups * a.dk);
  if (smem > 227 * 1024) return cudaErrorInvalidValue;
  if (smem > 48 * 1024) {
    cudaError_t e = set_max_smem((const void*)attn_decode_kernel<T, G, CH, NT, U, UV>);
    if (e != cudaSuccess) return e;
  }
  return launch_k(attn_decode_kernel<T, G, CH, NT, U, UV>, dim3(a.rows, a.heads), dim3(NT), smem,
                  s, a, qscale);
}

template <typename T, int G, int CH, int NT>
cudaError_t launch_dec_nt(const DecAttnArgs& a, float qscale, cudaStream_t s) {
  return launch_dec_nt_u<T, G, CH, NT, 2, 4>(a, qscale, s);
}

template <typename T, int G, int CH, int NT>
cudaError_t launch_dec_async(const DecAttnArgs& a, float qscale, cudaStream_t s) {
  constexpr int NW = NT / 32;
  const size_t smem = (size_t)NW * 8 * 32 * CH * 16 +
                      sizeof(float) * ((size_t)a.dk + a.max_k + 4 + (size_t)NW * a.dk);
  if (smem > 227 * 1024) return launch_dec_nt<T, G, CH, NT>(a, qscale, s);
  if (smem > 48 * 1024) {
    cudaError_t e = set_max_smem((const void*)attn_decode_async_kernel<T, G, CH, NT>);
    if (e != cudaSuccess) return e;
  }
  return launch_k(attn_decode_async_kernel<T, G, CH, NT>, dim3(a.rows, a.heads), dim3(NT), smem, s,
                  a, qscale);
}

// block width for the two-pass kernel: few (row, head) blocks -> wider blocks.
// FNMT_DEC_NT: 0 = auto (< FNMT_DEC_FEW rows x heads -> 512 threads, else 128;
// FEW default 600: r01 A/B 7.03 / 7.08 vs 6.97 / 6.99 M words/s for 1200),
// or a fixed 128 / 256 / 512.
int dec_nt_choice(int64_t blocks) {
  static int fixed = -1, few = -1;
  if (fixed < 0) {
    const char* e = getenv("FNMT_DEC_NT");
    fixed = e ? atoi(e) : 0;
    if (fixed != 128 && fixed != 256 && fixed != 512) fixed = 0;
    const char* f = getenv("FNMT_DEC_FEW");
    few = f ? atoi(f) : 600;
  }
  if (fixed) return fixed;
  return blocks < few ? 512 : 128;
}

template <typename T, int G, int CH>
cudaError_t launch_dec_wide(const DecAttnArgs& a, float qscale, cudaStream_t s) {
  switch (dec_nt_choice((int64_t)a.rows * a.heads)) {
    case 512: return launch_dec_nt<T, G, CH, 512>(a, qscale, s);
    case 256: return launch_dec_nt<T, G, CH, 256>(a, qscale, s);
    default: return launch_dec_nt<T, G, CH, 128>(a, qscale, s);
  }
}

template <typename T, int G, int CH>
cudaError_t launch_dec(const DecAttnArgs& a, float qscale, cudaStream_t s) {
  if (a.kc_off >= 0 || a.out_f32) {   // folded cross attention: two-pass kernel only
    if (G != 32 || a.heads != 1) return cudaErrorInvalidValue;
    return launch_dec_wide<T, G, CH>(a, qscale, s);
  }
  // few (row, head) blocks -> wide blocks so the SMs still have enough warps in flight
  // cp.async staging measured faster for 8 heads (dk=64) only (r01: 6-1-8 3.92M vs 3.67M
  // words/s; 6-1-1 3.92M vs 4.32M)
  if (G < 32) {
    if ((int64_t)a.rows * a.heads < 1200) return launch_dec_async<T, G, CH, 256>(a, qscale, s);
    return launch_dec_async<T, G, CH, 128>(a, qscale, s);
  }
  return launch_dec_wide<T, G, CH>(a, qscale, s);
}

bool dec_rows_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("FNMT_DEC_ROWS");
    on = !(e && e[0] == '0');
  }
  return on != 0;
}

template <typename T, int CH, int LPH>
cudaError_t launch_dec_rows(const DecAttnArgs& a, float qscale, cudaStream_t s) {
  constexpr int NT = 128;
  const int d = a.heads * a.dk;
  const int groups = NT / (d / Vec16<T>::N);
  const size_t smem = sizeof(float) * ((size_t)d + (size_t)a.heads * a.max_k + 4 +
                                       (size_t)groups * d + (LPH ? 0 : (NT / 32) * 2 * 32 * CH));
  if (smem > 227 * 1024) return cudaErrorInvalidValue;
  auto kern = attn_decode_rows_kernel<T, CH, NT, LPH>;
  if (smem > 48 * 1024) {
    cudaError_t e = set_max_smem((const void*)kern);
    if (e != cudaSuccess) return e;
  }
  return launch_k(kern, dim3(a.rows), dim3(NT), smem, s, a, qscale);
}

// Multi-head rows: heads of 8 / 16 / 32 lanes (fp16 dk 64 / 128 / 256), a row of
// 256 .. 512 elements per 128-thread CTA (CH 1 or 2 chunks per lane).
template <typename T>
cudaError_t try_dec_rows(const DecAttnArgs& a, float qscale, cudaStream_t s) {
  constexpr int VEC = Vec16<T>::N;
  if (sizeof(T) != 2 || a.heads < 2 || !dec_rows_enabled() || a.dk % VEC || (a.ldkv % VEC) ||
      (a.ldq % VEC))
    return cudaErrorNotSupported;
  const int lph = a.dk / VEC, d = a.heads * a.dk;
  if (d % (32 * VEC)) return cudaErrorNotSupported;
  const int ch = d / (32 * VEC);
  if (a.heads > 32) return cudaErrorNotSupported;
  if (ch == 1) {
    if (lph == 8) return launch_dec_rows<T, 1, 8>(a, qscale, s);
    if (lph == 16) return launch_dec_rows<T, 1, 16>(a, qscale, s);
    return launch_dec_rows<T, 1, 0>(a, qscale, s);
  } else if (ch == 2) {
    if (lph == 8) return launch_dec_rows<T, 2, 8>(a, qscale, s);
    if (lph == 16) return launch_dec_rows<T, 2, 16>(a, qscale, s);
    if (lph == 32) return launch_dec_rows<T, 2, 32>(a, qscale, s);
    return launch_dec_rows<T, 2, 0>(a, qscale, s);
  } else if (ch == 3) {
    return launch_dec_rows<T, 3, 0>(a, qscale, s);   // e.g. Deep-12-768: 8 heads x 96
  } else if (ch == 4) {
    if (lph == 8) return launch_dec_rows<T, 4, 8>(a, qscale, s);
    if (lph == 16) return launch_dec_rows<T, 4, 16>(a, qscale, s);
    if (lph == 32) return launch_dec_rows<T, 4, 32>(a, qscale, s);
    return launch_dec_rows<T, 4, 0>(a, qscale, s);
  }
  return cudaErrorNotSupported;
}

template <typename T>
cudaError_t decode_dispatch(const DecAttnArgs& a, cudaStream_t s) {
  constexpr int VEC = Vec16<T>::N;
  const float qscale = (float)(1.0 / sqrt((double)a.dk));
  if constexpr (sizeof(T) == 2) {
    cudaError_t e = try_dec_bulk<T>(a, qscale, s);
    if (e != cudaErrorNotSupported) return e;
    e = try_dec_rows<T>(a, qscale, s);
    if (e != cudaErrorNotSupported) return e;
  }
  const int nch = a.dk / VEC;
  const bool vec_ok = a.dk % VEC == 0 && nch <= kDThreads && (a.ldkv % VEC) == 0 &&
                      sizeof(float) * ((size_t)a.dk * 5 + a.max_k + 4) <= 227 * 1024;
  if (vec_ok) {
    if (nch <= 1) return launch_dec<T, 1, 1>(a, qscale, s);
    if (nch <= 2) return launch_dec<T, 2, 1>(a, qscale, s);
    if (nch <= 4) return launch_dec<T, 4, 1>(a, qscale, s);
    if (nch <= 8) return launch_dec<T, 8, 1>(a, qscale, s);
    if (nch <= 16) return launch_dec<T, 16, 1>(a, qscale, s);
    if (nch <= 32) return launch_dec<T, 32, 1>(a, qscale, s);
    if (nch <= 64) return launch_dec<T, 32, 2>(a, qscale, s);
    if (nch <= 96) return launch_dec<T, 32, 3>(a, qscale, s);
    return launch_dec<T, 32, 4>(a, qscale, s);
  }
  const size_t smem = sizeof(float) * ((size_t)a.dk + (size_t)a.max_k + 32);
  if (smem > 227 * 1024) return cudaErrorInvalidValue;
  if (smem > 48 * 1024) {
    cudaError_t e = set_max_smem((const void*)attn_decode_generic<T>);
    if (e != cudaSuccess) return e;
  }
  attn_decode_generic<T><<<dim3(a.rows, a.heads), kDThreads, smem, s>>>(a, qscale);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_attention_varlen(const AttnArgs& a, cudaStream_t s) {
  if (a.n_seq <= 0 || a.max_q <= 0) return cudaSuccess;
  if (attention_mma_ok(a)) return launch_attention_varlen_mma(a, s);
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
