// Fused decoder attention block for single-head folded decoders (Student-6-1-1
// and any 1-head decoder in fp16 / bf16): one kernel per decode step and
// layer replaces
//
//   self attention -> + residual -> norm1 -> cross attention -> + residual -> norm2
//
// (decode_step, model.py:321-338; _norm model.py:193-196 -> tensor.py:98-129).
// Both attentions are the folded forms the engine builds (engine.cu
// make_folded): every cached key row is [K~ (d) | V~ (d) | c | pad] with
// score_j = q . K~_j + c_j and the values already o-projected, so the
// attention output plus the o-projection bias is the residual branch itself.
//
// One CTA per query row, the whole decoder state of the row stays on chip:
//   * thread 0 streams the row's keys with cp.async.bulk (TMA engine) through
//     a double-buffered smem ring — the self cache slots r*cap + 0..t, then,
//     without a break in the ring, the sentence's cross keys (they do not
//     depend on the self phase, so the first cross chunks are in flight while
//     the self phase finishes);
//   * scores warp-per-key from smem, online softmax (running max / sum; one
//     chunk = the reference's max-shifted softmax, tensor.py:70-81), every
//     thread accumulates its CPT output columns;
//   * between the phases the residual add and LayerNorm run as a block
//     reduction (row mean in f64, eps on the deviation scale, exactly the
//     add_norm_kernel arithmetic), the norm1 output is rounded to the
//     activation type in smem and becomes the cross query;
//   * after the cross phase the second add + norm writes the fp32 residual
//     stream and its activation copy (the FFN GEMM's A operand).
// Rows of finished sentences exit at once (search.py:72 discards them).
#include <math.h>

#include <type_traits>

#include "common.cuh"
#include "kernels.h"

namespace fnmt {

namespace {

constexpr float kMaskValue = -1e9f;

template <typename T>
__device__ __forceinline__ void cvt8(const uint4& u, float (&f)[8]) {
  if constexpr (std::is_same<T, __half>::value) {
    const __half2* h = reinterpret_cast<const __half2*>(&u);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float2 x = __half22float2(h[i]);
      f[2 * i] = x.x;
      f[2 * i + 1] = x.y;
    }
  } else {
    const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float2 x = __bfloat1622float2(h[i]);
      f[2 * i] = x.x;
      f[2 * i + 1] = x.y;
    }
  }
}

// Residual add + LayerNorm of one row held CPT values per thread (add_norm_kernel
// arithmetic: f64 row mean cast to f32, f64 sum of squared (or absolute)
// deviations, scale = sqrt(mean) (l2) or mean (l1), y = g * dev / (scale + 1e-6) + b).
template <int NT, int CPT>
__device__ __forceinline__ void block_norm(float (&v)[CPT], const float* __restrict__ gain,
                                           const float* __restrict__ bias, int l1, double* red,
                                           int col) {
  constexpr int NW = NT / 32;
  constexpr int D = NT * CPT;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double s = 0.0;
#pragma unroll
  for (int i = 0; i < CPT; ++i) s += (double)v[i];
  s = warp_sum_d(s);
  if (lane == 0) red[warp] = s;
  __syncthreads();
  double tot = 0.0;
#pragma unroll
  for (int w = 0; w < NW; ++w) tot += red[w];
  const float mu = (float)(tot / (double)D);
  double q = 0.0;
#pragma unroll
  for (int i = 0; i < CPT; ++i) {
    v[i] -= mu;
    q += l1 ? (double)fabsf(v[i]) : (double)(v[i] * v[i]);
  }
  q = warp_sum_d(q);
  if (lane == 0) red[NW + warp] = q;
  __syncthreads();
  double qt = 0.0;
#pragma unroll
  for (int w = 0; w < NW; ++w) qt += red[NW + w];
  float sc = (float)(qt / (double)D);
  if (!l1) sc = sqrtf(sc);
  const float den = sc + 1e-6f;
#pragma unroll
  for (int i = 0; i < CPT; ++i) v[i] = gain[col + i] * v[i] / den + bias[col + i];
}

template <typename T, int NVL>
__device__ __forceinline__ void load_query(float (&qr)[NVL][8], const T* q, int D, float qscale) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int i = 0; i < NVL; ++i) {
    const int e0 = (lane + 32 * i) * 8;
    if (e0 < D) {
      float f[8];
      cvt8<T>(*reinterpret_cast<const uint4*>(q + e0), f);
#pragma unroll
      for (int k = 0; k < 8; ++k) qr[i][k] = f[k] * qscale;
    }
  }
}

template <typename T, int NT, int CPT>
__global__ void __launch_bounds__(NT) dec_layer_fused_kernel(DecLayerArgs a, float qscale,
                                                             int ch_s, int ch_c,
                                                             uint32_t buf_bytes) {
  pdl_trigger();
  pdl_wait();
  const int r = blockIdx.x;
  if (a.row_done && a.row_done[r]) return;
  constexpr int NW = NT / 32;
  constexpr int D = NT * CPT;                  // d_model (single head: dk == d)
  constexpr int NVL = (D / 8 + 31) / 32;       // 16-byte query vectors per lane
  extern __shared__ __align__(128) uint8_t smem_b[];
  uint8_t* buf0 = smem_b;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem_b + 2 * (size_t)buf_bytes);
  double* red = reinterpret_cast<double*>(bar + 2);           // [2 NW]
  T* xq = reinterpret_cast<T*>(red + 2 * NW);                 // [D] cross query
  float* S = reinterpret_cast<float*>(xq + D);                // [max(ch_s, ch_c)]
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int col = tid * CPT;

  const int t = *a.t_ptr;
  const int nk_s = t + 1;
  const int64_t row0_s = (int64_t)r * a.cap;
  const int seq = r / a.rows_per_seq;
  const int kl = a.k_len[seq];
  const bool all_masked = kl == 0;
  const int nk_c = all_masked ? a.k_pad : kl;
  const int64_t row0_c = a.k_start[seq];
  const int ns = (nk_s + ch_s - 1) / ch_s;
  const int ntot = ns + (nk_c + ch_c - 1) / ch_c;
  const T* ks = reinterpret_cast<const T*>(a.kself);
  const T* kc = reinterpret_cast<const T*>(a.kcross);
  const T* knew = reinterpret_cast<const T*>(a.knew);
  const size_t rb_s = (size_t)a.ld_self * sizeof(T), rb_c = (size_t)a.ld_cross * sizeof(T);

  auto issue = [&](int c) {
    uint8_t* dst = buf0 + (size_t)(c & 1) * buf_bytes;
    const T* src;
    uint32_t bytes;
    if (c < ns) {
      const int j0 = c * ch_s;
      const int n = min(ch_s, nk_s - j0);
      if (knew && c == ns - 1) {
        // last self chunk: keys j0..t-1 from the cache, key t from the GEMM's row
        mbar_expect_tx(bar + (c & 1), (uint32_t)(n * rb_s));
        if (n > 1) bulk_g2s(dst, ks + (row0_s + j0) * a.ld_self, (uint32_t)((n - 1) * rb_s), bar + (c & 1));
        bulk_g2s(dst + (size_t)(n - 1) * rb_s, knew + (size_t)r * a.ld_self, (uint32_t)rb_s,
                 bar + (c & 1));
        return;
      }
      src = ks + (row0_s + j0) * a.ld_self;
      bytes = (uint32_t)(n * rb_s);
    } else {
      const int j0 = (c - ns) * ch_c;
      src = kc + (row0_c + j0) * a.ld_cross;
      bytes = (uint32_t)(min(ch_c, nk_c - j0) * rb_c);
    }
    mbar_expect_tx(bar + (c & 1), bytes);
    bulk_g2s(dst, src, bytes, bar + (c & 1));
  };
  if (tid == 0) {
    mbar_init(bar, 1);
    mbar_init(bar + 1, 1);
    fence_mbar_init();
    issue(0);
    if (ntot > 1) issue(1);
  }
  float qr[NVL][8];
  load_query<T, NVL>(qr, reinterpret_cast<const T*>(a.q) + (size_t)r * a.ldq, D, qscale);
  float x[CPT];   // residual stream of this row (fp32), this thread's columns
  {
    const float* xr = a.x32 + (size_t)r * D + col;
#pragma unroll
    for (int i = 0; i < CPT; ++i) x[i] = xr[i];
  }
  __syncthreads();   // barrier init visible to all waiters

  float acc[CPT];
#pragma unroll
  for (int i = 0; i < CPT; ++i) acc[i] = 0.f;
  float m_run = -INFINITY, l_run = 0.f;
  for (int c = 0; c < ntot; ++c) {
    const bool self = c < ns;
    if (c == ns) {
      // self phase done: x = norm1(x + (attn + bo_self)); the rounded norm1
      // output is the cross query (the unfused path's activation copy)
      const float inv = 1.f / l_run;
#pragma unroll
      for (int i = 0; i < CPT; ++i) x[i] = x[i] + (acc[i] * inv + a.bo_self[col + i]);
      block_norm<NT, CPT>(x, a.g1, a.b1, a.l1, red, col);
#pragma unroll
      for (int i = 0; i < CPT; ++i) xq[col + i] = from_f32<T>(x[i]);
      __syncthreads();
      load_query<T, NVL>(qr, xq, D, qscale);
#pragma unroll
      for (int i = 0; i < CPT; ++i) acc[i] = 0.f;
      m_run = -INFINITY;
      l_run = 0.f;
    }
    const int n = self ? min(ch_s, nk_s - c * ch_s) : min(ch_c, nk_c - (c - ns) * ch_c);
    const size_t rb = self ? rb_s : rb_c;
    const int ld = self ? a.ld_self : a.ld_cross;
    const uint8_t* kbuf = buf0 + (size_t)(c & 1) * buf_bytes;
    mbar_wait(bar + (c & 1), (uint32_t)(c >> 1) & 1u);
    if (knew && c == ns - 1) {
      // append key t (now in smem) to the row's cache slot: coalesced 16-byte stores
      const uint4* srow = reinterpret_cast<const uint4*>(kbuf + (size_t)(n - 1) * rb);
      uint4* drow = reinterpret_cast<uint4*>(const_cast<T*>(ks) + (row0_s + t) * a.ld_self);
      for (int i = tid; i < (int)(rb / 16); i += NT) drow[i] = srow[i];
    }
    for (int j = warp; j < n; j += NW) {
      const T* kr = reinterpret_cast<const T*>(kbuf + (size_t)j * rb);
      float sacc = 0.f;
#pragma unroll
      for (int i = 0; i < NVL; ++i) {
        const int e0 = (lane + 32 * i) * 8;
        if (e0 < D) {
          float f[8];
          cvt8<T>(*reinterpret_cast<const uint4*>(kr + e0), f);
#pragma unroll
          for (int k = 0; k < 8; ++k) sacc = fmaf(qr[i][k], f[k], sacc);
        }
      }
      sacc = warp_sum(sacc);
      if (lane == 0) {
        sacc += qscale * to_f32(kr[a.kc_off]);
        S[j] = (!self && all_masked) ? sacc + kMaskValue : sacc;
      }
    }
    __syncthreads();
    float cmax = -INFINITY;
    for (int j = 0; j < n; ++j) cmax = fmaxf(cmax, S[j]);
    const float m_new = fmaxf(m_run, cmax);
    const float alpha = expf(m_run - m_new);
    l_run *= alpha;
#pragma unroll
    for (int i = 0; i < CPT; ++i) acc[i] *= alpha;
    const T* vrow0 = reinterpret_cast<const T*>(kbuf) + a.voff + col;
    for (int j = 0; j < n; ++j) {
      const float pj = expf(S[j] - m_new);
      l_run += pj;
      const T* vr = vrow0 + (size_t)j * ld;
      if constexpr (CPT == 2) {
        float2 v0;
        if constexpr (std::is_same<T, __half>::value)
          v0 = __half22float2(*reinterpret_cast<const __half2*>(vr));
        else
          v0 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(vr));
        acc[0] = fmaf(pj, v0.x, acc[0]);
        acc[1] = fmaf(pj, v0.y, acc[1]);
      } else if constexpr (CPT == 4) {
        const uint2 u = *reinterpret_cast<const uint2*>(vr);
        float2 v0, v1;
        if constexpr (std::is_same<T, __half>::value) {
          v0 = __half22float2(*reinterpret_cast<const __half2*>(&u.x));
          v1 = __half22float2(*reinterpret_cast<const __half2*>(&u.y));
        } else {
          v0 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.x));
          v1 = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&u.y));
        }
        acc[0] = fmaf(pj, v0.x, acc[0]);
        acc[1] = fmaf(pj, v0.y, acc[1]);
        acc[2] = fmaf(pj, v1.x, acc[2]);
        acc[3] = fmaf(pj, v1.y, acc[3]);
      } else {
#pragma unroll
        for (int i = 0; i < CPT; ++i) acc[i] = fmaf(pj, to_f32(vr[i]), acc[i]);
      }
    }
    m_run = m_new;
    __syncthreads();   // slot (c & 1) and S consumed
    if (tid == 0 && c + 2 < ntot) {
      fence_proxy_async_smem();
      issue(c + 2);
    }
  }
  // cross phase done: x = norm2(x + (attn + bo_cross)) -> residual stream + activation copy
  const float inv = 1.f / l_run;
#pragma unroll
  for (int i = 0; i < CPT; ++i) x[i] = x[i] + (acc[i] * inv + a.bo_cross[col + i]);
  block_norm<NT, CPT>(x, a.g2, a.b2, a.l1, red, col);
  float* xo = a.x32 + (size_t)r * D + col;
  T* xa = reinterpret_cast<T*>(a.xa) + (size_t)r * D + col;
#pragma unroll
  for (int i = 0; i < CPT; ++i) {
    xo[i] = x[i];
    xa[i] = from_f32<T>(x[i]);
  }
}

bool fused_layer_env() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("FNMT_FUSED_LAYER");
    on = !(e && e[0] == '0');
  }
  return on != 0;
}

// ring slot size (FNMT_LAYER_KB, default 16 KB: the bulk decode attention's A/B optimum)
uint32_t layer_buf_bytes() {
  static uint32_t b = 0;
  if (!b) {
    const char* e = getenv("FNMT_LAYER_KB");
    const int kb = e ? atoi(e) : 16;
    b = (uint32_t)std::max(4, std::min(100, kb)) * 1024u;
  }
  return b;
}

}  // namespace

bool dec_layer_fused_ok(int dtype, int d, int heads) {
  return fused_layer_env() && (dtype == kF16 || dtype == kBF16) && heads == 1 &&
         (d == 512 || d == 256 || d == 1024);
}

cudaError_t launch_dec_layer_fused(const DecLayerArgs& a, cudaStream_t s) {
  if (a.rows <= 0) return cudaSuccess;
  if (!dec_layer_fused_ok(a.dtype, a.d, 1)) return cudaErrorNotSupported;
  const size_t es = 2;
  const size_t rb_s = (size_t)a.ld_self * es, rb_c = (size_t)a.ld_cross * es;
  if (rb_s % 16 || rb_c % 16 || a.ldq % 8 || a.voff % 8 ||
      (reinterpret_cast<uintptr_t>(a.kself) & 15) || (reinterpret_cast<uintptr_t>(a.kcross) & 15) ||
      (reinterpret_cast<uintptr_t>(a.q) & 15) || (reinterpret_cast<uintptr_t>(a.knew) & 15))
    return cudaErrorNotSupported;
  const uint32_t buf = layer_buf_bytes();
  const int ch_s = (int)std::min<size_t>(64, buf / rb_s);
  const int ch_c = (int)std::min<size_t>(64, buf / rb_c);
  if (ch_s < 1 || ch_c < 1) return cudaErrorNotSupported;
  const int nw_max = 8;
  const size_t smem = 2 * (size_t)buf + 16 + sizeof(double) * 2 * nw_max + es * a.d +
                      sizeof(float) * std::max(ch_s, ch_c);
  const float qscale = (float)(1.0 / sqrt((double)a.d));
  auto go = [&](auto kern, int nt) -> cudaError_t {
    cudaError_t e = set_max_smem((const void*)kern);
    if (e != cudaSuccess) return e;
    return launch_k(kern, dim3(a.rows), dim3(nt), smem, s, a, qscale, ch_s, ch_c, buf);
  };
  static int nt = -1;
  if (nt < 0) {
    const char* e = getenv("FNMT_LAYER_NT");   // 128 (4 columns / thread) or 256 (2)
    nt = e ? atoi(e) : 128;
  }
  if (a.d == 512 && nt == 256)
    return a.dtype == kF16 ? go(dec_layer_fused_kernel<__half, 256, 2>, 256)
                           : go(dec_layer_fused_kernel<__nv_bfloat16, 256, 2>, 256);
  if (a.dtype == kF16) {
    if (a.d == 512) return go(dec_layer_fused_kernel<__half, 128, 4>, 128);
    if (a.d == 256) return go(dec_layer_fused_kernel<__half, 64, 4>, 64);
    return go(dec_layer_fused_kernel<__half, 256, 4>, 256);
  }
  if (a.d == 512) return go(dec_layer_fused_kernel<__nv_bfloat16, 128, 4>, 128);
  if (a.d == 256) return go(dec_layer_fused_kernel<__nv_bfloat16, 64, 4>, 64);
  return go(dec_layer_fused_kernel<__nv_bfloat16, 256, 4>, 256);
}

}  // namespace fnmt
