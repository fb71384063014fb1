// Persistent, warp-specialised decode attention fed by TMA (greedy decode,
// 16-bit KV caches).  Same contract as attn_decode_kernel (attention.cu):
// one query per (row, head) against the self-KV cache (keys 0..t, appended by
// the QKV GEMM epilogue) or the cached cross K/V (keys 0..S-1), reference
// arithmetic order (scores -> max-shifted softmax -> normalised weights ->
// value sum; model.py:199-240, tensor.py:70-81).
//
// Why: per-(row, head) CTAs are latency-bound (r01 ncu: 44% of DRAM peak,
// long-scoreboard stalls); a CTA can never prefetch the next row.  Here one
// CTA per SM walks a list of (row, head) items: warp 0 streams 2-D TMA boxes
// (KC keys x min(dk, 256) dims, ~16 KB) of every item's K chunks then V
// chunks through an NST-deep mbarrier ring, running ahead across item
// boundaries; warps 1..4 consume (q.K scores into smem, softmax, weights.V).
// HBM sees up to NST x 16 KB in flight per SM.
#include <math.h>

#include "common.cuh"
#include "kernels.h"

namespace fnmt {

namespace {

constexpr int kNCW = 4;                    // consumer warps
constexpr int kPThreads = 32 * (kNCW + 1);
constexpr int kStageBytes = 16384;
constexpr float kMask = -1e9f;

__device__ __forceinline__ void ld16(const __half* p, float (&f)[8]) {
  const uint4 u = *reinterpret_cast<const uint4*>(p);
  const __half2* h = reinterpret_cast<const __half2*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 x = __half22float2(h[i]);
    f[2 * i] = x.x;
    f[2 * i + 1] = x.y;
  }
}
__device__ __forceinline__ void ld16(const __nv_bfloat16* p, float (&f)[8]) {
  const uint4 u = *reinterpret_cast<const uint4*>(p);
  const __nv_bfloat162* h = reinterpret_cast<const __nv_bfloat162*>(&u);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const float2 x = __bfloat1622float2(h[i]);
    f[2 * i] = x.x;
    f[2 * i + 1] = x.y;
  }
}

__device__ __forceinline__ void mbar_arrive_cta(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void consumers_sync() {
  asm volatile("bar.sync 1, %0;" ::"n"(kNCW * 32) : "memory");
}

struct Item {
  int r, h, nk;
  bool all_masked;
  int64_t row0;
};

__device__ __forceinline__ Item item_of(const DecAttnArgs& a, int w, int t) {
  Item it;
  it.r = w / a.heads;
  it.h = w - it.r * a.heads;
  if (a.self_mode) {
    it.nk = t + 1;
    it.all_masked = false;
    it.row0 = (int64_t)it.r * a.cap;
  } else {
    const int seq = it.r / a.rows_per_seq;
    const int kl = a.k_len[seq];
    it.all_masked = kl == 0;
    it.nk = it.all_masked ? a.k_pad : kl;
    it.row0 = a.k_start[seq];
  }
  return it;
}

template <typename T, int NST>
__global__ void __launch_bounds__(kPThreads, 1)
    attn_decode_persist_kernel(const __grid_constant__ CUtensorMap tk,
                               const __grid_constant__ CUtensorMap tv, DecAttnArgs a, float qscale,
                               int KC, int k_col0, int v_col0) {
  constexpr int VEC = 8;
  extern __shared__ __align__(1024) uint8_t smem_p[];
  const int dk = a.dk;
  const int BC = dk < 256 ? dk : 256;
  const int chunk_elems = KC * dk;
  T* ring = reinterpret_cast<T*>(smem_p);
  float* qs = reinterpret_cast<float*>(smem_p + (size_t)NST * kStageBytes);
  float* S = qs + dk;
  const int nch = dk / VEC;
  const int groups = (kNCW * 32) / nch;
  float* red = S + a.max_k + 4;
  uint64_t* full = reinterpret_cast<uint64_t*>(
      (reinterpret_cast<uintptr_t>(red + (size_t)groups * dk) + 7) & ~static_cast<uintptr_t>(7));
  uint64_t* empty = full + NST;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int items = a.rows * a.heads;
  const int t = a.self_mode ? *a.t_ptr : 0;
  const uint32_t chunk_bytes = (uint32_t)chunk_elems * sizeof(T);

  if (threadIdx.x == 0) {
    tma_prefetch_desc(&tk);
    tma_prefetch_desc(&tv);
    for (int i = 0; i < NST; ++i) {
      mbar_init(full + i, 1);
      mbar_init(empty + i, kNCW);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == 0) {
    // ---------------- producer ----------------
    if (lane == 0) {
      int st = 0;
      uint32_t ph = 0;
      for (int w = blockIdx.x; w < items; w += gridDim.x) {
        const Item it = item_of(a, w, t);
        const int nchunks = (it.nk + KC - 1) / KC;
        for (int pass = 0; pass < 2; ++pass) {
          const CUtensorMap* map = pass == 0 ? &tk : &tv;
          const int col = (pass == 0 ? k_col0 : v_col0) + it.h * dk;
          for (int ck = 0; ck < nchunks; ++ck) {
            mbar_wait(empty + st, ph ^ 1);
            mbar_expect_tx(full + st, chunk_bytes);
            T* dst = ring + (size_t)st * (kStageBytes / sizeof(T));
            for (int b = 0; b < dk / BC; ++b)
              tma_load_2d(dst + (size_t)b * KC * BC, map, full + st, col + b * BC,
                          (int)(it.row0 + (int64_t)ck * KC));
            if (++st == NST) {
              st = 0;
              ph ^= 1;
            }
          }
        }
      }
    }
    return;
  }

  // ---------------- consumers (warps 1..kNCW) ----------------
  const int cw = warp - 1;
  const int ctid = threadIdx.x - 32;
  const int ch = ctid % nch, grp = ctid / nch;
  int st = 0;
  uint32_t ph = 0;
  for (int w = blockIdx.x; w < items; w += gridDim.x) {
    const Item it = item_of(a, w, t);
    const int nchunks = (it.nk + KC - 1) / KC;
    const T* q = reinterpret_cast<const T*>(a.q) + (size_t)it.r * a.ldq + it.h * dk;
    for (int e = ctid; e < dk; e += kNCW * 32) qs[e] = to_f32(q[e]) * qscale;
    consumers_sync();
    // pass 1: scores
    for (int ck = 0; ck < nchunks; ++ck) {
      mbar_wait(full + st, ph);
      const T* buf = ring + (size_t)st * (kStageBytes / sizeof(T));
      const int j0 = ck * KC;
      const int jn = min(KC, it.nk - j0);
      for (int jj = cw; jj < jn; jj += kNCW) {
        float s = 0.f;
        for (int e0 = lane * VEC; e0 < dk; e0 += 32 * VEC) {
          float f[VEC];
          ld16(buf + (size_t)(e0 / BC) * KC * BC + (size_t)jj * BC + (e0 % BC), f);
#pragma unroll
          for (int i = 0; i < VEC; ++i) s = fmaf(qs[e0 + i], f[i], s);
        }
        s = warp_sum(s);
        if (lane == 0) S[j0 + jj] = it.all_masked ? s + kMask : s;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive_cta(empty + st);
      if (++st == NST) {
        st = 0;
        ph ^= 1;
      }
    }
    consumers_sync();
    if (cw == 0) {
      float mx = -INFINITY;
      for (int j = lane; j < it.nk; j += 32) mx = fmaxf(mx, S[j]);
      mx = warp_max(mx);
      float sum = 0.f;
      for (int j = lane; j < it.nk; j += 32) {
        const float ex = expf(S[j] - mx);
        S[j] = ex;
        sum += ex;
      }
      sum = warp_sum(sum);
      for (int j = lane; j < it.nk; j += 32) S[j] = S[j] / sum;
    }
    consumers_sync();
    // pass 2: weights . V
    float acc[VEC];
#pragma unroll
    for (int i = 0; i < VEC; ++i) acc[i] = 0.f;
    for (int ck = 0; ck < nchunks; ++ck) {
      mbar_wait(full + st, ph);
      const T* buf = ring + (size_t)st * (kStageBytes / sizeof(T));
      const int j0 = ck * KC;
      const int jn = min(KC, it.nk - j0);
      if (grp < groups) {
        const int e0 = ch * VEC;
        const T* colp = buf + (size_t)(e0 / BC) * KC * BC + (e0 % BC);
        for (int jj = grp; jj < jn; jj += groups) {
          float f[VEC];
          ld16(colp + (size_t)jj * BC, f);
          const float wgt = S[j0 + jj];
#pragma unroll
          for (int i = 0; i < VEC; ++i) acc[i] = fmaf(wgt, f[i], acc[i]);
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive_cta(empty + st);
      if (++st == NST) {
        st = 0;
        ph ^= 1;
      }
    }
    if (grp < groups) {
#pragma unroll
      for (int i = 0; i < VEC; ++i) red[grp * dk + ch * VEC + i] = acc[i];
    }
    consumers_sync();
    T* out = reinterpret_cast<T*>(a.out) + (size_t)it.r * a.ldo + it.h * dk;
    for (int e = ctid; e < dk; e += kNCW * 32) {
      float sum = red[e];
      for (int gg = 1; gg < groups; ++gg) sum += red[gg * dk + e];
      out[e] = from_f32<T>(sum);
    }
    consumers_sync();   // qs / S / red reused by the next item
  }
}

int num_sms_attn() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

template <typename T>
cudaError_t launch_persist(const DecAttnArgs& a, const CUtensorMap& tk, const CUtensorMap& tv,
                           int k_col0, int v_col0, cudaStream_t s) {
  constexpr int NST = 12;
  const int KC = decode_tma_keys_per_chunk(a.dk, a.dtype);
  const int groups = (kNCW * 32) / (a.dk / 8);
  const size_t smem = (size_t)NST * kStageBytes +
                      sizeof(float) * ((size_t)a.dk + a.max_k + 4 + (size_t)groups * a.dk) + 8 +
                      16 * NST;
  if (smem > 227 * 1024) return cudaErrorInvalidValue;
  cudaError_t e = set_max_smem((const void*)attn_decode_persist_kernel<T, NST>);
  if (e != cudaSuccess) return e;
  const int items = a.rows * a.heads;
  const int grid = items < num_sms_attn() ? items : num_sms_attn();
  const float qscale = (float)(1.0 / sqrt((double)a.dk));
  attn_decode_persist_kernel<T, NST><<<grid, kPThreads, smem, s>>>(tk, tv, a, qscale, KC, k_col0,
                                                                    v_col0);
  return cudaGetLastError();
}

}  // namespace

// ~16 KB per ring stage: KC keys of dk 16-bit values (multiple of 8, <= 128 keys)
int decode_tma_keys_per_chunk(int dk, int dtype) {
  const int es = dtype == kF32 ? 4 : 2;
  int kc = kStageBytes / (dk * es);
  kc = kc > 128 ? 128 : kc;
  kc = (kc / 8) * 8;
  return kc < 8 ? 8 : kc;
}

cudaError_t launch_attention_decode_tma(const DecAttnArgs& a, const CUtensorMap& tk,
                                        const CUtensorMap& tv, int k_col0, int v_col0,
                                        cudaStream_t s) {
  if (a.rows <= 0) return cudaSuccess;
  if (a.anc || (a.dtype != kF16 && a.dtype != kBF16) || a.dk % 8 || a.new_k ||
      a.dk * 2 * decode_tma_keys_per_chunk(a.dk, a.dtype) > kStageBytes)
    return cudaErrorInvalidValue;
  if (a.dtype == kF16) return launch_persist<__half>(a, tk, tv, k_col0, v_col0, s);
  return launch_persist<__nv_bfloat16>(a, tk, tv, k_col0, v_col0, s);
}

}  // namespace fnmt
