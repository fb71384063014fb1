// Encoder self-attention on the tensor cores (fp16 / bf16 storage).
//
// Same contract as attn_varlen_kernel (attention.cu; model.py:199-245 via
// encode, model.py:279-281): packed varlen sequences, per-sequence keys only,
// the row softmax computed exactly like tensor.softmax (max shift, exp,
// divide by the in-order row sum, tensor.py:70-81), -1e9 offset when every
// key of a sequence is masked (model.py:37-38).
//
// The encoder sequences are short (newstest mean 24 tokens), so the two
// contractions are tiny per CTA (24 x 24 x 512); what matters is moving
// q/k/v through shared memory with 16-byte loads and doing the dot products
// on the tensor pipe instead of FMA-serial loops.  mma.sync m16n8k16
// (fp16/bf16 in, fp32 accumulate) is the right granularity here: a
// tcgen05 tile (M >= 64, TMEM allocation, mbarrier pipeline) would be
// mostly padding for a 24-row sequence.
//
//   CTA = (64-query tile, sequence, head), 4 warps x 16 query rows.
//   1. S = Q K^T: 64-key x 64-dim tiles of Q and K staged in smem (row
//      stride 72 halves: conflict-free 32-bit fragment loads); each warp
//      accumulates its 16 x 64 score block over the head dimension, scales
//      by 1/sqrt(dk) and writes fp32 scores to smem.
//   2. softmax per query row (one warp per row), probabilities kept fp32.
//   3. O = P V: V tiles [keys x 64 dims] staged row-major, B fragments via
//      ldmatrix.trans; P fragments converted from the fp32 rows.
//
// Numerics vs the fp32 reference: products of fp16 operands are exact and
// accumulate in fp32; the score scale is applied after the dot product
// (the reference scales q first, model.py:223) and P is rounded to the
// storage type for the second product — both well inside the fp16 logits
// tolerance (1e-2).  The fp32 parity mode keeps the SIMT kernel.
#include "common.cuh"
#include "kernels.h"

namespace fnmt {

namespace {

constexpr int kMQ = 64;          // queries per CTA
constexpr int kMK = 64;          // keys per tile
constexpr int kMD = 64;          // head dims per tile
constexpr int kMThreads = 128;   // 4 warps
constexpr int kLds = kMD + 8;    // smem row stride of Q / K / V tiles (halves)
constexpr float kMaskValue = -1e9f;
constexpr int kMaxKeys = 256;    // longer sequences use the SIMT kernel

template <typename T>
__device__ __forceinline__ void mma16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0,
                                         uint32_t b1);
template <>
__device__ __forceinline__ void mma16816<__half>(float (&c)[4], const uint32_t (&a)[4],
                                                 uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
template <>
__device__ __forceinline__ void mma16816<__nv_bfloat16>(float (&c)[4], const uint32_t (&a)[4],
                                                        uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
      "{%8,%9}, {%0,%1,%2,%3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}

template <typename T>
__device__ __forceinline__ uint32_t pack2(float x, float y);
template <>
__device__ __forceinline__ uint32_t pack2<__half>(float x, float y) {
  __half2 h = __floats2half2_rn(x, y);
  return *reinterpret_cast<uint32_t*>(&h);
}
template <>
__device__ __forceinline__ uint32_t pack2<__nv_bfloat16>(float x, float y) {
  __nv_bfloat162 h = __floats2bfloat162_rn(x, y);
  return *reinterpret_cast<uint32_t*>(&h);
}

__device__ __forceinline__ uint32_t lds32(const void* p) {
  return *reinterpret_cast<const uint32_t*>(p);
}

__device__ __forceinline__ void ldmatrix_x4_trans(uint32_t (&r)[4], const void* p) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(smem_u32(p)));
}

// rows [0, n) of a [rows x kMD] tile starting at column c0 of a row-major
// matrix (leading dim ld) into smem (stride kLds); zero outside.
template <typename T>
__device__ __forceinline__ void stage_tile(T* dst, const T* src, int64_t row0, int ld, int n,
                                           int c0, int dk) {
  for (int i = threadIdx.x; i < 64 * (kMD / 8); i += kMThreads) {
    const int r = i >> 3, c8 = (i & 7) * 8;
    uint4 v = make_uint4(0u, 0u, 0u, 0u);
    if (r < n && c0 + c8 < dk) v = *reinterpret_cast<const uint4*>(src + (row0 + r) * ld + c0 + c8);
    *reinterpret_cast<uint4*>(dst + r * kLds + c8) = v;
  }
}

template <typename T>
__global__ void __launch_bounds__(kMThreads)
    attn_varlen_mma_kernel(AttnArgs a, float qscale, int scap) {
  extern __shared__ __align__(16) uint8_t smraw[];
  float* S = reinterpret_cast<float*>(smraw);          // [kMQ][scap] fp32 scores / probabilities
  T* Qs = reinterpret_cast<T*>(S + kMQ * scap);        // [kMQ][kLds]
  T* Ks = Qs + kMQ * kLds;                             // [kMK][kLds]  (V tile in phase 3)
  const int b = blockIdx.y, h = blockIdx.z;
  const int q0 = blockIdx.x * kMQ;
  const int nq = a.q_len[b];
  if (q0 >= nq) return;
  const int kl = a.k_len[b];
  const bool all_masked = kl == 0;
  const int nk = all_masked ? a.k_pad : kl;
  const int qn = min(kMQ, nq - q0);
  const int64_t qrow0 = a.q_start[b] + q0;
  const int64_t krow0 = a.k_start[b];
  const int dk = a.dk;
  const T* q = reinterpret_cast<const T*>(a.q) + h * dk;
  const T* k = reinterpret_cast<const T*>(a.k) + h * dk;
  const T* v = reinterpret_cast<const T*>(a.v) + h * dk;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, tig = lane & 3;
  const int wr = warp * 16;
  const bool live = wr < qn;

  // ---- 1. scores ------------------------------------------------------------
  for (int kt = 0; kt < nk; kt += kMK) {
    float acc[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.f;
    for (int dc = 0; dc < dk; dc += kMD) {
      __syncthreads();
      stage_tile(Qs, q, qrow0, a.ldq, qn, dc, dk);
      stage_tile(Ks, k, krow0 + kt, a.ldkv, nk - kt, dc, dk);
      __syncthreads();
      if (live) {
#pragma unroll
        for (int kk = 0; kk < kMD; kk += 16) {
          uint32_t af[4];
          const T* qa = Qs + (wr + g) * kLds + kk + 2 * tig;
          af[0] = lds32(qa);
          af[1] = lds32(qa + 8 * kLds);
          af[2] = lds32(qa + 8);
          af[3] = lds32(qa + 8 * kLds + 8);
#pragma unroll
          for (int nt = 0; nt < 8; ++nt) {
            const T* kb = Ks + (nt * 8 + g) * kLds + kk + 2 * tig;
            mma16816<T>(acc[nt], af, lds32(kb), lds32(kb + 8));
          }
        }
      }
    }
    if (live) {
#pragma unroll
      for (int nt = 0; nt < 8; ++nt)
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          const int qi = wr + g + 8 * hh;
          const int kj = kt + nt * 8 + 2 * tig;
          float s0 = acc[nt][2 * hh] * qscale, s1 = acc[nt][2 * hh + 1] * qscale;
          if (all_masked) {
            s0 += kMaskValue;
            s1 += kMaskValue;
          }
          *reinterpret_cast<float2*>(S + qi * scap + kj) = make_float2(s0, s1);
        }
    }
  }
  __syncthreads();

  // ---- 2. softmax (tensor.py:70-81), zero past nk / qn ------------------------
  for (int qi = warp; qi < kMQ; qi += kMThreads / 32) {
    float* pr = S + qi * scap;
    if (qi >= qn) {
      if (qi < ((qn + 15) & ~15))
        for (int j = lane; j < scap; j += 32) pr[j] = 0.f;
      continue;
    }
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
    for (int j = nk + lane; j < scap; j += 32) pr[j] = 0.f;
  }

  // ---- 3. O = P V ----------------------------------------------------------------
  T* out = reinterpret_cast<T*>(a.out) + h * dk;
  for (int dc = 0; dc < dk; dc += kMD) {
    float o[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
    for (int kc = 0; kc < nk; kc += kMK) {
      __syncthreads();
      stage_tile(Ks, v, krow0 + kc, a.ldkv, nk - kc, dc, dk);
      __syncthreads();
      if (live) {
#pragma unroll
        for (int kk = 0; kk < kMK; kk += 16) {
          const float* p0 = S + (wr + g) * scap + kc + kk + 2 * tig;
          const float* p1 = p0 + 8 * scap;
          uint32_t af[4];
          af[0] = pack2<T>(p0[0], p0[1]);
          af[1] = pack2<T>(p1[0], p1[1]);
          af[2] = pack2<T>(p0[8], p0[9]);
          af[3] = pack2<T>(p1[8], p1[9]);
          // thread t addresses row (t & 7) of 8x8 matrix t >> 3:
          // m0 keys kk..+7 / dims n0..+7, m1 keys +8, m2 dims +8, m3 both
          const int mi = lane >> 3;
          const int key = kk + (lane & 7) + ((mi & 1) ? 8 : 0);
#pragma unroll
          for (int nt = 0; nt < 8; nt += 2) {
            uint32_t bf[4];
            ldmatrix_x4_trans(bf, Ks + key * kLds + nt * 8 + ((mi & 2) ? 8 : 0));
            mma16816<T>(o[nt], af, bf[0], bf[1]);
            mma16816<T>(o[nt + 1], af, bf[2], bf[3]);
          }
        }
      }
    }
    if (live) {
#pragma unroll
      for (int nt = 0; nt < 8; ++nt)
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          const int qi = wr + g + 8 * hh;
          const int dd = dc + nt * 8 + 2 * tig;
          if (qi < qn && dd < dk)
            *reinterpret_cast<uint32_t*>(out + (qrow0 + qi) * a.ldo + dd) =
                pack2<T>(o[nt][2 * hh], o[nt][2 * hh + 1]);
        }
    }
  }
}

// ---------------------------------------------------------------------------
// Pipelined variant for short sequences (<= 64 keys: the newstest batches).
// Same arithmetic as attn_varlen_mma_kernel (fragment order, fp32 scores,
// softmax, P rounded to T, identical outputs), but the operands stream
// through a 3-stage cp.async ring of head-dim chunks instead of synchronous
// loads: chunks 0..nd-1 carry the (Q, K) columns [64c, 64c+64) of the
// sequence, chunks nd..2nd-1 the V columns; while chunk c is in the tensor
// cores chunks c+1 and c+2 are in flight (the V chunks already load during
// the softmax).  Stages hold only the sequence's rows (RQ queries, RK keys,
// rounded to 16), so several CTAs share an SM.

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// rows [0, n) of the 64-column chunk c0 of a row-major matrix into a stage
// region (row stride kLds); columns past dk are zero-filled (plain stores)
template <typename T>
__device__ __forceinline__ void stage_async(T* dst, const T* src, int64_t row0, int ld, int n,
                                            int c0, int dk) {
  for (int i = threadIdx.x; i < n * (kMD / 8); i += kMThreads) {
    const int r = i >> 3, c8 = (i & 7) * 8;
    if (c0 + c8 < dk)
      cp_async16(dst + r * kLds + c8, src + (row0 + r) * ld + c0 + c8);
    else
      *reinterpret_cast<uint4*>(dst + r * kLds + c8) = make_uint4(0u, 0u, 0u, 0u);
  }
}

template <typename T>
__global__ void __launch_bounds__(kMThreads, 5)
    attn_enc_pipe_kernel(AttnArgs a, float qscale, int RQ, int RK) {
  extern __shared__ __align__(16) uint8_t smraw[];
  const int scap = RK + 4;                              // fp32 score row stride
  float* S = reinterpret_cast<float*>(smraw);           // [RQ][scap]
  T* ring = reinterpret_cast<T*>(S + RQ * scap);        // 3 x [(RQ + RK) x kLds]
  const int stage_elems = (RQ + RK) * kLds;
  const int b = blockIdx.y, h = blockIdx.z;
  const int q0 = blockIdx.x * kMQ;
  const int nq = a.q_len[b];
  if (q0 >= nq) return;
  const int kl = a.k_len[b];
  const bool all_masked = kl == 0;
  const int nk = all_masked ? a.k_pad : kl;
  const int nk16 = (nk + 15) & ~15;
  const int qn = min(kMQ, nq - q0);
  const int64_t qrow0 = a.q_start[b] + q0;
  const int64_t krow0 = a.k_start[b];
  const int dk = a.dk;
  const int nd = (dk + kMD - 1) / kMD;
  const T* q = reinterpret_cast<const T*>(a.q) + h * dk;
  const T* k = reinterpret_cast<const T*>(a.k) + h * dk;
  const T* v = reinterpret_cast<const T*>(a.v) + h * dk;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, tig = lane & 3;
  const int wr = warp * 16;
  const bool live = wr < qn;
  const int ntk = nk16 >> 3;                            // 8-key score tiles in use

  auto load = [&](int c) {
    if (c < 2 * nd) {
      T* st = ring + (c % 3) * stage_elems;
      if (c < nd) {
        stage_async(st, q, qrow0, a.ldq, qn, c * kMD, dk);
        stage_async(st + RQ * kLds, k, krow0, a.ldkv, nk, c * kMD, dk);
      } else {
        stage_async(st, v, krow0, a.ldkv, nk, (c - nd) * kMD, dk);
        // value rows [nk, nk16) meet zero probabilities: make them finite
        for (int i = threadIdx.x; i < (nk16 - nk) * (kMD / 8); i += kMThreads)
          *reinterpret_cast<uint4*>(st + (nk + (i >> 3)) * kLds + (i & 7) * 8) =
              make_uint4(0u, 0u, 0u, 0u);
      }
    }
    cp_async_commit();
  };
  load(0);
  load(1);

  float acc[8][4];
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i][0] = acc[i][1] = acc[i][2] = acc[i][3] = 0.f;
  T* out = reinterpret_cast<T*>(a.out) + h * dk;
  for (int c = 0; c < 2 * nd; ++c) {
    cp_async_wait<1>();
    __syncthreads();
    load(c + 2);
    const T* st = ring + (c % 3) * stage_elems;
    if (c < nd) {
      // ---- scores over head-dim chunk c ----
      if (live) {
        const T* Qs = st;
        const T* Ks = st + RQ * kLds;
#pragma unroll
        for (int kk = 0; kk < kMD; kk += 16) {
          uint32_t af[4];
          const T* qa = Qs + (wr + g) * kLds + kk + 2 * tig;
          af[0] = lds32(qa);
          af[1] = lds32(qa + 8 * kLds);
          af[2] = lds32(qa + 8);
          af[3] = lds32(qa + 8 * kLds + 8);
#pragma unroll
          for (int nt = 0; nt < 8; ++nt) {
            if (nt < ntk) {
              const T* kb = Ks + (nt * 8 + g) * kLds + kk + 2 * tig;
              mma16816<T>(acc[nt], af, lds32(kb), lds32(kb + 8));
            }
          }
        }
      }
      if (c == nd - 1) {
        if (live) {
#pragma unroll
          for (int nt = 0; nt < 8; ++nt)
            if (nt < ntk)
#pragma unroll
              for (int hh = 0; hh < 2; ++hh) {
                const int qi = wr + g + 8 * hh;
                const int kj = nt * 8 + 2 * tig;
                float s0 = acc[nt][2 * hh] * qscale, s1 = acc[nt][2 * hh + 1] * qscale;
                if (all_masked) {
                  s0 += kMaskValue;
                  s1 += kMaskValue;
                }
                *reinterpret_cast<float2*>(S + qi * scap + kj) = make_float2(s0, s1);
              }
        }
        __syncthreads();
        // softmax (tensor.py:70-81); probabilities of keys [nk, nk16) are zero
        for (int qi = warp; qi < RQ; qi += kMThreads / 32) {
          float* pr = S + qi * scap;
          if (qi >= qn) {
            for (int j = lane; j < nk16; j += 32) pr[j] = 0.f;
            continue;
          }
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
          for (int j = nk + lane; j < nk16; j += 32) pr[j] = 0.f;
        }
        __syncthreads();
      }
    } else if (live) {
      // ---- O[:, chunk] = P V[:, chunk] (all keys are in this stage) ----
      const int dc = (c - nd) * kMD;
      float o[8][4];
#pragma unroll
      for (int i = 0; i < 8; ++i) o[i][0] = o[i][1] = o[i][2] = o[i][3] = 0.f;
      for (int kk = 0; kk < nk16; kk += 16) {
        const float* p0 = S + (wr + g) * scap + kk + 2 * tig;
        const float* p1 = p0 + 8 * scap;
        uint32_t af[4];
        af[0] = pack2<T>(p0[0], p0[1]);
        af[1] = pack2<T>(p1[0], p1[1]);
        af[2] = pack2<T>(p0[8], p0[9]);
        af[3] = pack2<T>(p1[8], p1[9]);
        const int mi = lane >> 3;
        const int key = kk + (lane & 7) + ((mi & 1) ? 8 : 0);
#pragma unroll
        for (int nt = 0; nt < 8; nt += 2) {
          uint32_t bf[4];
          ldmatrix_x4_trans(bf, st + key * kLds + nt * 8 + ((mi & 2) ? 8 : 0));
          mma16816<T>(o[nt], af, bf[0], bf[1]);
          mma16816<T>(o[nt + 1], af, bf[2], bf[3]);
        }
      }
#pragma unroll
      for (int nt = 0; nt < 8; ++nt)
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          const int qi = wr + g + 8 * hh;
          const int dd = dc + nt * 8 + 2 * tig;
          if (qi < qn && dd < dk)
            *reinterpret_cast<uint32_t*>(out + (qrow0 + qi) * a.ldo + dd) =
                pack2<T>(o[nt][2 * hh], o[nt][2 * hh + 1]);
        }
    }
  }
  cp_async_wait<0>();
}

bool enc_pipe_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("FNMT_ATTN_PIPE");
    on = !(e && e[0] == '0');
  }
  return on != 0;
}

template <typename T>
cudaError_t pipe_dispatch(const AttnArgs& a, cudaStream_t s) {
  const int RQ = std::min(kMQ, (a.max_q + 15) & ~15);
  const int RK = (a.max_k + 15) & ~15;
  const size_t smem = sizeof(float) * (size_t)RQ * (RK + 4) +
                      sizeof(T) * 3 * (size_t)(RQ + RK) * kLds;
  cudaError_t e = set_max_smem((const void*)attn_enc_pipe_kernel<T>);
  if (e != cudaSuccess) return e;
  dim3 grid((a.max_q + kMQ - 1) / kMQ, a.n_seq, a.heads);
  const float qscale = (float)(1.0 / sqrt((double)a.dk));
  attn_enc_pipe_kernel<T><<<grid, kMThreads, smem, s>>>(a, qscale, RQ, RK);
  return cudaGetLastError();
}

template <typename T>
cudaError_t mma_dispatch(const AttnArgs& a, cudaStream_t s) {
  const int scap = ((a.max_k + kMK - 1) / kMK) * kMK;
  const size_t smem = sizeof(float) * (size_t)kMQ * scap + sizeof(T) * 2 * (size_t)64 * kLds;
  cudaError_t e = set_max_smem((const void*)attn_varlen_mma_kernel<T>);
  if (e != cudaSuccess) return e;
  dim3 grid((a.max_q + kMQ - 1) / kMQ, a.n_seq, a.heads);
  const float qscale = (float)(1.0 / sqrt((double)a.dk));
  attn_varlen_mma_kernel<T><<<grid, kMThreads, smem, s>>>(a, qscale, scap);
  return cudaGetLastError();
}

}  // namespace

bool attention_mma_ok(const AttnArgs& a) {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("FNMT_ATTN_MMA");
    on = !(e && e[0] == '0');
  }
  return on && (a.dtype == kF16 || a.dtype == kBF16) && a.dk % 16 == 0 &&
         a.max_k <= kMaxKeys && (a.ldq % 8) == 0 && (a.ldkv % 8) == 0 && (a.ldo % 2) == 0;
}

cudaError_t launch_attention_varlen_mma(const AttnArgs& a, cudaStream_t s) {
  if (a.n_seq <= 0 || a.max_q <= 0) return cudaSuccess;
  if (enc_pipe_enabled() && std::max(a.max_k, a.k_pad) <= kMK)
    return a.dtype == kF16 ? pipe_dispatch<__half>(a, s) : pipe_dispatch<__nv_bfloat16>(a, s);
  return a.dtype == kF16 ? mma_dispatch<__half>(a, s) : mma_dispatch<__nv_bfloat16>(a, s);
}

}  // namespace fnmt
