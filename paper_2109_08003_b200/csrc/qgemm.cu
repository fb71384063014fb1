// int8 projection GEMM: Projection.apply on a packed-int8 weight
// (model.py:84-90 -> quant8.quantize_activations + quant8.qgemm,
// quant8.py:171-195, :246-278), the paper's Eqs. 3-6 moved onto the B200
// integer tensor cores.
//
//   1. q_minmax_kernel: min / max of the f32 activations [M, K] (one
//      order-preserving 32-bit key each, atomicMax into 8 bytes of scratch).
//   2. q_quant_kernel: u8 activations with the reference's double arithmetic
//      (x / scale + zp, round half away from zero, clip to [0, 255]); row sums
//      in s32; K zero-padded to a multiple of 16 for TMA.
//   3. gemm_tc_kernel<.., I8 = true> (gemm.cu): TMA-fed tcgen05.mma
//      kind::i8 (u8 x s8 -> s32 in TMEM), epilogue expands the zeropoint
//      cross terms in double and rounds once to f32 (q_dequant_chunk), then
//      the usual bias / ReLU / store / argmax / fused-QKV epilogues.
//
// The integer core is exact (|acc| < 255 * 128 * K < 2^31 for K <= 65535),
// so the GEMM output is bit-identical to the reference's qgemm for the same
// quantized operands — independent of tile shape and batch size.
#include "common.cuh"
#include "kernels.h"

namespace fnmt {

namespace {

constexpr int kQThreads = 256;

__global__ void __launch_bounds__(kQThreads)
    q_minmax_kernel(const float* __restrict__ A, int lda, int M, int K, unsigned int* stats) {
  pdl_wait();
  unsigned int kmax = 0u, kmin = 0u;   // kmin holds ~key(min)
  const int64_t total = (int64_t)M * K;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  if ((lda & 3) == 0 && (K & 3) == 0 && (reinterpret_cast<uintptr_t>(A) & 15) == 0) {
    const int kq = K >> 2;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total / 4; i += stride) {
      const int64_t r = i / kq, c = (i - r * kq) * 4;
      const float4 x = *reinterpret_cast<const float4*>(A + r * lda + c);
      const float e[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const unsigned int k = f32_key(e[j]);
        kmax = max(kmax, k);
        kmin = max(kmin, ~k);
      }
    }
  } else {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += stride) {
      const int64_t r = i / K, c = i - r * K;
      const unsigned int k = f32_key(A[r * lda + c]);
      kmax = max(kmax, k);
      kmin = max(kmin, ~k);
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    kmax = max(kmax, __shfl_xor_sync(0xffffffffu, kmax, o));
    kmin = max(kmin, __shfl_xor_sync(0xffffffffu, kmin, o));
  }
  __shared__ unsigned int smax[kQThreads / 32], smin[kQThreads / 32];
  const int w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    smax[w] = kmax;
    smin[w] = kmin;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int i = 1; i < kQThreads / 32; ++i) {
      kmax = max(kmax, smax[i]);
      kmin = max(kmin, smin[i]);
    }
    atomicMax(stats, kmax);
    atomicMax(stats + 1, kmin);
  }
  pdl_trigger();
}

__device__ __forceinline__ uint32_t q_level(float x, double scale, double zp) {
  const double v = __dadd_rn(__ddiv_rn((double)x, scale), zp);
  double r = trunc(__dadd_rn(v, copysign(0.5, v)));
  r = fmin(fmax(r, 0.0), 255.0);
  return (uint32_t)r;
}

// One warp per row: u8 levels + s32 row sum; columns [K, Kp) zero.
__global__ void __launch_bounds__(kQThreads)
    q_quant_kernel(const float* __restrict__ A, int lda, int M, int K, int Kp,
                   const unsigned int* __restrict__ stats, uint8_t* __restrict__ qa,
                   int32_t* __restrict__ rowsum) {
  pdl_wait();
  double scale, zp;
  q_act_params(stats, scale, zp);
  const int lane = threadIdx.x & 31;
  const int warps = kQThreads / 32;
  for (int m = blockIdx.x * warps + (threadIdx.x >> 5); m < M; m += gridDim.x * warps) {
    const float* x = A + (int64_t)m * lda;
    uint8_t* q = qa + (int64_t)m * Kp;
    int sum = 0;
    for (int c = lane * 4; c < Kp; c += 128) {
      uint32_t packed = 0;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (c + j < K) {
          const uint32_t l = q_level(x[c + j], scale, zp);
          sum += (int)l;
          packed |= l << (8 * j);
        }
      }
      *reinterpret_cast<uint32_t*>(q + c) = packed;
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) sum += __shfl_xor_sync(0xffffffffu, sum, o);
    if (lane == 0) rowsum[m] = sum;
  }
  pdl_trigger();
}

int64_t align256(int64_t b) { return (b + 255) & ~int64_t(255); }

}  // namespace

int64_t qgemm_scratch_bytes(int64_t M, int K) {
  return align256(M * round_up16(K)) + align256(4 * M) + 256;
}

QScratch qgemm_scratch(void* base, int64_t M, int K) {
  QScratch q;
  uint8_t* p = reinterpret_cast<uint8_t*>(base);
  q.qa = p;
  q.qa_bytes = align256(M * round_up16(K));
  q.rowsum = reinterpret_cast<int32_t*>(p + q.qa_bytes);
  q.stats = reinterpret_cast<unsigned int*>(p + q.qa_bytes + align256(4 * M));
  q.rows = M;
  return q;
}

cudaError_t launch_qgemm(const GemmArgs& g, cudaStream_t s) {
  if (g.M <= 0 || g.N <= 0) return cudaSuccess;
  if (g.in_dtype != kF32 || !g.qs.qa || !g.qs.rowsum || !g.qs.stats || g.Kp != round_up16(g.K) ||
      g.qs.rows < g.M || g.qs.qa_bytes < (int64_t)g.M * g.Kp || !g.qscale || !g.qzp || !g.qcolsum)
    return cudaErrorInvalidValue;
  const float* A = reinterpret_cast<const float*>(g.A);
  cudaError_t e = cudaMemsetAsync(g.qs.stats, 0, 2 * sizeof(unsigned int), s);
  if (e != cudaSuccess) return e;
  const int64_t total = (int64_t)g.M * g.K;
  int blocks = (int)std::min<int64_t>((total / 4 + kQThreads - 1) / kQThreads + 1, 148 * 4);
  e = launch_k(q_minmax_kernel, dim3(blocks), dim3(kQThreads), 0, s, A, g.lda, g.M, g.K,
               g.qs.stats);
  if (e != cudaSuccess) return e;
  blocks = (int)std::min<int64_t>((g.M + 7) / 8, 148 * 8);
  e = launch_k(q_quant_kernel, dim3(blocks), dim3(kQThreads), 0, s, A, g.lda, g.M, g.K, g.Kp,
               (const unsigned int*)g.qs.stats, g.qs.qa, g.qs.rowsum);
  if (e != cudaSuccess) return e;
  CUtensorMap ta;
  if (!make_tmap_8(&ta, g.qs.qa, g.M, g.Kp, 128, nullptr)) return cudaErrorInvalidValue;
  return launch_tc_i8(ta, g, s);
}

}  // namespace fnmt
