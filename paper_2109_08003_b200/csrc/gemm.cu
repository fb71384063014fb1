// Projection GEMMs: C = A . W^T (+ bias, residual, ReLU) or fused vocab argmax.
//
// Replaces the reference's per-GEMM operator `Projection.apply`
// (model.py:84-90) -> `tensor.matmul` (tensor.py:46-57) and, with the argmax
// epilogue, the vocab projection + `np.argmax` of greedy search
// (model.py:344, search.py:71).
//
// * fp16 / bf16 path: hand-written tcgen05 kernel.  TMA (cp.async.bulk.tensor,
//   128 B swizzle) streams 128x64 A tiles and BNx64 W tiles through a
//   STAGES-deep mbarrier ring; one elected thread issues tcgen05.mma
//   (kind::f16, M=128, N=BN, K=16) into a TMEM fp32 accumulator; four warps
//   drain TMEM with tcgen05.ld and apply the fused epilogue.
// * fp32 path (parity mode, TF32 off): SIMT kernel, fp32 FMA in ascending-k
//   order.
//
// Both paths accumulate every output in a fixed k order that does not depend
// on M, so a sentence's result never depends on its batch neighbours
// (the reference's batch-invariance contract, tensor.py:8-12).
#include <cudaTypedefs.h>

#include <mutex>

#include "common.cuh"
#include "kernels.h"

namespace fnmt {

namespace {

constexpr int kBM = 128;
constexpr int kBK = 64;
constexpr int kBN = 128;
constexpr int kStages = 4;
constexpr int kABytes = kBM * kBK * 2;
constexpr int kBBytes = kBN * kBK * 2;
constexpr int kTcSmem = 1024 + kStages * (kABytes + kBBytes) + 256;

struct EpiParams {
  const float* bias;
  int M, N;
  int epi;
  void* C;
  int ldc;
  int c_dtype;
  int relu;
  const float* resid;
  int ld_resid;
  unsigned long long* keys;
};

__device__ __forceinline__ float epi_value(const EpiParams& e, int m, int n, float acc) {
  float v = acc;
  if (e.bias) v = v + e.bias[n];
  if (e.resid) v = e.resid[(size_t)m * e.ld_resid + n] + v;
  if (e.relu) v = fmaxf(v, 0.f);
  return v;
}

__device__ __forceinline__ void store_elem(const EpiParams& e, int m, int n, float v) {
  size_t off = (size_t)m * e.ldc + n;
  if (e.c_dtype == kF32)
    reinterpret_cast<float*>(e.C)[off] = v;
  else if (e.c_dtype == kF16)
    reinterpret_cast<__half*>(e.C)[off] = __float2half_rn(v);
  else
    reinterpret_cast<__nv_bfloat16*>(e.C)[off] = __float2bfloat16_rn(v);
}

// ---------------------------------------------------------------------------
// tcgen05 kernel

__global__ void __launch_bounds__(128, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tma, const __grid_constant__ CUtensorMap tmw,
                   int K, uint32_t idesc, EpiParams ep) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint8_t* sA = base;
  uint8_t* sB = base + kStages * kABytes;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + kStages * kBBytes);
  uint64_t* empty = full + kStages;
  uint64_t* done = empty + kStages;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(done + 1);

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int n0 = blockIdx.x * kBN;
  const int m0 = blockIdx.y * kBM;
  const int nk = (K + kBK - 1) / kBK;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tma);
    tma_prefetch_desc(&tmw);
    for (int s = 0; s < kStages; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, 1);
    }
    mbar_init(done, 1);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(tslot, kBN);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;

  if (warp == 0 && lane == 0) {
    // TMA producer
    for (int kb = 0; kb < nk; ++kb) {
      const int s = kb % kStages;
      const uint32_t ph = (kb / kStages) & 1;
      mbar_wait(empty + s, ph ^ 1);
      mbar_expect_tx(full + s, kABytes + kBBytes);
      tma_load_2d(sA + s * kABytes, &tma, full + s, kb * kBK, m0);
      tma_load_2d(sB + s * kBBytes, &tmw, full + s, kb * kBK, n0);
    }
  } else if (warp == 1 && lane == 0) {
    // MMA issuer (single thread)
    for (int kb = 0; kb < nk; ++kb) {
      const int s = kb % kStages;
      const uint32_t ph = (kb / kStages) & 1;
      mbar_wait(full + s, ph);
      tc_fence_after();
      const uint64_t ad = umma_desc_sw128(smem_u32(sA + s * kABytes));
      const uint64_t bd = umma_desc_sw128(smem_u32(sB + s * kBBytes));
#pragma unroll
      for (int kk = 0; kk < kBK / 16; ++kk)
        tc_mma_f16(tmem, ad + 2 * kk, bd + 2 * kk, idesc, (kb | kk) != 0 ? 1u : 0u);
      tc_commit(empty + s);
    }
    tc_commit(done);
  }
  __syncwarp();
  mbar_wait(done, 0);
  tc_fence_after();

  // Epilogue: warp w owns TMEM lanes [32w, 32w+32) == tile rows.
  const int m = m0 + warp * 32 + lane;
  const bool row_ok = m < ep.M;
  const uint32_t lane_addr = tmem + ((uint32_t)(warp * 32) << 16);
  unsigned long long best = 0ull;
#pragma unroll 1
  for (int c = 0; c < kBN / 32; ++c) {
    float v[32];
    tmem_ld32(lane_addr + c * 32, v);
    const int nb = n0 + c * 32;
    if (!row_ok || nb >= ep.N) continue;
    if (ep.epi == kEpiArgmax) {
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const int n = nb + i;
        if (n < ep.N) {
          unsigned long long key = argmax_key(v[i] + ep.bias[n], (uint32_t)n);
          best = key > best ? key : best;
        }
      }
      continue;
    }
    const bool full_chunk = nb + 32 <= ep.N;
    if (full_chunk && ep.c_dtype != kF32 && (ep.ldc % 8) == 0 && ep.resid == nullptr) {
      uint32_t packed[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        float a = v[2 * i] + (ep.bias ? ep.bias[nb + 2 * i] : 0.f);
        float b = v[2 * i + 1] + (ep.bias ? ep.bias[nb + 2 * i + 1] : 0.f);
        if (ep.relu) {
          a = fmaxf(a, 0.f);
          b = fmaxf(b, 0.f);
        }
        if (ep.c_dtype == kF16) {
          __half2 h = __floats2half2_rn(a, b);
          packed[i] = *reinterpret_cast<uint32_t*>(&h);
        } else {
          __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
          packed[i] = *reinterpret_cast<uint32_t*>(&h);
        }
      }
      uint4* dst = reinterpret_cast<uint4*>(reinterpret_cast<uint16_t*>(ep.C) +
                                            (size_t)m * ep.ldc + nb);
#pragma unroll
      for (int i = 0; i < 4; ++i)
        dst[i] = make_uint4(packed[4 * i], packed[4 * i + 1], packed[4 * i + 2], packed[4 * i + 3]);
    } else {
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const int n = nb + i;
        if (n < ep.N) store_elem(ep, m, n, epi_value(ep, m, n, v[i]));
      }
    }
  }
  if (ep.epi == kEpiArgmax && row_ok && best != 0ull) atomicMax(ep.keys + m, best);

  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, kBN);
}

// ---------------------------------------------------------------------------
// SIMT fp32 kernel (parity mode: true fp32, ascending-k FMA)

constexpr int kSB = 64, kSK = 16;

__global__ void __launch_bounds__(256)
    gemm_simt_kernel(const float* __restrict__ A, int lda, const float* __restrict__ W, int ldw,
                     int K, EpiParams ep) {
  __shared__ float As[kSK][kSB + 4];
  __shared__ float Ws[kSK][kSB + 4];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int m0 = blockIdx.y * kSB, n0 = blockIdx.x * kSB;
  float acc[4][4] = {};
  for (int k0 = 0; k0 < K; k0 += kSK) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int idx = threadIdx.x + 256 * i;
      const int r = idx >> 4, kk = idx & 15;
      const int gm = m0 + r, gn = n0 + r, gk = k0 + kk;
      As[kk][r] = (gm < ep.M && gk < K) ? A[(size_t)gm * lda + gk] : 0.f;
      Ws[kk][r] = (gn < ep.N && gk < K) ? W[(size_t)gn * ldw + gk] : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int kk = 0; kk < kSK; ++kk) {
      float a[4], w[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        a[i] = As[kk][ty * 4 + i];
        w[i] = Ws[kk][tx * 4 + i];
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fmaf(a[i], w[j], acc[i][j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int m = m0 + ty * 4 + i;
    if (m >= ep.M) continue;
    unsigned long long best = 0ull;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int n = n0 + tx * 4 + j;
      if (n >= ep.N) continue;
      if (ep.epi == kEpiArgmax) {
        unsigned long long key = argmax_key(acc[i][j] + ep.bias[n], (uint32_t)n);
        best = key > best ? key : best;
      } else {
        store_elem(ep, m, n, epi_value(ep, m, n, acc[i][j]));
      }
    }
    if (ep.epi == kEpiArgmax && best) atomicMax(ep.keys + m, best);
  }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

}  // namespace

int gemm_tile_n() { return kBN; }

bool make_tmap_16(CUtensorMap* out, const void* base, int dtype, int64_t rows, int64_t cols,
                  int64_t ld, int box_rows, std::string* err) {
  auto fn = encode_fn();
  if (!fn) {
    if (err) *err = "cuTensorMapEncodeTiled unavailable (driver too old?)";
    return false;
  }
  if ((reinterpret_cast<uintptr_t>(base) & 15) || ((ld * 2) & 15)) {
    if (err) *err = "TMA operand must be 16-byte aligned with a leading dimension multiple of 8";
    return false;
  }
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * 2)};
  cuuint32_t box[2] = {(cuuint32_t)kBK, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(out, dtype == kBF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16,
                  2, const_cast<void*>(base), dims, strides, box, estr,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    if (err) *err = "cuTensorMapEncodeTiled failed with CUresult " + std::to_string((int)r);
    return false;
  }
  return true;
}

cudaError_t launch_gemm(const GemmArgs& g, cudaStream_t s) {
  if (g.M <= 0 || g.N <= 0) return cudaSuccess;
  EpiParams ep{g.bias, g.M, g.N, g.epi, g.C, g.ldc, g.c_dtype, g.relu, g.resid, g.ld_resid, g.keys};
  if (g.in_dtype == kF32) {
    dim3 grid((g.N + kSB - 1) / kSB, (g.M + kSB - 1) / kSB);
    gemm_simt_kernel<<<grid, 256, 0, s>>>(reinterpret_cast<const float*>(g.A), g.lda,
                                          reinterpret_cast<const float*>(g.W), g.ldw, g.K, ep);
    return cudaGetLastError();
  }
  CUtensorMap ta, tw;
  const CUtensorMap* pa = g.tmap_a;
  const CUtensorMap* pw = g.tmap_w;
  if (!pa) {
    if (!make_tmap_16(&ta, g.A, g.in_dtype, g.M, g.K, g.lda, kBM, nullptr))
      return cudaErrorInvalidValue;
    pa = &ta;
  }
  if (!pw) {
    if (!make_tmap_16(&tw, g.W, g.in_dtype, g.N, g.K, g.ldw, kBN, nullptr))
      return cudaErrorInvalidValue;
    pw = &tw;
  }
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(gemm_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         kTcSmem);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  dim3 grid((g.N + kBN - 1) / kBN, (g.M + kBM - 1) / kBM);
  const uint32_t idesc = umma_idesc_f16(kBM, kBN, g.in_dtype == kBF16);
  gemm_tc_kernel<<<grid, 128, kTcSmem, s>>>(*pa, *pw, g.K, idesc, ep);
  return cudaGetLastError();
}

}  // namespace fnmt
