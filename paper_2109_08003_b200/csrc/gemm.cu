// Projection GEMMs: C = A . W^T (+ bias, residual, ReLU) or fused vocab argmax.
//
// Replaces the reference's per-GEMM operator `Projection.apply`
// (model.py:84-90) -> `tensor.matmul` (tensor.py:46-57) and, with the argmax
// epilogue, the vocab projection + `np.argmax` of greedy search
// (model.py:344, search.py:71).
//
// * fp16 / bf16 path: persistent, warp-specialised tcgen05 kernel.
//     warp 0      TMA producer: 128x64 A tiles and BNx64 W tiles
//                 (cp.async.bulk.tensor, 128 B swizzle) into a STAGES-deep
//                 mbarrier ring;
//     warp 1      one elected thread issues tcgen05.mma (kind::f16, M=128,
//                 N=BN, K=16) into one of two TMEM fp32 accumulators;
//     warps 2..5  epilogue: tcgen05.ld the finished accumulator, apply
//                 bias / residual / ReLU / dtype cast (or the argmax
//                 reduction), release the TMEM buffer.
//   The double-buffered accumulator lets the epilogue of tile i overlap the
//   MMAs of tile i+1.  BN (64/128/256) is chosen per problem so that skinny
//   decoder GEMMs still fill the 148 SMs.
// * fp32 path (parity mode, TF32 off): SIMT kernel, fp32 FMA in ascending-k
//   order.
//
// Every output is accumulated in a fixed k order that does not depend on M or
// on the tile shape, so a sentence's result never depends on its batch
// neighbours (the reference's batch-invariance contract, tensor.py:8-12).
#include <cudaTypedefs.h>

#include <mutex>

#include "common.cuh"
#include "kernels.h"

namespace fnmt {

namespace {

constexpr int kBM = 128;
constexpr int kBK = 64;
constexpr int kWBox = 64;   // W TMA box rows; BN/64 boxes per stage
constexpr int kABytes = kBM * kBK * 2;

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
  TopKPartials tk;
  void* kc;
  void* vc;
  int cap, seg;
  const int32_t* t_ptr;
  // int8 path: per-column weight scale / zeropoint / column sums, per-row
  // activation sums, activation min / max keys, real (unpadded) K
  const float* qscale;
  const float* qzp;
  const int32_t* qcolsum;
  const int32_t* rowsum;
  const unsigned int* stats;
  int qk;
  const int32_t* m_tab;   // GemmArgs::m_tab (with t_ptr)
};

// kEpiQKV destination of output element (m, n): q columns go to C, k / v
// columns to this step's KV-cache slot.
__device__ __forceinline__ void* qkv_dst(const EpiParams& ep, int m, int n, int t, int es) {
  const int sec = n / ep.seg, col = n - sec * ep.seg;
  if (sec == 0) return reinterpret_cast<uint8_t*>(ep.C) + ((size_t)m * ep.ldc + col) * es;
  uint8_t* cache = reinterpret_cast<uint8_t*>(sec == 1 ? ep.kc : ep.vc);
  return cache + (((size_t)m * ep.cap + t) * ep.seg + col) * es;
}

// Output row of accumulator row m: kEpiSlot writes row m into this step's
// cache slot m * cap + t (the folded self-attention cache, engine.cu).
__device__ __forceinline__ size_t out_row(const EpiParams& e, int m) {
  return e.epi == kEpiSlot ? (size_t)m * e.cap + *e.t_ptr : (size_t)m;
}

__device__ __forceinline__ float epi_value(const EpiParams& e, int m, int n, float acc) {
  float v = acc;
  if (e.bias) v = v + e.bias[n];
  if (e.resid) v = e.resid[(size_t)m * e.ld_resid + n] + v;
  if (e.relu) v = fmaxf(v, 0.f);
  return v;
}

__device__ __forceinline__ void store_elem(const EpiParams& e, int m, int n, float v) {
  if (e.epi == kEpiQKV) {
    void* p = qkv_dst(e, m, n, *e.t_ptr, e.c_dtype == kF32 ? 4 : 2);
    if (e.c_dtype == kF32)
      *reinterpret_cast<float*>(p) = v;
    else if (e.c_dtype == kF16)
      *reinterpret_cast<__half*>(p) = __float2half_rn(v);
    else
      *reinterpret_cast<__nv_bfloat16*>(p) = __float2bfloat16_rn(v);
    return;
  }
  size_t off = out_row(e, m) * e.ldc + n;
  if (e.c_dtype == kF32)
    reinterpret_cast<float*>(e.C)[off] = v;
  else if (e.c_dtype == kF16)
    reinterpret_cast<__half*>(e.C)[off] = __float2half_rn(v);
  else
    reinterpret_cast<__nv_bfloat16*>(e.C)[off] = __float2bfloat16_rn(v);
}

__device__ __forceinline__ void named_bar_sync(int id, int threads) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(threads) : "memory");
}

// Apply the epilogue to 32 consecutive accumulator columns of row m.  `bs`
// holds the bias of these columns in shared memory (zeros past N).  For the
// argmax epilogue the running (value, index) pair is kept in registers; a
// strict '>' over ascending columns keeps the lowest index on ties.
__device__ __forceinline__ void epilogue_chunk(const EpiParams& ep, int m, int nb,
                                               const float (&v)[32], const float* bs,
                                               float& best_v, int& best_i) {
  if (ep.epi == kEpiArgmax) {
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      const float x = v[i] + bs[i];
      if (nb + i < ep.N && x > best_v) {
        best_v = x;
        best_i = nb + i;
      }
    }
    return;
  }
  if (ep.epi == kEpiQKV) {
    const int t = *ep.t_ptr;
    const int es = ep.c_dtype == kF32 ? 4 : 2;
    const bool one_section = (nb % ep.seg) + 32 <= ep.seg && nb + 32 <= ep.N;
    if (one_section && es == 2 && (ep.seg % 8) == 0 && (ep.ldc % 8) == 0) {
      uint32_t packed[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const float a = v[2 * i] + bs[2 * i], b = v[2 * i + 1] + bs[2 * i + 1];
        if (ep.c_dtype == kF16) {
          __half2 hh = __floats2half2_rn(a, b);
          packed[i] = *reinterpret_cast<uint32_t*>(&hh);
        } else {
          __nv_bfloat162 hh = __floats2bfloat162_rn(a, b);
          packed[i] = *reinterpret_cast<uint32_t*>(&hh);
        }
      }
      uint4* dst = reinterpret_cast<uint4*>(qkv_dst(ep, m, nb, t, 2));
#pragma unroll
      for (int i = 0; i < 4; ++i)
        dst[i] = make_uint4(packed[4 * i], packed[4 * i + 1], packed[4 * i + 2], packed[4 * i + 3]);
      return;
    }
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      const int n = nb + i;
      if (n >= ep.N) continue;
      const float x = v[i] + bs[i];
      void* p = qkv_dst(ep, m, n, t, es);
      if (ep.c_dtype == kF32)
        *reinterpret_cast<float*>(p) = x;
      else if (ep.c_dtype == kF16)
        *reinterpret_cast<__half*>(p) = __float2half_rn(x);
      else
        *reinterpret_cast<__nv_bfloat16*>(p) = __float2bfloat16_rn(x);
    }
    return;
  }
  const bool full_chunk = nb + 32 <= ep.N;
  if (full_chunk && ep.c_dtype != kF32 && (ep.ldc % 8) == 0 && ep.resid == nullptr) {
    uint32_t packed[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      float a = v[2 * i] + bs[2 * i];
      float b = v[2 * i + 1] + bs[2 * i + 1];
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
    uint4* dst =
        reinterpret_cast<uint4*>(reinterpret_cast<uint16_t*>(ep.C) + out_row(ep, m) * ep.ldc + nb);
#pragma unroll
    for (int i = 0; i < 4; ++i)
      dst[i] = make_uint4(packed[4 * i], packed[4 * i + 1], packed[4 * i + 2], packed[4 * i + 3]);
    return;
  }
  if (full_chunk && ep.c_dtype == kF32 && (ep.ldc % 4) == 0 &&
      (ep.resid == nullptr || (ep.ld_resid % 4) == 0)) {
    float4* dst = reinterpret_cast<float4*>(reinterpret_cast<float*>(ep.C) + out_row(ep, m) * ep.ldc + nb);
    const float4* res = ep.resid ? reinterpret_cast<const float4*>(ep.resid + (size_t)m * ep.ld_resid + nb)
                                 : nullptr;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      float4 o;
      o.x = v[4 * i] + bs[4 * i];
      o.y = v[4 * i + 1] + bs[4 * i + 1];
      o.z = v[4 * i + 2] + bs[4 * i + 2];
      o.w = v[4 * i + 3] + bs[4 * i + 3];
      if (res) {
        const float4 r = res[i];
        o.x = r.x + o.x;
        o.y = r.y + o.y;
        o.z = r.z + o.z;
        o.w = r.w + o.w;
      }
      if (ep.relu) {
        o.x = fmaxf(o.x, 0.f);
        o.y = fmaxf(o.y, 0.f);
        o.z = fmaxf(o.z, 0.f);
        o.w = fmaxf(o.w, 0.f);
      }
      dst[i] = o;
    }
    return;
  }
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    const int n = nb + i;
    if (n < ep.N) {
      float x = v[i] + bs[i];
      if (ep.resid) x = ep.resid[(size_t)m * ep.ld_resid + n] + x;
      if (ep.relu) x = fmaxf(x, 0.f);
      store_elem(ep, m, n, x);
    }
  }
}

// int8 epilogue: turn 32 s32 accumulators of row m into the f32 value of
// quant8.qgemm (quant8.py:246-278) — the zeropoint cross terms expanded
// against the row / column sums, evaluated in double in the reference's
// operation order with explicit round-to-nearest ops (no FMA contraction),
// then rounded once to f32:
//   corr = ((acc - bzp*rowsum) - azp*colsum) + (K*azp)*bzp
//   out  = f32((ascale*bscale) * corr)
__device__ __forceinline__ void q_dequant_chunk(const EpiParams& ep, int m, float (&v)[32],
                                                const float* sc, const float* zp,
                                                const int32_t* cs) {
  double ascale, azp;
  q_act_params(ep.stats, ascale, azp);
  const double kazp = __dmul_rn((double)ep.qk, azp);
  const double rs = (double)ep.rowsum[m];
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    const double acc = (double)__float_as_int(v[i]);
    const double bz = (double)zp[i];
    double t = __dsub_rn(acc, __dmul_rn(bz, rs));
    t = __dsub_rn(t, __dmul_rn(azp, (double)cs[i]));
    t = __dadd_rn(t, __dmul_rn(kazp, bz));
    v[i] = __double2float_rn(__dmul_rn(__dmul_rn(ascale, (double)sc[i]), t));
  }
}

constexpr int kEpiWarps = 8;                       // 2 per TMEM lane quarter
constexpr int kTcThreads = 64 + kEpiWarps * 32;    // producer + MMA warps, epilogue

// ---------------------------------------------------------------------------
// persistent tcgen05 kernel

// Every stage row is 128 bytes of K: 64 fp16/bf16 elements, or 128 int8.
// TS (TMA-store epilogue): every epilogue warp owns two 4 KB staging buffers
// (a 32-row x 32-column chunk, swizzled) that TMA stores to global memory
constexpr int kStageWarpBytes = 2 * 4096;

template <int BN, int STAGES, bool I8 = false, int TK = 0, int NACC = 2, bool TS = false>
struct TcCfg {
  // TK (beam top-K epilogue): per-row exchange of the two column halves' partials
  static constexpr int kTkBytes = TK ? kBM * (4 + 8 + 8 * TK) : 0;
  static constexpr int kBKe = I8 ? 2 * kBK : kBK;   // K elements per stage
  static constexpr int kBBytes = BN * kBK * 2;
  static constexpr int kStage = kABytes + kBBytes;
  static constexpr int kTmemCols = NACC * BN;   // NACC = 2: double-buffered accumulator
  static constexpr int kColBytes = I8 ? 16 : 4;   // bias (+ scale, zeropoint, column sum)
  static constexpr int kOut = TS ? 1024 + kEpiWarps * kStageWarpBytes : 0;
  static constexpr int kSmem = 1024 + STAGES * kStage + 2 * BN * kColBytes + kTkBytes + 256 + kOut;
};

// Tile of this CTA's it-th iteration (-1 when done): a grid-stride walk.
__device__ __forceinline__ int tile_at(int it, int tiles) {
  const int t = blockIdx.x + it * gridDim.x;
  return t < tiles ? t : -1;
}

// tile -> (row block, column block)
__device__ __forceinline__ void tile_coords(int tile, int tiles_n, int BN, int& m0, int& n0) {
  m0 = (tile / tiles_n) * kBM;
  n0 = (tile % tiles_n) * BN;
}


__device__ __forceinline__ float4 lds_f4(const float* p) {
  float4 r;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "r"(smem_u32(p)));
  return r;
}

__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Beam epilogue for one row of a 256-column tile (kTopKTile): each of the two
// warps of a TMEM lane quarter makes two passes over its 128-column half (max
// + running top-K, then sum of exp(x - max)); the half-1 warp hands its
// partial to the half-0 warp through shared memory, which merges them (max,
// rescaled sum, top-K in (value desc, index asc) order — half 0 holds the
// lower indices, so a strict '>' keeps ties on the lower id) and writes one
// partial per (row, tile) for beam_row_reduce (beam.cu).
template <int BN, int TOPK>
__device__ __forceinline__ void topk_epilogue(const EpiParams& ep, uint32_t taddr, const float* bs,
                                              int m, bool row_ok, int n0, int half, int row,
                                              uint8_t* scratch) {
  static_assert(BN == kTopKTile, "a 256-column tile per top-K partial");
  float mx = -INFINITY;
  float tv[TOPK];
  int ti[TOPK];
#pragma unroll
  for (int j = 0; j < TOPK; ++j) {
    tv[j] = -INFINITY;
    ti[j] = -1;
  }
  // pass 1: half-tile max and running top-K.  A chunk whose max does not beat
  // the current K-th value cannot change the top-K, so the insertion network
  // runs only for the (rare, after the first chunk) chunks that can.  The
  // bias chunk comes from shared memory as 16-byte vectors.
  constexpr float kLog2e = 1.4426950408889634f;
#pragma unroll 1
  for (int c = 0; c < BN / 64; ++c) {
    float v[32];
    tmem_ld32(taddr + c * 32, v);
    const int nb = n0 + c * 32;
    const int nv = min(32, ep.N - nb);   // valid columns of this chunk (may be <= 0)
    float cm = -INFINITY;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const float4 b = lds_f4(bs + c * 32 + 4 * q);
      v[4 * q] += b.x;
      v[4 * q + 1] += b.y;
      v[4 * q + 2] += b.z;
      v[4 * q + 3] += b.w;
    }
    if (nv < 32) {
#pragma unroll
      for (int i = 0; i < 32; ++i)
        if (i >= nv) v[i] = -INFINITY;
    }
#pragma unroll
    for (int i = 0; i < 32; ++i) cm = fmaxf(cm, v[i]);
    mx = fmaxf(mx, cm);
    if (cm > tv[TOPK - 1]) {
#pragma unroll
      for (int i = 0; i < 32; ++i) {
        const float x = v[i];
        if (x > tv[TOPK - 1]) {
          tv[TOPK - 1] = x;
          ti[TOPK - 1] = nb + i;
#pragma unroll
          for (int j = TOPK - 1; j > 0; --j) {
            if (tv[j] > tv[j - 1]) {
              const float fv = tv[j];
              tv[j] = tv[j - 1];
              tv[j - 1] = fv;
              const int iv = ti[j];
              ti[j] = ti[j - 1];
              ti[j - 1] = iv;
            }
          }
        }
      }
    }
  }
  // pass 2: sum of exp(x - max) over the valid columns, exp as 2^(x log2e -
  // max log2e) on the MUFU (flush-to-zero: terms below 2^-126 vanish next to
  // the max's 1)
  double sum = 0.0;
  const float mxl = mx * kLog2e;
#pragma unroll 1
  for (int c = 0; c < BN / 64; ++c) {
    float v[32];
    tmem_ld32(taddr + c * 32, v);
    const int nv = min(32, ep.N - (n0 + c * 32));
    float cs = 0.f;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      const float4 b = lds_f4(bs + c * 32 + 4 * q);
      const float x[4] = {v[4 * q] + b.x, v[4 * q + 1] + b.y, v[4 * q + 2] + b.z,
                          v[4 * q + 3] + b.w};
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const float e = ex2_approx(fmaf(x[k], kLog2e, -mxl));
        cs += (4 * q + k < nv) ? e : 0.f;
      }
    }
    sum += (double)cs;
  }
  float* smx = reinterpret_cast<float*>(scratch);                 // [kBM]
  double* ssum = reinterpret_cast<double*>(scratch + 4 * kBM);     // [kBM]
  float* stv = reinterpret_cast<float*>(scratch + 12 * kBM);       // [TOPK][kBM]
  int* sti = reinterpret_cast<int*>(scratch + (12 + 4 * TOPK) * kBM);
  if (half == 1) {
    smx[row] = mx;
    ssum[row] = sum;
#pragma unroll
    for (int j = 0; j < TOPK; ++j) {
      stv[j * kBM + row] = tv[j];
      sti[j * kBM + row] = ti[j];
    }
  }
  named_bar_sync(1, kEpiWarps * 32);
  if (half != 0) return;
  const float m1 = smx[row];
  const float M = fmaxf(mx, m1);
  double tot = 0.0;
  if (mx > -INFINITY) tot += sum * exp((double)mx - (double)M);
  if (m1 > -INFINITY) tot += ssum[row] * exp((double)m1 - (double)M);
#pragma unroll
  for (int k = 0; k < TOPK; ++k) {
    const float x = stv[k * kBM + row];
    if (x > tv[TOPK - 1]) {
      tv[TOPK - 1] = x;
      ti[TOPK - 1] = sti[k * kBM + row];
#pragma unroll
      for (int j = TOPK - 1; j > 0; --j) {
        if (tv[j] > tv[j - 1]) {
          const float fv = tv[j];
          tv[j] = tv[j - 1];
          tv[j - 1] = fv;
          const int iv = ti[j];
          ti[j] = ti[j - 1];
          ti[j - 1] = iv;
        }
      }
    }
  }
  if (row_ok && n0 < ep.N) {
    const size_t o = (size_t)m * ep.tk.tiles + n0 / kTopKTile;
    ep.tk.pmax[o] = M;
    ep.tk.psum[o] = tot;
#pragma unroll
    for (int j = 0; j < TOPK; ++j) {
      ep.tk.pval[o * TOPK + j] = tv[j];
      ep.tk.pidx[o * TOPK + j] = ti[j];
    }
  }
}

// TMA-store epilogue (Projection.apply's output, model.py:84-90): stage 32
// rows x 32 columns of output (row = lane) into a swizzled chunk buffer and
// TMA-store it at (column nb, row m0r).  fp16 / bf16: 64-byte rows,
// SWIZZLE_64B (16-byte unit k of row r at k ^ ((r >> 1) & 3)); fp32: 128-byte
// rows, SWIZZLE_128B (unit k at k ^ (r & 7)) -- conflict-free shared stores.
__device__ __forceinline__ void ts_store_chunk(const EpiParams& ep, const CUtensorMap* tmc,
                                               uint8_t* buf, int lane, int nb, int m0r,
                                               const float (&v)[32], const float* bs) {
  bulk_wait_read<1>();   // this buffer's previous store (two chunks ago) has been read
  __syncwarp();
  if (ep.c_dtype == kF32) {
    uint4* row = reinterpret_cast<uint4*>(buf + lane * 128);
#pragma unroll
    for (int k = 0; k < 8; ++k) {
      float o[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        o[i] = v[4 * k + i] + bs[4 * k + i];
        if (ep.relu) o[i] = fmaxf(o[i], 0.f);
      }
      row[k ^ (lane & 7)] = make_uint4(__float_as_uint(o[0]), __float_as_uint(o[1]),
                                       __float_as_uint(o[2]), __float_as_uint(o[3]));
    }
  } else {
    uint4* row = reinterpret_cast<uint4*>(buf + lane * 64);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      uint32_t pk[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        float a = v[8 * k + 2 * i] + bs[8 * k + 2 * i];
        float b = v[8 * k + 2 * i + 1] + bs[8 * k + 2 * i + 1];
        if (ep.relu) {
          a = fmaxf(a, 0.f);
          b = fmaxf(b, 0.f);
        }
        if (ep.c_dtype == kF16) {
          __half2 h = __floats2half2_rn(a, b);
          pk[i] = *reinterpret_cast<uint32_t*>(&h);
        } else {
          __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
          pk[i] = *reinterpret_cast<uint32_t*>(&h);
        }
      }
      row[k ^ ((lane >> 1) & 3)] = make_uint4(pk[0], pk[1], pk[2], pk[3]);
    }
  }
  fence_proxy_async_smem();   // generic-proxy writes -> visible to the TMA engine
  __syncwarp();
  if (lane == 0) {
    tma_store_2d(tmc, buf, nb, m0r);
    bulk_commit();
  }
}

template <int BN, int STAGES, int TOPK, bool I8 = false, int MINB = 1, int NACC = 2,
          bool TS = false>
__global__ void __launch_bounds__(kTcThreads, MINB)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tma, const __grid_constant__ CUtensorMap tmw,
                   const __grid_constant__ CUtensorMap tmc, int K, uint32_t idesc, EpiParams ep,
                   int tiles_n, int tiles) {
  using Cfg = TcCfg<BN, STAGES, I8, TOPK, NACC, TS>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* base = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  uint8_t* sA = base;
  uint8_t* sB = base + STAGES * kABytes;
  float* bias_s = reinterpret_cast<float*>(sB + STAGES * Cfg::kBBytes);   // [2][BN]
  // int8: [2][BN] column scale, zeropoint, column sum after the bias
  float* qsc_s = bias_s + 2 * BN;
  float* qzp_s = qsc_s + (I8 ? 2 * BN : 0);
  int32_t* qcs_s = reinterpret_cast<int32_t*>(qzp_s + (I8 ? 2 * BN : 0));
  // TOPK: half exchange (8-byte aligned: everything before is a multiple of 8 bytes)
  uint8_t* tks = reinterpret_cast<uint8_t*>(bias_s + (Cfg::kColBytes / 4) * 2 * BN);
  uint64_t* full = reinterpret_cast<uint64_t*>(tks + Cfg::kTkBytes);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tslot = reinterpret_cast<uint32_t*>(tempty + 2);
  // TS staging: 1024-byte aligned (the 128-byte swizzle period), after the barriers
  uint8_t* ostage = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(tslot) + 16 + 1023) & ~static_cast<uintptr_t>(1023));

  const int warp = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int nk = (K + Cfg::kBKe - 1) / Cfg::kBKe;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tma);
    tma_prefetch_desc(&tmw);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full + s, 1);
      mbar_init(empty + s, 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(tfull + b, 1);
      mbar_init(tempty + b, kEpiWarps);
    }
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc(tslot, Cfg::kTmemCols);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  // PDL: barrier init / TMEM alloc / descriptor prefetch above overlap the
  // predecessor's tail; A (and everything else) is read only after this.
  pdl_trigger();
  pdl_wait();
  // greedy decode: only the row blocks that still hold rows inside their budget
  if (ep.m_tab) {
    const int mv = min(ep.M, ep.m_tab[*ep.t_ptr]);
    tiles = tiles_n * ((mv + kBM - 1) / kBM);
  }

  if (warp == 0) {
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      for (int it = 0;; ++it) {
        const int tile = tile_at(it, tiles);
        if (tile < 0) break;
        int m0, n0;
        tile_coords(tile, tiles_n, BN, m0, n0);
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait(empty + s, ph ^ 1);
          mbar_expect_tx(full + s, Cfg::kStage);
          tma_load_2d(sA + s * kABytes, &tma, full + s, kb * Cfg::kBKe, m0);
#pragma unroll
          for (int j = 0; j < BN / kWBox; ++j)
            tma_load_2d(sB + s * Cfg::kBBytes + j * kWBox * 128, &tmw, full + s, kb * Cfg::kBKe,
                        n0 + j * kWBox);
          if (++s == STAGES) {
            s = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      int s = 0;
      uint32_t ph = 0;
      int acc = 0;
      uint32_t aph = 0;
      for (int it = 0;; ++it) {
        const int tile = tile_at(it, tiles);
        if (tile < 0) break;
        // last N tile: the MMA covers only the valid columns (rounded to 16),
        // e.g. the 8-column tail of the folded [K~ | V~ | c] cache rows
        uint32_t id = idesc;
        int m0, n0;
        tile_coords(tile, tiles_n, BN, m0, n0);
        const int rem = ep.N - n0;
        if (rem < BN) {
          const int nt = rem < 16 ? 16 : (rem + 15) & ~15;
          id = (idesc & ~(0x3Fu << 17)) | ((uint32_t)(nt >> 3) << 17);
        }
        mbar_wait(tempty + acc, aph ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + acc * BN;
        for (int kb = 0; kb < nk; ++kb) {
          mbar_wait(full + s, ph);
          tc_fence_after();
          const uint64_t ad = umma_desc_sw128(smem_u32(sA + s * kABytes));
          const uint64_t bd = umma_desc_sw128(smem_u32(sB + s * Cfg::kBBytes));
          // 4 MMAs of 32 bytes of K each (K = 16 fp16 or K = 32 int8)
#pragma unroll
          for (int kk = 0; kk < 4; ++kk) {
            if constexpr (I8)
              tc_mma_i8(d, ad + 2 * kk, bd + 2 * kk, id, (kb | kk) != 0 ? 1u : 0u);
            else
              tc_mma_f16(d, ad + 2 * kk, bd + 2 * kk, id, (kb | kk) != 0 ? 1u : 0u);
          }
          tc_commit(empty + s);
          if (++s == STAGES) {
            s = 0;
            ph ^= 1;
          }
        }
        tc_commit(tfull + acc);
        if (++acc == NACC) {
          acc = 0;
          aph ^= 1;
        }
      }
    }
  } else {
    // epilogue warps 2..9: TMEM lane quarter = warp % 4 (hardware rule), and
    // the two warps of a quarter split the tile's columns in halves.
    const int quarter = warp & 3;
    const int half = (warp - 2) >> 2;
    int acc = 0;
    uint32_t aph = 0;
    for (int it = 0;; ++it) {
      const int tile = tile_at(it, tiles);
      if (tile < 0) break;
      int m0, n0;
      tile_coords(tile, tiles_n, BN, m0, n0);
      // stage this tile's bias while the MMAs run (double-buffered by acc)
      float* bs = bias_s + acc * BN;
      for (int i = threadIdx.x - 64; i < BN; i += kEpiWarps * 32) {
        const bool in = n0 + i < ep.N;
        bs[i] = (ep.bias && in) ? ep.bias[n0 + i] : 0.f;
        if constexpr (I8) {
          qsc_s[acc * BN + i] = in ? ep.qscale[n0 + i] : 0.f;
          qzp_s[acc * BN + i] = in ? ep.qzp[n0 + i] : 0.f;
          qcs_s[acc * BN + i] = in ? ep.qcolsum[n0 + i] : 0;
        }
      }
      named_bar_sync(1, kEpiWarps * 32);
      mbar_wait(tfull + acc, aph);
      tc_fence_after();
      const int m = m0 + quarter * 32 + lane;
      const bool row_ok = m < ep.M;
      const int col0 = half * (BN / 2);
      const uint32_t taddr = tmem + acc * BN + col0 + ((uint32_t)(quarter * 32) << 16);
      if constexpr (TOPK > 0) {
        topk_epilogue<BN, TOPK>(ep, taddr, bs + col0, m, row_ok, n0 + col0, half,
                                quarter * 32 + lane, tks);
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(tempty + acc);
      } else {
        float best_v = -INFINITY;
        int best_i = -1;
        if constexpr (TS) {
          uint8_t* stg = ostage + (warp - 2) * kStageWarpBytes;
#pragma unroll 1
          for (int c = 0; c < BN / 64; ++c) {
            float v[32];
            tmem_ld32(taddr + c * 32, v);
            const int nb = n0 + col0 + c * 32;
            if (nb < ep.N)
              ts_store_chunk(ep, &tmc, stg + (c & 1) * 4096, lane, nb, m0 + quarter * 32, v,
                             bs + col0 + c * 32);
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(tempty + acc);
        } else {
#pragma unroll 1
          for (int c = 0; c < BN / 64; ++c) {
            float v[32];
            tmem_ld32(taddr + c * 32, v);
            const int nb = n0 + col0 + c * 32;
            if constexpr (I8) {
              if (row_ok && nb < ep.N) {
                const int o = acc * BN + col0 + c * 32;
                q_dequant_chunk(ep, m, v, qsc_s + o, qzp_s + o, qcs_s + o);
              }
            }
            if (row_ok && nb < ep.N)
              epilogue_chunk(ep, m, nb, v, bs + col0 + c * 32, best_v, best_i);
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(tempty + acc);
          if (ep.epi == kEpiArgmax && row_ok && best_i >= 0)
            atomicMax(ep.keys + m, argmax_key(best_v, (uint32_t)best_i));
        }
      }
      if (++acc == NACC) {
        acc = 0;
        aph ^= 1;
      }
    }
  }
  if constexpr (TS) {
    if (warp >= 2 && lane == 0) bulk_wait_all();   // output stores complete before exit
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, Cfg::kTmemCols);
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

int num_sms() {
  static int n = 0;
  if (!n) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    if (n <= 0) n = 148;
  }
  return n;
}

// MINB = 2: two co-resident CTAs per SM (half-depth stage ring, <= 96
// registers) for the skinny decoder GEMMs, so a second tile (or another
// decode lane's kernel) hides the TMA / MMA / epilogue latency of the first.
template <int BN, int STAGES, int TOPK = 0, bool I8 = false, int MINB = 1, int NACC = 2,
          bool TS = false>
cudaError_t launch_tc(const CUtensorMap& ta, const CUtensorMap& tw, const GemmArgs& g,
                      const EpiParams& ep, cudaStream_t s, const CUtensorMap* tc = nullptr) {
  using Cfg = TcCfg<BN, STAGES, I8, TOPK, NACC, TS>;
  static_assert(Cfg::kSmem <= 227 * 1024, "GEMM stage ring exceeds shared memory");
  static_assert(MINB == 1 || MINB * (Cfg::kSmem + 1024) <= 228 * 1024, "MINB CTAs do not fit");
  static_assert(MINB * NACC * BN <= 512, "co-resident CTAs exceed TMEM");
  auto kern = gemm_tc_kernel<BN, STAGES, TOPK, I8, MINB, NACC, TS>;
  cudaError_t e = set_max_smem((const void*)kern);
  if (e != cudaSuccess) return e;
  const int tiles_n = (g.N + BN - 1) / BN;
  const int tiles = tiles_n * ((g.M + kBM - 1) / kBM);
  const int grid = tiles < MINB * num_sms() ? tiles : MINB * num_sms();
  const uint32_t idesc = I8 ? umma_idesc_i8(kBM, BN) : umma_idesc_f16(kBM, BN, g.in_dtype == kBF16);
  return launch_k(kern, dim3(grid), dim3(kTcThreads),
                  (size_t)Cfg::kSmem, s, ta, tw, tc ? *tc : tw, I8 ? g.Kp : g.K, idesc, ep,
                  tiles_n, tiles);
}


}  // namespace

int gemm_tile_n() { return kWBox; }

bool dual_cta_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("FNMT_GEMM_DUAL");
    on = !(e && e[0] == '0');
  }
  return on != 0;
}

bool pdl_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("FNMT_PDL");
    on = !(e && e[0] == '0');
  }
  return on != 0;
}

bool tma_store_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("FNMT_TMA_STORE");
    on = !(e && e[0] == '0');
  }
  return on != 0;
}

// Output tensor map of a kEpiStore GEMM: [M, N] with leading dimension ldc,
// box 32 columns x 32 rows, swizzled like ts_store_chunk writes the chunk.
bool make_tmap_out(CUtensorMap* out, const void* base, int dtype, int64_t rows, int64_t cols,
                   int64_t ld) {
  auto fn = encode_fn();
  const int es = dtype == kF32 ? 4 : 2;
  if (!fn || (reinterpret_cast<uintptr_t>(base) & 15) || ((ld * es) & 15)) return false;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * es)};
  cuuint32_t box[2] = {32u, 32u};
  cuuint32_t estr[2] = {1, 1};
  const CUtensorMapDataType t = dtype == kF32    ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32
                                : dtype == kBF16 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16
                                                 : CU_TENSOR_MAP_DATA_TYPE_FLOAT16;
  return fn(out, t, 2, const_cast<void*>(base), dims, strides, box, estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE,
            dtype == kF32 ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_64B,
            CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

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

// N tile: the largest of 256/128/64 that still gives >= FNMT_BN_WAVE x SMs
// tiles (default 0.15: r02 A/B of the 6-1-1 bench with 4 decode lanes, 0.6 /
// 0.3 / 0.15 -> 7.72 / 7.86 / 7.92 M words/s — bigger N tiles re-read A less
// often and leave SMs to the other lanes; r01 single-lane 9216-row steps
// favoured 0.6 over 0.9-2.0).
int pick_bn(int M, int N, int K) {
  static double wave = -1.0, wave_k = -1.0;
  if (wave < 0) {
    const char* e = getenv("FNMT_BN_WAVE");
    wave = e ? atof(e) : 0.15;
    if (!(wave > 0.0 && wave < 4.0)) wave = 0.15;
    // long-K GEMMs (decoder FFN2, K = 2048): a tile's MMA time grows with K, so
    // they get their own threshold (FNMT_BN_WAVE_LONGK)
    const char* f = getenv("FNMT_BN_WAVE_LONGK");
    wave_k = f ? atof(f) : wave;
    if (!(wave_k > 0.0 && wave_k < 4.0)) wave_k = wave;
  }
  const int mt = (M + kBM - 1) / kBM;
  const double need = (K >= 1024 ? wave_k : wave) * num_sms();
  for (int bn : {256, 128}) {
    if ((double)mt * ((N + bn - 1) / bn) >= need) return bn;
  }
  return 64;
}

cudaError_t launch_gemm(const GemmArgs& g, cudaStream_t s) {
  if (g.M <= 0 || g.N <= 0) return cudaSuccess;
  if (g.qw) return launch_qgemm(g, s);
  EpiParams ep{g.bias, g.M, g.N, g.epi, g.C, g.ldc, g.c_dtype, g.relu, g.resid, g.ld_resid,
               g.keys, g.topk, g.kc, g.vc, g.cap, g.seg, g.t_ptr,
               nullptr, nullptr, nullptr, nullptr, nullptr, 0, g.m_tab};
  if (g.m_tab && (!g.t_ptr || g.epi == kEpiTopK)) return cudaErrorInvalidValue;
  if (g.epi == kEpiQKV && (!g.kc || !g.vc || !g.t_ptr || g.seg <= 0 || g.N != 3 * g.seg))
    return cudaErrorInvalidValue;
  if (g.epi == kEpiSlot && (!g.t_ptr || g.cap <= 0 || g.resid)) return cudaErrorInvalidValue;
  if (g.epi == kEpiTopK && (g.in_dtype == kF32 || (g.topk.K != 4 && g.topk.K != 8)))
    return cudaErrorInvalidValue;   // fp32 path: store logits + launch_logits_topk_partials
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
    if (!make_tmap_16(&tw, g.W, g.in_dtype, g.N, g.K, g.ldw, kWBox, nullptr))
      return cudaErrorInvalidValue;
    pw = &tw;
  }
  if (g.epi == kEpiTopK) {
    static_assert(kTopKTile == 256, "one top-K partial per BN = 256 tile");
    return g.topk.K == 4 ? launch_tc<256, 4, 4>(*pa, *pw, g, ep, s)
                         : launch_tc<256, 4, 8>(*pa, *pw, g, ep, s);
  }
  const int bn = pick_bn(g.M, g.N, g.K);
  CUtensorMap tc;
  if (g.epi == kEpiStore && !g.resid && tma_store_enabled() &&
      make_tmap_out(&tc, g.C, g.c_dtype, g.M, g.N, g.ldc)) {
    switch (bn) {
      case 256: return launch_tc<256, 3, 0, false, 1, 2, true>(*pa, *pw, g, ep, s, &tc);
      case 128: return launch_tc<128, 4, 0, false, 1, 2, true>(*pa, *pw, g, ep, s, &tc);
      default: return launch_tc<64, 5, 0, false, 1, 2, true>(*pa, *pw, g, ep, s, &tc);
    }
  }
  switch (bn) {
    case 256: return launch_tc<256, 4>(*pa, *pw, g, ep, s);
    case 128: return launch_tc<128, 6>(*pa, *pw, g, ep, s);
    default:
      if (g.K <= 1024 && dual_cta_enabled()) return launch_tc<64, 4, 0, false, 2>(*pa, *pw, g, ep, s);
      return launch_tc<64, 8>(*pa, *pw, g, ep, s);
  }
}

// int8 tcgen05 GEMM over activations already quantized into g.qs (qgemm.cu).
cudaError_t launch_tc_i8(const CUtensorMap& ta, const GemmArgs& g, cudaStream_t s) {
  if (g.epi == kEpiTopK || !g.qtmap_w) return cudaErrorInvalidValue;
  EpiParams ep{g.bias, g.M, g.N, g.epi, g.C, g.ldc, g.c_dtype, g.relu, g.resid, g.ld_resid,
               g.keys, g.topk, g.kc, g.vc, g.cap, g.seg, g.t_ptr,
               g.qscale, g.qzp, g.qcolsum, g.qs.rowsum, g.qs.stats, g.K};
  switch (pick_bn(g.M, g.N, g.K)) {
    case 256: return launch_tc<256, 4, 0, true>(ta, *g.qtmap_w, g, ep, s);
    case 128: return launch_tc<128, 6, 0, true>(ta, *g.qtmap_w, g, ep, s);
    default: return launch_tc<64, 8, 0, true>(ta, *g.qtmap_w, g, ep, s);
  }
}

bool make_tmap_8(CUtensorMap* out, const void* base, int64_t rows, int64_t kp, int box_rows,
                 std::string* err) {
  auto fn = encode_fn();
  if (!fn) {
    if (err) *err = "cuTensorMapEncodeTiled unavailable (driver too old?)";
    return false;
  }
  if ((reinterpret_cast<uintptr_t>(base) & 15) || (kp & 15)) {
    if (err) *err = "int8 TMA operand must be 16-byte aligned with K padded to 16";
    return false;
  }
  cuuint64_t dims[2] = {(cuuint64_t)kp, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)kp};
  cuuint32_t box[2] = {128u, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = fn(out, CU_TENSOR_MAP_DATA_TYPE_UINT8, 2, const_cast<void*>(base), dims, strides,
                  box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    if (err) *err = "cuTensorMapEncodeTiled (int8) failed with CUresult " + std::to_string((int)r);
    return false;
  }
  return true;
}

}  // namespace fnmt
