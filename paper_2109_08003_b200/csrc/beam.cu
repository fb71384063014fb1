// Batched beam search on the device — the reference's per-sentence
// `_beam_one` (search.py:114-147) for a whole batch at once.
//
// Row layout: row = sentence * k + slot.  Per step:
//  1. the vocab GEMM epilogue (gemm.cu, kEpiTopK) leaves, for every
//     (row, 256-column tile), the tile max, sum exp(x - max) and its top-K
//     logits (or, in fp32 parity mode, logits_topk_partials builds the same
//     partials from stored logits);
//  2. beam_row_reduce merges them per row into logZ (log-sum-exp, f64) and
//     the row's top-k (logit desc, id asc);
//  3. beam_select, one warp per sentence, forms candidates
//     score(parent) + logit - logZ in f64 (search.py:125-129: log-softmax
//     scores, no length normalisation), orders them (score desc, token asc,
//     parent asc) (search.py:131), sends EOS picks to the finished pool —
//     each consumes a beam slot (search.py:134-139) — stops a sentence when
//     no actives remain, k hypotheses finished or the budget is spent
//     (search.py:140-142), records back-pointers, and rebuilds the self-KV
//     ancestor table instead of gathering caches (DecodeCache.select,
//     model.py:170-181).  The last CTA bumps the step counter.
//  4. after the loop beam_final picks max(pool, key=(score, -tokens))
//     (search.py:145-147) and backtracks the tokens.
// Only a sentence's own rows are touched, so results do not depend on the
// batch composition.
#include <math.h>

#include "common.cuh"
#include "kernels.h"

namespace fnmt {

namespace {

constexpr int kWarpsPerCta = 8;

__global__ void beam_init_kernel(BeamState b, int bos) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < b.rows) {
    const int slot = i % b.k;
    b.prev[i] = slot == 0 ? bos : b.pad;
    b.score[i] = 0.0;
    b.active[i] = slot == 0;
  }
  if (i < b.nS) {
    b.finished[i] = 0;
    b.n_done[i] = 0;
    b.fin_t[i] = -1;
    b.fin_n[i] = 0;
  }
  if (i == 0) {
    *b.t = 0;
    *b.alive = b.nS;
    b.ticket[0] = 0;
    b.ticket[1] = 0;
  }
}

// insert (v, i) into a list sorted by (value desc, index asc) of length L
template <int L>
__device__ __forceinline__ void topk_insert(float (&tv)[L], int (&ti)[L], float v, int i) {
  if (!(v > tv[L - 1] || (v == tv[L - 1] && i >= 0 && (ti[L - 1] < 0 || i < ti[L - 1])))) return;
  tv[L - 1] = v;
  ti[L - 1] = i;
#pragma unroll
  for (int j = L - 1; j > 0; --j) {
    const bool up = tv[j] > tv[j - 1] || (tv[j] == tv[j - 1] && ti[j] >= 0 &&
                                          (ti[j - 1] < 0 || ti[j] < ti[j - 1]));
    if (up) {
      const float fv = tv[j];
      tv[j] = tv[j - 1];
      tv[j - 1] = fv;
      const int iv = ti[j];
      ti[j] = ti[j - 1];
      ti[j - 1] = iv;
    }
  }
}

// fp32 parity path: partials from stored logits, one warp per (row, tile)
__global__ void logits_topk_partials_kernel(const float* __restrict__ logits, int rows, int n,
                                            TopKPartials p) {
  const int wid = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (wid >= rows * p.tiles) return;
  const int r = wid / p.tiles, tile = wid % p.tiles;
  const float* row = logits + (size_t)r * n;
  const int c0 = tile * kTopKTile;
  float mx = -INFINITY;
  float tv[kTopKMax];
  int ti[kTopKMax];
#pragma unroll
  for (int j = 0; j < kTopKMax; ++j) {
    tv[j] = -INFINITY;
    ti[j] = -1;
  }
  for (int c = c0 + lane; c < min(n, c0 + kTopKTile); c += 32) {
    const float x = row[c];
    mx = fmaxf(mx, x);
    topk_insert(tv, ti, x, c);
  }
  mx = warp_max(mx);
  double s = 0.0;
  for (int c = c0 + lane; c < min(n, c0 + kTopKTile); c += 32) s += (double)expf(row[c] - mx);
  s = warp_sum_d(s);
  const size_t o = (size_t)r * p.tiles + tile;
  for (int round = 0; round < p.K; ++round) {
    unsigned long long key = ti[0] >= 0 ? argmax_key(tv[0], (uint32_t)ti[0]) : 0ull;
    unsigned long long best = key;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const unsigned long long o2 = __shfl_xor_sync(0xffffffffu, best, off);
      best = o2 > best ? o2 : best;
    }
    if (best != 0ull && key == best) {   // winner pops its head
#pragma unroll
      for (int j = 0; j < kTopKMax - 1; ++j) {
        tv[j] = tv[j + 1];
        ti[j] = ti[j + 1];
      }
      tv[kTopKMax - 1] = -INFINITY;
      ti[kTopKMax - 1] = -1;
    }
    if (lane == 0) {
      p.pval[o * p.K + round] = best ? float_from_order_key((uint32_t)(best >> 32)) : -INFINITY;
      p.pidx[o * p.K + round] = best ? (int)argmax_key_index(best) : -1;
    }
  }
  if (lane == 0) {
    p.pmax[o] = mx;
    p.psum[o] = s;
  }
}

// one warp per row: logZ and the row's top-k
__global__ void beam_row_reduce_kernel(BeamState b) {
  pdl_trigger();
  pdl_wait();
  const int r = blockIdx.x * kWarpsPerCta + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (r >= b.rows || !b.active[r]) return;
  const TopKPartials& p = b.part;
  const int T = p.tiles;
  float M = -INFINITY;
  for (int i = lane; i < T; i += 32) M = fmaxf(M, p.pmax[(size_t)r * T + i]);
  M = warp_max(M);
  double z = 0.0;
  for (int i = lane; i < T; i += 32) {
    const size_t o = (size_t)r * T + i;
    z += p.psum[o] * exp((double)p.pmax[o] - (double)M);
  }
  z = warp_sum_d(z);
  float tv[kTopKMax];
  int ti[kTopKMax];
#pragma unroll
  for (int j = 0; j < kTopKMax; ++j) {
    tv[j] = -INFINITY;
    ti[j] = -1;
  }
  for (int i = lane; i < T * p.K; i += 32) {
    const size_t o = (size_t)r * T * p.K + i;
    const int id = p.pidx[o];
    if (id >= 0) topk_insert(tv, ti, p.pval[o], id);
  }
  for (int round = 0; round < b.k; ++round) {
    const unsigned long long key = ti[0] >= 0 ? argmax_key(tv[0], (uint32_t)ti[0]) : 0ull;
    unsigned long long best = key;
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
      const unsigned long long o2 = __shfl_xor_sync(0xffffffffu, best, off);
      best = o2 > best ? o2 : best;
    }
    if (best != 0ull && key == best) {
#pragma unroll
      for (int j = 0; j < kTopKMax - 1; ++j) {
        tv[j] = tv[j + 1];
        ti[j] = ti[j + 1];
      }
      tv[kTopKMax - 1] = -INFINITY;
      ti[kTopKMax - 1] = -1;
    }
    if (lane == 0) {
      b.rval[(size_t)r * b.k + round] = best ? float_from_order_key((uint32_t)(best >> 32)) : -INFINITY;
      b.ridx[(size_t)r * b.k + round] = best ? (int)argmax_key_index(best) : -1;
    }
  }
  if (lane == 0) b.rlogz[r] = (double)M + log(z);
}

// candidate order: score desc, token asc, parent asc (search.py:131)
__device__ __forceinline__ bool cand_before(double s1, int t1, int p1, double s2, int t2, int p2) {
  if (s1 != s2) return s1 > s2;
  if (t1 != t2) return t1 < t2;
  return p1 < p2;
}

__global__ void beam_select_kernel(BeamState b) {
  constexpr int KM = kTopKMax;
  __shared__ int sh_new_n[kWarpsPerCta];
  __shared__ int sh_par[kWarpsPerCta][KM];
  __shared__ int sh_stop[kWarpsPerCta];
  __shared__ int cta_alive;
  pdl_trigger();
  pdl_wait();
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int s = blockIdx.x * kWarpsPerCta + warp;
  const int t = *b.t;
  const int k = b.k;
  if (threadIdx.x == 0) cta_alive = 0;
  __syncthreads();
  const bool live = s < b.nS && !b.finished[s];
  if (live) {
    const int base = s * k;
    if (lane == 0) {
      double cs[KM];
      int ct[KM], cp[KM];
      int count = 0;
      for (int a = 0; a < k; ++a) {
        if (!b.active[base + a]) continue;
        const double sa = b.score[base + a];
        const double lz = b.rlogz[base + a];
        for (int j = 0; j < k; ++j) {
          const int v = b.ridx[(size_t)(base + a) * k + j];
          if (v < 0) continue;
          const double sc = sa + ((double)b.rval[(size_t)(base + a) * k + j] - lz);
          // insertion into the sorted candidate list (length <= k)
          int pos = count < k ? count : k;
          while (pos > 0 && cand_before(sc, v, a, cs[pos - 1], ct[pos - 1], cp[pos - 1])) {
            if (pos < k) {
              cs[pos] = cs[pos - 1];
              ct[pos] = ct[pos - 1];
              cp[pos] = cp[pos - 1];
            }
            --pos;
          }
          if (pos < k) {
            cs[pos] = sc;
            ct[pos] = v;
            cp[pos] = a;
            if (count < k) ++count;
          }
        }
      }
      int nd = b.n_done[s];
      int new_n = 0;
      double nsc[KM];
      int ntk[KM], npr[KM];
      for (int i = 0; i < count; ++i) {
        if (ct[i] == b.eos) {
          if (nd < 2 * k) {
            b.done_score[s * 2 * k + nd] = cs[i];
            b.done_t[s * 2 * k + nd] = t;
            b.done_slot[s * 2 * k + nd] = cp[i];
          }
          ++nd;
        } else {
          nsc[new_n] = cs[i];
          ntk[new_n] = ct[i];
          npr[new_n] = cp[i];
          ++new_n;
        }
      }
      b.n_done[s] = nd < 2 * k ? nd : 2 * k;
      const bool stop = new_n == 0 || nd >= k || t + 1 >= b.budget[s];
      for (int i = 0; i < new_n; ++i) {
        b.tok_hist[(size_t)t * b.rows + base + i] = ntk[i];
        b.par_hist[(size_t)t * b.rows + base + i] = npr[i];
      }
      for (int i = 0; i < k; ++i) {
        const bool on = !stop && i < new_n;
        b.active[base + i] = on;
        b.score[base + i] = i < new_n ? nsc[i] : 0.0;
        b.prev[base + i] = on ? ntk[i] : b.pad;
      }
      if (stop) {
        b.finished[s] = 1;
        b.fin_t[s] = t;
        b.fin_n[s] = new_n;
      }
      sh_new_n[warp] = new_n;
      sh_stop[warp] = stop;
      for (int i = 0; i < new_n; ++i) sh_par[warp][i] = npr[i];
    }
    __syncwarp();
    if (!sh_stop[warp]) {
      const int32_t* cur = b.anc + (size_t)(t & 1) * b.rows * b.cap;
      int32_t* nxt = b.anc + (size_t)((t + 1) & 1) * b.rows * b.cap;
      for (int i = 0; i < sh_new_n[warp]; ++i) {
        const int parent_row = base + sh_par[warp][i];
        for (int j = lane; j <= t; j += 32)
          nxt[(size_t)(base + i) * b.cap + j] =
              j < t ? cur[(size_t)parent_row * b.cap + j] : parent_row;
      }
      if (lane == 0) atomicAdd(&cta_alive, 1);
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (cta_alive) atomicAdd(reinterpret_cast<int*>(&b.ticket[1]), cta_alive);
    __threadfence();
    const unsigned int done = atomicAdd(&b.ticket[0], 1u);
    if (done == gridDim.x - 1) {
      __threadfence();
      *b.alive = atomicExch(reinterpret_cast<int*>(&b.ticket[1]), 0);
      b.ticket[0] = 0;
      *b.t = t + 1;
    }
  }
}

__global__ void beam_final_kernel(BeamState b) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int s = blockIdx.x * kWarpsPerCta + warp;
  if (s >= b.nS) return;
  const int k = b.k, base = s * k;
  const int nd = b.n_done[s];
  const bool use_done = nd > 0;
  const int npool = use_done ? nd : b.fin_n[s];
  int32_t* scr = b.scratch + (size_t)s * 2 * k * b.cap;
  // lane c backtracks candidate c
  int my_len = 0;
  double my_score = -INFINITY;
  if (lane < npool) {
    int slot, L;
    if (use_done) {
      my_score = b.done_score[s * 2 * k + lane];
      L = b.done_t[s * 2 * k + lane];
      slot = b.done_slot[s * 2 * k + lane];
    } else {
      my_score = b.score[base + lane];
      L = b.fin_t[s] + 1;
      slot = lane;
    }
    my_len = L;
    int cur = slot;
    for (int tt = L - 1; tt >= 0; --tt) {
      const size_t h = (size_t)tt * b.rows + base + cur;
      scr[(size_t)lane * b.cap + tt] = b.tok_hist[h];
      cur = b.par_hist[h];
    }
  }
  __syncwarp();
  int best = 0;
  __shared__ double sh_score[kWarpsPerCta][32];
  __shared__ int sh_len[kWarpsPerCta][32];
  sh_score[warp][lane] = my_score;
  sh_len[warp][lane] = my_len;
  __syncwarp();
  if (lane == 0) {
    for (int c = 1; c < npool; ++c) {
      const double sc = sh_score[warp][c], sb = sh_score[warp][best];
      bool better = sc > sb;
      if (sc == sb) {   // tuple(-tokens) larger wins (search.py:146)
        const int lc = sh_len[warp][c], lb = sh_len[warp][best];
        const int m = lc < lb ? lc : lb;
        int i = 0;
        while (i < m && scr[(size_t)c * b.cap + i] == scr[(size_t)best * b.cap + i]) ++i;
        better = i < m ? scr[(size_t)c * b.cap + i] < scr[(size_t)best * b.cap + i] : lc > lb;
      }
      if (better) best = c;
    }
  }
  best = __shfl_sync(0xffffffffu, best, 0);
  const int L = sh_len[warp][best];
  for (int i = lane; i < L; i += 32) b.out_ids[(size_t)s * b.cap + i] = scr[(size_t)best * b.cap + i];
  if (lane == 0) b.out_len[s] = npool > 0 ? L : 0;
}

}  // namespace

cudaError_t launch_beam_init(const BeamState& b, int bos, cudaStream_t s) {
  const int n = b.rows > b.nS ? b.rows : b.nS;
  beam_init_kernel<<<(n + 255) / 256, 256, 0, s>>>(b, bos);
  return cudaGetLastError();
}

cudaError_t launch_logits_topk_partials(const float* logits, int rows, int n,
                                        const TopKPartials& p, cudaStream_t s) {
  const int64_t warps = (int64_t)rows * p.tiles;
  if (warps <= 0) return cudaSuccess;
  logits_topk_partials_kernel<<<(unsigned)((warps + 7) / 8), 256, 0, s>>>(logits, rows, n, p);
  return cudaGetLastError();
}

cudaError_t launch_beam_row_reduce(const BeamState& b, cudaStream_t s) {
  return launch_k(beam_row_reduce_kernel, dim3((b.rows + kWarpsPerCta - 1) / kWarpsPerCta),
                  dim3(32 * kWarpsPerCta), 0, s, b);
}

cudaError_t launch_beam_select(const BeamState& b, cudaStream_t s) {
  return launch_k(beam_select_kernel, dim3((b.nS + kWarpsPerCta - 1) / kWarpsPerCta),
                  dim3(32 * kWarpsPerCta), 0, s, b);
}

cudaError_t launch_beam_final(const BeamState& b, cudaStream_t s) {
  beam_final_kernel<<<(b.nS + kWarpsPerCta - 1) / kWarpsPerCta, 32 * kWarpsPerCta, 0, s>>>(b);
  return cudaGetLastError();
}

}  // namespace fnmt
