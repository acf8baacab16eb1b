// Integer/selection kernels of the SBO iteration:
//  * stable counting sort of signals by assigned block (sbo.py:231-249) and the
//    per-block segment table the coding/outer-product kernels run over;
//  * worst-W set by radix select on float64 residual keys (sbo.py:223-228);
//  * deterministic float64 reductions (sbo.py:295-296, linalg.py:81-86, 148-162).
#include "common.cuh"

namespace sbo {

constexpr int kGroupTile = 1024;  // signals per CTA of the grouping kernels (32 warps)
constexpr int kSumTile = 1024;

// ---------------------------------------------------------------------------
// grouping
// ---------------------------------------------------------------------------
// Per warp, the distinct block values and their counts; used for stable
// intra-tile ranks without a K-sized table.
struct WarpRuns {
  int val[32];
  int cnt[32];
  int n;
};

__device__ void warp_runs(int b, bool valid, WarpRuns* wr, int* rank_in_warp) {
  const int lane = threadIdx.x & 31;
  const unsigned act = __ballot_sync(0xffffffffu, valid);
  const unsigned peers = __match_any_sync(0xffffffffu, valid ? b : -1) & act;
  *rank_in_warp = __popc(peers & ((1u << lane) - 1u));
  const bool leader = valid && (__ffs(peers) - 1 == lane);
  const unsigned lead = __ballot_sync(0xffffffffu, leader);
  if (leader) {
    const int slot = __popc(lead & ((1u << lane) - 1u));
    wr->val[slot] = b;
    wr->cnt[slot] = __popc(peers);
  }
  if (lane == 0) wr->n = __popc(lead);
}

__global__ void __launch_bounds__(kGroupTile) k_group_count(const int32_t* __restrict__ best,
                                                           int64_t m, int K, int32_t* cnt) {
  __shared__ WarpRuns runs[kGroupTile / 32];
  const int64_t j = static_cast<int64_t>(blockIdx.x) * kGroupTile + threadIdx.x;
  const bool valid = j < m;
  const int b = valid ? best[j] : -1;
  int r;
  warp_runs(b, valid, &runs[threadIdx.x >> 5], &r);
  __syncthreads();
  // one thread per warp-run entry accumulates into the tile's count row
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l < runs[w].n) atomicAdd(&cnt[static_cast<int64_t>(blockIdx.x) * K + runs[w].val[l]],
                               runs[w].cnt[l]);
}

// exclusive scan of column b over tiles -> tile offsets; total count per block
__global__ void k_group_scan(int32_t* cnt, int64_t ntiles, int K, int64_t* total) {
  const int b = blockIdx.x;
  __shared__ int64_t carry;
  __shared__ int64_t wsum[32];
  if (threadIdx.x == 0) carry = 0;
  __syncthreads();
  for (int64_t base = 0; base < ntiles; base += blockDim.x) {
    const int64_t t = base + threadIdx.x;
    const int64_t v = t < ntiles ? cnt[t * K + b] : 0;
    // block-wide inclusive scan
    int64_t x = v;
    const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t n = __shfl_up_sync(0xffffffffu, x, o);
      if (lane >= o) x += n;
    }
    if (lane == 31) wsum[w] = x;
    __syncthreads();
    if (w == 0) {
      int64_t s = lane < static_cast<int>(blockDim.x >> 5) ? wsum[lane] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int64_t n = __shfl_up_sync(0xffffffffu, s, o);
        if (lane >= o) s += n;
      }
      wsum[lane] = s;
    }
    __syncthreads();
    const int64_t incl = x + (w > 0 ? wsum[w - 1] : 0) + carry;
    if (t < ntiles) cnt[t * K + b] = static_cast<int32_t>(incl - v);
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) carry = incl;
    __syncthreads();
  }
  if (threadIdx.x == 0) total[b] = carry;
}

// bounds = exclusive scan of totals; the segment table per block
__global__ void k_group_bounds(const int64_t* total, int K, int seg_len, int64_t* bounds,
                               int32_t* seg_block, int64_t* seg_lo, int64_t* seg_hi,
                               int32_t* nseg, int64_t* seg_first) {
  if (threadIdx.x == 0) {
    int64_t acc = 0, sacc = 0;
    for (int b = 0; b < K; ++b) {
      bounds[b] = acc;
      seg_first[b] = sacc;
      acc += total[b];
      sacc += ceil_div(total[b], seg_len);
    }
    bounds[K] = acc;
    seg_first[K] = sacc;
    *nseg = static_cast<int32_t>(sacc);
  }
  __syncthreads();
  for (int b = threadIdx.x; b < K; b += blockDim.x) {
    const int64_t lo = bounds[b], hi = bounds[b + 1];
    int64_t s = seg_first[b];
    for (int64_t a = lo; a < hi; a += seg_len, ++s) {
      seg_block[s] = b;
      seg_lo[s] = a;
      seg_hi[s] = min64(a + seg_len, hi);
    }
  }
}

__global__ void __launch_bounds__(kGroupTile) k_group_scatter(const int32_t* __restrict__ best,
                                                             int64_t m, int K,
                                                             const int32_t* __restrict__ off,
                                                             const int64_t* __restrict__ bounds,
                                                             int32_t* perm) {
  __shared__ WarpRuns runs[kGroupTile / 32];
  __shared__ int before[kGroupTile / 32][65];  // K <= 64: per-warp exclusive block counts
  const int64_t j = static_cast<int64_t>(blockIdx.x) * kGroupTile + threadIdx.x;
  const bool valid = j < m;
  const int b = valid ? best[j] : -1;
  int r;
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  warp_runs(b, valid, &runs[w], &r);
  if (K <= 64) {
    for (int e = threadIdx.x; e < (kGroupTile / 32) * 64; e += kGroupTile) before[e >> 6][e & 63] = 0;
    __syncthreads();
    if (l < runs[w].n) before[w][runs[w].val[l]] = runs[w].cnt[l];
    __syncthreads();
    if (threadIdx.x < K) {  // exclusive scan over warps, one block per thread
      int acc = 0;
      for (int v = 0; v < kGroupTile / 32; ++v) {
        const int c = before[v][threadIdx.x];
        before[v][threadIdx.x] = acc;
        acc += c;
      }
    }
    __syncthreads();
    if (!valid) return;
    r += before[w][b];
  } else {
    __syncthreads();
    if (!valid) return;
    for (int v = 0; v < w; ++v)
      for (int e = 0; e < runs[v].n; ++e)
        if (runs[v].val[e] == b) r += runs[v].cnt[e];
  }
  perm[bounds[b] + off[static_cast<int64_t>(blockIdx.x) * K + b] + r] = static_cast<int32_t>(j);
}

// ---------------------------------------------------------------------------
// worst set: radix select over 64-bit keys (residual desc, index asc)
// ---------------------------------------------------------------------------
struct SelectState {
  unsigned long long prefix;
  long long need;  // members still to take at/below the current prefix
};

__global__ void k_select_init(SelectState* st, long long need) {
  if (threadIdx.x == 0) {
    st->prefix = 0ull;
    st->need = need;
  }
}

__global__ void k_key_hist(const double* __restrict__ r, int64_t m, const SelectState* st,
                           unsigned long long prefix_arg, int shift, long long* hist) {
  __shared__ unsigned int h[256];
  for (int i = threadIdx.x; i < 256; i += blockDim.x) h[i] = 0;
  __syncthreads();
  const unsigned long long prefix = st ? st->prefix : prefix_arg;
  const int hs = shift + 8;
  const int lane = threadIdx.x & 31;
  // warp-aggregated: keys share few digits (the high bytes of similar floats), so
  // one shared atomic per distinct digit per warp instead of one per key
  for (int64_t base = static_cast<int64_t>(blockIdx.x) * blockDim.x; base < m;
       base += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t j = base + threadIdx.x;
    int bin = -1;
    if (j < m) {
      const unsigned long long key = key_of(r[j]);
      if (hs >= 64 || (key >> hs) == (prefix >> hs)) bin = static_cast<int>((key >> shift) & 255u);
    }
    const unsigned peers = __match_any_sync(0xffffffffu, bin);
    if (bin >= 0 && __ffs(peers) - 1 == lane) atomicAdd(&h[bin], static_cast<unsigned>(__popc(peers)));
  }
  __syncthreads();
  for (int i = threadIdx.x; i < 256; i += blockDim.x)
    if (h[i]) atomicAdd(reinterpret_cast<unsigned long long*>(hist + i),
                        static_cast<unsigned long long>(h[i]));
}

// the digit d of the need-th largest key: with suffix sums S[d] = sum_{d' >= d} h[d'],
// the largest d with S[d] >= need (256 threads, one bin each, block scan)
__global__ void __launch_bounds__(256) k_key_pick(SelectState* st, long long* hist, int shift) {
  __shared__ long long wsum[8];
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const int d = 255 - t;  // thread t owns bin 255 - t: a prefix over t is a suffix over d
  const long long v = hist[d];
  long long x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const long long n = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += n;
  }
  if (lane == 31) wsum[w] = x;
  __syncthreads();
  long long before = 0;
  for (int i = 0; i < w; ++i) before += wsum[i];
  const long long incl = x + before;  // S[d]
  const long long excl = incl - v;    // S[d + 1]
  const long long need = st->need;
  __syncthreads();  // every thread has read st->need
  if (incl >= need && excl < need) {
    st->need = need - excl;
    st->prefix |= static_cast<unsigned long long>(d) << shift;
  }
  hist[d] = 0;
}

// per-tile (greater, equal) counts against the threshold
__global__ void k_worst_count(const double* __restrict__ r, int64_t m, const SelectState* st,
                              unsigned long long thr_arg, long long* gt, long long* eq) {
  const unsigned long long thr = st ? st->prefix : thr_arg;
  const int64_t j = static_cast<int64_t>(blockIdx.x) * kSumTile + threadIdx.x;
  unsigned long long key = j < m ? key_of(r[j]) : 0ull;
  const int g = (j < m && key > thr), e = (j < m && key == thr);
  __shared__ int sg[32], se[32];
  const int wg = warp_sum_int(g), we = warp_sum_int(e);
  if ((threadIdx.x & 31) == 0) {
    sg[threadIdx.x >> 5] = wg;
    se[threadIdx.x >> 5] = we;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    long long a = 0, b = 0;
    for (int w = 0; w < kSumTile / 32; ++w) {
      a += sg[w];
      b += se[w];
    }
    gt[blockIdx.x] = a;
    eq[blockIdx.x] = b;
  }
}

// exclusive scans of the per-tile counts (single CTA, sequential over chunks)
__global__ void k_worst_scan(long long* gt, long long* eq, int64_t ntiles, long long* total) {
  __shared__ long long carry_g, carry_e;
  __shared__ long long wg[32], we[32];
  if (threadIdx.x == 0) carry_g = carry_e = 0;
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int64_t base = 0; base < ntiles; base += blockDim.x) {
    const int64_t t = base + threadIdx.x;
    const long long vg = t < ntiles ? gt[t] : 0, ve = t < ntiles ? eq[t] : 0;
    long long xg = vg, xe = ve;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const long long a = __shfl_up_sync(0xffffffffu, xg, o);
      const long long b = __shfl_up_sync(0xffffffffu, xe, o);
      if (lane >= o) {
        xg += a;
        xe += b;
      }
    }
    if (lane == 31) {
      wg[w] = xg;
      we[w] = xe;
    }
    __syncthreads();
    if (w == 0) {
      long long sg = lane < static_cast<int>(blockDim.x >> 5) ? wg[lane] : 0;
      long long se = lane < static_cast<int>(blockDim.x >> 5) ? we[lane] : 0;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const long long a = __shfl_up_sync(0xffffffffu, sg, o);
        const long long b = __shfl_up_sync(0xffffffffu, se, o);
        if (lane >= o) {
          sg += a;
          se += b;
        }
      }
      wg[lane] = sg;
      we[lane] = se;
    }
    __syncthreads();
    const long long ig = xg + (w > 0 ? wg[w - 1] : 0) + carry_g;
    const long long ie = xe + (w > 0 ? we[w - 1] : 0) + carry_e;
    if (t < ntiles) {
      gt[t] = ig - vg;
      eq[t] = ie - ve;
    }
    __syncthreads();
    if (threadIdx.x == blockDim.x - 1) {
      carry_g = ig;
      carry_e = ie;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0 && total) {
    total[0] = carry_g;
    total[1] = carry_e;
  }
}

__global__ void k_worst_write(const double* __restrict__ r, int64_t m, const SelectState* st,
                              unsigned long long thr_arg, long long take_arg,
                              const long long* gt, const long long* eq, int32_t* members) {
  const unsigned long long thr = st ? st->prefix : thr_arg;
  const long long take = st ? st->need : take_arg;
  const int64_t j = static_cast<int64_t>(blockIdx.x) * kSumTile + threadIdx.x;
  const unsigned long long key = j < m ? key_of(r[j]) : 0ull;
  const int g = (j < m && key > thr), e = (j < m && key == thr);
  // intra-tile exclusive ranks
  __shared__ int sg[32], se[32];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const unsigned lt = (1u << lane) - 1u;
  const unsigned bg = __ballot_sync(0xffffffffu, g), be = __ballot_sync(0xffffffffu, e);
  if (lane == 0) {
    sg[w] = __popc(bg);
    se[w] = __popc(be);
  }
  __syncthreads();
  long long rg = __popc(bg & lt), re = __popc(be & lt);
  for (int v = 0; v < w; ++v) {
    rg += sg[v];
    re += se[v];
  }
  rg += gt[blockIdx.x];
  re += eq[blockIdx.x];
  const long long eq_taken_before = re < take ? re : take;
  if (g) members[rg + eq_taken_before] = static_cast<int32_t>(j);
  if (e && re < take) members[rg + re] = static_cast<int32_t>(j);
}

// ---------------------------------------------------------------------------
// deterministic float64 sums
// ---------------------------------------------------------------------------
__global__ void k_sum_tiles(const double* __restrict__ x, int64_t n, double* partial) {
  __shared__ double red[32];
  const int64_t j = static_cast<int64_t>(blockIdx.x) * kSumTile + threadIdx.x;
  double v = j < n ? x[j] : 0.0;
  v = block_sum<kSumTile>(v, red);
  if (threadIdx.x == 0) partial[blockIdx.x] = v;
}

__global__ void k_sum_final(const double* partial, int64_t n, double* out) {
  __shared__ double red[32];
  // fixed assignment of partials to threads, fixed tree
  double acc = 0.0;
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) acc += partial[i];
  acc = block_sum<1024>(acc, red);
  if (threadIdx.x == 0) *out = acc;
}

__global__ void k_defect(const double* __restrict__ Q, int p, double* out) {
  __shared__ double red[32];
  const double* q = Q + static_cast<int64_t>(blockIdx.x) * p * p;
  double acc = 0.0;
  for (int e = threadIdx.x; e < p * p; e += blockDim.x) {
    const int a = e / p, b = e % p;  // (Q^T Q)[a][b] = sum_k Q[k][a] Q[k][b]
    double g = 0.0;
    for (int k = 0; k < p; ++k) g = fma(q[k * p + a], q[k * p + b], g);
    g -= (a == b) ? 1.0 : 0.0;
    acc = fma(g, g, acc);
  }
  acc = block_sum<256>(acc, red);
  if (threadIdx.x == 0) out[blockIdx.x] = sqrt(acc);
}

// ||y_j - Q_b x_j||^2 per signal, warp per signal; CTA partial sums
template <typename TY>
__global__ void k_frob(const TY* __restrict__ y, int64_t m, int p,
                       const double* __restrict__ blocks, const int32_t* __restrict__ block,
                       int k, int64_t ld, const int16_t* __restrict__ idx,
                       const double* __restrict__ val, double* partial) {
  __shared__ double red[32];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t j = static_cast<int64_t>(blockIdx.x) * (blockDim.x / 32) + warp;
  double acc = 0.0;
  if (j < m) {
    const double* q = blocks + static_cast<int64_t>(block[j]) * p * p;
    for (int d = lane; d < p; d += 32) {
      double r = y[j * p + d];
      for (int t = 0; t < k; ++t) r -= q[d * p + idx[t * ld + j]] * val[t * ld + j];
      acc = fma(r, r, acc);
    }
  }
  acc = block_sum<256>(acc, red);
  if (threadIdx.x == 0) partial[blockIdx.x] = acc;
}

}  // namespace sbo

using namespace sbo;

extern "C" size_t sbo_group_workspace_bytes(int64_t m, int K) {
  const int64_t ntiles = ceil_div(m, kGroupTile);
  return sizeof(int32_t) * ntiles * K + sizeof(int64_t) * (2 * K + 2) + 256;
}

extern "C" int64_t sbo_max_segments(int64_t m, int K, int seg_len) {
  return ceil_div(m, seg_len) + K;
}

extern "C" int sbo_group(const int32_t* best, int64_t m, int K, int seg_len, int32_t* perm,
                         int64_t* bounds, int32_t* seg_block, int64_t* seg_lo, int64_t* seg_hi,
                         int32_t* nseg, void* ws, size_t ws_bytes, void* stream) {
  if (K < 1) return fail(SBO_EINVAL, "K must be at least 1");
  if (seg_len < kTile || seg_len % kTile) return fail(SBO_EINVAL, "seg_len must be a multiple of 64");
  if (ws_bytes < sbo_group_workspace_bytes(m, K)) return fail(SBO_EINVAL, "group workspace too small");
  cudaStream_t st = as_stream(stream);
  const int64_t ntiles = ceil_div(m, kGroupTile);
  int32_t* cnt = static_cast<int32_t*>(ws);
  int64_t* total = reinterpret_cast<int64_t*>(
      (reinterpret_cast<uintptr_t>(cnt + ntiles * K) + 15) & ~uintptr_t(15));
  int64_t* seg_first = total + K;
  if (ntiles > 0) {
    SBO_CHECK_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int32_t) * ntiles * K, st));
    k_group_count<<<static_cast<unsigned>(ntiles), kGroupTile, 0, st>>>(best, m, K, cnt);
    int rc = check_launch("k_group_count");
    if (rc) return rc;
  }
  k_group_scan<<<K, 1024, 0, st>>>(cnt, ntiles, K, total);
  int rc = check_launch("k_group_scan");
  if (rc) return rc;
  k_group_bounds<<<1, 256, 0, st>>>(total, K, seg_len, bounds, seg_block, seg_lo, seg_hi, nseg,
                                    seg_first);
  rc = check_launch("k_group_bounds");
  if (rc || ntiles == 0) return rc;
  k_group_scatter<<<static_cast<unsigned>(ntiles), kGroupTile, 0, st>>>(best, m, K, cnt, bounds,
                                                                       perm);
  return check_launch("k_group_scatter");
}

extern "C" size_t sbo_worst_workspace_bytes(int64_t m) {
  const int64_t ntiles = ceil_div(m, kSumTile);
  return sizeof(SelectState) + sizeof(long long) * (256 + 2 * ntiles + 2) + 64;
}

extern "C" int sbo_worst_set(const double* residual_sq, int64_t m, int64_t w, int32_t* members,
                             void* ws, size_t ws_bytes, void* stream) {
  if (w < 1) return fail(SBO_EINVAL, "worst-set size must be at least 1");
  if (ws_bytes < sbo_worst_workspace_bytes(m)) return fail(SBO_EINVAL, "worst workspace too small");
  if (m == 0) return SBO_OK;
  cudaStream_t st = as_stream(stream);
  SelectState* S = static_cast<SelectState*>(ws);
  long long* hist = reinterpret_cast<long long*>(S + 1);
  long long* gt = hist + 256;
  const int64_t ntiles = ceil_div(m, kSumTile);
  long long* eq = gt + ntiles;
  const long long take = w < m ? w : m;
  // state set by a kernel, not a host copy: capturable in a CUDA graph and no
  // pageable transfer competing with other streams' copies
  k_select_init<<<1, 32, 0, st>>>(S, take);
  SBO_CHECK_CUDA(cudaMemsetAsync(hist, 0, sizeof(long long) * 256, st));
  if (w >= m) {
    // everything: threshold 0 and all zero-keys taken (need = m, prefix 0)
  } else {
    const int grid = static_cast<int>(ceil_div(m, 256) < 1184 ? ceil_div(m, 256) : 1184);
    for (int shift = 56; shift >= 0; shift -= 8) {
      k_key_hist<<<grid, 256, 0, st>>>(residual_sq, m, S, 0ull, shift, hist);
      k_key_pick<<<1, 256, 0, st>>>(S, hist, shift);
    }
    int rc = check_launch("k_key_hist/pick");
    if (rc) return rc;
  }
  k_worst_count<<<static_cast<unsigned>(ntiles), kSumTile, 0, st>>>(residual_sq, m, S, 0ull, gt, eq);
  k_worst_scan<<<1, 1024, 0, st>>>(gt, eq, ntiles, nullptr);
  k_worst_write<<<static_cast<unsigned>(ntiles), kSumTile, 0, st>>>(residual_sq, m, S, 0ull, 0,
                                                                    gt, eq, members);
  return check_launch("k_worst_*");
}

// ---------------------------------------------------------------------------
// Device-resident radix select for signal shards (the sharded worst set): the
// select state lives in the worst-set workspace; the caller allreduces each
// pass's histogram in device memory (NCCL) between sbo_select_hist and
// sbo_select_pick, and allgathers the per-rank tie counts before
// sbo_select_write — no host round trip.
// ---------------------------------------------------------------------------
__global__ void k_select_take(SelectState* st, const long long* eq_all, int rank,
                              const long long* gt_eq, long long* count) {
  if (threadIdx.x == 0) {
    long long before = 0;
    for (int q = 0; q < rank; ++q) before += eq_all[q];
    long long take = st->need - before;  // threshold ties go to lower ranks first
    if (take < 0) take = 0;
    if (take > eq_all[rank]) take = eq_all[rank];
    st->need = take;
    *count = gt_eq[0] + take;
  }
}

extern "C" int sbo_select_begin(void* ws, int64_t need, void* stream) {
  k_select_init<<<1, 32, 0, as_stream(stream)>>>(static_cast<SelectState*>(ws), need);
  return check_launch("k_select_init");
}

extern "C" int sbo_select_hist(const double* residual_sq, int64_t m, void* ws, int shift,
                               int64_t* hist256, void* stream) {
  if (shift < 0 || shift > 56 || shift % 8) return fail(SBO_EINVAL, "shift must be 0, 8, .., 56");
  cudaStream_t st = as_stream(stream);
  SBO_CHECK_CUDA(cudaMemsetAsync(hist256, 0, sizeof(int64_t) * 256, st));
  if (m == 0) return SBO_OK;
  const int grid = static_cast<int>(ceil_div(m, 256) < 1184 ? ceil_div(m, 256) : 1184);
  k_key_hist<<<grid, 256, 0, st>>>(residual_sq, m, static_cast<const SelectState*>(ws), 0ull,
                                   shift, reinterpret_cast<long long*>(hist256));
  return check_launch("k_key_hist");
}

extern "C" int sbo_select_pick(void* ws, int64_t* hist256, int shift, void* stream) {
  k_key_pick<<<1, 256, 0, as_stream(stream)>>>(static_cast<SelectState*>(ws),
                                               reinterpret_cast<long long*>(hist256), shift);
  return check_launch("k_key_pick");
}

extern "C" int sbo_select_counts(const double* residual_sq, int64_t m, void* ws, size_t ws_bytes,
                                 int64_t* gt_eq, void* stream) {
  if (ws_bytes < sbo_worst_workspace_bytes(m)) return fail(SBO_EINVAL, "worst workspace too small");
  cudaStream_t st = as_stream(stream);
  SelectState* S = static_cast<SelectState*>(ws);
  long long* gt = reinterpret_cast<long long*>(S + 1) + 256;
  const int64_t ntiles = ceil_div(m > 0 ? m : 1, kSumTile);
  long long* eq = gt + ntiles;
  if (m == 0) return cudaMemsetAsync(gt_eq, 0, 2 * sizeof(int64_t), st) == cudaSuccess ? SBO_OK
                                                                                : fail(SBO_ECUDA, "memset");
  k_worst_count<<<static_cast<unsigned>(ntiles), kSumTile, 0, st>>>(residual_sq, m, S, 0ull, gt, eq);
  k_worst_scan<<<1, 1024, 0, st>>>(gt, eq, ntiles, reinterpret_cast<long long*>(gt_eq));
  return check_launch("k_worst_count/scan");
}

extern "C" int sbo_select_write(const double* residual_sq, int64_t m, void* ws, size_t ws_bytes,
                                const int64_t* gt_eq, const int64_t* eq_all, int rank,
                                int32_t* members, int64_t* count, void* stream) {
  if (ws_bytes < sbo_worst_workspace_bytes(m)) return fail(SBO_EINVAL, "worst workspace too small");
  cudaStream_t st = as_stream(stream);
  SelectState* S = static_cast<SelectState*>(ws);
  long long* gt = reinterpret_cast<long long*>(S + 1) + 256;
  const int64_t ntiles = ceil_div(m > 0 ? m : 1, kSumTile);
  long long* eq = gt + ntiles;
  k_select_take<<<1, 32, 0, st>>>(S, reinterpret_cast<const long long*>(eq_all), rank,
                                  reinterpret_cast<const long long*>(gt_eq),
                                  reinterpret_cast<long long*>(count));
  if (m > 0)
    k_worst_write<<<static_cast<unsigned>(ntiles), kSumTile, 0, st>>>(residual_sq, m, S, 0ull, 0,
                                                                      gt, eq, members);
  return check_launch("k_worst_write");
}

extern "C" int sbo_key_histogram(const double* residual_sq, int64_t m, uint64_t prefix, int shift,
                                 int64_t* hist256, void* stream) {
  if (shift < 0 || shift > 56 || shift % 8) return fail(SBO_EINVAL, "shift must be 0, 8, .., 56");
  if (m == 0) return SBO_OK;
  const int grid = static_cast<int>(ceil_div(m, 256) < 1184 ? ceil_div(m, 256) : 1184);
  k_key_hist<<<grid, 256, 0, as_stream(stream)>>>(residual_sq, m, nullptr, prefix, shift,
                                                  reinterpret_cast<long long*>(hist256));
  return check_launch("k_key_hist");
}

extern "C" int sbo_worst_collect(const double* residual_sq, int64_t m, uint64_t threshold_key,
                                 int64_t take_equal, int32_t* members, int64_t* count, void* ws,
                                 size_t ws_bytes, void* stream) {
  if (ws_bytes < sbo_worst_workspace_bytes(m)) return fail(SBO_EINVAL, "worst workspace too small");
  if (m == 0) return SBO_OK;
  cudaStream_t st = as_stream(stream);
  long long* gt = reinterpret_cast<long long*>(static_cast<SelectState*>(ws) + 1) + 256;
  const int64_t ntiles = ceil_div(m, kSumTile);
  long long* eq = gt + ntiles;
  k_worst_count<<<static_cast<unsigned>(ntiles), kSumTile, 0, st>>>(residual_sq, m, nullptr,
                                                                    threshold_key, gt, eq);
  k_worst_scan<<<1, 1024, 0, st>>>(gt, eq, ntiles, reinterpret_cast<long long*>(count));
  k_worst_write<<<static_cast<unsigned>(ntiles), kSumTile, 0, st>>>(
      residual_sq, m, nullptr, threshold_key, take_equal, gt, eq, members);
  return check_launch("k_worst_collect");
}

// ---------------------------------------------------------------------------
// ordering of the flagged signals by their two lowest candidate blocks
// ---------------------------------------------------------------------------
constexpr int kCandKeys = 64 * 65;

__device__ __forceinline__ int cand_key(uint64_t mask) {
  const int lo = mask ? __ffsll(static_cast<long long>(mask)) - 1 : 0;
  const uint64_t rest = mask & (mask - 1ull);
  const int hi = rest ? __ffsll(static_cast<long long>(rest)) - 1 : 64;
  return lo * 65 + hi;
}

__global__ void k_cand_hist(const uint64_t* __restrict__ cand, const int32_t* nflag, int* cnt) {
  __shared__ int h[kCandKeys];
  for (int i = threadIdx.x; i < kCandKeys; i += blockDim.x) h[i] = 0;
  __syncthreads();
  const int n = *nflag;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    atomicAdd(&h[cand_key(cand[i])], 1);
  __syncthreads();
  for (int i = threadIdx.x; i < kCandKeys; i += blockDim.x)
    if (h[i]) atomicAdd(&cnt[i], h[i]);
}

__global__ void __launch_bounds__(1024) k_cand_scan(int* cnt) {
  __shared__ int wsum[32];
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  constexpr int PER = (kCandKeys + 1023) / 1024;  // keys per thread (5)
  int v[PER], tot = 0;
#pragma unroll
  for (int u = 0; u < PER; ++u) {
    const int i = t * PER + u;
    v[u] = i < kCandKeys ? cnt[i] : 0;
    tot += v[u];
  }
  int x = tot;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int n = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += n;
  }
  if (lane == 31) wsum[w] = x;
  __syncthreads();
  if (w == 0) {
    int s2 = wsum[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int n = __shfl_up_sync(0xffffffffu, s2, o);
      if (lane >= o) s2 += n;
    }
    wsum[lane] = s2;
  }
  __syncthreads();
  int off = x - tot + (w > 0 ? wsum[w - 1] : 0);
#pragma unroll
  for (int u = 0; u < PER; ++u) {
    const int i = t * PER + u;
    if (i < kCandKeys) cnt[i] = off;
    off += v[u];
  }
}

__global__ void k_cand_scatter(const int32_t* __restrict__ flags, const uint64_t* __restrict__ cand,
                               const int32_t* nflag, int* off, int32_t* flags_out,
                               uint64_t* cand_out) {
  const int n = *nflag;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const uint64_t mk = cand[i];
    const int at = atomicAdd(&off[cand_key(mk)], 1);
    flags_out[at] = flags[i];
    cand_out[at] = mk;
  }
}

extern "C" size_t sbo_cand_workspace_bytes(void) { return sizeof(int) * kCandKeys + 64; }

extern "C" int sbo_cand_sort(const int32_t* flags, const uint64_t* cand, const int32_t* nflag,
                             int64_t max_list, int32_t* flags_out, uint64_t* cand_out, void* ws,
                             size_t ws_bytes, void* stream) {
  if (ws_bytes < sbo_cand_workspace_bytes()) return fail(SBO_EINVAL, "cand workspace too small");
  if (!flags || !cand || !nflag || !flags_out || !cand_out) return fail(SBO_EINVAL, "null list");
  if (max_list <= 0) return SBO_OK;
  cudaStream_t st = as_stream(stream);
  int* cnt = static_cast<int*>(ws);
  SBO_CHECK_CUDA(cudaMemsetAsync(cnt, 0, sizeof(int) * kCandKeys, st));
  const int grid = static_cast<int>(ceil_div(max_list, 256) < 296 ? ceil_div(max_list, 256) : 296);
  k_cand_hist<<<grid, 256, 0, st>>>(cand, nflag, cnt);
  k_cand_scan<<<1, 1024, 0, st>>>(cnt);
  k_cand_scatter<<<grid, 256, 0, st>>>(flags, cand, nflag, cnt, flags_out, cand_out);
  return check_launch("k_cand_sort");
}

extern "C" size_t sbo_sum_workspace_bytes(int64_t n) {
  return sizeof(double) * (ceil_div(n, kSumTile) + 1) + 64;
}

extern "C" int sbo_sum(const double* x, int64_t n, double* total, void* ws, size_t ws_bytes,
                       void* stream) {
  if (ws_bytes < sbo_sum_workspace_bytes(n)) return fail(SBO_EINVAL, "sum workspace too small");
  cudaStream_t st = as_stream(stream);
  double* partial = static_cast<double*>(ws);
  const int64_t nt = ceil_div(n, kSumTile);
  if (nt == 0) {
    SBO_CHECK_CUDA(cudaMemsetAsync(total, 0, sizeof(double), st));
    return SBO_OK;
  }
  k_sum_tiles<<<static_cast<unsigned>(nt), kSumTile, 0, st>>>(x, n, partial);
  k_sum_final<<<1, 1024, 0, st>>>(partial, nt, total);
  return check_launch("k_sum_tiles");
}

extern "C" int sbo_defect(const double* Q, int K, int p, double* out, void* stream) {
  if (K < 1 || p < 1) return fail(SBO_EINVAL, "bad defect shape");
  k_defect<<<K, 256, 0, as_stream(stream)>>>(Q, p, out);
  return check_launch("k_defect");
}

extern "C" int sbo_frobenius_sq(const void* y, int dtype, int64_t m, int p, const double* blocks,
                                const int32_t* block, int s0, int64_t ld, const int16_t* idx,
                                const double* val, double* total, void* ws, size_t ws_bytes,
                                void* stream) {
  const int64_t n = ceil_div(m, 8);
  if (ws_bytes < sizeof(double) * (n + 1)) return fail(SBO_EINVAL, "frobenius workspace too small");
  cudaStream_t st = as_stream(stream);
  double* partial = static_cast<double*>(ws);
  if (n == 0) {
    SBO_CHECK_CUDA(cudaMemsetAsync(total, 0, sizeof(double), st));
    return SBO_OK;
  }
  const int k = s0 < p ? s0 : p;
  if (dtype == SBO_F32)
    k_frob<float><<<static_cast<unsigned>(n), 256, 0, st>>>(static_cast<const float*>(y), m, p,
                                                            blocks, block, k, ld, idx, val, partial);
  else
    k_frob<double><<<static_cast<unsigned>(n), 256, 0, st>>>(static_cast<const double*>(y), m, p,
                                                             blocks, block, k, ld, idx, val, partial);
  k_sum_final<<<1, 1024, 0, st>>>(partial, n, total);
  return check_launch("k_frob");
}
