// Exact warp-cooperative top-k of one float64 coefficient row (onb.py:58-76).
#pragma once

#include "common.cuh"

namespace sbo {

// Exact top-k of one coefficient row, warp-cooperative.  Lane l owns the
// coefficients i = l + 32 t.  Returns the selected mask bit t in `sel`.
struct RowPick {
  unsigned sel;     // bit t: coefficient lane+32t kept
  double score;     // warp-reduced: sum of kept c^2 (kind 0) or |c| (kind 1)
  double rest_sq;   // warp-reduced: sum of the DISCARDED c^2 = ||y - Q x||^2
};

__device__ inline RowPick pick_row_rank(const double* Cs, int p, int k, int kind) {
  const int lane = threadIdx.x & 31;
  const int T = (p + 31) >> 5;
  double a[8];
  int rank[8];
#pragma unroll
  for (int t = 0; t < 8; ++t) {
    const int i = lane + 32 * t;
    a[t] = (t < T && i < p) ? fabs(Cs[i]) : -1.0;
    rank[t] = 0;
  }
  for (int j = 0; j < p; ++j) {
    const double cj = fabs(Cs[j]);
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      if (t < T) {
        const int i = lane + 32 * t;
        rank[t] += (cj > a[t]) || (cj == a[t] && j < i);
      }
    }
  }
  RowPick r;
  r.sel = 0u;
  // The squared residual is accumulated from the discarded coefficients: equal
  // to ||y||^2 - sum(kept^2) by Parseval (the reference's formula, sbo.py:218)
  // but without its cancellation when the kept energy is close to ||y||^2.
  double sc = 0.0, sq = 0.0, rest = 0.0;
#pragma unroll
  for (int t = 0; t < 8; ++t) {
    const int i = lane + 32 * t;
    if (t < T && i < p) {
      const double c = Cs[i];
      if (rank[t] < k) {
        r.sel |= 1u << t;
        sq = fma(c, c, sq);
        sc += fabs(c);
      } else {
        rest = fma(c, c, rest);
      }
    }
  }
  r.score = warp_sum(kind == SBO_KIND_SQUARED_SUM ? sq : sc);
  r.rest_sq = warp_sum(rest);
  return r;
}

// Same result, faster for large p: the k-th largest fp32 magnitude T by bisection on
// its bit pattern (non-negative floats order like their bits; warp-wide counts by
// __reduce_add_sync).  fp32 rounding is monotone, so when exactly k magnitudes are
// >= T the kept set is the float64 one; otherwise (a tie at fp32 precision) the rank
// method decides.
__device__ inline RowPick pick_row(const double* Cs, int p, int k, int kind) {
  const int lane = threadIdx.x & 31;
  const int T = (p + 31) >> 5;
  uint32_t key[8];
  unsigned valid = 0u;
#pragma unroll
  for (int t = 0; t < 8; ++t) {
    const int i = lane + 32 * t;
    const bool on = t < T && i < p;
    key[t] = on ? __float_as_uint(static_cast<float>(fabs(Cs[i]))) : 0u;
    valid |= (on ? 1u : 0u) << t;
  }
  uint32_t th = 0u;
  for (int bit = 30; bit >= 0; --bit) {
    const uint32_t cand = th | (1u << bit);
    unsigned c = 0u;
#pragma unroll
    for (int t = 0; t < 8; ++t) c += ((valid >> t) & 1u) && key[t] >= cand;
    if (static_cast<int>(__reduce_add_sync(0xffffffffu, c)) >= k) th = cand;
  }
  unsigned sel = 0u, c = 0u;
#pragma unroll
  for (int t = 0; t < 8; ++t)
    if (((valid >> t) & 1u) && key[t] >= th) {
      sel |= 1u << t;
      ++c;
    }
  if (static_cast<int>(__reduce_add_sync(0xffffffffu, c)) != k) return pick_row_rank(Cs, p, k, kind);
  RowPick r;
  r.sel = sel;
  double sq = 0.0, sc = 0.0, rest = 0.0;
#pragma unroll
  for (int t = 0; t < 8; ++t) {
    if ((valid >> t) & 1u) {
      const double v = Cs[lane + 32 * t];
      if ((sel >> t) & 1u) {
        sq = fma(v, v, sq);
        sc += fabs(v);
      } else {
        rest = fma(v, v, rest);
      }
    }
  }
  r.score = warp_sum(kind == SBO_KIND_SQUARED_SUM ? sq : sc);
  r.rest_sq = warp_sum(rest);
  return r;
}

}  // namespace sbo

namespace sbo {

// Per-warp shared scratch of pick_row_cand.
struct PickScratch {
  double v[64];
  int16_t i[64];
  uint32_t bm[8];
};

// pick_row for p = 256, k <= 32 with fewer instructions: the k-th largest of the
// 32 lane maxima (a shuffle bitonic sort) bounds the k-th largest magnitude from
// below (k distinct coefficients reach it), so the kept set lies among the
// coefficients >= that bound — typically 20-30.  They are compacted to shared
// memory and ranked exactly (|c| descending, index ascending: the rule of
// pick_row_rank) in float64; more than 64 candidates fall back to pick_row.
__device__ inline RowPick pick_row_cand64(const double* Cs, int k, int kind, PickScratch& w) {
  const int lane = threadIdx.x & 31;
  const unsigned full = 0xffffffffu, lt = (1u << lane) - 1u;
  double a[8];
  double lm = 0.0;
#pragma unroll
  for (int t = 0; t < 8; ++t) {
    a[t] = fabs(Cs[lane + 32 * t]);
    lm = fmax(lm, a[t]);
  }
  // descending bitonic sort of the lane maxima
#pragma unroll
  for (int size = 2; size <= 32; size <<= 1) {
#pragma unroll
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      const double o = __shfl_xor_sync(full, lm, stride);
      const bool desc = size == 32 || (lane & size) == 0;
      const bool lower = (lane & stride) == 0;
      lm = (lower == desc) ? fmax(lm, o) : fmin(lm, o);
    }
  }
  const double lo = __shfl_sync(full, lm, k - 1);
  unsigned bal[8];
  int n = 0;
#pragma unroll
  for (int t = 0; t < 8; ++t) {
    bal[t] = __ballot_sync(full, a[t] >= lo);
    n += __popc(bal[t]);
  }
  if (n > 64) return pick_row(Cs, 256, k, kind);
  __syncwarp();
  if (lane < 8) w.bm[lane] = 0u;
  int base = 0;
#pragma unroll
  for (int t = 0; t < 8; ++t) {
    if ((bal[t] >> lane) & 1u) {
      const int at = base + __popc(bal[t] & lt);
      w.v[at] = a[t];
      w.i[at] = static_cast<int16_t>(lane + 32 * t);
    }
    base += __popc(bal[t]);
  }
  __syncwarp();
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int c = lane + 32 * h;
    if (c < n) {
      const double v = w.v[c];
      const int id = w.i[c];
      int rank = 0;
      for (int j = 0; j < n; ++j) {
        const double u = w.v[j];
        rank += (u > v) || (u == v && w.i[j] < id);
      }
      if (rank < k) atomicOr(&w.bm[id >> 5], 1u << (id & 31));
    }
  }
  __syncwarp();
  RowPick r;
  r.sel = 0u;
  double sq = 0.0, sc = 0.0, rest = 0.0;
#pragma unroll
  for (int t = 0; t < 8; ++t) {
    if ((w.bm[t] >> lane) & 1u) {
      r.sel |= 1u << t;
      sq = fma(a[t], a[t], sq);
      sc += a[t];
    } else {
      rest = fma(a[t], a[t], rest);
    }
  }
  __syncwarp();  // the scratch is reused by the warp's next row
  r.score = warp_sum(kind == SBO_KIND_SQUARED_SUM ? sq : sc);
  r.rest_sq = warp_sum(rest);
  return r;
}

// The same with 32-bit keys (|c| rounded toward zero to float32: monotone, so the
// bound from the lane maxima still admits every kept coefficient): the bound by a
// bitonic sort of integer keys, the candidates (at most 32, one per lane, in
// index order) ranked by shuffles.  When the kept set's smallest key is shared
// with a discarded candidate, the float32 keys cannot order them: pick_row_cand64
// decides (exact float64 ranking).
__device__ inline RowPick pick_row_cand(const double* Cs, int k, int kind, PickScratch& w) {
  const int lane = threadIdx.x & 31;
  const unsigned full = 0xffffffffu, lt = (1u << lane) - 1u;
  double a[8];
  uint32_t key[8];
  uint32_t lm = 0u;
#pragma unroll
  for (int t = 0; t < 8; ++t) {
    a[t] = fabs(Cs[lane + 32 * t]);
    key[t] = __float_as_uint(__double2float_rz(a[t]));
    lm = max(lm, key[t]);
  }
#pragma unroll
  for (int size = 2; size <= 32; size <<= 1) {
#pragma unroll
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      const uint32_t o = __shfl_xor_sync(full, lm, stride);
      const bool desc = size == 32 || (lane & size) == 0;
      const bool lower = (lane & stride) == 0;
      lm = (lower == desc) ? max(lm, o) : min(lm, o);
    }
  }
  const uint32_t lo = __shfl_sync(full, lm, k - 1);
  unsigned bal[8];
  int n = 0;
#pragma unroll
  for (int t = 0; t < 8; ++t) {
    bal[t] = __ballot_sync(full, key[t] >= lo);
    n += __popc(bal[t]);
  }
  if (n > 32) return pick_row_cand64(Cs, k, kind, w);
  // compaction in index order (index = lane + 32 t: t-major, lanes ascending)
  __syncwarp();
  int base = 0;
#pragma unroll
  for (int t = 0; t < 8; ++t) {
    if ((bal[t] >> lane) & 1u) {
      const int at = base + __popc(bal[t] & lt);
      w.i[at] = static_cast<int16_t>(lane + 32 * t);
      reinterpret_cast<uint32_t*>(w.v)[at] = key[t];
    }
    base += __popc(bal[t]);
  }
  if (lane < 8) w.bm[lane] = 0u;
  __syncwarp();
  const bool has = lane < n;
  const uint32_t ck = has ? reinterpret_cast<const uint32_t*>(w.v)[lane] : 0u;
  int rank = 0;
  for (int j = 0; j < n; ++j) {
    const uint32_t kj = __shfl_sync(full, ck, j);
    rank += (kj > ck) || (kj == ck && j < lane);
  }
  const bool sel = has && rank < k;
  const uint32_t tmin = __reduce_min_sync(full, sel ? ck : 0xffffffffu);
  if (__any_sync(full, has && !sel && ck == tmin)) return pick_row_cand64(Cs, k, kind, w);
  if (sel) {
    const int id = w.i[lane];
    atomicOr(&w.bm[id >> 5], 1u << (id & 31));
  }
  __syncwarp();
  RowPick r;
  r.sel = 0u;
  double sq = 0.0, sc = 0.0, rest = 0.0;
#pragma unroll
  for (int t = 0; t < 8; ++t) {
    if ((w.bm[t] >> lane) & 1u) {
      r.sel |= 1u << t;
      sq = fma(a[t], a[t], sq);
      sc += a[t];
    } else {
      rest = fma(a[t], a[t], rest);
    }
  }
  __syncwarp();  // the scratch is reused by the warp's next row
  r.score = warp_sum(kind == SBO_KIND_SQUARED_SUM ? sq : sc);
  r.rest_sq = warp_sum(rest);
  return r;
}

}  // namespace sbo
