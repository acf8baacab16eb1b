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
