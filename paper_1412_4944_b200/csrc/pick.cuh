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

__device__ inline RowPick pick_row(const double* Cs, int p, int k, int kind) {
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

}  // namespace sbo
