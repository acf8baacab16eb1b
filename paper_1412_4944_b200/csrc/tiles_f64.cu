// Float64 tile kernels: projection onto orthonormal blocks, exact hard-threshold
// selection, energy/argmax, own-block coding and sparse outer products.
//
// These are the exact (float64, CUDA-core) implementations of the reference's
// represent / select_top / sparse_outer (sbo.py:138-220, onb.py:58-76, 127-134).
// They serve every signal dimension p <= 256 and every s0, and they are the
// certification path of the tensor-core kernels (tc_represent.cu).
//
// Tile geometry: a CTA of 256 threads owns 64 signals.  C = Y_tile . Q_b is
// built in 64x64 chunks with a 4x4 register tile per thread (y and q staged in
// shared memory as float64), then each warp ranks its signals' coefficients:
// coefficient i is kept iff fewer than k coefficients beat it under the key
// (|c| descending, index ascending) — the stable-argsort rule of onb.py:73.
#include "common.cuh"
#include "pick.cuh"
#include "topk.cuh"

namespace sbo {

constexpr int kSyLd = kTile + 2;  // float64 row stride of the staged y chunk (16B aligned rows)

// p <= 64 tiles use the float64 tensor cores (DMMA) with 68-double rows
constexpr int kDmmaLd = 68;

struct TileLayout {
  int p, ldc;
  size_t c_off, y_off, q_off, rows_off, misc_off, bytes;
  __host__ __device__ explicit TileLayout(int p_) : p(p_) {
    ldc = p <= 64 ? kDmmaLd : p + 1;
    c_off = 0;
    y_off = c_off + sizeof(double) * kTile * ldc;
    y_off = (y_off + 15) & ~size_t(15);
    q_off = y_off + sizeof(double) * 64 * kDmmaLd;
    rows_off = q_off + sizeof(double) * 64 * kDmmaLd;
    misc_off = rows_off + sizeof(int64_t) * kTile;
    bytes = misc_off + sizeof(double) * kTile * 3 + 2 * sizeof(int) * kTile + 64;
  }
};

__device__ __forceinline__ void dmma8(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// p <= 64 staging, zero padded to 64: signals signal-major sY[s][k], block sQ[k][i]
template <typename TY>
__device__ void stage_y64(const TY* __restrict__ y, int p, const int64_t* rows, double* sY) {
  for (int e = threadIdx.x; e < kTile * 64; e += kThreads) {
    const int s = e >> 6, kk = e & 63;
    const int64_t r = rows[s];
    sY[s * kDmmaLd + kk] = (r >= 0 && kk < p) ? static_cast<double>(__ldg(y + r * p + kk)) : 0.0;
  }
}
__device__ void stage_q64(const double* __restrict__ q, int p, double* sQ) {
  for (int e = threadIdx.x; e < 64 * 64; e += kThreads) {
    const int kk = e >> 6, ii = e & 63;
    sQ[kk * kDmmaLd + ii] = (kk < p && ii < p) ? __ldg(q + kk * p + ii) : 0.0;
  }
}
// C[s][i] = sum_k sY[s][k] sQ[k][i] on DMMA; warp w: signals [8w, 8w+8) x 64 atoms
__device__ void project64_dmma(const double* sY, const double* sQ, double* C) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, g = lane >> 2, t4 = lane & 3;
  double c[8][2];
#pragma unroll
  for (int n = 0; n < 8; ++n) c[n][0] = c[n][1] = 0.0;
  const double* ya = sY + (8 * warp + g) * kDmmaLd + t4;
#pragma unroll 4
  for (int k0 = 0; k0 < 64; k0 += 4) {
    const double a = ya[k0];
    const double* qb = sQ + (k0 + t4) * kDmmaLd + g;
#pragma unroll
    for (int n = 0; n < 8; ++n) dmma8(c[n][0], c[n][1], a, qb[8 * n]);
  }
  double* crow = C + (8 * warp + g) * kDmmaLd + 2 * t4;
#pragma unroll
  for (int n = 0; n < 8; ++n)
    *reinterpret_cast<double2*>(crow + 8 * n) = make_double2(c[n][0], c[n][1]);
}

// p > 64: C[s][i] = sum_k y[rows[s]][k] Q[k][i] on DMMA in 64 x 64 chunks — per
// 64-atom column chunk, the 64-wide K chunks are staged (sY[s][k], sQ[k][i], row
// stride 68) and accumulated in the warps' fragments (warp w: signals 8w..8w+8).
template <typename TY>
__device__ void project_tile_dmma(const TY* __restrict__ y, int p, const int64_t* rows,
                                  const double* __restrict__ q, double* C, int ldc, double* sY,
                                  double* sQ) {
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t4 = lane & 3;
  for (int ic = 0; ic < p; ic += 64) {
    double c[8][2];
#pragma unroll
    for (int n = 0; n < 8; ++n) c[n][0] = c[n][1] = 0.0;
    for (int kc = 0; kc < p; kc += 64) {
      __syncthreads();
      // the chunk's loads in batches of 8 per thread, all in flight before the
      // batch's stores (a load-store loop pays one memory latency per element,
      // 16 of them per chunk and 16 chunks per tile at p = 256)
      constexpr int PER = kTile * 64 / kThreads, BATCH = 8;
#pragma unroll
      for (int u0 = 0; u0 < PER; u0 += BATCH) {
        double vy[BATCH], vq[BATCH];
#pragma unroll
        for (int u = 0; u < BATCH; ++u) {
          const int e = tid + (u0 + u) * kThreads, s = e >> 6, kk = e & 63;
          const int64_t r = rows[s];
          vy[u] = (r >= 0 && kc + kk < p) ? static_cast<double>(__ldg(y + r * p + kc + kk)) : 0.0;
          vq[u] = (kc + s < p && ic + kk < p)
                      ? __ldg(q + static_cast<int64_t>(kc + s) * p + ic + kk)
                      : 0.0;
        }
#pragma unroll
        for (int u = 0; u < BATCH; ++u) {
          const int e = tid + (u0 + u) * kThreads, s = e >> 6, kk = e & 63;
          sY[s * kDmmaLd + kk] = vy[u];
          sQ[s * kDmmaLd + kk] = vq[u];
        }
      }
      __syncthreads();
      const double* ya = sY + (8 * warp + g) * kDmmaLd + t4;
#pragma unroll 4
      for (int k0 = 0; k0 < 64; k0 += 4) {
        const double a = ya[k0];
        const double* qb = sQ + (k0 + t4) * kDmmaLd + g;
#pragma unroll
        for (int n = 0; n < 8; ++n) dmma8(c[n][0], c[n][1], a, qb[8 * n]);
      }
    }
    double* crow = C + (8 * warp + g) * ldc + ic + 2 * t4;
#pragma unroll
    for (int n = 0; n < 8; ++n)
#pragma unroll
      for (int h = 0; h < 2; ++h)
        if (ic + 8 * n + 2 * t4 + h < p) crow[8 * n + h] = c[n][h];
  }
  __syncthreads();
}

// Fast exact selection for p <= 64, k <= 15: four lanes per signal (a quad);
// lane q owns coefficients i = q + 4u, u < 16.  The fp32 magnitudes are a
// monotone rounding of the float64 ones, so when the k-th and (k+1)-th largest
// fp32 magnitudes differ, the kept set is exactly {i : fp32|c_i| >= t_k} — the
// same set as the float64 stable-argsort rule.  Otherwise ok = false and the
// caller re-decides that signal with pick_row.  All 32 lanes must call this.
struct QuadPick {
  bool ok;
  uint32_t mask;  // bit u: coefficient q + 4u kept
  double score, rest_sq;
};

__device__ __forceinline__ double quad_sum(double v) {
  v += __shfl_xor_sync(0xffffffffu, v, 1);
  v += __shfl_xor_sync(0xffffffffu, v, 2);
  return v;
}

__device__ QuadPick quad_pick(const double* Cs, int p, int k, int kind, bool active) {
  const int q = threadIdx.x & 3;
  double c[16];
  float a[16], srt[16];
#pragma unroll
  for (int u = 0; u < 16; ++u) {
    const int i = q + 4 * u;
    const bool on = active && i < p;
    c[u] = on ? Cs[i] : 0.0;
    a[u] = on ? static_cast<float>(fabs(c[u])) : -1.0f;
    srt[u] = a[u];
  }
  topk::sort_desc<16>(srt);
#pragma unroll
  for (int x = 1; x <= 2; x <<= 1) {
    float other[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) other[u] = __shfl_xor_sync(0xffffffffu, srt[u], x);
    topk::merge_top<16>(srt, other);
  }
  float tk = srt[0], tk1 = srt[1];
#pragma unroll
  for (int u = 1; u < 16; ++u) {
    if (u == k - 1) tk = srt[u];
    if (u == k) tk1 = srt[u];
  }
  QuadPick r;
  r.ok = tk > tk1;
  r.mask = 0u;
  double sq = 0.0, sa = 0.0, rest = 0.0;
#pragma unroll
  for (int u = 0; u < 16; ++u) {
    if (q + 4 * u < p) {
      if (a[u] >= tk) {
        r.mask |= 1u << u;
        sq = fma(c[u], c[u], sq);
        sa += fabs(c[u]);
      } else {
        rest = fma(c[u], c[u], rest);
      }
    }
  }
  sq = quad_sum(sq);
  sa = quad_sum(sa);
  r.rest_sq = quad_sum(rest);
  r.score = kind == SBO_KIND_SQUARED_SUM ? sq : sa;
  return r;
}

// ascending position of kept coefficient i among the quad's kept set
__device__ __forceinline__ int quad_position(const uint32_t (&masks)[4], int i) {
  int pos = 0;
#pragma unroll
  for (int q2 = 0; q2 < 4; ++q2) {
    const int below = i > q2 ? (i - q2 + 3) >> 2 : 0;  // u' with q2 + 4u' < i
    pos += __popc(masks[q2] & ((below >= 32) ? 0xffffffffu : ((1u << below) - 1u)));
  }
  return pos;
}

// ---------------------------------------------------------------------------
// energy pass (sbo.py:177-194), fresh or incremental
// ---------------------------------------------------------------------------
template <typename TY>
__global__ void __launch_bounds__(kThreads) k_energy_f64(
    const TY* __restrict__ y, int64_t m, int p, const double* __restrict__ blocks, int b0,
    int b1, int k, int kind, int accumulate, const int32_t* __restrict__ list,
    const int32_t* __restrict__ nlist, int32_t* best, double* score, double* rest_sq,
    double* norm_sq, const uint64_t* __restrict__ cand) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ unsigned long long tile_cand;  // union of the tile's candidate blocks (bit b - b0)
  const TileLayout L(p);
  double* C = reinterpret_cast<double*>(smem + L.c_off);
  double* sY = reinterpret_cast<double*>(smem + L.y_off);
  double* sQ = reinterpret_cast<double*>(smem + L.q_off);
  int64_t* rows = reinterpret_cast<int64_t*>(smem + L.rows_off);
  double* bscore = reinterpret_cast<double*>(smem + L.misc_off);
  double* brest = bscore + kTile;
  double* bnorm = brest + kTile;
  int* bbest = reinterpret_cast<int*>(bnorm + kTile);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // signals: [0, m), or list[0 .. *nlist) (the float64 re-decision of flagged signals)
  const int64_t count = list ? static_cast<int64_t>(*nlist) : m;
  for (int64_t base = static_cast<int64_t>(blockIdx.x) * kTile; base < count;
       base += static_cast<int64_t>(gridDim.x) * kTile) {
    __syncthreads();
    if (threadIdx.x < kTile) {
      const int64_t t = base + threadIdx.x;
      const int64_t j = t < count ? (list ? static_cast<int64_t>(list[t]) : t) : -1;
      rows[threadIdx.x] = j;
      if (accumulate && j >= 0) {
        bbest[threadIdx.x] = best[j];
        bscore[threadIdx.x] = score[j];
        brest[threadIdx.x] = rest_sq[j];
      } else {
        bbest[threadIdx.x] = -1;
        bscore[threadIdx.x] = -1.0;
        brest[threadIdx.x] = 0.0;
      }
    }
    if (threadIdx.x == 0) tile_cand = cand ? 0ull : ~0ull;
    __syncthreads();
    if (cand && threadIdx.x < kTile && base + threadIdx.x < count)
      atomicOr(&tile_cand, static_cast<unsigned long long>(cand[base + threadIdx.x]));
    __syncthreads();
    const unsigned long long tcand = tile_cand;
    int* fb = bbest + kTile;  // per-signal "needs the exact rank method" marks
    if (p <= 64) stage_y64(y, p, rows, sY);
    for (int b = b0; b < b1; ++b) {
      if (b - b0 < 64 && !((tcand >> (b - b0)) & 1ull)) continue;  // no signal of the tile can win here
      if (p <= 64) {
        __syncthreads();
        stage_q64(blocks + static_cast<int64_t>(b) * p * p, p, sQ);
        __syncthreads();
        project64_dmma(sY, sQ, C);
        __syncthreads();
      } else {
        project_tile_dmma(y, p, rows, blocks + static_cast<int64_t>(b) * p * p, C, L.ldc, sY, sQ);
      }
      if (p <= 64 && k < 16) {
        const int s = threadIdx.x >> 2;
        const bool act = rows[s] >= 0;
        const QuadPick r = quad_pick(C + s * L.ldc, p, k, kind, act);
        if ((threadIdx.x & 3) == 0) {
          fb[s] = act && !r.ok;
          if (act && r.ok && r.score > bscore[s]) {  // strict: first maximum wins (sbo.py:191)
            bscore[s] = r.score;
            brest[s] = r.rest_sq;
            bbest[s] = b;
          }
        }
        __syncthreads();
      }
      for (int s = warp; s < kTile; s += kThreads / 32) {
        if (rows[s] < 0 || (p <= 64 && k < 16 && !fb[s])) continue;
        const RowPick r = pick_row(C + s * L.ldc, p, k, kind);
        if (lane == 0 && r.score > bscore[s]) {
          bscore[s] = r.score;
          brest[s] = r.rest_sq;
          bbest[s] = b;
        }
      }
      __syncthreads();
    }
    // ||y||^2 in float64
    for (int s = warp; s < kTile; s += kThreads / 32) {
      const int64_t j = rows[s];
      if (j < 0) continue;
      double acc = 0.0;
      for (int kk = lane; kk < p; kk += 32) {
        const double v = y[j * p + kk];
        acc = fma(v, v, acc);
      }
      acc = warp_sum(acc);
      if (lane == 0) bnorm[s] = acc;
    }
    __syncthreads();
    if (threadIdx.x < kTile && rows[threadIdx.x] >= 0) {
      const int64_t j = rows[threadIdx.x];
      best[j] = bbest[threadIdx.x];
      score[j] = bscore[threadIdx.x];
      rest_sq[j] = brest[threadIdx.x];
      if (norm_sq) norm_sq[j] = bnorm[threadIdx.x];
    }
  }
}

// ---------------------------------------------------------------------------
// own-block coding over segments (sbo.py:196-211, onb.py:170)
// ---------------------------------------------------------------------------
template <typename TY>
__global__ void __launch_bounds__(kThreads) k_code_f64(
    const TY* __restrict__ y, int p, const int32_t* __restrict__ order,
    const int32_t* __restrict__ seg_block, const int64_t* __restrict__ seg_lo,
    const int64_t* __restrict__ seg_hi, const int32_t* __restrict__ nseg,
    const double* __restrict__ blocks, int block_override, int k, int kind, int out_by_signal,
    int64_t ld, int16_t* idx, double* val, double* energy, double* rest_sq) {
  if (static_cast<int>(blockIdx.x) >= *nseg) return;
  extern __shared__ __align__(16) unsigned char smem[];
  const TileLayout L(p);
  double* C = reinterpret_cast<double*>(smem + L.c_off);
  double* sY = reinterpret_cast<double*>(smem + L.y_off);
  double* sQ = reinterpret_cast<double*>(smem + L.q_off);
  int64_t* rows = reinterpret_cast<int64_t*>(smem + L.rows_off);

  const int seg = blockIdx.x;
  const int b = block_override >= 0 ? block_override : seg_block[seg];
  const int64_t lo = seg_lo[seg], hi = seg_hi[seg];
  const double* q = blocks + static_cast<int64_t>(b) * p * p;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const unsigned lt = (1u << lane) - 1u;
  if (p <= 64) stage_q64(q, p, sQ);  // the segment's block, staged once
  for (int64_t t0 = lo; t0 < hi; t0 += kTile) {
    __syncthreads();
    if (threadIdx.x < kTile) {
      const int64_t t = t0 + threadIdx.x;
      rows[threadIdx.x] = t < hi ? (order ? static_cast<int64_t>(order[t]) : t) : -1;
    }
    __syncthreads();
    if (p <= 64) {
      stage_y64(y, p, rows, sY);
      __syncthreads();
      project64_dmma(sY, sQ, C);
      __syncthreads();
    } else {
      project_tile_dmma(y, p, rows, q, C, L.ldc, sY, sQ);
    }
    int* fb = reinterpret_cast<int*>(smem + L.misc_off);
    const bool quad = p <= 64 && k < 16;
    if (quad) {
      const int s = threadIdx.x >> 2, qd = threadIdx.x & 3;
      const bool act = rows[s] >= 0;
      const double* Cs = C + s * L.ldc;
      const QuadPick r = quad_pick(Cs, p, k, kind, act);
      uint32_t masks[4];
#pragma unroll
      for (int x = 0; x < 4; ++x)
        masks[x] = __shfl_sync(0xffffffffu, r.mask, (threadIdx.x & 31 & ~3) | x);
      if (qd == 0) fb[s] = act && !r.ok;
      if (act && r.ok) {
        const int64_t col = out_by_signal ? rows[s] : (t0 + s);
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          if (idx && ((r.mask >> u) & 1u)) {  // idx == NULL: residuals only
            const int i = qd + 4 * u;
            const int at = quad_position(masks, i);
            idx[at * ld + col] = static_cast<int16_t>(i);
            val[at * ld + col] = Cs[i];
          }
        }
        if (qd == 0) {
          if (energy) energy[col] = r.score;
          if (rest_sq) rest_sq[col] = r.rest_sq;
        }
      }
      __syncthreads();
    }
    for (int s = warp; s < kTile; s += kThreads / 32) {
      if (rows[s] < 0 || (quad && !fb[s])) continue;
      const double* Cs = C + s * L.ldc;
      const RowPick r = pick_row(Cs, p, k, kind);
      const int64_t col = out_by_signal ? rows[s] : (t0 + s);
      int pos = 0;
      const int T = (p + 31) >> 5;
      for (int t = 0; t < T; ++t) {
        const bool on = (r.sel >> t) & 1u;
        const unsigned bal = __ballot_sync(0xffffffffu, on);
        if (on && idx) {
          const int at = pos + __popc(bal & lt);
          idx[at * ld + col] = static_cast<int16_t>(lane + 32 * t);
          val[at * ld + col] = Cs[lane + 32 * t];
        }
        pos += __popc(bal);
      }
      if (lane == 0) {
        if (energy) energy[col] = r.score;
        if (rest_sq) rest_sq[col] = r.rest_sq;
      }
    }
  }
}

// ---------------------------------------------------------------------------
// sparse outer products P = Y X^T per segment (onb.py:127-134) and the Gram
// matrix of a member list (X = Y).  The code block is densified per 64-column
// chunk in shared memory; P is accumulated in registers (4x4 per thread) in
// signal order, so partials are deterministic.
// ---------------------------------------------------------------------------
struct OuterLayout {
  size_t yt_off, x_off, rows_off, bytes;
  __host__ __device__ OuterLayout() {
    yt_off = 0;
    x_off = yt_off + sizeof(double) * kTile * kSyLd;
    rows_off = x_off + sizeof(double) * kTile * kSyLd;
    bytes = rows_off + sizeof(int64_t) * kTile;
  }
};

template <typename TY>
__global__ void __launch_bounds__(kThreads) k_outer_f64(
    const TY* __restrict__ y, int p, const int32_t* __restrict__ order,
    const int64_t* __restrict__ seg_lo, const int64_t* __restrict__ seg_hi,
    const int32_t* __restrict__ nseg, int k, int64_t ld, const int16_t* __restrict__ idx,
    const double* __restrict__ val, int dense_self, double* partial) {
  if (static_cast<int>(blockIdx.x) >= *nseg) return;
  extern __shared__ __align__(16) unsigned char smem[];
  const OuterLayout L;
  double* sYt = reinterpret_cast<double*>(smem + L.yt_off);  // [s][kk]
  double* sX = reinterpret_cast<double*>(smem + L.x_off);    // [s][ii]
  int64_t* rows = reinterpret_cast<int64_t*>(smem + L.rows_off);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t4 = lane & 3;
  const int seg = blockIdx.x;
  const int64_t lo = seg_lo[seg], hi = seg_hi[seg];
  double* out = partial + static_cast<int64_t>(seg) * p * p;

  // one 64 x 64 output tile (kc, ic) of the segment's partial per CTA (blockIdx.y)
  const int nic = (p + 63) / 64;
  {
    const int kc = 64 * (static_cast<int>(blockIdx.y) / nic), ic = 64 * (static_cast<int>(blockIdx.y) % nic);
    const int kn = min(64, p - kc);
    {
      const int in = min(64, p - ic);
      // P[kc + 8 warp + g][ic + 8 n + 2 t4 + h] on DMMA (m8n8k4): A = Y^T (rows kk,
      // k = signals), B = X (signals x atoms), signals in order 4 at a time
      double acc[8][2];
#pragma unroll
      for (int n = 0; n < 8; ++n) acc[n][0] = acc[n][1] = 0.0;
      for (int64_t t0 = lo; t0 < hi; t0 += kTile) {
        __syncthreads();
        if (tid < kTile) {
          const int64_t t = t0 + tid;
          rows[tid] = t < hi ? (order ? static_cast<int64_t>(order[t]) : t) : -1;
        }
        __syncthreads();
        for (int e = tid; e < kTile * 64; e += kThreads) {
          const int s = e >> 6, kk = e & 63;
          const int64_t r = rows[s];
          double v = 0.0, x = 0.0;
          if (r >= 0) {
            if (kk < kn) v = static_cast<double>(__ldg(y + r * p + kc + kk));
            if (dense_self && kk < in) x = static_cast<double>(__ldg(y + r * p + ic + kk));
          }
          sYt[s * kSyLd + kk] = v;
          sX[s * kSyLd + kk] = x;
        }
        if (!dense_self) {
          __syncthreads();
          for (int e = tid; e < kTile * k; e += kThreads) {
            const int s = e / k, rr = e % k;
            if (rows[s] < 0) continue;
            const int64_t col = t0 + s;
            const int i = idx[rr * ld + col];
            if (i >= ic && i < ic + in) sX[s * kSyLd + (i - ic)] = val[rr * ld + col];
          }
        }
        __syncthreads();
        // rows of signals beyond the segment are zero in both staged operands
        const double* ya = sYt + t4 * kSyLd + 8 * warp + g;
        const double* xb = sX + t4 * kSyLd + g;
#pragma unroll 4
        for (int s4 = 0; s4 < kTile; s4 += 4) {
          const double av = ya[s4 * kSyLd];
#pragma unroll
          for (int n = 0; n < 8; ++n) dmma8(acc[n][0], acc[n][1], av, xb[s4 * kSyLd + 8 * n]);
        }
      }
      const int row = 8 * warp + g;
#pragma unroll
      for (int n = 0; n < 8; ++n)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int col = 8 * n + 2 * t4 + h;
          if (row < kn && col < in) out[static_cast<int64_t>(kc + row) * p + ic + col] = acc[n][h];
        }
    }
  }
}

// Sparse outer products for p = 256 (config D), k <= 32 kept atoms per signal:
// P[d][a] = sum over the segment's signals of y[d] x[a], on the CUDA cores in
// float64 with only the kept pairs multiplied (k / p = 1/16 of the dense DMMA
// product's work).  CTA (segment, dim quarter): 32 warps, warp w owns atoms
// w + 32 j, lane the dims 64 q + 2 lane + {0, 1} — 16 float64 accumulators in
// registers.  Per chunk of 64 signals: the quarter's y rows as float64 and the
// codes densified per atom in shared memory with a 64-bit signal mask per atom
// (atomicOr: order-free); each warp walks its atoms' masks in ascending signal
// order, so the summation order — and the partial — is deterministic.  The next
// chunk's y and codes are prefetched into registers during the FMAs; the
// partial leaves through shared memory as coalesced 2-KB rows.
namespace osp {
constexpr int P = 256, DQ = 64, C = 64, THREADS = 1024, WARPS = 32, AW = P / WARPS;
constexpr int YPT = C * DQ / THREADS;  // y values per thread per chunk
constexpr int TLD = P + 1;             // row stride of the transposed partial
constexpr int KMAX = 32, CODES = C * KMAX / THREADS;  // code entries per thread
struct Smem {
  double ys[C][DQ];
  double xval[P][C];
  uint32_t mask[2][P][C / 32];
};
static_assert(C * DQ + P * C >= DQ * TLD, "the transposed partial fits in ys + xval");
}  // namespace osp

template <typename TY>
__global__ void __launch_bounds__(osp::THREADS, 1) k_outer_sparse256(
    const TY* __restrict__ y, const int32_t* __restrict__ order,
    const int64_t* __restrict__ seg_lo, const int64_t* __restrict__ seg_hi,
    const int32_t* __restrict__ nseg, int k, int64_t ld, const int16_t* __restrict__ idx,
    const double* __restrict__ val, double* partial) {
  using namespace osp;
  if (static_cast<int>(blockIdx.x) >= *nseg) return;
  extern __shared__ __align__(16) unsigned char smem[];
  Smem& S = *reinterpret_cast<Smem*>(smem);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int seg = blockIdx.x, d0 = DQ * static_cast<int>(blockIdx.y);
  const int64_t lo = seg_lo[seg], hi = seg_hi[seg];
  reinterpret_cast<uint32_t*>(S.mask)[tid] = 0u;  // both mask buffers: 2 x 256 x 2 words
  // prefetch: y row tid / 16, dims d0 + 4 (tid % 16) .. + 3; code entries
  // e = tid + 1024 i (signal e % 64, slot e / 64)
  const int yr = tid >> 4, yc = YPT * (tid & 15);
  double yv[YPT];
  int ci[CODES];
  double cv[CODES];
  auto prefetch = [&](int64_t t0) {
    const int64_t t = t0 + yr;
    if (t < hi) {
      const int64_t r = order ? static_cast<int64_t>(order[t]) : t;
      const TY* src = y + r * P + d0 + yc;
#pragma unroll
      for (int i = 0; i < YPT; ++i) yv[i] = static_cast<double>(__ldg(src + i));
    } else {
#pragma unroll
      for (int i = 0; i < YPT; ++i) yv[i] = 0.0;
    }
#pragma unroll
    for (int i = 0; i < CODES; ++i) {
      const int e = tid + THREADS * i, s = e % C, u = e / C;
      const int64_t col = t0 + s;
      ci[i] = -1;
      if (u < k && col < hi) {
        ci[i] = idx[u * ld + col];
        cv[i] = val[u * ld + col];
      }
    }
  };
  double acc[AW][2];
#pragma unroll
  for (int j = 0; j < AW; ++j) acc[j][0] = acc[j][1] = 0.0;
  int buf = 0;
  if (lo < hi) prefetch(lo);
  __syncthreads();
  for (int64_t t0 = lo; t0 < hi; t0 += C) {
    // stage the prefetched chunk (the previous chunk's FMAs are done: sync below)
#pragma unroll
    for (int i = 0; i < YPT; i += 2)
      *reinterpret_cast<double2*>(&S.ys[yr][yc + i]) = make_double2(yv[i], yv[i + 1]);
#pragma unroll
    for (int i = 0; i < CODES; ++i) {
      if (ci[i] >= 0) {
        const int s = (tid + THREADS * i) % C;
        S.xval[ci[i]][s] = cv[i];
        atomicOr(&S.mask[buf][ci[i]][s >> 5], 1u << (s & 31));
      }
    }
    __syncthreads();
    if (t0 + C < hi) prefetch(t0 + C);
    if (tid < P * (C / 32)) reinterpret_cast<uint32_t*>(S.mask[buf ^ 1])[tid] = 0u;  // next chunk's
#pragma unroll
    for (int j = 0; j < AW; ++j) {
      const int a = warp + WARPS * j;
#pragma unroll
      for (int w = 0; w < C / 32; ++w) {
        for (uint32_t m = S.mask[buf][a][w]; m; m &= m - 1) {
          const int s = 32 * w + __ffs(m) - 1;
          const double x = S.xval[a][s];
          const double2 yy = *reinterpret_cast<const double2*>(&S.ys[s][2 * lane]);
          acc[j][0] = fma(yy.x, x, acc[j][0]);
          acc[j][1] = fma(yy.y, x, acc[j][1]);
        }
      }
    }
    buf ^= 1;
    __syncthreads();
  }
  // transpose through shared memory (ys + xval, free after the loop's last sync)
  double* T = &S.ys[0][0];
#pragma unroll
  for (int j = 0; j < AW; ++j) {
    const int a = warp + WARPS * j;
    T[(2 * lane) * TLD + a] = acc[j][0];
    T[(2 * lane + 1) * TLD + a] = acc[j][1];
  }
  __syncthreads();
  double* out = partial + static_cast<int64_t>(seg) * P * P + static_cast<int64_t>(d0) * P;
  for (int e = tid; e < DQ * P; e += THREADS) out[e] = T[(e / P) * TLD + e % P];
}

// P_b = sum of block b's segment partials.  A CTA owns 32 consecutive elements;
// its 8 warps take the segments s0 + w, s0 + w + 8, ... (coalesced 256-B rows),
// and the 8 slice sums are added in slice order: a fixed summation order, so the
// result is deterministic, with 8x the memory-level parallelism of one thread
// per element.
__global__ void __launch_bounds__(256) k_reduce_segments(const double* __restrict__ partial,
                                                        const int32_t* __restrict__ seg_block,
                                                        const int32_t* __restrict__ nseg, int K,
                                                        int p, double* P) {
  __shared__ double part[8][33];
  __shared__ int range[2];
  const int b = blockIdx.y;
  const int64_t pp = static_cast<int64_t>(p) * p;
  const int el = threadIdx.x & 31, sl = threadIdx.x >> 5;
  const int64_t e = static_cast<int64_t>(blockIdx.x) * 32 + el;
  if (threadIdx.x < 32) {
    // segments are sorted by block: block b's range [s0, s1) by a 32-way search
    // (each round narrows [lo, hi) to one of 32 slices with one load per lane:
    // two or three dependent loads instead of a binary search's ~11)
    const int lane32 = threadIdx.x;
    const int n = *nseg;
    int s0 = 0, s1 = n;
    if (seg_block) {
      for (int pass = 0; pass < 2; ++pass) {  // pass 0: first s with block >= b; 1: > b
        const int key = b + pass;
        int lo = 0, hi = n;  // answer in [lo, hi]
        while (hi - lo > 0) {
          const int step = (hi - lo + 31) / 32;
          const int probe = lo + lane32 * step;
          const bool below = probe < hi && seg_block[probe] < key;
          const unsigned bal = __ballot_sync(0xffffffffu, below);
          const int cnt = __popc(bal);  // probes below key: a prefix of the lanes
          const int nlo = cnt == 0 ? lo : lo + (cnt - 1) * step + 1;
          const int nhi = cnt == 0 ? lo : min(hi, lo + cnt * step);
          if (step == 1) {
            lo = hi = lo + cnt;
            break;
          }
          lo = nlo;
          hi = nhi;
        }
        if (pass == 0) s0 = lo;
        else s1 = lo;
      }
    } else if (b != 0) {
      s1 = 0;
    }
    if (lane32 == 0) {
      range[0] = s0;
      range[1] = s1;
    }
  }
  __syncthreads();
  const int s0 = range[0], s1 = range[1];
  double acc = 0.0;
  if (e < pp) {
    int s = s0 + sl;
    for (; s + 24 < s1; s += 32) {  // 4 independent loads in flight
      const double v0 = __ldcs(partial + static_cast<int64_t>(s) * pp + e);
      const double v1 = __ldcs(partial + static_cast<int64_t>(s + 8) * pp + e);
      const double v2 = __ldcs(partial + static_cast<int64_t>(s + 16) * pp + e);
      const double v3 = __ldcs(partial + static_cast<int64_t>(s + 24) * pp + e);
      acc += v0;
      acc += v1;
      acc += v2;
      acc += v3;
    }
    for (; s < s1; s += 8) acc += __ldcs(partial + static_cast<int64_t>(s) * pp + e);
  }
  part[sl][el] = acc;
  __syncthreads();
  if (sl == 0 && e < pp) {
    double t = part[0][el];
#pragma unroll
    for (int w = 1; w < 8; ++w) t += part[w][el];
    P[b * pp + e] = t;
  }
}

// Gram partials over chunks of a member list, then the ordered reduction
// (count, optional: the list length on the device, at most w — a sharded
// worst set's local member count, never read back to the host)
__global__ void k_chunk_segments(int64_t w, const int64_t* count, int chunk, int64_t* lo,
                                 int64_t* hi, int32_t* nseg) {
  if (count) w = min64(w, max(*count, int64_t(0)));
  const int64_t n = ceil_div(w, chunk);
  for (int64_t s = threadIdx.x; s < n; s += blockDim.x) {
    lo[s] = s * chunk;
    hi[s] = min64(w, (s + 1) * chunk);
  }
  if (threadIdx.x == 0) *nseg = static_cast<int32_t>(n);
}

}  // namespace sbo

using namespace sbo;


namespace {
template <typename TY>
int energy_impl(const void* yv, int64_t m, int p, const double* blocks, int b0, int b1, int k,
                int kind, int accumulate, const int32_t* list, const int32_t* nlist,
                int64_t max_list, int32_t* best, double* score, double* rest_sq,
                double* norm_sq, cudaStream_t st, const uint64_t* cand = nullptr) {
  const TileLayout L(p);
  cudaFuncSetAttribute(k_energy_f64<TY>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       static_cast<int>(L.bytes));
  int64_t tiles = ceil_div(list ? max_list : m, kTile);
  if (list && tiles > 1184) tiles = 1184;  // grid-stride over the (device-sized) list
  if (tiles < 1) tiles = 1;
  k_energy_f64<TY><<<static_cast<unsigned>(tiles), kThreads, L.bytes, st>>>(
      static_cast<const TY*>(yv), m, p, blocks, b0, b1, k, kind, accumulate, list, nlist, best,
      score, rest_sq, norm_sq, cand);
  return check_launch("k_energy_f64");
}

template <typename TY>
int code_impl(const void* yv, int p, const int32_t* order, const int32_t* seg_block,
              const int64_t* seg_lo, const int64_t* seg_hi, const int32_t* nseg,
              int64_t max_seg, const double* blocks, int block_override, int k, int kind,
              int out_by_signal, int64_t ld, int16_t* idx, double* val, double* energy,
              double* rest_sq, cudaStream_t st) {
  const TileLayout L(p);
  cudaFuncSetAttribute(k_code_f64<TY>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       static_cast<int>(L.bytes));
  k_code_f64<TY><<<static_cast<unsigned>(max_seg), kThreads, L.bytes, st>>>(
      static_cast<const TY*>(yv), p, order, seg_block, seg_lo, seg_hi, nseg, blocks,
      block_override, k, kind, out_by_signal, ld, idx, val, energy, rest_sq);
  return check_launch("k_code_f64");
}

template <typename TY>
int outer_impl(const void* yv, int p, const int32_t* order, const int64_t* seg_lo,
               const int64_t* seg_hi, const int32_t* nseg, int64_t max_seg, int k, int64_t ld,
               const int16_t* idx, const double* val, int dense_self, double* partial,
               cudaStream_t st) {
  if (p == osp::P && !dense_self && k <= osp::KMAX) {
    cudaFuncSetAttribute(k_outer_sparse256<TY>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(sizeof(osp::Smem)));
    k_outer_sparse256<TY><<<dim3(static_cast<unsigned>(max_seg), osp::P / osp::DQ),
                            osp::THREADS, sizeof(osp::Smem), st>>>(
        static_cast<const TY*>(yv), order, seg_lo, seg_hi, nseg, k, ld, idx, val, partial);
    return check_launch("k_outer_sparse256");
  }
  const OuterLayout L;
  cudaFuncSetAttribute(k_outer_f64<TY>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       static_cast<int>(L.bytes));
  const unsigned nt = static_cast<unsigned>((p + 63) / 64);
  k_outer_f64<TY><<<dim3(static_cast<unsigned>(max_seg), nt * nt), kThreads, L.bytes, st>>>(
      static_cast<const TY*>(yv), p, order, seg_lo, seg_hi, nseg, k, ld, idx, val, dense_self,
      partial);
  return check_launch("k_outer_f64");
}

int check_common(int dtype, int p, int s0) {
  if (dtype != SBO_F32 && dtype != SBO_F64) return fail(SBO_EINVAL, "dtype must be SBO_F32 or SBO_F64");
  if (p < 1 || p > kPMax) return fail(SBO_EINVAL, "p must be in [1, 256]");
  if (s0 < 1) return fail(SBO_EINVAL, "s0 must be at least 1");
  return SBO_OK;
}
}  // namespace

extern "C" int sbo_energy_pass(const void* y, int dtype, int64_t m, int p, const double* blocks,
                               int b0, int b1, int s0, int kind, int accumulate, int32_t* best,
                               double* score, double* rest_sq, double* norm_sq, void* stream) {
  if (int rc = check_common(dtype, p, s0)) return rc;
  if (b0 < 0 || b1 < b0 || (!accumulate && b0 != 0))
    return fail(SBO_EINVAL, "bad block range for the energy pass");
  if (m == 0 || b1 == b0) return SBO_OK;
  const int k = s0 < p ? s0 : p;
  return dtype == SBO_F32
             ? energy_impl<float>(y, m, p, blocks, b0, b1, k, kind, accumulate, nullptr,
                                  nullptr, 0, best, score, rest_sq, norm_sq, as_stream(stream))
             : energy_impl<double>(y, m, p, blocks, b0, b1, k, kind, accumulate, nullptr,
                                   nullptr, 0, best, score, rest_sq, norm_sq, as_stream(stream));
}

extern "C" int sbo_energy_recheck(const void* y, int dtype, int64_t m, int p,
                                  const double* blocks, int b0, int K, int s0, int kind,
                                  const int32_t* list, const int32_t* nlist, int64_t max_list,
                                  int32_t* best, double* score, double* residual_sq,
                                  void* stream) {
  if (int rc = check_common(dtype, p, s0)) return rc;
  if (K < 1 || !list || !nlist) return fail(SBO_EINVAL, "recheck needs K >= 1 and a list");
  if (b0 < 0 || b0 >= K) return fail(SBO_EINVAL, "recheck needs 0 <= b0 < K");
  if (max_list <= 0) return SBO_OK;
  const int k = s0 < p ? s0 : p;
  const int acc = b0 > 0 ? 1 : 0;
  return dtype == SBO_F32
             ? energy_impl<float>(y, m, p, blocks, b0, K, k, kind, acc, list, nlist, max_list,
                                  best, score, residual_sq, nullptr, as_stream(stream))
             : energy_impl<double>(y, m, p, blocks, b0, K, k, kind, acc, list, nlist, max_list,
                                   best, score, residual_sq, nullptr, as_stream(stream));
}

extern "C" int sbo_energy_recheck_cand(const void* y, int dtype, int64_t m, int p,
                                       const double* blocks, int K, int s0, int kind,
                                       const int32_t* list, const uint64_t* cand,
                                       const int32_t* nlist, int64_t max_list, int32_t* best,
                                       double* score, double* residual_sq, void* stream) {
  if (int rc = check_common(dtype, p, s0)) return rc;
  if (K < 1 || K > 64 || !list || !cand || !nlist)
    return fail(SBO_EINVAL, "candidate recheck needs 1 <= K <= 64, a list and its masks");
  if (max_list <= 0) return SBO_OK;
  const int k = s0 < p ? s0 : p;
  return dtype == SBO_F32
             ? energy_impl<float>(y, m, p, blocks, 0, K, k, kind, 0, list, nlist, max_list,
                                  best, score, residual_sq, nullptr, as_stream(stream), cand)
             : energy_impl<double>(y, m, p, blocks, 0, K, k, kind, 0, list, nlist, max_list,
                                   best, score, residual_sq, nullptr, as_stream(stream), cand);
}

extern "C" int sbo_code_segments(const void* y, int dtype, int p, const int32_t* order,
                                 const int32_t* seg_block, const int64_t* seg_lo,
                                 const int64_t* seg_hi, const int32_t* nseg, int64_t max_seg,
                                 const double* blocks, int block_override, int s0, int kind,
                                 int out_by_signal, int64_t ld, int16_t* idx, double* val,
                                 double* energy, double* rest_sq, void* stream) {
  if (int rc = check_common(dtype, p, s0)) return rc;
  if (max_seg <= 0) return SBO_OK;
  const int k = s0 < p ? s0 : p;
  return dtype == SBO_F32
             ? code_impl<float>(y, p, order, seg_block, seg_lo, seg_hi, nseg, max_seg, blocks,
                                block_override, k, kind, out_by_signal, ld, idx, val, energy,
                                rest_sq, as_stream(stream))
             : code_impl<double>(y, p, order, seg_block, seg_lo, seg_hi, nseg, max_seg, blocks,
                                 block_override, k, kind, out_by_signal, ld, idx, val, energy,
                                 rest_sq, as_stream(stream));
}

extern "C" int sbo_outer_segments(const void* y, int dtype, int p, const int32_t* order,
                                  const int64_t* seg_lo, const int64_t* seg_hi,
                                  const int32_t* nseg, int64_t max_seg, int s0, int64_t ld,
                                  const int16_t* idx, const double* val, double* partial,
                                  void* stream) {
  if (int rc = check_common(dtype, p, s0)) return rc;
  if (max_seg <= 0) return SBO_OK;
  const int k = s0 < p ? s0 : p;
  return dtype == SBO_F32
             ? outer_impl<float>(y, p, order, seg_lo, seg_hi, nseg, max_seg, k, ld, idx, val, 0,
                                 partial, as_stream(stream))
             : outer_impl<double>(y, p, order, seg_lo, seg_hi, nseg, max_seg, k, ld, idx, val,
                                  0, partial, as_stream(stream));
}

extern "C" int sbo_reduce_segments(const double* partial, const int32_t* seg_block,
                                   const int32_t* nseg, int64_t max_seg, int K, int p,
                                   double* P, void* stream) {
  if (K < 1 || p < 1) return fail(SBO_EINVAL, "bad reduce shape");
  (void)max_seg;
  const int64_t pp = static_cast<int64_t>(p) * p;
  dim3 grid(static_cast<unsigned>(ceil_div(pp, 32)), static_cast<unsigned>(K));
  k_reduce_segments<<<grid, 256, 0, as_stream(stream)>>>(partial, seg_block, nseg, K, p, P);
  return check_launch("k_reduce_segments");
}

extern "C" size_t sbo_gram_workspace_bytes(int64_t w, int chunk, int p) {
  const int64_t n = ceil_div(w > 0 ? w : 1, chunk > 0 ? chunk : 1);
  return sizeof(double) * n * p * p + sizeof(int64_t) * 2 * n + 64;
}

extern "C" int sbo_gram_counted(const void* y, int dtype, int p, const int32_t* members,
                                int64_t w, const int64_t* count, int chunk, double* G, void* ws,
                                size_t ws_bytes, void* stream) {
  if (int rc = check_common(dtype, p, 1)) return rc;
  if (chunk < kTile || chunk % kTile) return fail(SBO_EINVAL, "chunk must be a multiple of 64");
  if (ws_bytes < sbo_gram_workspace_bytes(w, chunk, p))
    return fail(SBO_EINVAL, "gram workspace too small");
  cudaStream_t st = as_stream(stream);
  if (w <= 0) {
    SBO_CHECK_CUDA(cudaMemsetAsync(G, 0, sizeof(double) * p * p, st));
    return SBO_OK;
  }
  const int64_t n = ceil_div(w, chunk);
  double* partial = static_cast<double*>(ws);
  int64_t* lo = reinterpret_cast<int64_t*>(partial + n * p * p);
  int64_t* hi = lo + n;
  int32_t* ns = reinterpret_cast<int32_t*>(hi + n);
  k_chunk_segments<<<1, 256, 0, st>>>(w, count, chunk, lo, hi, ns);
  int rc = p <= 64 ? sbo_gram_partials64(y, dtype, p, members, lo, hi, ns, n, partial, st)
           : dtype == SBO_F32 ? outer_impl<float>(y, p, members, lo, hi, ns, n, 1, 0, nullptr,
                                                  nullptr, 1, partial, st)
                              : outer_impl<double>(y, p, members, lo, hi, ns, n, 1, 0, nullptr,
                                                   nullptr, 1, partial, st);
  if (rc) return rc;
  const int64_t pp = static_cast<int64_t>(p) * p;
  k_reduce_segments<<<dim3(static_cast<unsigned>(ceil_div(pp, 32)), 1), 256, 0, st>>>(
      partial, nullptr, ns, 1, p, G);
  return check_launch("k_reduce_segments(gram)");
}

extern "C" int sbo_gram(const void* y, int dtype, int p, const int32_t* members, int64_t w,
                        int chunk, double* G, void* ws, size_t ws_bytes, void* stream) {
  return sbo_gram_counted(y, dtype, p, members, w, nullptr, chunk, G, ws, ws_bytes, stream);
}

extern "C" int sbo_chunk_segments(int64_t w, const int64_t* count, int chunk, int64_t* seg_lo,
                                  int64_t* seg_hi, int32_t* nseg, void* stream) {
  if (chunk < 1 || !seg_lo || !seg_hi || !nseg) return fail(SBO_EINVAL, "bad arguments");
  k_chunk_segments<<<1, 256, 0, as_stream(stream)>>>(w > 0 ? w : 0, count, chunk, seg_lo,
                                                     seg_hi, nseg);
  return check_launch("k_chunk_segments");
}

// select_top on explicit float64 coefficients (onb.py:58-76): coefficient
// vectors are rows of `coeffs` (t x p); warp per vector.
__global__ void k_select_rows(const double* __restrict__ coeffs, int64_t t, int p, int k,
                              int64_t ld, int16_t* idx, double* val) {
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t j = static_cast<int64_t>(blockIdx.x) * (blockDim.x / 32) + warp;
  if (j >= t) return;
  const double* Cs = coeffs + j * p;
  const RowPick r = pick_row(Cs, p, k, SBO_KIND_SQUARED_SUM);
  const unsigned lt = (1u << lane) - 1u;
  int pos = 0;
  const int T = (p + 31) >> 5;
  for (int q = 0; q < T; ++q) {
    const bool on = (r.sel >> q) & 1u;
    const unsigned bal = __ballot_sync(0xffffffffu, on);
    if (on) {
      const int at = pos + __popc(bal & lt);
      idx[at * ld + j] = static_cast<int16_t>(lane + 32 * q);
      val[at * ld + j] = Cs[lane + 32 * q];
    }
    pos += __popc(bal);
  }
}

extern "C" int sbo_select_top(const double* coeffs, int64_t t, int p, int s0, int64_t ld,
                              int16_t* idx, double* val, void* stream) {
  if (p < 1 || p > kPMax) return fail(SBO_EINVAL, "p must be in [1, 256]");
  if (s0 < 1) return fail(SBO_EINVAL, "s0 must be at least 1");
  if (t == 0) return SBO_OK;
  const int k = s0 < p ? s0 : p;
  k_select_rows<<<static_cast<unsigned>(ceil_div(t, 8)), 256, 0, as_stream(stream)>>>(
      coeffs, t, p, k, ld, idx, val);
  return check_launch("k_select_rows");
}

// The coding step of k_code_f64 (sbo.py:196-211) on coefficient rows computed
// elsewhere (coef_i8.cu): row j is position j of a segment table whose count is
// *n (device), its output column is order[j] (out_by_signal) or j.  Same
// selection (pick_row, any kind), same outputs (kept pairs, score, discarded
// energy); rows at or past *n are skipped.
__global__ void k_select_coded(const double* __restrict__ coeffs, const int64_t* __restrict__ n,
                               int64_t t, int p, int k, int kind,
                               const int32_t* __restrict__ order, int64_t ld, int16_t* idx,
                               double* val, double* energy, double* rest_sq) {
  __shared__ PickScratch scr[8];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t rows = n ? min64(t, *n) : t;
  for (int64_t j = static_cast<int64_t>(blockIdx.x) * (blockDim.x / 32) + warp; j < rows;
       j += static_cast<int64_t>(gridDim.x) * (blockDim.x / 32)) {
  const double* Cs = coeffs + j * p;
  const RowPick r = (p == 256 && k <= 32) ? pick_row_cand(Cs, k, kind, scr[warp])
                                          : pick_row(Cs, p, k, kind);
  const int64_t col = order ? order[j] : j;
  const unsigned lt = (1u << lane) - 1u;
  int pos = 0;
  const int T = (p + 31) >> 5;
  for (int q = 0; q < T; ++q) {
    const bool on = (r.sel >> q) & 1u;
    const unsigned bal = __ballot_sync(0xffffffffu, on);
    if (on && idx) {
      const int at = pos + __popc(bal & lt);
      idx[at * ld + col] = static_cast<int16_t>(lane + 32 * q);
      val[at * ld + col] = Cs[lane + 32 * q];
    }
    pos += __popc(bal);
  }
  if (lane == 0) {
    if (energy) energy[col] = r.score;
    if (rest_sq) rest_sq[col] = r.rest_sq;
  }
  }
}

extern "C" int sbo_select_coded(const double* coeffs, const int64_t* n, int64_t t, int p, int s0,
                                int kind, const int32_t* order, int64_t ld, int16_t* idx,
                                double* val, double* energy, double* rest_sq, void* stream) {
  if (p < 1 || p > kPMax) return fail(SBO_EINVAL, "p must be in [1, 256]");
  if (s0 < 1) return fail(SBO_EINVAL, "s0 must be at least 1");
  if (idx && !val) return fail(SBO_EINVAL, "idx without val");
  if (t <= 0) return SBO_OK;
  const int k = s0 < p ? s0 : p;
  // grid-stride over the rows (t may be a capacity, the count on the device)
  k_select_coded<<<static_cast<unsigned>(min64(ceil_div(t, 8), 148 * 64)), 256, 0,
                   as_stream(stream)>>>(
      coeffs, n, t, p, k, kind, order, ld, idx, val, energy, rest_sq);
  return check_launch("k_select_coded");
}
