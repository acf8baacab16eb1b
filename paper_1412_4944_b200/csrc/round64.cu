// The 1ONB round for p <= 64 (onb.py:170-171), any s0, fused per block
// segment: float64 projection on the DMMA tensor cores, exact top-k selection
// in registers, and the sparse outer product P += Y X^T in signal order.
//
// * Projection: warp w computes signals [8w, 8w+8) x 64 atoms of a 64-signal
//   tile with mma.sync m8n8k4 f64; the accumulator fragment leaves each quad
//   of lanes (t4 = lane & 3) holding one signal's 64 coefficients, 16 per lane
//   (atoms 8n + 2 t4 + h).  Nothing is written back to shared memory.
// * Selection (select_top, onb.py:58-76): the high 32 bits of |c| (sign
//   cleared) are a monotone key of the float64 magnitude, so when exactly k keys
//   reach the k-th largest key t_k the kept set is {i : key_i >= t_k} — the
//   float64 stable-argsort set.  Quad networks find t_k (top-8 lists for k <= 8,
//   top-16 for k < 16, bisection on the key bits for k >= 16); a signal with a
//   key tie at the threshold (a 2^-20 relative gap) is re-decided by its warp with
//   the exact rank rule (pick_row).  Keys need no float64 -> float32 conversion:
//   the XU pipe is left to the signal conversions (it ran at 81 % with them).
// * Outer product (sparse_outer, onb.py:127-134): the kept values are written as
//   a dense X tile (zeros elsewhere) and P += Y^T X runs on DMMA in signal order
//   (deterministic partials, no atomics).  A sparse DFMA form (2 p k flop per
//   signal) was measured 1.6x slower: its per-signal bookkeeping is instruction-
//   bound, while the dense DMMA form issues 1 instruction per 512 flop.
// * Residual mode (represent's residual, sbo.py:213-218): the same projection and
//   selection, writing the energy of the discarded coefficients per signal.
#include "common.cuh"
#include "pick.cuh"
#include "topk.cuh"

namespace sbo {
namespace r64 {

constexpr int LD = 68;  // float64 row stride of the block / X tiles (conflict-free fragments)

// Signal tiles are staged in their storage type: float32 rows (stride 72 floats,
// conflict-free DMMA fragment loads, double-buffered: the next tile's cp.async
// copies fly during this tile) or float64 rows (stride 68, single buffer).
template <typename TY>
struct Stage {
  static constexpr int NB = sizeof(TY) == 4 ? 2 : 1;
  static constexpr int YLD = sizeof(TY) == 4 ? 72 : 68;
};

template <typename TY>
struct Layout {
  size_t y_off, q_off, x_off, rows_off, scr_off, flag_off, bytes;
  __host__ __device__ Layout() {
    y_off = 0;                                                        // sY[buf][s][kk]
    q_off = y_off + sizeof(TY) * Stage<TY>::NB * kTile * Stage<TY>::YLD;
    q_off = (q_off + 15) & ~size_t(15);                               // sQ[kk][i] float64
    x_off = q_off + sizeof(double) * 64 * LD;                         // X[s][i]
    rows_off = x_off + sizeof(double) * kTile * LD;                   // rows[buf][s]
    scr_off = rows_off + sizeof(int64_t) * Stage<TY>::NB * kTile;     // per-warp fallback row
    flag_off = scr_off + sizeof(double) * 8 * 64;
    bytes = flag_off + 8 * 64;
  }
};

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ void cp_async16(void* dst, const void* src, bool valid) {
  const unsigned sa = static_cast<unsigned>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(sa), "l"(src),
               "r"(valid ? 16 : 0));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;"); }

__device__ __forceinline__ float select_f(bool c, float a, float b) {
  float r;
  asm("{\n\t.reg .pred q;\n\tsetp.ne.s32 q, %3, 0;\n\tselp.f32 %0, %1, %2, q;\n\t}"
      : "=f"(r)
      : "f"(a), "f"(b), "r"(static_cast<int>(c)));
  return r;
}

__device__ __forceinline__ int select_i(bool c, int a, int b) {
  int r;
  asm("{\n\t.reg .pred q;\n\tsetp.ne.s32 q, %3, 0;\n\tselp.b32 %0, %1, %2, q;\n\t}"
      : "=r"(r)
      : "r"(a), "r"(b), "r"(static_cast<int>(c)));
  return r;
}

__device__ __forceinline__ int atom_of(int u, int t4) { return 8 * (u >> 1) + 2 * t4 + (u & 1); }

// MODE_ROUND: coding + P partials; MODE_RESID: coding + squared residuals and
// scores; MODE_GRAM: P partials with X = Y (the Gram matrix of a member list,
// onb.py:79-95 via thin_svd(ysub) — no block, no coding)
// MODE_CODE: coding only, the kept (index, value) pairs written at the signal's
// segment position (the layout sbo_code_segments writes with out_by_signal = 0),
// for the tensor-core outer product (outer_i8.cu)
constexpr int MODE_ROUND = 0, MODE_RESID = 1, MODE_GRAM = 2, MODE_CODE = 3;

// ascending position of atom a = atom_of(u, t4) among the quad's kept atoms
// (masks[t'] = kept bits of quad lane t', bit u' <-> atom_of(u', t'))
__device__ __forceinline__ int kept_rank(const uint32_t (&masks)[4], int u, int t4) {
  const int n = u >> 1, h = u & 1;
  const uint32_t lower = (1u << (2 * n)) - 1u;  // atoms of column groups < n
  int r = 0;
#pragma unroll
  for (int t2 = 0; t2 < 4; ++t2) {
    uint32_t below = lower;
    if (2 * t2 < 2 * t4 + h) below |= 1u << (2 * n);
    if (2 * t2 + 1 < 2 * t4 + h) below |= 1u << (2 * n + 1);
    r += __popc(masks[t2] & below);
  }
  return r;
}

template <typename TY, int MODE>
__global__ void __launch_bounds__(kThreads, 2) k_round64(
    const TY* __restrict__ y, int p, const int32_t* __restrict__ order,
    const int32_t* __restrict__ seg_block, const int64_t* __restrict__ seg_lo,
    const int64_t* __restrict__ seg_hi, const int32_t* __restrict__ nseg,
    const double* __restrict__ blocks, int block_override, int k, double* partial,
    double* rest_sq, int kind, double* score, int64_t ld, int16_t* cidx, double* cval) {
  constexpr int NB = Stage<TY>::NB, YLD = Stage<TY>::YLD;
  constexpr bool kResid = MODE == MODE_RESID;
  constexpr bool kCode = MODE == MODE_CODE;
  constexpr bool kOuter = MODE == MODE_ROUND || MODE == MODE_GRAM;
  if (static_cast<int>(blockIdx.x) >= *nseg) return;
  extern __shared__ __align__(16) unsigned char smem[];
  const Layout<TY> L;
  TY* sYall = reinterpret_cast<TY*>(smem + L.y_off);
  double* sQ = reinterpret_cast<double*>(smem + L.q_off);
  double* X = reinterpret_cast<double*>(smem + L.x_off);
  int64_t* rowsall = reinterpret_cast<int64_t*>(smem + L.rows_off);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int g = lane >> 2, t4 = lane & 3;
  double* scr = reinterpret_cast<double*>(smem + L.scr_off) + warp * 64;
  unsigned char* fl = smem + L.flag_off + warp * 64;
  const int seg = blockIdx.x;
  const int64_t lo = seg_lo[seg], hi = seg_hi[seg];
  // P accumulator (outer mode), DMMA fragments: warp w owns rows [8w, 8w+8) x 64 atoms
  double acc[8][2];
#pragma unroll
  for (int j = 0; j < 8; ++j) acc[j][0] = acc[j][1] = 0.0;

  // stage tile [base, base + 64) into buffer `buf`; rows beyond hi / coordinates
  // beyond p are zero.  p = 64: 16-B cp.async copies of whole rows (async);
  // otherwise element loads (synchronous).
  auto stage = [&](int64_t base, int buf) {
    TY* sY = sYall + buf * kTile * YLD;
    int64_t* rows = rowsall + buf * kTile;
    if (tid < kTile) {
      const int64_t t = base + tid;
      rows[tid] = t < hi ? (order ? static_cast<int64_t>(order[t]) : t) : -1;
    }
    constexpr int CH = 64 * static_cast<int>(sizeof(TY)) / 16;  // 16-B chunks per row
    if (p == 64) {
      for (int e = tid; e < kTile * CH; e += kThreads) {
        const int sl = e / CH, c = e % CH;
        const int64_t t = base + sl;
        const int64_t r = t < hi ? (order ? static_cast<int64_t>(order[t]) : t) : -1;
        cp_async16(sY + sl * YLD + c * (16 / sizeof(TY)), r >= 0 ? y + r * 64 + c * (16 / sizeof(TY)) : y,
                   r >= 0);
      }
      cp_async_commit();
    } else {
      for (int e = tid; e < kTile * 64; e += kThreads) {
        const int sl = e >> 6, kk = e & 63;
        const int64_t t = base + sl;
        const int64_t r = t < hi ? (order ? static_cast<int64_t>(order[t]) : t) : -1;
        sY[sl * YLD + kk] = (r >= 0 && kk < p) ? __ldg(y + r * p + kk) : TY(0);
      }
    }
  };
  if (NB == 2) stage(lo, 0);
  // (the first tile's copies are in flight while the block is loaded)
  if constexpr (MODE != MODE_GRAM) {
    const int b = block_override >= 0 ? block_override : seg_block[seg];
    const double* q = blocks + static_cast<int64_t>(b) * p * p;
    // the block, zero padded to 64 x 64: all 16 loads per thread in flight at
    // once (a load-store loop would pay one L2 latency per element)
    constexpr int PER = 64 * 64 / kThreads;
    double v[PER];
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int e = tid + u * kThreads, kk = e >> 6, ii = e & 63;
      v[u] = (kk < p && ii < p) ? __ldg(q + kk * p + ii) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int e = tid + u * kThreads;
      sQ[(e >> 6) * LD + (e & 63)] = v[u];
    }
  }
  int it = 0;
  for (int64_t t0 = lo; t0 < hi; t0 += kTile, ++it) {
    const int buf = NB == 2 ? (it & 1) : 0;
    if (NB == 1) {
      __syncthreads();  // the previous tile is done with the buffer
      stage(t0, 0);
    }
    cp_async_wait_all();
    __syncthreads();  // tile `buf` landed everywhere; the previous tile is done with X / buf^1
    if (NB == 2 && t0 + kTile < hi) stage(t0 + kTile, buf ^ 1);  // in flight during this tile
    const TY* sY = sYall + buf * kTile * YLD;
    const int64_t* rows = rowsall + buf * kTile;
    const int s = 8 * warp + g;
    if constexpr (MODE == MODE_GRAM) {
      // X = Y (zero rows for inactive signals are already zero in sY)
      double* xr = X + s * LD + 2 * t4;
      const TY* yr = sY + s * YLD + 2 * t4;
#pragma unroll
      for (int n = 0; n < 8; ++n)
        *reinterpret_cast<double2*>(xr + 8 * n) =
            make_double2(static_cast<double>(yr[8 * n]), static_cast<double>(yr[8 * n + 1]));
    } else {
    // C = Y_tile . Q: this quad's signal s = 8 warp + g, coefficients c[n][h] of
    // atoms 8n + 2 t4 + h
    double c[8][2];
#pragma unroll
    for (int n = 0; n < 8; ++n) c[n][0] = c[n][1] = 0.0;
    {
      const TY* ya = sY + s * YLD + t4;
#pragma unroll 4
      for (int k0 = 0; k0 < 64; k0 += 4) {
        const double a = static_cast<double>(ya[k0]);
        const double* qb = sQ + (k0 + t4) * LD + g;
#pragma unroll
        for (int n = 0; n < 8; ++n) dmma(c[n][0], c[n][1], a, qb[8 * n]);
      }
    }
    // exact selection in registers
    const bool act = rows[s] >= 0;
    // magnitudes are recomputed from c where needed (register pressure)
    // selection keys: the high word of |c| (sign cleared) orders like |c| — no
    // float64 -> float32 conversion (the XU pipe the Y conversions already load);
    // 20 mantissa bits, so a key tie (re-decided exactly) is a 2^-20 relative gap.
    // -1: inactive signal or atom beyond p.
    auto key = [&](int u) -> int {
      return (act && atom_of(u, t4) < p) ? (__double2hiint(c[u >> 1][u & 1]) & 0x7FFFFFFF) : -1;
    };
    uint32_t mask = 0u;
    unsigned need;
    if (k <= 8) {
      // top-8 keys per lane (two sorted 8s merged), merged across the quad: the
      // k-th largest key t_k; the kept set is {key >= t_k} when exactly k keys
      // reach it (no tie at the threshold) — half the comparators of the 16-wide
      // network below
      int srt[8], oth[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        srt[u] = key(u);
        oth[u] = key(u + 8);
      }
      topk::sort8_desc(srt);
      topk::sort8_desc(oth);
      topk::merge_top<8>(srt, oth);
#pragma unroll
      for (int x = 1; x <= 2; x <<= 1) {
#pragma unroll
        for (int u = 0; u < 8; ++u) oth[u] = __shfl_xor_sync(0xffffffffu, srt[u], x);
        topk::merge_top<8>(srt, oth);
      }
      int tk = srt[0];
#pragma unroll
      for (int u = 1; u < 8; ++u) tk = select_i(u == k - 1, srt[u], tk);
      int cnt = 0;
#pragma unroll
      for (int u = 0; u < 16; ++u)
        if (key(u) >= tk && key(u) >= 0) {
          mask |= 1u << u;
          ++cnt;
        }
      cnt += __shfl_xor_sync(0xffffffffu, cnt, 1);
      cnt += __shfl_xor_sync(0xffffffffu, cnt, 2);
      need = __ballot_sync(0xffffffffu, act && cnt != k && t4 == 0);
    } else if (k < 16) {
      int srt[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) srt[u] = key(u);
      topk::sort_desc<16>(srt);
#pragma unroll
      for (int x = 1; x <= 2; x <<= 1) {
        int other[16];
#pragma unroll
        for (int u = 0; u < 16; ++u) other[u] = __shfl_xor_sync(0xffffffffu, srt[u], x);
        topk::merge_top<16>(srt, other);
      }
      // the k-th / (k+1)-th largest by register selects (a plain srt[k - 1] with
      // runtime k would go through local memory)
      int tk = srt[0], tk1 = srt[1];
#pragma unroll
      for (int u = 1; u < 16; ++u) {
        tk = select_i(u == k - 1, srt[u], tk);
        tk1 = select_i(u == k, srt[u], tk1);
      }
#pragma unroll
      for (int u = 0; u < 16; ++u)
        if (key(u) >= tk && key(u) >= 0) mask |= 1u << u;
      // key ties at the threshold: the warp re-decides those signals exactly
      need = __ballot_sync(0xffffffffu, act && !(tk > tk1) && t4 == 0);
    } else {
      // k >= 16: the k-th largest key of the quad's 64 by bisection on its bits:
      // the largest T
      // with #{|c| >= T} >= k.  Exactly k at or above T: the kept set; otherwise a
      // tie at the threshold, re-decided by the warp's exact rank rule.
      uint32_t ukey[16];
#pragma unroll
      for (int u = 0; u < 16; ++u) ukey[u] = key(u) >= 0 ? static_cast<uint32_t>(key(u)) : 0u;
      const uint32_t vmask = [&] {
        uint32_t v = 0u;
#pragma unroll
        for (int u = 0; u < 16; ++u) v |= (act && atom_of(u, t4) < p ? 1u : 0u) << u;
        return v;
      }();
      uint32_t T = 0u;
#pragma unroll 1
      for (int bit = 30; bit >= 0; --bit) {
        const uint32_t cand = T | (1u << bit);
        int cnt = 0;
#pragma unroll
        for (int u = 0; u < 16; ++u) cnt += ((vmask >> u) & 1u) && ukey[u] >= cand;
        cnt += __shfl_xor_sync(0xffffffffu, cnt, 1);
        cnt += __shfl_xor_sync(0xffffffffu, cnt, 2);
        if (cnt >= k) T = cand;
      }
      int cnt = 0;
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const bool on = ((vmask >> u) & 1u) && ukey[u] >= T;
        cnt += on;
        if (on) mask |= 1u << u;
      }
      cnt += __shfl_xor_sync(0xffffffffu, cnt, 1);
      cnt += __shfl_xor_sync(0xffffffffu, cnt, 2);
      need = __ballot_sync(0xffffffffu, act && cnt != k && t4 == 0);
    }
    double rest = -1.0, fscore = 0.0;  // rest < 0: not decided by the fallback
    while (need) {
      const int gg = (__ffs(need) - 1) >> 2;
      need &= need - 1;
      if (g == gg) {
#pragma unroll
        for (int u = 0; u < 16; ++u) scr[atom_of(u, t4)] = c[u >> 1][u & 1];
      }
      __syncwarp();
      const RowPick r = pick_row(scr, p, k, kind);
      fl[lane] = r.sel & 1u;
      fl[lane + 32] = (r.sel >> 1) & 1u;
      __syncwarp();
      if (g == gg) {
        mask = 0u;
#pragma unroll
        for (int u = 0; u < 16; ++u)
          if (fl[atom_of(u, t4)]) mask |= 1u << u;
        rest = r.rest_sq;
        fscore = r.score;
      }
      __syncwarp();
    }
    if constexpr (kCode) {
      // the kept pairs in ascending atom order at column t of the segment order
      uint32_t masks[4];
#pragma unroll
      for (int x = 0; x < 4; ++x) masks[x] = __shfl_sync(0xffffffffu, mask, (lane & ~3) | x);
      if (act) {
        const int64_t col = t0 + s;
#pragma unroll
        for (int u = 0; u < 16; ++u) {
          if ((mask >> u) & 1u) {
            const int at = kept_rank(masks, u, t4);
            cidx[at * ld + col] = static_cast<int16_t>(atom_of(u, t4));
            cval[at * ld + col] = c[u >> 1][u & 1];
          }
        }
      }
    } else if constexpr (kResid) {
      // every lane takes part in the quad sum (full-mask shuffles), the
      // fallback's exact value wins where it was computed
      double d = 0.0, e = 0.0;
#pragma unroll
      for (int u = 0; u < 16; ++u) {
        const double v = c[u >> 1][u & 1];
        if ((mask >> u) & 1u) e = kind == SBO_KIND_SQUARED_SUM ? fma(v, v, e) : e + fabs(v);
        else if (act && atom_of(u, t4) < p) d = fma(v, v, d);
      }
      d += __shfl_xor_sync(0xffffffffu, d, 1);
      d += __shfl_xor_sync(0xffffffffu, d, 2);
      e += __shfl_xor_sync(0xffffffffu, e, 1);
      e += __shfl_xor_sync(0xffffffffu, e, 2);
      if (rest < 0.0) rest = d;
      else e = fscore;
      if (act && t4 == 0) {
        rest_sq[rows[s]] = rest;
        if (score) score[rows[s]] = e;
      }
    } else if constexpr (MODE == MODE_ROUND) {
      // X = the kept coefficients, zeros elsewhere (fragment layout -> rows of X)
      double* xr = X + s * LD + 2 * t4;
#pragma unroll
      for (int n = 0; n < 8; ++n)
        *reinterpret_cast<double2*>(xr + 8 * n) =
            make_double2(((mask >> (2 * n)) & 1u) ? c[n][0] : 0.0,
                         ((mask >> (2 * n + 1)) & 1u) ? c[n][1] : 0.0);
    }
    }  // MODE != MODE_GRAM
    if constexpr (kOuter) {
      __syncthreads();
      // P[kk][i] += sum_s Y[s][kk] X[s][i] on DMMA, signals in order (inactive
      // rows are zero in both Y and X)
      const TY* ya = sY + t4 * YLD + 8 * warp + g;
      const double* xb = X + t4 * LD + g;
#pragma unroll 4
      for (int s4 = 0; s4 < kTile; s4 += 4) {
        const double av = static_cast<double>(ya[s4 * YLD]);
#pragma unroll
        for (int n = 0; n < 8; ++n) dmma(acc[n][0], acc[n][1], av, xb[s4 * LD + 8 * n]);
      }
    }
  }
  if constexpr (kOuter) {
    double* out = partial + static_cast<int64_t>(seg) * p * p;
    const int row = 8 * warp + g;
#pragma unroll
    for (int n = 0; n < 8; ++n)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int col = 8 * n + 2 * t4 + h;
        if (row < p && col < p) out[row * p + col] = acc[n][h];
      }
  }
}

template <typename TY, int MODE>
int launch(const void* yv, int p, const int32_t* order, const int32_t* seg_block,
           const int64_t* seg_lo, const int64_t* seg_hi, const int32_t* nseg, int64_t max_seg,
           const double* blocks, int block_override, int k, double* partial, double* rest_sq,
           int kind, double* score, cudaStream_t st, int64_t ld = 0, int16_t* cidx = nullptr,
           double* cval = nullptr) {
  const Layout<TY> L;
  cudaFuncSetAttribute(k_round64<TY, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       static_cast<int>(L.bytes));
  k_round64<TY, MODE><<<static_cast<unsigned>(max_seg), kThreads, L.bytes, st>>>(
      static_cast<const TY*>(yv), p, order, seg_block, seg_lo, seg_hi, nseg, blocks,
      block_override, k, partial, rest_sq, kind, score, ld, cidx, cval);
  return check_launch(MODE == MODE_RESID ? "k_round64<resid>"
                      : MODE == MODE_GRAM ? "k_round64<gram>"
                      : MODE == MODE_CODE ? "k_round64<code>" : "k_round64");
}

int check(int dtype, int p, int s0) {
  if (dtype != SBO_F32 && dtype != SBO_F64) return fail(SBO_EINVAL, "bad dtype");
  if (p < 1 || p > 64) return fail(SBO_EINVAL, "the fused round needs p <= 64");
  const int k = s0 < p ? s0 : p;
  if (s0 < 1) return fail(SBO_EINVAL, "s0 must be at least 1");
  return SBO_OK;
}

}  // namespace r64
}  // namespace sbo

using namespace sbo;

extern "C" int sbo_round_segments(const void* y, int dtype, int p, const int32_t* order,
                                  const int32_t* seg_block, const int64_t* seg_lo,
                                  const int64_t* seg_hi, const int32_t* nseg, int64_t max_seg,
                                  const double* blocks, int block_override, int s0,
                                  double* partial, void* stream) {
  if (int rc = r64::check(dtype, p, s0)) return rc;
  if (max_seg <= 0) return SBO_OK;
  const int k = s0 < p ? s0 : p;
  return dtype == SBO_F32
             ? r64::launch<float, r64::MODE_ROUND>(y, p, order, seg_block, seg_lo, seg_hi, nseg, max_seg,
                                         blocks, block_override, k, partial, nullptr,
                                         SBO_KIND_SQUARED_SUM, nullptr, as_stream(stream))
             : r64::launch<double, r64::MODE_ROUND>(y, p, order, seg_block, seg_lo, seg_hi, nseg, max_seg,
                                          blocks, block_override, k, partial, nullptr,
                                          SBO_KIND_SQUARED_SUM, nullptr, as_stream(stream));
}

extern "C" int sbo_residual_segments(const void* y, int dtype, int p, const int32_t* order,
                                     const int32_t* seg_block, const int64_t* seg_lo,
                                     const int64_t* seg_hi, const int32_t* nseg,
                                     int64_t max_seg, const double* blocks, int s0, int kind,
                                     double* rest_sq, double* score, void* stream) {
  if (int rc = r64::check(dtype, p, s0)) return rc;
  if (!rest_sq) return fail(SBO_EINVAL, "rest_sq is required");
  if (kind != SBO_KIND_SQUARED_SUM && kind != SBO_KIND_ABS_SUM) return fail(SBO_EINVAL, "bad kind");
  if (max_seg <= 0) return SBO_OK;
  const int k = s0 < p ? s0 : p;
  return dtype == SBO_F32
             ? r64::launch<float, r64::MODE_RESID>(y, p, order, seg_block, seg_lo, seg_hi, nseg, max_seg,
                                        blocks, -1, k, nullptr, rest_sq, kind, score,
                                        as_stream(stream))
             : r64::launch<double, r64::MODE_RESID>(y, p, order, seg_block, seg_lo, seg_hi, nseg, max_seg,
                                         blocks, -1, k, nullptr, rest_sq, kind, score,
                                         as_stream(stream));
}

// Gram partials of a member list for p <= 64 on DMMA (used by sbo_gram): one
// p x p partial per segment of the list, in member order.
int sbo_gram_partials64(const void* y, int dtype, int p, const int32_t* members,
                        const int64_t* seg_lo, const int64_t* seg_hi, const int32_t* nseg,
                        int64_t max_seg, double* partial, void* stream) {
  if (max_seg <= 0) return SBO_OK;
  return dtype == SBO_F32
             ? r64::launch<float, r64::MODE_GRAM>(y, p, members, nullptr, seg_lo, seg_hi, nseg,
                                                  max_seg, nullptr, 0, 1, partial, nullptr,
                                                  SBO_KIND_SQUARED_SUM, nullptr,
                                                  as_stream(stream))
             : r64::launch<double, r64::MODE_GRAM>(y, p, members, nullptr, seg_lo, seg_hi,
                                                   nseg, max_seg, nullptr, 0, 1, partial,
                                                   nullptr, SBO_KIND_SQUARED_SUM, nullptr,
                                                   as_stream(stream));
}

extern "C" int sbo_round_code_segments(const void* y, int dtype, int p, const int32_t* order,
                                       const int32_t* seg_block, const int64_t* seg_lo,
                                       const int64_t* seg_hi, const int32_t* nseg,
                                       int64_t max_seg, const double* blocks, int block_override,
                                       int s0, int64_t ld, int16_t* idx, double* val,
                                       void* stream) {
  if (int rc = r64::check(dtype, p, s0)) return rc;
  if (!idx || !val) return fail(SBO_EINVAL, "idx and val are required");
  if (max_seg <= 0) return SBO_OK;
  const int k = s0 < p ? s0 : p;
  return dtype == SBO_F32
             ? r64::launch<float, r64::MODE_CODE>(y, p, order, seg_block, seg_lo, seg_hi, nseg,
                                                  max_seg, blocks, block_override, k, nullptr,
                                                  nullptr, SBO_KIND_SQUARED_SUM, nullptr,
                                                  as_stream(stream), ld, idx, val)
             : r64::launch<double, r64::MODE_CODE>(y, p, order, seg_block, seg_lo, seg_hi, nseg,
                                                   max_seg, blocks, block_override, k, nullptr,
                                                   nullptr, SBO_KIND_SQUARED_SUM, nullptr,
                                                   as_stream(stream), ld, idx, val);
}
