// Sparse outer products P = Y X^T per segment (onb.py:127-134, the training
// round's P_b = Y_b X_b^T, north_star item 3) on the 5th-gen tensor cores,
// exactly: both operands are cut into 7-bit integer digits and every digit
// product is accumulated in int32 TMEM by tcgen05.mma kind::i8.
//
// Number formats (scales are per call, chosen on the host from sbo_i8_scan):
//   y  = Y_int 2^-Sy, Y_int = sum_a Y_a 128^(4-a), a = 0..4, |Y_a| <= 127
//        (sign-magnitude digits; exact for float32 signals whose values all sit
//        on the 2^-Sy grid below 2^(35-Sy) — e.g. unit-range image patches)
//   x  = X_int 2^-Sx, X_int = sum_b X_b 128^(7-b), b = 0..7: two's-complement
//        digits of the rounded fixed-point code value (X_0 = X_int >> 49 signed,
//        X_b = 7-bit fields in [0, 127] below it: 8 independent shift-and-mask
//        extractions, no carry chain); |X_int| < 2^54, resolution 2^-Sx: far
//        below the float64 rounding of P's sums)
//   P[i][j] = 2^(77-Sy-Sx) sum_L D_L[i][j] 128^-L, D_L = sum_{a+b=L} Y_a X_b^T,
//   levels L <= 7 kept (the dropped levels weigh <= 2^-56 of the product).
// Every sum is exact integer arithmetic: TMEM int32 per run of consecutive
// segments of one block (a TMEM column takes <= 4 digit pairs of <= 127 x 127
// per signal, runs bounded to 2^14 signals: < 2^30), then int64 global
// accumulators per block (levels 0-3 and 4-7
// each folded into one int64), so P does not depend on the order of the
// signals, the segmentation or the grid: bit-identical for any CTA count.
//
// Tiles: 128 signals = K of the MMAs (one 128-B swizzled row of int8).  Digit
// planes (64 rows x 128 signals, K-major, SW128): X planes ordered X0 X4 X1 X5
// X2 X6 X3 X7 so that [X_b; X_b+4] is one M = 128 operand (rows = atom, digit
// b in lanes 0-63 and b+4 in lanes 64-127); Y planes Y0..Y4 stack along N.
// TMEM (512 columns x 128 lanes):
//   set 1, columns 64c + dim (c = 0..3): lanes 0-63 hold level c (pairs b + a = c,
//     b <= 3), lanes 64-127 level c + 4 (pairs (b + 4) + a);
//   set 2, columns 256 + 64(c - 4) + dim (c = 4..7): lanes 0-63 level c for the
//     pairs b <= 3, a >= 1 with b + a >= 4 (lanes 64-127: levels >= 8, unused).
// Warp roles (512 threads, one CTA per SM; CTA c takes a contiguous range of
// segments, i.e. mostly one block's signals):
//   warp 0 lane 0  MMA issuer (8 MMAs per 32-signal k-step)
//   warps 0-3      epilogue at the end of each run (block change): TMEM -> int64
//                  red.add into the block's accumulators (k_i8_finalize -> P)
//   warps 4-15     producers: digit planes of the next tile (double-buffered)
#include "common.cuh"
#include "sm100.cuh"

namespace sbo {
namespace oi8 {

constexpr int P = 64;
constexpr int TS = 128;                 // signals per tile
constexpr int YD = 5, XD = 8;
constexpr int PLANE = P * TS;           // 8 KB
constexpr int THREADS = 512;
constexpr int NPROD = THREADS - 128;    // producer threads (warps 4-15)
constexpr int EPI_DIMS = 8;             // dims per TMEM read batch of the epilogue
constexpr int64_t RUN_MAX = 1 << 14;    // signals per TMEM accumulation (int32 bound:
                                        // <= 4 digit pairs x 127 x 127 per signal and region)

constexpr uint32_t YTILE = YD * PLANE;  // one transposed Y digit tile: 40 KB

struct Smem {
  int8_t x[2][XD * PLANE];
  int8_t y[2][YTILE];
  uint64_t full[2], fully[2], empty[2], run_done;
  uint32_t tmem;
  int base;
};

// the CTA's contiguous range of segments: range r of nr (default: the CTA index)
__device__ __forceinline__ void seg_range(int nseg, int& s0, int& s1, int r = -1, int nr = 0) {
  if (r < 0) {
    r = static_cast<int>(blockIdx.x);
    nr = static_cast<int>(gridDim.x);
  }
  s0 = static_cast<int>(static_cast<int64_t>(nseg) * r / nr);
  s1 = static_cast<int>(static_cast<int64_t>(nseg) * (r + 1) / nr);
}

// tile slot of segment s0's first tile: tiles of the segments before it (each
// segment's tiles start at a fresh 128-signal slot); every thread of the CTA
// calls it, the result is valid in all of them
__device__ int tile_base(const int64_t* seg_lo, const int64_t* seg_hi, int s0, int* slot) {
  if (threadIdx.x == 0) *slot = 0;
  __syncthreads();
  int mine = 0;
  for (int s = threadIdx.x; s < s0; s += blockDim.x)
    mine += static_cast<int>(ceil_div(seg_hi[s] - seg_lo[s], TS));
  for (int o = 16; o > 0; o >>= 1) mine += __shfl_xor_sync(0xffffffffu, mine, o);
  if ((threadIdx.x & 31) == 0 && mine) atomicAdd(slot, mine);
  __syncthreads();
  const int b = *slot;
  __syncthreads();
  return b;
}
constexpr size_t SMEM_BYTES = sizeof(Smem) + 1024;

__device__ __forceinline__ Smem* smem_of(unsigned char* raw) {
  const uint32_t a = sm100::smem_u32(raw);
  return reinterpret_cast<Smem*>(raw + ((1024u - (a & 1023u)) & 1023u));
}

// instruction descriptor: kind::i8, A = B = s8 (K-major), D = s32, M x N
__host__ __device__ constexpr uint32_t idesc_i8(int m, int n) {
  return (2u << 4) | (1u << 7) | (1u << 10) | (static_cast<uint32_t>(n >> 3) << 17) |
         (static_cast<uint32_t>(m >> 4) << 24);
}

__device__ __forceinline__ void umma_i8(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc,
                                        uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

// memory slot of X digit plane b: [X_b; X_b+4] adjacent
__device__ __forceinline__ int xslot(int b) { return b < 4 ? 2 * b : 2 * (b - 4) + 1; }

// byte offset of (row r, signal column s) inside a 64 x 128 plane
__device__ __forceinline__ uint32_t plane_off(int r, int s) {
  return static_cast<uint32_t>(r >> 3) * 1024u + sm100::sw128_offset(r & 7, s);
}

// int32 TMEM word -> double exactly, without the conversion pipe
__device__ __forceinline__ double i2d(uint32_t v) {
  return __hiloint2double(0x43300000, static_cast<int>(v ^ 0x80000000u)) - 4503601774854144.0;
}

struct Ring {
  int i = 0;
  uint32_t ph = 0;
  __device__ __forceinline__ void next() {
    if (++i == 2) {
      i = 0;
      ph ^= 1u;
    }
  }
};

// PD = 256 (config D): CTA (range, combo = blockIdx.x % 16): atom group ag = combo / 4 and
// dim group dg = combo % 4 of 64 each — the p = 64 product on the 64 x 64 slice,
// the Y tile of the dim group (a 40-KB image of its own) and the X planes of the
// atom group's kept pairs.
template <int PD>
__global__ void __launch_bounds__(THREADS, 1)
k_outer_i8(const int8_t* __restrict__ ytiles, const int32_t* __restrict__ seg_block,
           const int64_t* __restrict__ seg_lo,
           const int64_t* __restrict__ seg_hi, const int32_t* __restrict__ nseg_p, int k,
           int64_t ld, const int16_t* __restrict__ idx, const double* __restrict__ val,
           double xscale, unsigned long long* __restrict__ acc64) {
  extern __shared__ unsigned char raw[];
  Smem* S = smem_of(raw);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nseg = *nseg_p;
  if (tid == 0) {
    for (int s = 0; s < 2; ++s) {
      sm100::mbar_init(&S->full[s], 1);
      sm100::mbar_init(&S->fully[s], 1);
      sm100::mbar_init(&S->empty[s], 1);
    }
    sm100::mbar_init(&S->run_done, 1);
    sm100::fence_barrier_init();
  }
  if (warp == 1) sm100::tmem_alloc(&S->tmem, 512);
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem = S->tmem;
  // PD = 256: the 16 slices of one segment range are consecutive CTAs, so they
  // run together and share the range's Y tiles and codes in L2
  constexpr int NG = PD / P;  // 64-wide groups per dimension
  const int combo = static_cast<int>(blockIdx.x) % (NG * NG);
  const int ag = combo / NG, dg = combo % NG;
  int sa, sb;
  seg_range(nseg, sa, sb, static_cast<int>(blockIdx.x) / (NG * NG),
            static_cast<int>(gridDim.x) / (NG * NG));
  const int slot0 = tile_base(seg_lo, seg_hi, sa, &S->base);

  if (warp >= 4) {  // ------------------------------------------------ producers
    //   Y: the tile's transposed digit planes (sbo_y_tiles, once per grouping)
    //      arrive by one bulk copy on fully[stage];
    //   X: zero planes, then each kept pair's 8 balanced digits; thread (sl, r0)
    //      takes code rows r0, r0 + 3, ... of signal sl.  The first code rows of
    //      the next tile are loaded before the wait for its stage.
    const int pt = tid - 128;
    constexpr int XPRE = 3;                                  // code rows preloaded
    const int sl_x = pt & (TS - 1), r0_x = pt >> 7;          // 384 = 3 x 128
    Ring r;
    int slot = slot0;
    for (int seg = sa; seg < sb; ++seg) {
      const int64_t lo = seg_lo[seg], hi = seg_hi[seg];
      for (int64_t t0 = lo; t0 < hi; t0 += TS, ++slot) {
        const int n = static_cast<int>(min64(TS, hi - t0));
        int pj[XPRE];
        double pv[XPRE];
#pragma unroll
        for (int c = 0; c < XPRE; ++c) {
          const int rr = r0_x + 3 * c;
          pj[c] = -1;
          pv[c] = 0.0;
          if (rr < k && sl_x < n) {
            const int64_t col = rr * ld + t0 + sl_x;
            pj[c] = __ldg(idx + col);
            pv[c] = __ldg(val + col);
          }
        }
        sm100::mbar_wait(&S->empty[r.i], r.ph ^ 1u);
        if (pt == 0) {
          sm100::mbar_expect_tx(&S->fully[r.i], YTILE);
          sm100::bulk_g2s(S->y[r.i], ytiles + (static_cast<int64_t>(slot) * NG + dg) * YTILE,
                          YTILE, &S->fully[r.i]);
        }
        int8_t* xs = S->x[r.i];
        {
          uint4* z = reinterpret_cast<uint4*>(xs);
          for (int e = pt; e < XD * PLANE / 16; e += NPROD) z[e] = make_uint4(0, 0, 0, 0);
        }
        asm volatile("bar.sync 2, %0;" ::"r"(NPROD));  // X planes zeroed
        auto put = [&](int j, double x, int sl) {
          j -= P * ag;  // the atom group's slice
          if (NG > 1 && (j < 0 || j >= P)) return;
          const long long v = __double2ll_rn(x * xscale);
          const uint32_t off = plane_off(j, sl);
          xs[xslot(0) * PLANE + off] = static_cast<int8_t>(v >> 49);
#pragma unroll
          for (int b = 1; b < XD; ++b)
            xs[xslot(b) * PLANE + off] = static_cast<int8_t>((v >> (7 * (XD - 1 - b))) & 127);
        };
#pragma unroll
        for (int c = 0; c < XPRE; ++c)
          if (pj[c] >= 0) put(pj[c], pv[c], sl_x);
        if (sl_x < n) {
          for (int rr = r0_x + 3 * XPRE; rr < k; rr += 3) {
            const int64_t col = rr * ld + t0 + sl_x;
            put(__ldg(idx + col), __ldg(val + col), sl_x);
          }
        }
        // generic-proxy writes -> visible to the tensor core (async proxy)
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        asm volatile("bar.sync 2, %0;" ::"r"(NPROD));
        if (pt == 0) sm100::mbar_arrive(&S->full[r.i]);
        r.next();
      }
    }
  } else {  // ---------------------------------- warps 0-3: issuer + epilogue
    // runs: maximal stretches of the CTA's segments with one block (and at most
    // RUN_MAX signals); TMEM accumulates a run, the epilogue folds it into the
    // block's int64 accumulators
    Ring r;
    uint32_t run_ph = 0;
    const int e = tid;  // TMEM lane of this epilogue thread
    int seg = sa;
    while (seg < sb) {
      const int blk = seg_block ? seg_block[seg] : 0;
      int send = seg;
      int64_t cnt = 0;
      while (send < sb && (seg_block ? seg_block[send] : 0) == blk &&
             cnt + (seg_hi[send] - seg_lo[send]) <= RUN_MAX) {
        cnt += seg_hi[send] - seg_lo[send];
        ++send;
      }
      if (send == seg) {  // a single segment longer than RUN_MAX (not produced by sbo_group)
        cnt = seg_hi[seg] - seg_lo[seg];
        send = seg + 1;
      }
      if (warp == 0) {
        if (lane == 0) {
          bool first = true;
          for (int sg = seg; sg < send; ++sg) {
            for (int64_t t0 = seg_lo[sg]; t0 < seg_hi[sg]; t0 += TS) {
              sm100::mbar_wait(&S->full[r.i], r.ph);
              sm100::mbar_wait(&S->fully[r.i], r.ph);
              sm100::tc_fence_after();
              const uint32_t xb = sm100::smem_u32(S->x[r.i]);
              const uint32_t yb = sm100::smem_u32(S->y[r.i]);
#pragma unroll
              for (int kk = 0; kk < TS / 32; ++kk) {
                const uint32_t ko = kk * 32;
                const uint32_t init = first && kk == 0 ? 0u : 1u;
                // set 1: [X_b; X_b+4] x [Y_0 .. Y_3-b] -> columns 64 b
#pragma unroll
                for (int b = 0; b < 4; ++b)
                  umma_i8(tmem + 64 * b, sm100::desc_sw128(xb + 2 * b * PLANE + ko),
                          sm100::desc_sw128(yb + ko), idesc_i8(128, 64 * (4 - b)),
                          b == 0 ? init : 1u);
                // set 2: [X_b; X_b+4] x [Y_4-b .. Y_4] -> columns 256 (levels 4..7)
#pragma unroll
                for (int bb = 0; bb < 4; ++bb) {
                  const int b = 3 - bb;  // b = 3 first: its N = 256 initialises 256-511
                  const int a0 = 4 - b;
                  umma_i8(tmem + 256, sm100::desc_sw128(xb + 2 * b * PLANE + ko),
                          sm100::desc_sw128(yb + a0 * PLANE + ko), idesc_i8(128, 64 * (5 - a0)),
                          bb == 0 ? init : 1u);
                }
              }
              first = false;
              sm100::umma_commit(&S->empty[r.i]);
              r.next();
            }
          }
          sm100::umma_commit(&S->run_done);
        }
        __syncwarp();
      }
      // ------------------------------------------------------------- epilogue
      sm100::mbar_wait(&S->run_done, run_ph);
      run_ph ^= 1u;
      sm100::tc_fence_after();
      if (cnt > 0) {
        const bool top = e < 64;
        const int j = e & 63;
        const uint32_t lane_base = tmem + (static_cast<uint32_t>(32 * warp) << 16);
        // block accumulators: [blk][0: levels 0-3 | 1: levels 4-7][dim][atom]
        unsigned long long* out = acc64 + static_cast<int64_t>(blk) * 2 * PD * PD +
                                  static_cast<int64_t>(P * dg) * PD + P * ag;
        for (int d0 = 0; d0 < P; d0 += EPI_DIMS) {
          uint32_t v[8][EPI_DIMS];  // [slot][dim]: top slots = levels 0..7, bottom = 4..7
#pragma unroll
          for (int L = 0; L < 8; ++L) {
            if (!top && L < 4) continue;
            const uint32_t col = top ? (L < 4 ? 64 * L : 256 + 64 * (L - 4)) : 64 * (L - 4);
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                : "=r"(v[L][0]), "=r"(v[L][1]), "=r"(v[L][2]), "=r"(v[L][3]), "=r"(v[L][4]),
                  "=r"(v[L][5]), "=r"(v[L][6]), "=r"(v[L][7])
                : "r"(lane_base + col + d0));
          }
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
          for (int q = 0; q < EPI_DIMS; ++q) {
            // fold four levels into one int64: sum_L D_L 128^(3-L) (exact, < 2^62)
            long long lo = 0;
#pragma unroll
            for (int L = 4; L < 8; ++L) lo = lo * 128 + static_cast<int>(v[L][q]);
            unsigned long long* o = out + (d0 + q) * PD + j;
            atomicAdd(o + PD * PD, static_cast<unsigned long long>(lo));
            if (top) {
              long long hi = 0;
#pragma unroll
              for (int L = 0; L < 4; ++L) hi = hi * 128 + static_cast<int>(v[L][q]);
              atomicAdd(o, static_cast<unsigned long long>(hi));
            }
          }
        }
      }
      sm100::tc_fence_before();
      // all TMEM reads of this run are done before the next run's MMAs
      asm volatile("bar.sync 1, 128;");
      seg = send;
    }
  }
  __syncthreads();
  if (warp == 1) sm100::tmem_dealloc(tmem, 512);
}

// Transposed Y digit tiles, once per grouping (the order does not change across
// a grouping's training rounds): tile slot = (segment, 128-position chunk) in
// segment order, 5 planes x [64 dims][128 signals] int8, SW128-swizzled: the
// exact shared-memory image k_outer_i8 bulk-copies.  Item = (signal quad q, dim
// word w): 5 planes x 4 signals words of the signal-major digit rows, each 4 x 4
// byte block transposed with PRMT.
constexpr int YT_THREADS = 256;

// PD = 256: per tile, four consecutive 40-KB images, one per 64-dim group.
template <int PD>
__global__ void __launch_bounds__(YT_THREADS)
k_y_tiles(const int8_t* __restrict__ ydig, const int32_t* __restrict__ order,
          const int64_t* __restrict__ seg_lo, const int64_t* __restrict__ seg_hi,
          const int32_t* __restrict__ nseg_p, int8_t* __restrict__ tiles) {
  __shared__ __align__(16) int8_t st[YTILE];
  __shared__ int64_t srow[TS];
  __shared__ int base;
  const int nseg = *nseg_p;
  int sa, sb;
  seg_range(nseg, sa, sb);
  int slot = tile_base(seg_lo, seg_hi, sa, &base);
  const int tid = threadIdx.x;
  for (int seg = sa; seg < sb; ++seg) {
    const int64_t lo = seg_lo[seg], hi = seg_hi[seg];
    for (int64_t t0 = lo; t0 < hi; t0 += TS, ++slot) {
      const int n = static_cast<int>(min64(TS, hi - t0));
      if (tid < TS) srow[tid] = tid < n ? (order ? static_cast<int64_t>(order[t0 + tid]) : t0 + tid)
                                        : -1;
      __syncthreads();
      for (int dg = 0; dg < PD / P; ++dg) {
      for (int it = tid; it < (TS / 4) * (P / 4); it += YT_THREADS) {
        const int w = it & 15, q = it >> 4;
        uint32_t wv[YD][4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int sl = 4 * q + u;
          const uint32_t* src =
              reinterpret_cast<const uint32_t*>(ydig + (sl < n ? srow[sl] : 0) * (YD * PD) +
                                                P * dg) + w;
#pragma unroll
          for (int a = 0; a < YD; ++a) wv[a][u] = sl < n ? __ldg(src + a * (PD / 4)) : 0u;
        }
#pragma unroll
        for (int a = 0; a < YD; ++a) {
          const uint32_t t0_ = __byte_perm(wv[a][0], wv[a][1], 0x5140);
          const uint32_t t1_ = __byte_perm(wv[a][2], wv[a][3], 0x5140);
          const uint32_t t2_ = __byte_perm(wv[a][0], wv[a][1], 0x7362);
          const uint32_t t3_ = __byte_perm(wv[a][2], wv[a][3], 0x7362);
          const uint32_t c[4] = {__byte_perm(t0_, t1_, 0x5410), __byte_perm(t0_, t1_, 0x7632),
                                 __byte_perm(t2_, t3_, 0x5410), __byte_perm(t2_, t3_, 0x7632)};
#pragma unroll
          for (int d = 0; d < 4; ++d)
            *reinterpret_cast<uint32_t*>(st + a * PLANE + plane_off(4 * w + d, 4 * q)) = c[d];
        }
      }
      __syncthreads();
      uint4* dst = reinterpret_cast<uint4*>(
          tiles + (static_cast<int64_t>(slot) * (PD / P) + dg) * YTILE);
      const uint4* srcs = reinterpret_cast<const uint4*>(st);
      for (int e = tid; e < static_cast<int>(YTILE / 16); e += YT_THREADS) dst[e] = srcs[e];
      __syncthreads();
      }
    }
  }
}

// P[b][i][j] = 2^(77-sy-sx) (HI 128^-3 + LO 128^-7) from the int64 accumulators
template <int PD>
__global__ void k_i8_finalize(const unsigned long long* __restrict__ acc64, int nblocks,
                              double pscale, double* __restrict__ Pout) {
  const int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (e >= static_cast<int64_t>(nblocks) * PD * PD) return;
  const int64_t b = e / (PD * PD), ij = e % (PD * PD);
  const long long hi = static_cast<long long>(acc64[(2 * b) * PD * PD + ij]);
  const long long lo = static_cast<long long>(acc64[(2 * b + 1) * PD * PD + ij]);
  Pout[e] = fma(static_cast<double>(hi), 4.76837158203125e-07,
                static_cast<double>(lo) * 1.7763568394002505e-15) * pscale;
}

}  // namespace oi8

// ---------------------------------------------------------------------------
// signal-major digit rows: row s = 5 planes x p dims of Y_a (y = Y_int 2^-sy,
// Y_int = sum_a Y_a 128^(4-a), sign-magnitude), one thread per (signal, dim);
// p = 64 (outer_i8.cu, round_i8.cu) or 256 (coef_i8.cu)
template <int PD>
__global__ void k_y_digits(const float* __restrict__ y, int64_t m, int sy, int8_t* ydig) {
  const int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (e >= m * PD) return;
  const int64_t s = e / PD;
  const int i = static_cast<int>(e % PD);
  const uint32_t bits = __float_as_uint(y[e]);
  const uint32_t ex = (bits >> 23) & 255u;
  const uint32_t mant = (bits & 0x7FFFFFu) | (ex ? 0x800000u : 0u);
  const int sh = static_cast<int>(ex ? ex : 1u) - 150 + sy;  // Y_int = mant * 2^sh
  uint32_t lo28, top;
  if (sh >= 0) {
    lo28 = (mant << sh) & 0x0FFFFFFFu;
    top = sh >= 5 ? (mant >> (28 - sh)) : 0u;
  } else {
    lo28 = sh > -24 ? (mant >> -sh) : 0u;
    top = 0u;
  }
  const uint32_t d[oi8::YD] = {top, lo28 >> 21, (lo28 >> 14) & 127u, (lo28 >> 7) & 127u,
                               lo28 & 127u};
  const bool neg = bits >> 31;
  int8_t* row = ydig + s * (oi8::YD * PD);
#pragma unroll
  for (int a = 0; a < oi8::YD; ++a)
    row[a * PD + i] = static_cast<int8_t>(neg ? -static_cast<int>(d[a]) : static_cast<int>(d[a]));
}

// ---------------------------------------------------------------------------
// scan of the signal matrix for the digit formats: [0] = smallest E with every
// |y| < 2^E (int), [1] = smallest exponent of a set mantissa bit over the
// nonzero values (int), [2..3] = largest ||y||^2 (double bits)
__global__ void k_i8_scan(const float* __restrict__ y, int64_t m, int p, int* emax, int* lsb,
                          unsigned long long* norm2) {
  int my_e = -1000, my_l = 1000;
  double my_n = 0.0;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t r = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; r < m;
       r += stride) {
    double nn = 0.0;
    for (int i = 0; i < p; ++i) {
      const float f = y[r * p + i];
      nn = fma(static_cast<double>(f), static_cast<double>(f), nn);
      const uint32_t bits = __float_as_uint(f) & 0x7FFFFFFFu;
      if (!bits) continue;
      const int e = static_cast<int>(bits >> 23);
      const uint32_t mant = (bits & 0x7FFFFFu) | (e ? 0x800000u : 0u);
      const int ee = (e ? e : 1) - 150;  // value = mant * 2^ee
      my_e = max(my_e, ee + 32 - __clz(mant));
      my_l = min(my_l, ee + __ffs(mant) - 1);
    }
    my_n = fmax(my_n, nn);
  }
  for (int o = 16; o > 0; o >>= 1) {
    my_e = max(my_e, __shfl_xor_sync(0xffffffffu, my_e, o));
    my_l = min(my_l, __shfl_xor_sync(0xffffffffu, my_l, o));
    my_n = fmax(my_n, __shfl_xor_sync(0xffffffffu, my_n, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMax(emax, my_e);
    atomicMin(lsb, my_l);
    atomicMax(norm2, static_cast<unsigned long long>(__double_as_longlong(my_n)));
  }
}

}  // namespace sbo

using namespace sbo;

extern "C" int sbo_i8_scan(const void* y, int dtype, int64_t m, int p, int32_t* out,
                           void* stream) {
  if (dtype != SBO_F32) return fail(SBO_EINVAL, "the digit scan needs float32 signals");
  if (!out || p < 1) return fail(SBO_EINVAL, "bad arguments");
  cudaStream_t st = as_stream(stream);
  const int init[4] = {-1000, 1000, 0, 0};
  SBO_CHECK_CUDA(cudaMemcpyAsync(out, init, sizeof(init), cudaMemcpyHostToDevice, st));
  if (m <= 0) return SBO_OK;
  const int blocks = static_cast<int>(min64(ceil_div(m, 256), 148 * 8));
  k_i8_scan<<<blocks, 256, 0, st>>>(static_cast<const float*>(y), m, p, out, out + 1,
                                    reinterpret_cast<unsigned long long*>(out + 2));
  return check_launch("k_i8_scan");
}

extern "C" int sbo_y_digits(const void* y, int dtype, int64_t m, int p, int sy, void* ydig,
                            void* stream) {
  if (dtype != SBO_F32 || (p != 64 && p != 256))
    return fail(SBO_EINVAL, "digit rows need float32, p = 64 or 256");
  if (m <= 0) return SBO_OK;
  const int64_t n = m * p;
  const unsigned grid = static_cast<unsigned>(ceil_div(n, 256));
  if (p == 64)
    k_y_digits<64><<<grid, 256, 0, as_stream(stream)>>>(static_cast<const float*>(y), m, sy,
                                                         static_cast<int8_t*>(ydig));
  else
    k_y_digits<256><<<grid, 256, 0, as_stream(stream)>>>(static_cast<const float*>(y), m, sy,
                                                          static_cast<int8_t*>(ydig));
  return check_launch("k_y_digits");
}

extern "C" size_t sbo_y_tiles_bytes(int64_t n, int64_t max_seg, int p) {
  return static_cast<size_t>(ceil_div(n > 0 ? n : 0, oi8::TS) + (max_seg > 0 ? max_seg : 0)) *
         oi8::YTILE * (p == 256 ? 4 : 1);
}

extern "C" int sbo_y_tiles(const void* ydig, int p, const int32_t* order, const int64_t* seg_lo,
                           const int64_t* seg_hi, const int32_t* nseg, int64_t max_seg,
                           void* tiles, void* stream) {
  if (!ydig || !tiles) return fail(SBO_EINVAL, "bad arguments");
  if (p != 64 && p != 256) return fail(SBO_EINVAL, "digit tiles need p = 64 or 256");
  if (max_seg <= 0) return SBO_OK;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const unsigned grid = static_cast<unsigned>(min64(max_seg, 4 * sms));
  auto kern = p == 256 ? oi8::k_y_tiles<256> : oi8::k_y_tiles<64>;
  kern<<<grid, oi8::YT_THREADS, 0, as_stream(stream)>>>(
      static_cast<const int8_t*>(ydig), order, seg_lo, seg_hi, nseg, static_cast<int8_t*>(tiles));
  return check_launch("k_y_tiles");
}

extern "C" size_t sbo_outer_i8_workspace_bytes(int nblocks, int p) {
  return static_cast<size_t>(nblocks > 0 ? nblocks : 0) * 2 * p * p * sizeof(long long);
}

extern "C" int sbo_outer_i8_segments(const void* ytiles, int p, const int32_t* seg_block,
                                     const int64_t* seg_lo,
                                     const int64_t* seg_hi, const int32_t* nseg,
                                     int64_t max_seg, int nblocks, int s0, int64_t ld,
                                     const int16_t* idx, const double* val, int sy, int sx,
                                     double* P, void* workspace, size_t ws_bytes,
                                     void* stream) {
  if (p != 64 && p != 256) return fail(SBO_EINVAL, "the tensor-core outer product needs p = 64 or 256");
  if (s0 < 1 || !idx || !val || !P || nblocks < 1) return fail(SBO_EINVAL, "bad arguments");
  if (ws_bytes < sbo_outer_i8_workspace_bytes(nblocks, p) || !workspace)
    return fail(SBO_EINVAL, "outer_i8 workspace too small");
  const int k = s0 < p ? s0 : p;
  cudaStream_t st = as_stream(stream);
  SBO_CHECK_CUDA(cudaMemsetAsync(workspace, 0, sbo_outer_i8_workspace_bytes(nblocks, p), st));
  auto* acc = static_cast<unsigned long long*>(workspace);
  if (max_seg > 0) {
    auto kern = p == 256 ? oi8::k_outer_i8<256> : oi8::k_outer_i8<64>;
    static bool attr[2] = {false, false};
    if (!attr[p == 256]) {
      SBO_CHECK_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                          static_cast<int>(oi8::SMEM_BYTES)));
      attr[p == 256] = true;
    }
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const unsigned grid = static_cast<unsigned>(min64(max_seg, sms)) * (p == 256 ? 16u : 1u);
    kern<<<grid, oi8::THREADS, oi8::SMEM_BYTES, st>>>(
        static_cast<const int8_t*>(ytiles), seg_block, seg_lo, seg_hi, nseg, k, ld, idx,
        val, ldexp(1.0, sx), acc);
    if (int rc = check_launch("k_outer_i8")) return rc;
  }
  const int64_t n = static_cast<int64_t>(nblocks) * p * p;
  auto fin = p == 256 ? oi8::k_i8_finalize<256> : oi8::k_i8_finalize<64>;
  fin<<<static_cast<unsigned>(ceil_div(n, 256)), 256, 0, st>>>(acc, nblocks,
                                                               ldexp(1.0, 77 - sy - sx), P);
  return check_launch("k_i8_finalize");
}
