// Exact float64 coefficients C = Q^T y for p = 256 (config D) on the tcgen05
// tensor cores, from integer digits: the Ozaki split of round_i8.cu (y = Y_int
// 2^-sy in 5 sign-magnitude 7-bit digits, each block entry rounded to 2^-54 in
// 8 balanced digits, digit products of level <= 7 accumulated exactly in int32
// TMEM, recombined in float64) at four times the depth and width:
//
// * K = 256 dims = 4 K-blocks of 64; the atoms = 4 quarters of 64.  Per
//   128-signal tile and quarter q, the 4 K-blocks accumulate into one 512-column
//   TMEM image (8 levels x 64 atoms, even levels in columns 0-255, odd in 256-511,
//   exactly round_i8's layout) — |D_L| <= 5 x 256 x 127 x 64 < 2^24, and the
//   paired levels D_L 128 + D_L+1 < 2^31 stay exact in int32.
// * Per (quarter, K-block) stage: the tile's digit rows of the K-block (5 planes
//   x 64 B per signal, gathered through the segment order with 16-B cp.async into
//   the SW128 slabs [Y0|Y1] [Y2|Y3] [Y4|-]) and the block's digit image of that
//   (quarter, K-block) (4 slabs [Q_2s|Q_2s+1] of 64 atoms x 128 B, one bulk copy).
// * The epilogue drains a quarter (8 warps: rows 32 (w % 4), atoms 32 (w / 4)),
//   recombines, and writes the float64 coefficients as rows of 256 at the
//   segment position; sbo_select_top then selects on them.
//
// This replaces the float64 DMMA projection of the p = 256 rounds (k_code_f64);
// the selection and the outer product stay float64.
#include "common.cuh"
#include "pick.cuh"
#include "sm100.cuh"

namespace sbo {
namespace ci8 {

constexpr int P = 256, TS = 128, YD = 5, QDIM = 64;
constexpr int A_SLAB = TS * 128;               // 16 KB: [Y_2j | Y_2j+1], 128-B swizzle
constexpr int A_BYTES = 2 * A_SLAB + TS * 64;  // 40 KB: + Y4 alone, 64-B swizzle
constexpr int NST = 3;                         // pipeline stages
constexpr int B_SLAB = QDIM * 128;   // 8 KB
constexpr int B_BYTES = 4 * B_SLAB;  // 32 KB: one (quarter, K-block) digit image
constexpr int EPI_THREADS = 256, MMA_WARP = 8, PROD_WARP0 = 9, NPROD = 64;
constexpr int THREADS = 352;
constexpr int64_t QDIG_BLOCK = 16 * static_cast<int64_t>(B_BYTES);  // 512 KB per block

struct Smem {
  int8_t a[NST][A_BYTES];
  int8_t b[NST][B_BYTES];
  uint64_t full[NST], empty[NST], acc_full, acc_empty;
  uint32_t tmem;
};
constexpr size_t SMEM_BYTES = sizeof(Smem) + 1024;

__device__ __forceinline__ Smem* smem_of(unsigned char* raw) {
  const uint32_t a = sm100::smem_u32(raw);
  return reinterpret_cast<Smem*>(raw + ((1024u - (a & 1023u)) & 1023u));
}

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

__device__ __forceinline__ uint32_t slab_off(int row, int byte) {
  return static_cast<uint32_t>(row >> 3) * 1024u + sm100::sw128_offset(row & 7, byte);
}

// Y4's slab: rows of 64 B, 64-B swizzle (16-B chunk ^= (row / 2) % 4), 8-row
// groups 512 B apart
__device__ __forceinline__ uint32_t sw64_off(int row, int byte) {
  return static_cast<uint32_t>(row) * 64u + ((((byte >> 4) ^ ((row >> 1) & 3)) << 4) | (byte & 15));
}

__device__ __forceinline__ uint64_t desc_sw64(uint32_t addr) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((addr >> 4) & 0x3FFF);  // start address
  d |= static_cast<uint64_t>(1) << 16;               // LBO (unused, swizzled K-major)
  d |= static_cast<uint64_t>(512 >> 4) << 32;        // SBO: 8 rows x 64 B
  d |= static_cast<uint64_t>(1) << 46;               // descriptor version (sm_100)
  d |= static_cast<uint64_t>(4) << 61;               // SWIZZLE_64B
  return d;
}

// A operand of y digit a at K offset ko (bytes) of the stage at ab
__device__ __forceinline__ uint64_t a_desc(uint32_t ab, int a, uint32_t ko) {
  return a < 4 ? sm100::desc_sw128(ab + (a >> 1) * A_SLAB + (a & 1) * 64 + ko)
               : desc_sw64(ab + 2 * A_SLAB + ko);
}

__device__ __forceinline__ double l2d(long long v) {
  const int hi = static_cast<int>(v >> 32) + 0x43380000;
  return __hiloint2double(hi, static_cast<int>(v)) - 6755399441055744.0;
}

__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src),
               "r"(valid ? 16 : 0));
}

__device__ __forceinline__ void seg_range(int nseg, int& s0, int& s1) {
  s0 = static_cast<int>(static_cast<int64_t>(nseg) * blockIdx.x / gridDim.x);
  s1 = static_cast<int>(static_cast<int64_t>(nseg) * (blockIdx.x + 1) / gridDim.x);
}

struct Ring {
  int i = 0;
  uint32_t ph = 0;
  __device__ __forceinline__ void next() {
    if (++i == NST) {
      i = 0;
      ph ^= 1u;
    }
  }
};

// producers: one (quarter, K-block) stage — the block image slice by one bulk
// copy, the tile's digit rows of the K-block by 16-B cp.async; the stage's full
// barrier gets this warp's arrival one stage later (cp.async.wait_group 1)
struct Producer {
  int pw, pt, lane, rj[5], cj[5], prev = -1;
  __device__ explicit Producer(int warp, int tid) {
    pw = warp - PROD_WARP0;
    pt = tid - PROD_WARP0 * 32;
    lane = tid & 31;
#pragma unroll
    for (int j = 0; j < 5; ++j) {
      rj[j] = (lane + 32 * j) / 20;
      cj[j] = (lane + 32 * j) % 20;
    }
  }
  // warp pw gathers rows [64 pw, 64 pw + 64): lane l takes 16-B chunk
  // c = l + 32 j of each 8-row group (row c / 20, plane (c % 20) / 4)
  __device__ __forceinline__ void stage(Smem* S, Ring& r, const int8_t* qimg,
                                        const int8_t* __restrict__ ydig, const int (&o)[2], int n,
                                        int kb) {
    sm100::mbar_wait(&S->empty[r.i], r.ph ^ 1u);
    if (pt == 0) {
      asm volatile("mbarrier.expect_tx.shared::cta.b64 [%0], %1;" ::"r"(
                       sm100::smem_u32(&S->full[r.i])),
                   "r"(B_BYTES)
                   : "memory");
      sm100::bulk_g2s(S->b[r.i], qimg, B_BYTES, &S->full[r.i]);
    }
    const uint32_t base = sm100::smem_u32(S->a[r.i]);
#pragma unroll
    for (int g = 0; g < 8; ++g) {
#pragma unroll
      for (int j = 0; j < 5; ++j) {
        const int rl = 8 * g + rj[j], row = 64 * pw + rl;
        const int sig = __shfl_sync(0xffffffffu, o[g >> 2], rl & 31);
        const int c = cj[j], a = c >> 2;
        const uint32_t dst = a < 4 ? base + (a >> 1) * A_SLAB + slab_off(row, (a & 1) * 64 + (c & 3) * 16)
                                   : base + 2 * A_SLAB + sw64_off(row, (c & 3) * 16);
        cp_async16(dst,
                   ydig + static_cast<int64_t>(sig) * (YD * P) + a * P + kb * QDIM + (c & 3) * 16,
                   row < n);
      }
    }
    asm volatile("cp.async.commit_group;");
    if (prev >= 0) {
      asm volatile("cp.async.wait_group 1;" ::: "memory");
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      sm100::mbar_arrive(&S->full[prev]);
    }
    prev = r.i;
    r.next();
  }
  __device__ __forceinline__ void finish(Smem* S) {
    if (prev >= 0) {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      sm100::mbar_arrive(&S->full[prev]);
    }
  }
};

// issuer (one thread): the 10 digit-pair MMAs of both 32-deep k-steps of a
// stage; a quarter's accumulators are initialised at K-block 0 (after the
// epilogue drained the previous quarter) and committed after K-block 3
__device__ __forceinline__ void mma_stage(Smem* S, uint32_t tmem, Ring& r, int kb,
                                          uint32_t& acc_ph) {
  sm100::mbar_wait(&S->full[r.i], r.ph);
  if (kb == 0) sm100::mbar_wait(&S->acc_empty, acc_ph ^ 1u);
  sm100::tc_fence_after();
  const uint32_t ab = sm100::smem_u32(S->a[r.i]), bb = sm100::smem_u32(S->b[r.i]);
#pragma unroll
  for (int kk = 0; kk < 2; ++kk) {
    const uint32_t ko = kk * 32;
    const uint32_t init = (kb == 0 && kk == 0) ? 0u : 1u;
    // (y digit A_, Q parity PI_, N, TMEM column): levels A_ + PI_ + 2i of one parity
#define CI8_MMA(A_, PI_, N_, COL_, ACC_)                                                    \
  umma_i8(tmem + (COL_), a_desc(ab, (A_), ko),                                             \
          sm100::desc_sw128(bb + (PI_)*64 + ko), idesc_i8(128, (N_)), (ACC_))
    CI8_MMA(0, 0, 256, 0, init);    // levels 0 2 4 6
    CI8_MMA(0, 1, 256, 256, init);  // levels 1 3 5 7
    CI8_MMA(1, 0, 256, 256, 1u);
    CI8_MMA(1, 1, 192, 64, 1u);
    CI8_MMA(2, 0, 192, 64, 1u);
    CI8_MMA(2, 1, 192, 320, 1u);
    CI8_MMA(3, 0, 192, 320, 1u);
    CI8_MMA(3, 1, 128, 128, 1u);
    CI8_MMA(4, 0, 128, 128, 1u);
    CI8_MMA(4, 1, 128, 384, 1u);
#undef CI8_MMA
  }
  sm100::umma_commit(&S->empty[r.i]);
  if (kb == 3) {
    sm100::umma_commit(&S->acc_full);
    acc_ph ^= 1u;
  }
  r.next();
}

// epilogue warp: one quarter's 32 atoms (a0 ..) of its 32 rows out of TMEM,
// recombined to float64 and stored at out[64 q + a0 ..] (out NULL: discarded)
__device__ __forceinline__ void drain_quarter(Smem* S, uint32_t lane_base, int a0, int q,
                                              uint32_t& acc_ph, double cscale, double* out) {
  const int lane = threadIdx.x & 31;
  sm100::mbar_wait(&S->acc_full, acc_ph);
  acc_ph ^= 1u;
  sm100::tc_fence_after();
#pragma unroll
  for (int ch = 0; ch < 4; ++ch) {
    uint32_t v[8][8];  // [level][atom]
#pragma unroll
    for (int L = 0; L < 8; ++L) {
      const uint32_t col = (L & 1 ? 256u + 64u * (L >> 1) : 64u * (L >> 1)) + a0 + 8 * ch;
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
          : "=r"(v[L][0]), "=r"(v[L][1]), "=r"(v[L][2]), "=r"(v[L][3]), "=r"(v[L][4]),
            "=r"(v[L][5]), "=r"(v[L][6]), "=r"(v[L][7])
          : "r"(lane_base + col));
    }
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    double c[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int e0 = static_cast<int>(v[0][u]) * 128 + static_cast<int>(v[1][u]);
      const int e1 = static_cast<int>(v[2][u]) * 128 + static_cast<int>(v[3][u]);
      const int e2 = static_cast<int>(v[4][u]) * 128 + static_cast<int>(v[5][u]);
      const int e3 = static_cast<int>(v[6][u]) * 128 + static_cast<int>(v[7][u]);
      const double hi_ = l2d(static_cast<long long>(e0) * 16384 + e1);
      const double lo_ = l2d(static_cast<long long>(e2) * 16384 + e3);
      c[u] = fma(hi_, 268435456.0, lo_) * cscale;
    }
    if (out) {
      double2* o2 = reinterpret_cast<double2*>(out + QDIM * q + a0 + 8 * ch);
#pragma unroll
      for (int u = 0; u < 4; ++u) o2[u] = make_double2(c[2 * u], c[2 * u + 1]);
    }
  }
  sm100::tc_fence_before();
  __syncwarp();
  if (lane == 0) sm100::mbar_arrive(&S->acc_empty);
}

__device__ __forceinline__ void setup(Smem* S, int warp) {
  if (threadIdx.x == 0) {
    for (int s = 0; s < NST; ++s) {
      sm100::mbar_init(&S->full[s], NPROD);  // producer arrivals + the B bulk copy's bytes
      sm100::mbar_init(&S->empty[s], 1);
    }
    sm100::mbar_init(&S->acc_full, 1);
    sm100::mbar_init(&S->acc_empty, EPI_THREADS / 32);
    sm100::fence_barrier_init();
  }
  if (warp == MMA_WARP) sm100::tmem_alloc(&S->tmem, 512);
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
}

__global__ void __launch_bounds__(THREADS, 1)
k_coef_i8(const int8_t* __restrict__ ydig, const int32_t* __restrict__ order,
          const int32_t* __restrict__ seg_block, const int64_t* __restrict__ seg_lo,
          const int64_t* __restrict__ seg_hi, const int32_t* __restrict__ nseg_p,
          const int8_t* __restrict__ qdig, int block_override, double cscale,
          double* __restrict__ coef) {
  extern __shared__ unsigned char raw[];
  Smem* S = smem_of(raw);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nseg = *nseg_p;
  setup(S, warp);
  const uint32_t tmem = S->tmem;
  int sa, sb;
  seg_range(nseg, sa, sb);
  auto block_of = [&](int seg) { return block_override >= 0 ? block_override : seg_block[seg]; };

  if (warp >= PROD_WARP0) {  // ------------------------------------------ producers
    Producer pr(warp, tid);
    Ring r;
    for (int seg = sa; seg < sb; ++seg) {
      const int64_t lo = seg_lo[seg], hi = seg_hi[seg];
      const int8_t* qb = qdig + static_cast<int64_t>(block_of(seg)) * QDIG_BLOCK;
      for (int64_t t0 = lo; t0 < hi; t0 += TS) {
        const int n = static_cast<int>(min64(TS, hi - t0));
        int o[2];
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int row = 64 * pr.pw + 32 * h + lane;
          o[h] = row < n ? (order ? order[t0 + row] : static_cast<int>(t0 + row)) : 0;
        }
        for (int st = 0; st < 16; ++st)  // st = 4 quarter + K-block
          pr.stage(S, r, qb + st * static_cast<int64_t>(B_BYTES), ydig, o, n, st & 3);
      }
    }
    pr.finish(S);
  } else if (warp == MMA_WARP) {  // --------------------------------------- issuer
    if (lane == 0) {
      Ring r;
      uint32_t acc_ph = 0;
      for (int seg = sa; seg < sb; ++seg) {
        const int64_t lo = seg_lo[seg], hi = seg_hi[seg];
        for (int64_t t0 = lo; t0 < hi; t0 += TS)
          for (int st = 0; st < 16; ++st) mma_stage(S, tmem, r, st & 3, acc_ph);
      }
    }
  } else {  // ------------------------------------------------------------ epilogue
    const int q4 = warp & 3;
    const int row = 32 * q4 + lane;
    const uint32_t lane_base = tmem + (static_cast<uint32_t>(32 * q4) << 16);
    const int a0 = 32 * (warp >> 2);
    uint32_t acc_ph = 0;
    for (int seg = sa; seg < sb; ++seg) {
      const int64_t lo = seg_lo[seg], hi = seg_hi[seg];
      for (int64_t t0 = lo; t0 < hi; t0 += TS) {
        double* out = t0 + row < hi ? coef + (t0 + row) * P : nullptr;
        for (int q = 0; q < 4; ++q) drain_quarter(S, lane_base, a0, q, acc_ph, cscale, out);
      }
    }
  }
  __syncthreads();
  if (warp == MMA_WARP) sm100::tmem_dealloc(tmem, 512);
}

// union of the candidate masks of a tile's rows (every lane of the warp calls it)
__device__ __forceinline__ uint64_t tile_union(const uint64_t* __restrict__ cand, int64_t base,
                                               int n) {
  uint64_t u = 0;
  for (int i = threadIdx.x & 31; i < n; i += 32) u |= cand[base + i];
  const uint32_t lo = __reduce_or_sync(0xffffffffu, static_cast<uint32_t>(u));
  const uint32_t hi = __reduce_or_sync(0xffffffffu, static_cast<uint32_t>(u >> 32));
  return (static_cast<uint64_t>(hi) << 32) | lo;
}

// The float64 re-decision of the signals the tensor-core energy pass flagged
// (sbo.py:177-194 over each signal's candidate blocks; the role of
// sbo_energy_recheck_cand, tiles_f64.cu): tiles of 128 flagged signals (sorted by
// candidate mask, so a tile's masks mostly agree); for each block of the tile's
// union, the exact digit projection of the tile as above, its four quarters
// drained to a per-CTA float64 row buffer (L2-resident, double-buffered across
// blocks), then each epilogue warp ranks its rows whose mask holds the block
// (pick_row, the exact selection) and keeps the first maximum (blocks ascending:
// ties -> lower block, sbo.py:191).
__global__ void __launch_bounds__(THREADS, 1)
k_recheck_i8(const int8_t* __restrict__ ydig, const int32_t* __restrict__ list,
             const uint64_t* __restrict__ cand, const int32_t* __restrict__ nlist,
             const int8_t* __restrict__ qdig, int k, int kind, double cscale, double* scratch,
             int32_t* best, double* score, double* residual) {
  extern __shared__ unsigned char raw[];
  Smem* S = smem_of(raw);
  __shared__ double bscore[TS], brest[TS];
  __shared__ int bbest[TS];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int64_t count = *nlist;
  const int64_t ntiles = (count + TS - 1) / TS;
  setup(S, warp);
  const uint32_t tmem = S->tmem;

  if (warp >= PROD_WARP0) {  // ------------------------------------------ producers
    Producer pr(warp, tid);
    Ring r;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      const int64_t t0 = tile * TS;
      const int n = static_cast<int>(min64(TS, count - t0));
      int o[2];
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int row = 64 * pr.pw + 32 * h + lane;
        o[h] = row < n ? list[t0 + row] : 0;
      }
      for (uint64_t u = tile_union(cand, t0, n); u; u &= u - 1) {
        const int8_t* qb = qdig + static_cast<int64_t>(__ffsll(u) - 1) * QDIG_BLOCK;
        for (int st = 0; st < 16; ++st)
          pr.stage(S, r, qb + st * static_cast<int64_t>(B_BYTES), ydig, o, n, st & 3);
      }
    }
    pr.finish(S);
  } else if (warp == MMA_WARP) {  // --------------------------------------- issuer
    Ring r;
    uint32_t acc_ph = 0;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      const int64_t t0 = tile * TS;
      const int n = static_cast<int>(min64(TS, count - t0));
      const int nb = __popcll(tile_union(cand, t0, n));
      if (lane == 0)
        for (int i = 0; i < 16 * nb; ++i) mma_stage(S, tmem, r, i & 3, acc_ph);
      __syncwarp();
    }
  } else {  // ------------------------------------------------------------ epilogue
    const int q4 = warp & 3;
    const int row = 32 * q4 + lane;
    const uint32_t lane_base = tmem + (static_cast<uint32_t>(32 * q4) << 16);
    const int a0 = 32 * (warp >> 2);
    uint32_t acc_ph = 0;
    int buf = 0;
    double* scr = scratch + static_cast<int64_t>(blockIdx.x) * 2 * TS * P;
    for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
      const int64_t t0 = tile * TS;
      const int n = static_cast<int>(min64(TS, count - t0));
      for (int rr = warp; rr < TS; rr += EPI_THREADS / 32) {  // this warp's selection rows
        if (lane == 0) {
          bscore[rr] = -1.0;
          brest[rr] = 0.0;
          bbest[rr] = -1;
        }
      }
      for (uint64_t u = tile_union(cand, t0, n); u; u &= u - 1) {
        const int b = __ffsll(u) - 1;
        double* rows = scr + buf * TS * P;
        for (int q = 0; q < 4; ++q)
          drain_quarter(S, lane_base, a0, q, acc_ph, cscale, row < n ? rows + row * P : nullptr);
        __threadfence_block();
        asm volatile("bar.sync 1, %0;" ::"r"(EPI_THREADS) : "memory");
        for (int rr = warp; rr < n; rr += EPI_THREADS / 32) {
          if (!((cand[t0 + rr] >> b) & 1ull)) continue;
          const RowPick pk = pick_row(rows + rr * P, P, k, kind);
          if (lane == 0 && pk.score > bscore[rr]) {  // strict: first maximum wins
            bscore[rr] = pk.score;
            brest[rr] = pk.rest_sq;
            bbest[rr] = b;
          }
        }
        buf ^= 1;
      }
      __syncwarp();
      for (int rr = warp; rr < n; rr += EPI_THREADS / 32) {
        if (lane == 0) {
          const int64_t j = list[t0 + rr];
          best[j] = bbest[rr];
          score[j] = bscore[rr];
          residual[j] = brest[rr];
        }
      }
    }
  }
  __syncthreads();
  if (warp == MMA_WARP) sm100::tmem_dealloc(tmem, 512);
}

// The block's digit images for k_coef_i8: per (quarter q, K-block kb) 32 KB =
// 4 SW128 slabs [Q_2s | Q_2s+1] of 64 atom rows x 128 B (dims 64 kb .. + 63);
// Q_int = rint(q 2^54) in 8 balanced 7-bit digits.  One thread per entry.
__global__ void k_q_digits256(const double* __restrict__ blocks, int b0, int nb,
                              int8_t* __restrict__ qdig) {
  const int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (e >= static_cast<int64_t>(nb) * P * P) return;
  const int b = b0 + static_cast<int>(e / (P * P));
  const int rem = static_cast<int>(e % (P * P));
  const int dim = rem / P, atom = rem % P;  // q[dim][atom]: atom = column (numpy layout)
  long long v = __double2ll_rn(blocks[static_cast<int64_t>(b) * P * P + rem] * 18014398509481984.0);
  int8_t* out = qdig + static_cast<int64_t>(b) * QDIG_BLOCK +
                (4 * (atom / QDIM) + dim / QDIM) * static_cast<int64_t>(B_BYTES);
  const int ar = atom % QDIM, dk = dim % QDIM;
#pragma unroll
  for (int d = 7; d >= 0; --d) {
    const int dd = ((static_cast<int>(v) + 64) & 127) - 64;
    v = (v - dd) >> 7;
    out[(d >> 1) * B_SLAB + slab_off(ar, (d & 1) * 64 + dk)] = static_cast<int8_t>(dd);
  }
}

}  // namespace ci8
}  // namespace sbo

using namespace sbo;

namespace {
int sm_count() {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms;
}
}  // namespace

extern "C" size_t sbo_coef_i8_workspace_bytes(int nblocks) {
  return static_cast<size_t>(nblocks > 0 ? nblocks : 0) * ci8::QDIG_BLOCK;
}

extern "C" int sbo_coef_i8_segments(const void* ydig, int sy, const int32_t* order,
                                    const int32_t* seg_block, const int64_t* seg_lo,
                                    const int64_t* seg_hi, const int32_t* nseg,
                                    int64_t max_seg, const double* blocks, int nblocks,
                                    int block_override, double* coef, void* workspace,
                                    size_t ws_bytes, void* stream) {
  if (!ydig || !blocks || !coef || nblocks < 1) return fail(SBO_EINVAL, "bad arguments");
  if (block_override >= nblocks) return fail(SBO_EINVAL, "block_override out of range");
  if (!workspace || ws_bytes < sbo_coef_i8_workspace_bytes(nblocks))
    return fail(SBO_EINVAL, "coef_i8 workspace too small");
  if (max_seg <= 0) return SBO_OK;
  cudaStream_t st = as_stream(stream);
  auto* qdig = static_cast<int8_t*>(workspace);
  const int b0 = block_override >= 0 ? block_override : 0;
  const int nb = block_override >= 0 ? 1 : nblocks;
  const int64_t ne = static_cast<int64_t>(nb) * ci8::P * ci8::P;
  ci8::k_q_digits256<<<static_cast<unsigned>(ceil_div(ne, 256)), 256, 0, st>>>(blocks, b0, nb,
                                                                                qdig);
  if (int rc = check_launch("k_q_digits256")) return rc;
  static bool attr = false;
  if (!attr) {
    SBO_CHECK_CUDA(cudaFuncSetAttribute(ci8::k_coef_i8, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(ci8::SMEM_BYTES)));
    attr = true;
  }
  const unsigned grid = static_cast<unsigned>(min64(max_seg, sm_count()));
  ci8::k_coef_i8<<<grid, ci8::THREADS, ci8::SMEM_BYTES, st>>>(
      static_cast<const int8_t*>(ydig), order, seg_block, seg_lo, seg_hi, nseg, qdig,
      block_override, ldexp(1.0, -sy - 26), coef);
  return check_launch("k_coef_i8");
}

extern "C" size_t sbo_recheck_i8_workspace_bytes(int K) {
  return static_cast<size_t>(K > 0 ? K : 0) * ci8::QDIG_BLOCK +
         static_cast<size_t>(sm_count()) * 2 * ci8::TS * ci8::P * sizeof(double);
}

extern "C" int sbo_energy_recheck_i8(const void* ydig, int sy, const double* blocks, int K,
                                     int s0, int kind, const int32_t* list,
                                     const uint64_t* cand, const int32_t* nlist,
                                     int64_t max_list, int32_t* best, double* score,
                                     double* residual, void* workspace, size_t ws_bytes,
                                     void* stream) {
  if (!ydig || !blocks || !list || !cand || !nlist || !best || !score || !residual)
    return fail(SBO_EINVAL, "bad arguments");
  if (K < 1 || K > 64) return fail(SBO_EINVAL, "the candidate recheck needs 1 <= K <= 64");
  if (s0 < 1) return fail(SBO_EINVAL, "s0 must be at least 1");
  if (!workspace || ws_bytes < sbo_recheck_i8_workspace_bytes(K))
    return fail(SBO_EINVAL, "recheck_i8 workspace too small");
  if (max_list <= 0) return SBO_OK;
  cudaStream_t st = as_stream(stream);
  auto* qdig = static_cast<int8_t*>(workspace);
  const int64_t ne = static_cast<int64_t>(K) * ci8::P * ci8::P;
  ci8::k_q_digits256<<<static_cast<unsigned>(ceil_div(ne, 256)), 256, 0, st>>>(blocks, 0, K,
                                                                                qdig);
  if (int rc = check_launch("k_q_digits256")) return rc;
  static bool attr = false;
  if (!attr) {
    SBO_CHECK_CUDA(cudaFuncSetAttribute(ci8::k_recheck_i8,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(ci8::SMEM_BYTES)));
    attr = true;
  }
  const int sms = sm_count();
  const unsigned grid =
      static_cast<unsigned>(min64(ceil_div(max_list, static_cast<int64_t>(ci8::TS)), sms));
  auto* scratch = reinterpret_cast<double*>(qdig + K * ci8::QDIG_BLOCK);
  ci8::k_recheck_i8<<<grid, ci8::THREADS, ci8::SMEM_BYTES, st>>>(
      static_cast<const int8_t*>(ydig), list, cand, nlist, qdig, s0 < ci8::P ? s0 : ci8::P, kind,
      ldexp(1.0, -sy - 26), scratch, best, score, residual);
  return check_launch("k_recheck_i8");
}

// ---------------------------------------------------------------------------
// The float64 re-decision over (signal, candidate block) pairs: the flagged
// signals are bucketed per candidate block, each block's list is projected
// (k_coef_i8) and ranked (sbo_select_coded) on its own — only the pairs a
// signal's mask names are computed, where k_recheck_i8 projects every row of a
// tile onto the union of the tile's masks — and a last pass keeps each signal's
// first maximum over its candidate blocks in ascending order (sbo.py:191).
// ---------------------------------------------------------------------------
namespace sbo {
namespace ci8 {

__global__ void k_pair_lists(const int32_t* __restrict__ list, const uint64_t* __restrict__ cand,
                             const int32_t* __restrict__ nlist, int64_t cap,
                             unsigned long long* cnt, int32_t* pl_sig, int32_t* pl_f) {
  // per CTA: a shared histogram of the tile's pairs per block, one global
  // reservation per (CTA, block), then the scatter (positions within a block's
  // list are unordered: each pair's result does not depend on them)
  __shared__ unsigned long long base[64];
  __shared__ unsigned int hist[64];
  const int64_t n = *nlist;
  for (int64_t f0 = static_cast<int64_t>(blockIdx.x) * blockDim.x; f0 < n;
       f0 += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    if (threadIdx.x < 64) hist[threadIdx.x] = 0u;
    __syncthreads();
    const int64_t f = f0 + threadIdx.x;
    const uint64_t mask = f < n ? cand[f] : 0ull;
    for (uint64_t m = mask; m; m &= m - 1) atomicAdd(&hist[__ffsll(static_cast<long long>(m)) - 1], 1u);
    __syncthreads();
    if (threadIdx.x < 64) {
      base[threadIdx.x] = hist[threadIdx.x] ? atomicAdd(cnt + threadIdx.x,
                                                        static_cast<unsigned long long>(hist[threadIdx.x]))
                                            : 0ull;
      hist[threadIdx.x] = 0u;
    }
    __syncthreads();
    if (f < n) {
      const int32_t j = list[f];
      for (uint64_t m = mask; m; m &= m - 1) {
        const int b = __ffsll(static_cast<long long>(m)) - 1;
        const int64_t pos = static_cast<int64_t>(base[b] + atomicAdd(&hist[b], 1u));
        pl_sig[b * cap + pos] = j;
        pl_f[b * cap + pos] = static_cast<int32_t>(f);
      }
    }
    __syncthreads();
  }
}

__global__ void k_pair_reduce(const int32_t* __restrict__ list, const uint64_t* __restrict__ cand,
                              const int32_t* __restrict__ nlist, int64_t cap,
                              const double* __restrict__ s_score,
                              const double* __restrict__ s_rest, int32_t* best, double* score,
                              double* residual) {
  const int64_t n = *nlist;
  for (int64_t f = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; f < n;
       f += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    double bs = -1.0, br = 0.0;
    int bb = -1;
    for (uint64_t m = cand[f]; m; m &= m - 1) {  // blocks ascending: first maximum wins
      const int b = __ffsll(static_cast<long long>(m)) - 1;
      const double sc = s_score[b * cap + f];
      if (sc > bs) {
        bs = sc;
        br = s_rest[b * cap + f];
        bb = b;
      }
    }
    const int64_t j = list[f];
    best[j] = bb;
    score[j] = bs;
    residual[j] = br;
  }
}

constexpr int PAIR_CHUNK = 512;  // positions per segment of a block's pair list

struct PairWs {
  unsigned long long* cnt;
  int64_t *seg_lo, *seg_hi;
  int32_t *nseg, *seg_block, *pl_sig, *pl_f;
  double *s_score, *s_rest, *coef;
  int8_t* qdig;
  size_t bytes;
  int64_t max_seg;
  PairWs(void* base, int K, int64_t cap) {
    auto* p = static_cast<unsigned char*>(base);
    size_t off = 0;
    auto take = [&](size_t n) {
      unsigned char* r = p ? p + off : nullptr;
      off += (n + 255) & ~size_t(255);
      return r;
    };
    max_seg = (cap + PAIR_CHUNK - 1) / PAIR_CHUNK;
    if (max_seg < 1) max_seg = 1;
    cnt = reinterpret_cast<unsigned long long*>(take(64 * 8));
    seg_lo = reinterpret_cast<int64_t*>(take(max_seg * 8));
    seg_hi = reinterpret_cast<int64_t*>(take(max_seg * 8));
    nseg = reinterpret_cast<int32_t*>(take(4));
    seg_block = reinterpret_cast<int32_t*>(take(max_seg * 4));
    pl_sig = reinterpret_cast<int32_t*>(take(static_cast<size_t>(K) * cap * 4));
    pl_f = reinterpret_cast<int32_t*>(take(static_cast<size_t>(K) * cap * 4));
    s_score = reinterpret_cast<double*>(take(static_cast<size_t>(K) * cap * 8));
    s_rest = reinterpret_cast<double*>(take(static_cast<size_t>(K) * cap * 8));
    qdig = reinterpret_cast<int8_t*>(take(static_cast<size_t>(K) * QDIG_BLOCK));
    coef = reinterpret_cast<double*>(take(static_cast<size_t>(cap) * P * 8));
    bytes = off;
  }
};

}  // namespace ci8
}  // namespace sbo

extern "C" size_t sbo_recheck_pairs_workspace_bytes(int K, int64_t max_list) {
  return ci8::PairWs(nullptr, K, max_list > 0 ? max_list : 1).bytes;
}

extern "C" int sbo_energy_recheck_pairs(const void* ydig, int sy, const double* blocks, int K,
                                        int s0, int kind, const int32_t* list,
                                        const uint64_t* cand, const int32_t* nlist,
                                        int64_t max_list, int32_t* best, double* score,
                                        double* residual, void* workspace, size_t ws_bytes,
                                        void* stream) {
  if (!ydig || !blocks || !list || !cand || !nlist || !best || !score || !residual)
    return fail(SBO_EINVAL, "bad arguments");
  if (K < 1 || K > 64) return fail(SBO_EINVAL, "the candidate recheck needs 1 <= K <= 64");
  if (s0 < 1) return fail(SBO_EINVAL, "s0 must be at least 1");
  if (max_list <= 0) return SBO_OK;
  ci8::PairWs w(workspace, K, max_list);
  if (!workspace || ws_bytes < w.bytes) return fail(SBO_EINVAL, "recheck_pairs workspace too small");
  cudaStream_t st = as_stream(stream);
  const int64_t cap = max_list;
  SBO_CHECK_CUDA(cudaMemsetAsync(w.cnt, 0, 64 * 8, st));
  SBO_CHECK_CUDA(cudaMemsetAsync(w.seg_block, 0, w.max_seg * 4, st));
  const unsigned grid = static_cast<unsigned>(min64(ceil_div(cap, 256), 148 * 8));
  ci8::k_pair_lists<<<grid, 256, 0, st>>>(list, cand, nlist, cap, w.cnt, w.pl_sig, w.pl_f);
  if (int rc = check_launch("k_pair_lists")) return rc;
  const size_t qbytes = static_cast<size_t>(K) * ci8::QDIG_BLOCK;
  for (int b = 0; b < K; ++b) {
    const int64_t* cnt_b = reinterpret_cast<const int64_t*>(w.cnt + b);
    if (int rc = sbo_chunk_segments(cap, cnt_b, ci8::PAIR_CHUNK, w.seg_lo, w.seg_hi, w.nseg,
                                    stream))
      return rc;
    if (int rc = sbo_coef_i8_segments(ydig, sy, w.pl_sig + b * cap, w.seg_block, w.seg_lo,
                                      w.seg_hi, w.nseg, w.max_seg, blocks, K, b, w.coef, w.qdig,
                                      qbytes, stream))
      return rc;
    if (int rc = sbo_select_coded(w.coef, cnt_b, cap, ci8::P, s0, kind, w.pl_f + b * cap, cap,
                                  nullptr, nullptr, w.s_score + b * cap, w.s_rest + b * cap,
                                  stream))
      return rc;
  }
  ci8::k_pair_reduce<<<grid, 256, 0, st>>>(list, cand, nlist, cap, w.s_score, w.s_rest, best,
                                           score, residual);
  return check_launch("k_pair_reduce");
}
