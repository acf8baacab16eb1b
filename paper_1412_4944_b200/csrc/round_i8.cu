// The 1ONB round's coding step for p = 64 (onb.py:170-171: C = Q^T Y, then
// select_top, onb.py:58-76) and represent's residual pass (sbo.py:207-218) on
// the 5th-gen tensor cores: the float64-accurate projection is computed EXACTLY
// from integer digits by tcgen05.mma kind::i8 (an Ozaki split), not on DMMA.
//
// Number formats (the signal format is the one of outer_i8.cu, sbo_i8_scan):
//   y = Y_int 2^-sy,  Y_int = sum_a Y_a 128^(4-a), a = 0..4, |Y_a| <= 127
//       (sign-magnitude digits, the signal-major rows of sbo_y_digits)
//   q = Q_int 2^-54,  Q_int = sum_b Q_b 128^(7-b), b = 0..7, Q_b in [-64, 63]
//       (balanced digits of the block entries rounded to 2^-54; |q| <= 1)
//   c = sum_i y_i q_i = 2^(-sy-54) sum_L D_L 128^(11-L), D_L = sum_{a+b=L} Y_a Q_b^T
//   Levels L <= 7 are kept (the dropped ones weigh < 2^-47 absolute at the
//   unit-range scale sy = 35, typically ~1e-17): c = 2^(-sy-26) (HI 2^28 + LO),
//   HI = sum_{L<=3} D_L 128^(3-L), LO = sum_{4<=L<=7} D_L 128^(7-L), all exact
//   integer arithmetic in int32 TMEM (|D_L| <= 5 * 64 * 127 * 64 < 2^22) and
//   exact float64 integers; the only rounding is HI 2^28 + LO.
//
// MMA schedule (M = 128 signals, K = 64 dims as 2 k-steps of 32): the 8 Q digit
// planes are stored as 4 slabs [Q0|Q1] [Q2|Q3] [Q4|Q5] [Q6|Q7] of 64 atom rows x
// 128 B (SW128), so at K offset 0 the slabs stack the even digits Q0 Q2 Q4 Q6
// along N and at K offset 64 the odd ones.  Y_a x (even or odd digits) therefore
// produces levels of one parity in consecutive 64-column groups: TMEM columns
// 0-255 hold the even levels 0 2 4 6, columns 256-511 the odd levels 1 3 5 7.
// Ten MMAs per k-step (N = 256, 256, 256, 192 x 4, 128 x 3: 1920 columns, the
// 30 digit pairs of level <= 7), all at N >= 128.
//
// Selection: the high word of |c| (sign cleared) is a monotone key of |c|; the
// top-k threshold t_k comes from register networks (each of the two epilogue
// warpgroups owns 32 atoms of every row, their top-G lists are merged through
// shared memory); when exactly k keys reach t_k the kept set is {key >= t_k},
// the float64 stable-argsort set.  Otherwise (a key tie at the threshold, a
// 2^-20 relative gap) the row is re-decided with the exact rank rule on its
// float64 coefficients: the tied atoms ordered by the low word of |c|, equal
// magnitudes by atom (ties -> lower atom), all in registers + shared-memory
// exchanges between the two halves of the row.
//
// Warp roles (352 threads, one CTA per SM, a contiguous range of segments):
//   warps 0-7   epilogue: warp w reads TMEM lanes 32 (w % 4) .. +31 (its rows),
//               atoms 32 (w / 4) .. +31 (its half)
//   warp 8      MMA issuer (lane 0); the block's digit slabs by one bulk copy
//               when the block changes
//   warps 9-10  producers: each tile's 128 digit rows (320 B) gathered with
//               16-B cp.async into the SW128 A slabs [Y0|Y1] [Y2|Y3] [Y4|-]
#include "common.cuh"
#include "sm100.cuh"
#include "topk.cuh"

namespace sbo {
namespace ri8 {

constexpr int P = 64;
constexpr int TS = 128;                 // signals per tile (M)
constexpr int YD = 5;
constexpr int A_SLAB = TS * 128;        // 16 KB
constexpr int A_BYTES = 3 * A_SLAB;     // 48 KB
constexpr int B_SLAB = P * 128;         // 8 KB
constexpr int B_BYTES = 4 * B_SLAB;     // 32 KB: the block's digit image
constexpr int MODE_CODE = 0, MODE_RESID = 1;

// Role layout for NQ epilogue atom parts (NQ = 2: 32 atoms per thread, any
// k <= 32; NQ = 4: 16 atoms per thread, k <= 16, twice the epilogue warps for
// latency hiding): warps [0, 4 NQ) epilogue, then the MMA issuer, then the
// producers.
template <int NQ>
struct Roles {
  static constexpr int AQ = 64 / NQ;                 // atoms per epilogue thread
  static constexpr int EPI_WARPS = 4 * NQ;
  static constexpr int EPI_THREADS = 32 * EPI_WARPS;
  static constexpr int MMA_WARP = EPI_WARPS;
  static constexpr int PROD_WARP0 = EPI_WARPS + 1;
  static constexpr int PROD_WARPS = 2;
  static constexpr int NPROD = 32 * PROD_WARPS;
  static constexpr int THREADS = 32 * (EPI_WARPS + 1 + PROD_WARPS);
  static constexpr int GMAX = NQ == 2 ? 32 : 16;     // largest top-G list (k <= GMAX)
};

// shared memory, top-G lists of length G
template <int NQ, int G>
struct Smem {
  int8_t a[2][A_BYTES];
  int8_t b[B_BYTES];
  int32_t lists[NQ][G][TS];     // [part][rank][row]: per-part top-G keys
  int32_t cnt[2][NQ][TS];       // exchange buffers [parity][part][row]
  double part[NQ][2][TS];       // [part][rest | score][row]
  int16_t oidx[G][TS];          // code outputs staged per (slot, row)
  double oval[G][TS];
  uint64_t full[2], empty[2], acc_full, acc_empty, b_full;
  uint32_t tmem;
};
template <int NQ, int G>
constexpr size_t smem_bytes() { return sizeof(Smem<NQ, G>) + 1024; }

template <int NQ, int G>
__device__ __forceinline__ Smem<NQ, G>* smem_of(unsigned char* raw) {
  const uint32_t a = sm100::smem_u32(raw);
  return reinterpret_cast<Smem<NQ, G>*>(raw + ((1024u - (a & 1023u)) & 1023u));
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

// byte offset of (row, byte) inside a slab of 128-B SW128 rows
__device__ __forceinline__ uint32_t slab_off(int row, int byte) {
  return static_cast<uint32_t>(row >> 3) * 1024u + sm100::sw128_offset(row & 7, byte);
}

// integer |v| < 2^51 -> double exactly, without the conversion pipe: the bits
// of 1.5 2^52 + v, minus 1.5 2^52
__device__ __forceinline__ double l2d(long long v) {
  // (the magic's low word is 0: only the high word needs the add, no carry)
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
    if (++i == 2) {
      i = 0;
      ph ^= 1u;
    }
  }
};

__device__ __forceinline__ int sel_i(bool c, int a, int b) { return c ? a : b; }

template <int G, int MODE, int NQ>
__global__ void __launch_bounds__(Roles<NQ>::THREADS, 1)
k_round_i8(const int8_t* __restrict__ ydig, const int32_t* __restrict__ order,
           const int32_t* __restrict__ seg_block, const int64_t* __restrict__ seg_lo,
           const int64_t* __restrict__ seg_hi, const int32_t* __restrict__ nseg_p,
           const int8_t* __restrict__ qdig, int block_override, int k, int kind,
           double cscale, int64_t ld, int16_t* __restrict__ cidx, double* __restrict__ cval,
           double* __restrict__ rest_sq, double* __restrict__ score) {
  using R = Roles<NQ>;
  constexpr int AQ = R::AQ, EPI_THREADS = R::EPI_THREADS, MMA_WARP = R::MMA_WARP;
  constexpr int PROD_WARP0 = R::PROD_WARP0, NPROD = R::NPROD;
  static_assert(G <= R::GMAX, "top-G list longer than the part lists");
  extern __shared__ unsigned char raw[];
  using SM = Smem<NQ, G>;
  SM* S = smem_of<NQ, G>(raw);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int nseg = *nseg_p;
  if (tid == 0) {
    for (int s = 0; s < 2; ++s) {
      sm100::mbar_init(&S->full[s], NPROD);
      sm100::mbar_init(&S->empty[s], 1);
    }
    sm100::mbar_init(&S->acc_full, 1);
    sm100::mbar_init(&S->acc_empty, EPI_THREADS / 32);
    sm100::mbar_init(&S->b_full, 1);
    sm100::fence_barrier_init();
  }
  if (warp == MMA_WARP) sm100::tmem_alloc(&S->tmem, 512);
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem = S->tmem;
  int sa, sb;
  seg_range(nseg, sa, sb);
  auto block_of = [&](int seg) { return block_override >= 0 ? block_override : seg_block[seg]; };

  if (warp >= PROD_WARP0) {  // ------------------------------------------ producers
    // producer warp pw gathers rows [RPW pw, RPW pw + RPW) of each tile, 8 rows
    // (160 16-B chunks) per 5 copy rounds: lane l takes chunk q = l + 32 j of
    // the group, row q / 20, chunk q % 20 (digit (q % 20) / 4).  The rows'
    // signal ids are loaded before the stage wait and shuffled to the copies.
    constexpr int RPW = TS / R::PROD_WARPS, OR = RPW / 32;
    const int pw = warp - PROD_WARP0;
    int rj[5], cj[5];
#pragma unroll
    for (int j = 0; j < 5; ++j) {
      rj[j] = (lane + 32 * j) / 20;
      cj[j] = (lane + 32 * j) % 20;
    }
    Ring r;
    int prev = -1;  // stage of the previous tile (its arrival waits for this tile's issue)
    for (int seg = sa; seg < sb; ++seg) {
      const int64_t lo = seg_lo[seg], hi = seg_hi[seg];
      for (int64_t t0 = lo; t0 < hi; t0 += TS) {
        const int n = static_cast<int>(min64(TS, hi - t0));
        int o[OR];
#pragma unroll
        for (int h = 0; h < OR; ++h) {
          const int row = RPW * pw + 32 * h + lane;
          o[h] = row < n ? (order ? order[t0 + row] : static_cast<int>(t0 + row)) : 0;
        }
        sm100::mbar_wait(&S->empty[r.i], r.ph ^ 1u);
        const uint32_t base = sm100::smem_u32(S->a[r.i]);
#pragma unroll
        for (int g = 0; g < RPW / 8; ++g) {
#pragma unroll
          for (int j = 0; j < 5; ++j) {
            const int rl = 8 * g + rj[j], row = RPW * pw + rl;
            const int sig = __shfl_sync(0xffffffffu, o[g >> 2], rl & 31);
            const int c = cj[j], a = c >> 2;
            cp_async16(base + (a >> 1) * A_SLAB + slab_off(row, (a & 1) * 64 + (c & 3) * 16),
                       ydig + static_cast<int64_t>(sig) * (YD * P) + c * 16, row < n);
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
    }
    if (prev >= 0) {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      sm100::mbar_arrive(&S->full[prev]);
    }
  } else if (warp == MMA_WARP) {  // --------------------------------------- issuer
    if (lane == 0) {
      Ring r;
      uint32_t acc_ph = 0, b_ph = 0;
      int cur = -1;
      const uint32_t bb = sm100::smem_u32(S->b);
      for (int seg = sa; seg < sb; ++seg) {
        const int blk = block_of(seg);
        const int64_t lo = seg_lo[seg], hi = seg_hi[seg];
        for (int64_t t0 = lo; t0 < hi; t0 += TS) {
          sm100::mbar_wait(&S->full[r.i], r.ph);
          // the epilogue drained the previous tile, so its MMAs (the last readers
          // of the B slabs) have completed
          sm100::mbar_wait(&S->acc_empty, acc_ph ^ 1u);
          if (blk != cur) {
            sm100::mbar_expect_tx(&S->b_full, B_BYTES);
            sm100::bulk_g2s(S->b, qdig + static_cast<int64_t>(blk) * B_BYTES, B_BYTES, &S->b_full);
            sm100::mbar_wait(&S->b_full, b_ph);
            b_ph ^= 1u;
            cur = blk;
          }
          sm100::tc_fence_after();
          const uint32_t ab = sm100::smem_u32(S->a[r.i]);
#pragma unroll
          for (int kk = 0; kk < 2; ++kk) {
            const uint32_t ko = kk * 32;
            // (a, parity pi, N, TMEM column): levels a + pi + 2i of one parity
            // y digit a at slab a/2, K offset 64 (a % 2); Q parity pi at K offset 64 pi
#define RI8_MMA(A_, PI_, N_, COL_, ACC_)                                                    \
  umma_i8(tmem + (COL_), sm100::desc_sw128(ab + ((A_) >> 1) * A_SLAB + ((A_)&1) * 64 + ko), \
          sm100::desc_sw128(bb + (PI_)*64 + ko), idesc_i8(128, (N_)), (ACC_))
            RI8_MMA(0, 0, 256, 0, kk);     // levels 0 2 4 6 (initialises 0-255)
            RI8_MMA(0, 1, 256, 256, kk);   // levels 1 3 5 7 (initialises 256-511)
            RI8_MMA(1, 0, 256, 256, 1u);   // 1 3 5 7
            RI8_MMA(1, 1, 192, 64, 1u);    // 2 4 6
            RI8_MMA(2, 0, 192, 64, 1u);    // 2 4 6
            RI8_MMA(2, 1, 192, 320, 1u);   // 3 5 7
            RI8_MMA(3, 0, 192, 320, 1u);   // 3 5 7
            RI8_MMA(3, 1, 128, 128, 1u);   // 4 6
            RI8_MMA(4, 0, 128, 128, 1u);   // 4 6
            RI8_MMA(4, 1, 128, 384, 1u);   // 5 7
#undef RI8_MMA
          }
          sm100::umma_commit(&S->empty[r.i]);
          sm100::umma_commit(&S->acc_full);
          r.next();
          acc_ph ^= 1u;
        }
      }
    }
  } else {  // ------------------------------------------------------------ epilogue
    const int q4 = warp & 3, part = warp >> 2;
    const int row = 32 * q4 + lane;
    const uint32_t lane_base = tmem + (static_cast<uint32_t>(32 * q4) << 16);
    const int a0 = AQ * part;  // this thread's atoms [a0, a0 + AQ)
    int xb = 0;  // exchange buffer parity
    uint32_t acc_ph = 0;
    // every exchange is between the NQ warps that hold the same 32 rows (warps
    // q4, q4 + 4, ...): a named barrier per row group (ids 1-4 sync, 5-8 vote),
    // so row groups never wait for each other
    constexpr int GROUP = 32 * NQ;
    const int bar_id = 1 + q4, vote_id = 5 + q4;
    auto bar = [&]() { asm volatile("bar.sync %0, %1;" ::"r"(bar_id), "r"(GROUP) : "memory"); };
    auto any_of = [&](bool pr) {
      int r;
      asm volatile(
          "{\n\t.reg .pred p, q;\n\tsetp.ne.s32 p, %1, 0;\n\t"
          "bar.red.or.pred q, %2, %3, p;\n\tselp.s32 %0, 1, 0, q;\n\t}"
          : "=r"(r)
          : "r"(static_cast<int>(pr)), "r"(vote_id), "r"(GROUP)
          : "memory");
      return r != 0;
    };
    // the row's per-part values (a barrier: called by every epilogue thread);
    // returns the total and, in `before`, the sum over the parts below this one
    auto gather = [&](int mine, int& before) {
      S->cnt[xb][part][row] = mine;
      bar();
      int tot = 0;
      before = 0;
#pragma unroll
      for (int q = 0; q < NQ; ++q) {
        const int x = S->cnt[xb][q][row];
        tot += x;
        before += q < part ? x : 0;
      }
      xb ^= 1;
      return tot;
    };
    for (int seg = sa; seg < sb; ++seg) {
      const int64_t lo = seg_lo[seg], hi = seg_hi[seg];
      for (int64_t t0 = lo; t0 < hi; t0 += TS) {
        const bool act = t0 + row < hi;
        // the signal id (resid mode) is loaded before the wait
        int64_t sig = 0;
        if (MODE == MODE_RESID && act) sig = order ? static_cast<int64_t>(order[t0 + row]) : t0 + row;
        sm100::mbar_wait(&S->acc_full, acc_ph);
        acc_ph ^= 1u;
        sm100::tc_fence_after();
        double c[AQ];
        // selection key of atom a0 + i: the high word of |c| (an inactive row's
        // keys are garbage: its outputs are never written)
        auto key = [&](int i) { return __double2hiint(c[i]) & 0x7FFFFFFF; };
#pragma unroll
        for (int q = 0; q < AQ / 8; ++q) {
          uint32_t v[8][8];  // [level][atom]: 8 atoms per TMEM round trip
#pragma unroll
          for (int L = 0; L < 8; ++L) {
            const uint32_t col = (L & 1 ? 256u + 64u * (L >> 1) : 64u * (L >> 1)) + a0 + 8 * q;
            asm volatile(
                "tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                : "=r"(v[L][0]), "=r"(v[L][1]), "=r"(v[L][2]), "=r"(v[L][3]), "=r"(v[L][4]),
                  "=r"(v[L][5]), "=r"(v[L][6]), "=r"(v[L][7])
                : "r"(lane_base + col));
          }
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            // pairs of levels in int32 (|D_L 128 + D_L+1| < 2^29), HI / LO in int64, exact doubles
            const int e0 = static_cast<int>(v[0][u]) * 128 + static_cast<int>(v[1][u]);
            const int e1 = static_cast<int>(v[2][u]) * 128 + static_cast<int>(v[3][u]);
            const int e2 = static_cast<int>(v[4][u]) * 128 + static_cast<int>(v[5][u]);
            const int e3 = static_cast<int>(v[6][u]) * 128 + static_cast<int>(v[7][u]);
            const double hi_ = l2d(static_cast<long long>(e0) * 16384 + e1);
            const double lo_ = l2d(static_cast<long long>(e2) * 16384 + e3);
            c[8 * q + u] = fma(hi_, 268435456.0, lo_) * cscale;
          }
        }
        sm100::tc_fence_before();
        __syncwarp();
        if (lane == 0) sm100::mbar_arrive(&S->acc_empty);  // TMEM free for the next tile

        // ---- selection (select_top, onb.py:58-76): the k-th largest key over
        // the row's parts; exactly k keys at or above it -> the kept set.
        // kk-th largest of the row's 64 keys (kk <= G): per-part top-G lists
        // merged through shared memory
        auto kth = [&](auto keyf, int kk) {
          int v[AQ >= G ? AQ : G];
#pragma unroll
          for (int i = 0; i < AQ; ++i) v[i] = keyf(i);
#pragma unroll
          for (int i = AQ; i < G; ++i) v[i] = static_cast<int>(0x80000000u);
          constexpr int W = AQ >= G ? G : AQ;  // sorted run length
          if constexpr (AQ >= G) {
#pragma unroll
            for (int g = 0; g < AQ; g += G) topk::sort_desc<G>(v + g);
#pragma unroll
            for (int step = G; step < AQ; step <<= 1) {
#pragma unroll
              for (int g = 0; g + step < AQ; g += 2 * step) topk::merge_top<G>(v + g, v + g + step);
            }
          } else {
            topk::sort_desc<W>(v);  // the whole part (padding stays at the end)
          }
#pragma unroll
          for (int i = 0; i < G; ++i) S->lists[part][i][row] = v[i];
          bar();
#pragma unroll
          for (int q = 1; q < NQ; ++q) {
            const int o = (part + q) % NQ;
#pragma unroll
            for (int i = 0; i < G; ++i) v[i] = topk::vmax(v[i], S->lists[o][G - 1 - i][row]);
            topk::merge_desc<G>(v);
          }
          int t = v[0];
#pragma unroll
          for (int i = 1; i < G; ++i) t = sel_i(i == kk - 1, v[i], t);
          return t;
        };
        const int t1 = kth(key, k);
        uint32_t mask = 0u;
#pragma unroll
        for (int i = 0; i < AQ; ++i)
          if (key(i) >= t1) mask |= 1u << i;
        int before;
        const int kept_all = gather(__popc(mask), before);  // (unconditional: a barrier)
        const bool need = act && kept_all != k;
        if (any_of(need)) {
          // a key tie at the threshold (a 2^-20 relative gap): the tied atoms
          // are ordered by the low word of |c| (the full float64 magnitude),
          // then, for equal magnitudes, by atom (stable argsort: lower first).
          // Every gather is a barrier: called unconditionally by all threads.
          uint32_t gt1 = 0u, tie = 0u;
#pragma unroll
          for (int i = 0; i < AQ; ++i) {
            gt1 |= (key(i) > t1 ? 1u : 0u) << i;
            tie |= (key(i) == t1 ? 1u : 0u) << i;
          }
          int dummy;
          const int gt1_all = gather(__popc(gt1), dummy);
          const int r = need ? k - gt1_all : 1;
          auto key2 = [&](int i) {
            return need && ((tie >> i) & 1u)
                       ? (__double2loint(c[i]) ^ static_cast<int>(0x80000000u))
                       : static_cast<int>(0x80000000u);
          };
          const int t2 = kth(key2, r);
          uint32_t ge2 = 0u, gt2 = 0u;
#pragma unroll
          for (int i = 0; i < AQ; ++i) {
            ge2 |= (((tie >> i) & 1u) && key2(i) >= t2 ? 1u : 0u) << i;
            gt2 |= (((tie >> i) & 1u) && key2(i) > t2 ? 1u : 0u) << i;
          }
          const int ge2_all = gather(__popc(ge2), dummy);
          const bool need3 = need && ge2_all != r;
          uint32_t take = ge2;
          if (any_of(need3)) {
            // equal float64 magnitudes at the threshold: the lowest atoms first
            const int nd = r - gather(__popc(gt2), dummy);
            const uint32_t eq = ge2 & ~gt2;
            int eq_before;
            gather(__popc(eq), eq_before);
            int mine = min(max(nd - eq_before, 0), __popc(eq));
            if (need3) {
              take = gt2;
              uint32_t e = eq;
              while (mine-- > 0 && e) {
                take |= e & (0u - e);
                e &= e - 1u;
              }
            }
          }
          if (need) mask = gt1 | take;
          int b2;
          gather(__popc(mask), b2);
          if (need) before = b2;
        }
        // ---- outputs
        if constexpr (MODE == MODE_CODE) {
          // the kept pairs in ascending atom order, staged per (slot, row) in
          // shared memory, then written as coalesced rows of the code matrices
          if (act) {
            int at = before;
#pragma unroll
            for (int i = 0; i < AQ; ++i) {
              if ((mask >> i) & 1u) {
                S->oidx[at][row] = static_cast<int16_t>(a0 + i);
                S->oval[at][row] = c[i];
                ++at;
              }
            }
          }
          bar();
          const int n = static_cast<int>(min64(TS, hi - t0));
          // this row group's 32 rows, slot by slot (32 consecutive columns)
          for (int e = 32 * part + lane; e < k * 32; e += GROUP) {
            const int at = e >> 5, rr = 32 * q4 + (e & 31);
            if (rr < n) {
              cidx[at * ld + t0 + rr] = S->oidx[at][rr];
              cval[at * ld + t0 + rr] = S->oval[at][rr];
            }
          }
        } else {
          // discarded energy (no kept-sum cancellation) and the kept score,
          // summed over the parts in a fixed order
          double rest = 0.0, sc = 0.0;
#pragma unroll
          for (int i = 0; i < AQ; ++i) {
            const double x = c[i];
            if ((mask >> i) & 1u) sc = kind == SBO_KIND_SQUARED_SUM ? fma(x, x, sc) : sc + fabs(x);
            else rest = fma(x, x, rest);
          }
          S->part[part][0][row] = rest;
          S->part[part][1][row] = sc;
          bar();
          if (part == 0 && act) {
            double rs = 0.0, ss = 0.0;
#pragma unroll
            for (int q = 0; q < NQ; ++q) {
              rs += S->part[q][0][row];
              ss += S->part[q][1][row];
            }
            rest_sq[sig] = rs;
            if (score) score[sig] = ss;
          }
          bar();
        }
      }
    }
  }
  __syncthreads();
  if (warp == MMA_WARP) sm100::tmem_dealloc(tmem, 512);
}

// The block's digit image for k_round_i8: 4 SW128 slabs [Q_2s | Q_2s+1] of 64
// atom rows x 128 B; Q_int = rint(q 2^54) in 8 balanced 7-bit digits.  One
// thread per (block, atom, dim).
__global__ void k_q_digits(const double* __restrict__ blocks, int b0, int nb,
                           int8_t* __restrict__ qdig) {
  const int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x;
  if (e >= static_cast<int64_t>(nb) * P * P) return;
  const int b = b0 + static_cast<int>(e / (P * P));
  const int rem = static_cast<int>(e % (P * P));
  const int dim = rem >> 6, atom = rem & 63;  // q[dim][atom]: atom = column (numpy layout)
  long long v = __double2ll_rn(blocks[static_cast<int64_t>(b) * P * P + rem] * 18014398509481984.0);
  int8_t* out = qdig + static_cast<int64_t>(b) * B_BYTES;
#pragma unroll
  for (int d = 7; d >= 0; --d) {
    const int dd = ((static_cast<int>(v) + 64) & 127) - 64;
    v = (v - dd) >> 7;
    out[(d >> 1) * B_SLAB + slab_off(atom, (d & 1) * 64 + dim)] = static_cast<int8_t>(dd);
  }
}

}  // namespace ri8
}  // namespace sbo

using namespace sbo;

#ifndef RI8_NQ
#define RI8_NQ 2  // epilogue atom parts of the code mode for s0 <= 16
#endif
#ifndef RI8_NQ_RESID
#define RI8_NQ_RESID 4  // epilogue atom parts of the residual mode for s0 <= 16
#endif

extern "C" size_t sbo_round_i8_workspace_bytes(int nblocks) {
  return static_cast<size_t>(nblocks > 0 ? nblocks : 0) * ri8::B_BYTES;
}

template <int G, int MODE, int NQ>
static int launch_ri8(unsigned grid, cudaStream_t st, const int8_t* ydig, const int32_t* order,
                      const int32_t* seg_block, const int64_t* seg_lo, const int64_t* seg_hi,
                      const int32_t* nseg, const int8_t* qdig, int ov, int k, int kind,
                      double cscale, int64_t ld, int16_t* idx, double* val, double* rest_sq,
                      double* score) {
  static bool attr = false;
  constexpr size_t smem = ri8::smem_bytes<NQ, G>();
  static_assert(smem <= 232448, "shared memory over the 227-KB limit");
  if (!attr) {
    SBO_CHECK_CUDA(cudaFuncSetAttribute(ri8::k_round_i8<G, MODE, NQ>,
                                        cudaFuncAttributeMaxDynamicSharedMemorySize,
                                        static_cast<int>(smem)));
    attr = true;
  }
  ri8::k_round_i8<G, MODE, NQ><<<grid, ri8::Roles<NQ>::THREADS, smem, st>>>(
      ydig, order, seg_block, seg_lo, seg_hi, nseg, qdig, ov, k, kind, cscale, ld, idx, val,
      rest_sq, score);
  return check_launch(MODE == ri8::MODE_CODE ? "k_round_i8<code>" : "k_round_i8<resid>");
}

extern "C" int sbo_round_i8_segments(const void* ydig, int sy, const int32_t* order,
                                     const int32_t* seg_block, const int64_t* seg_lo,
                                     const int64_t* seg_hi, const int32_t* nseg,
                                     int64_t max_seg, const double* blocks, int nblocks,
                                     int block_override, int s0, int mode, int kind, int64_t ld,
                                     int16_t* idx, double* val, double* rest_sq, double* score,
                                     void* workspace, size_t ws_bytes, void* stream) {
  if (!ydig || !blocks || nblocks < 1) return fail(SBO_EINVAL, "bad arguments");
  if (s0 < 1 || s0 > 32) return fail(SBO_EINVAL, "the integer-digit round needs 1 <= s0 <= 32");
  if (block_override >= nblocks) return fail(SBO_EINVAL, "block_override out of range");
  if (mode == ri8::MODE_CODE && (!idx || !val)) return fail(SBO_EINVAL, "idx and val are required");
  if (mode == ri8::MODE_RESID && !rest_sq) return fail(SBO_EINVAL, "rest_sq is required");
  if (mode != ri8::MODE_CODE && mode != ri8::MODE_RESID) return fail(SBO_EINVAL, "bad mode");
  if (kind != SBO_KIND_SQUARED_SUM && kind != SBO_KIND_ABS_SUM) return fail(SBO_EINVAL, "bad kind");
  if (!workspace || ws_bytes < sbo_round_i8_workspace_bytes(nblocks))
    return fail(SBO_EINVAL, "round_i8 workspace too small");
  if (max_seg <= 0) return SBO_OK;
  cudaStream_t st = as_stream(stream);
  auto* qdig = static_cast<int8_t*>(workspace);
  const int b0 = block_override >= 0 ? block_override : 0;
  const int nb = block_override >= 0 ? 1 : nblocks;
  const int64_t ne = static_cast<int64_t>(nb) * 64 * 64;
  ri8::k_q_digits<<<static_cast<unsigned>(ceil_div(ne, 256)), 256, 0, st>>>(blocks, b0, nb, qdig);
  if (int rc = check_launch("k_q_digits")) return rc;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const unsigned grid = static_cast<unsigned>(min64(max_seg, sms));
  const double cscale = ldexp(1.0, -sy - 26);
  const auto* yd = static_cast<const int8_t*>(ydig);
// code mode: 2 atom parts (8 epilogue warps); residual mode (no staged code
// outputs): 4 parts (16 epilogue warps) for s0 <= 16 — measured per mode
// (A/B per iteration: code 29.2 vs 37.0 ms of retrain with 2 vs 4 parts,
// residual 20.4 vs 21.6 ms of represent #2 with 4 vs 2)
#define RI8_GO(G_, NQC_, NQR_)                                                                \
  return mode == ri8::MODE_CODE                                                                \
             ? launch_ri8<G_, ri8::MODE_CODE, NQC_>(grid, st, yd, order, seg_block, seg_lo,    \
                                                    seg_hi, nseg, qdig, block_override, s0,    \
                                                    kind, cscale, ld, idx, val, rest_sq,       \
                                                    score)                                     \
             : launch_ri8<G_, ri8::MODE_RESID, NQR_>(grid, st, yd, order, seg_block, seg_lo,   \
                                                     seg_hi, nseg, qdig, block_override, s0,   \
                                                     kind, cscale, ld, idx, val, rest_sq,      \
                                                     score)
  if (s0 <= 8) RI8_GO(8, RI8_NQ, RI8_NQ_RESID);
  if (s0 <= 16) RI8_GO(16, RI8_NQ, RI8_NQ_RESID);
  RI8_GO(32, 2, 2);
#undef RI8_GO
}
