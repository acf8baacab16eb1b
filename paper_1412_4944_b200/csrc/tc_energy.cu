// Tensor-core representation energy pass for p = 64 (sbo.py:177-194 on tcgen05).
//
// C = Y_tile . [Q_b0 .. Q_b1) is computed on the 5th-gen tensor cores with a
// split-fp16 scheme: every signal and every block is scaled by a power of two
// into [16, 32), split into fp16 hi + lo (22 significant bits), and the three
// products lo.hi + hi.lo + hi.hi are accumulated in fp32 TMEM — the accuracy
// of 3xTF32 at the fp16 rate.  Signals sit on M (TMEM lane = signal), so each
// epilogue thread owns one signal's 64 coefficients per block: squares, a
// bitonic top-k network (topk.cuh), the block's kept energy E and discarded
// energy R = S - E, and the running best / second-best block.  The argmax is
// certified with an error bound; near-ties are appended to a list that the
// float64 kernel re-decides exactly (tiles_f64.cu), so decisions equal the
// float64 reference's.
//
// Warp roles (persistent CTA per SM, 384 threads):
//   warp 0      bulk-async producer: A tiles (128 signals x 64 fp16, hi+lo) and
//               B chunks (4 blocks = 256 atoms x 64 fp16, hi+lo), 2 stages each
//   warp 1      single-thread UMMA issuer, 128x256x16, 2 TMEM accumulator stages
//   warps 4-11  epilogue; warps w and w+4 share TMEM lane quarter w%4 and take
//               blocks {0,1} / {2,3} of each 4-block chunk
// Global operands are stored pre-swizzled (128-B rows, 16-B chunk ^ row%8), so
// a plain cp.async.bulk lands them MMA-ready in shared memory.
#include "common.cuh"
#include "sm100.cuh"
#include "topk.cuh"

namespace sbo {
namespace tc {

constexpr int P = 64;
constexpr int M = 128;
constexpr int CHUNK = 4;           // blocks per accumulator stage
constexpr int EPI_WARPS = 8;
constexpr int THREADS = 128 + 32 * EPI_WARPS;
constexpr uint32_t A_BYTES = M * P * 2;          // one fp16 tile: 16 KB
constexpr uint32_t B_BLOCK_BYTES = P * P * 2;    // one block in fp16: 8 KB

struct Smem {
  __half a[2][2][M * P];            // [stage][hi, lo]
  __half b[2][2][CHUNK * P * P];    // [stage][hi, lo]
  uint64_t a_full[2], a_empty[2], b_full[2], b_empty[2], acc_full[2], acc_empty[2];
  uint32_t tmem;
  float x_r1[M], x_r2[M], x_s[M], x_rb[M], x_eb[M];
  int x_b1[M];
  // decision value per (block - b0, signal) for the candidate masks: fp32 up to
  // 32 blocks, fp16 up to 64 (compared with a 2^-10 relative margin, so the masks
  // stay supersets; wider than the fp32 ones, hence only above 32 blocks)
  union {
    float f[32][M];
    __half h[64][M];
  } x_dec;
};
constexpr size_t SMEM_BYTES = sizeof(Smem) + 1024;

__device__ __forceinline__ Smem* smem_of(unsigned char* raw) {
  const uint32_t a = sm100::smem_u32(raw);
  return reinterpret_cast<Smem*>(raw + ((1024u - (a & 1023u)) & 1023u));
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

// error bound of one coefficient (absolute, unscaled units), DESIGN.md section 3.  The
// measured kind::f16 MMA aligns its 17 addends (16 exact products + the accumulator) to the
// largest nominal exponent, truncates each toward zero 25 bits below it, and truncates the
// sum toward zero to fp32 (tools/f16acc_micro.cu, tools/f16acc_fit2.py: every result of
// 23,040 random dot products reproduced).  Per MMA the error is < (17 2^-25 + 2^-23) T with
// T = sum |y_k q_k| <= ||y||.  The 8 cross-term MMAs run first, at 2^-10 of the scale, and the
// 4 hi.hi MMAs give 4 (17 2^-25 + 2^-23) = 2.50e-6; the split adds 3 2^-22 = 0.72e-6.
// That totals 3.23e-6 ||y||.
__device__ __forceinline__ float coef_err(float s_norm) { return 3.3e-6f * sqrtf(s_norm); }

// bound on |R_hat - R| for a block with n discarded coefficients: coefficient
// errors (Cauchy-Schwarz over the discarded set, which may differ from the exact
// one only among near-equal magnitudes) plus the fp32 sum of <= 64 small terms
__device__ __forceinline__ float resid_err(float r, float s, float d, int n) {
  (void)s;
  return 2.0f * d * sqrtf(static_cast<float>(n) * fmaxf(r, 0.0f)) + n * d * d + 8e-6f * fmaxf(r, 0.0f);
}

// candidate mask of a signal flagged by an incremental pass over [b0, b1)
// (b1 <= 64): its incoming winner and every appended block
__device__ __forceinline__ uint64_t accum_cand(int prev, int b0, int b1) {
  const uint64_t app = (b1 - b0 >= 64 ? ~0ull : ((1ull << (b1 - b0)) - 1ull)) << b0;
  return (prev >= 0 && prev < 64 ? 1ull << prev : 0ull) | app;
}

template <int G, bool ABS>
__global__ void __launch_bounds__(THREADS, 1)
k_energy_tc(const __half* __restrict__ yh, const __half* __restrict__ yl,
            const int16_t* __restrict__ escale, int64_t m, const __half* __restrict__ qh,
            const __half* __restrict__ ql, const int16_t* __restrict__ fscale, int b0, int b1,
            int ksel, int accumulate, int32_t* best, double* score, double* residual,
            int32_t* flags, int32_t* nflag, uint64_t* cand) {
  extern __shared__ unsigned char raw[];
  Smem* S = smem_of(raw);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t ntiles = ceil_div(m, M);
  const int nblk = b1 - b0;
  const int nchunks = (nblk + CHUNK - 1) / CHUNK;

  if (threadIdx.x == 0) {
    for (int s = 0; s < 2; ++s) {
      sm100::mbar_init(&S->a_full[s], 1);
      sm100::mbar_init(&S->a_empty[s], 1);
      sm100::mbar_init(&S->b_full[s], 1);
      sm100::mbar_init(&S->b_empty[s], 1);
      sm100::mbar_init(&S->acc_full[s], 1);
      // one block: each epilogue group takes alternate tiles (and one stage)
      sm100::mbar_init(&S->acc_empty[s], nblk == 1 ? EPI_WARPS / 2 : EPI_WARPS);
    }
    sm100::fence_barrier_init();
  }
  if (warp == 2) sm100::tmem_alloc(&S->tmem, 512);
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem = S->tmem;

  if (warp == 0) {
    if (lane == 0) {  // ---------------------------------------------- producer
      Ring ra, rb;
      for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        sm100::mbar_wait(&S->a_empty[ra.i], ra.ph ^ 1u);
        sm100::mbar_expect_tx(&S->a_full[ra.i], 2 * A_BYTES);
        sm100::bulk_g2s(S->a[ra.i][0], yh + t * M * P, A_BYTES, &S->a_full[ra.i]);
        sm100::bulk_g2s(S->a[ra.i][1], yl + t * M * P, A_BYTES, &S->a_full[ra.i]);
        ra.next();
        for (int c = 0; c < nchunks; ++c) {
          const int nb = min(CHUNK, nblk - c * CHUNK);
          const uint32_t bytes = nb * B_BLOCK_BYTES;
          const int64_t off = static_cast<int64_t>(b0 + c * CHUNK) * P * P;
          sm100::mbar_wait(&S->b_empty[rb.i], rb.ph ^ 1u);
          sm100::mbar_expect_tx(&S->b_full[rb.i], 2 * bytes);
          sm100::bulk_g2s(S->b[rb.i][0], qh + off, bytes, &S->b_full[rb.i]);
          sm100::bulk_g2s(S->b[rb.i][1], ql + off, bytes, &S->b_full[rb.i]);
          rb.next();
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ------------------------------------------- MMA issuer
      Ring ra, rb, racc;
      for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        sm100::mbar_wait(&S->a_full[ra.i], ra.ph);
        sm100::tc_fence_after();
        const uint32_t a_hi = sm100::smem_u32(S->a[ra.i][0]);
        const uint32_t a_lo = sm100::smem_u32(S->a[ra.i][1]);
        for (int c = 0; c < nchunks; ++c) {
          const int nb = min(CHUNK, nblk - c * CHUNK);
          sm100::mbar_wait(&S->b_full[rb.i], rb.ph);
          sm100::mbar_wait(&S->acc_empty[racc.i], racc.ph ^ 1u);
          sm100::tc_fence_after();
          const uint32_t b_hi = sm100::smem_u32(S->b[rb.i][0]);
          const uint32_t b_lo = sm100::smem_u32(S->b[rb.i][1]);
          const uint32_t d = tmem + racc.i * 256;
          const uint32_t idesc = sm100::idesc_f16(M, nb * P);
          // the small cross terms first, then hi.hi: each MMA truncates its addends to
          // 2^-25 of the largest one (measured), so only the 4 hi.hi
          // MMAs lose bits at the scale of the coefficient (coef_err)
#pragma unroll
          for (int kk = 0; kk < P / 16; ++kk) {
            const uint32_t ko = kk * 32;  // 16 fp16 along K inside the 128-B swizzle atom
            sm100::umma_f16(d, sm100::desc_sw128(a_lo + ko), sm100::desc_sw128(b_hi + ko), idesc,
                            kk > 0);
            sm100::umma_f16(d, sm100::desc_sw128(a_hi + ko), sm100::desc_sw128(b_lo + ko), idesc, 1);
          }
#pragma unroll
          for (int kk = 0; kk < P / 16; ++kk) {
            const uint32_t ko = kk * 32;
            sm100::umma_f16(d, sm100::desc_sw128(a_hi + ko), sm100::desc_sw128(b_hi + ko), idesc, 1);
          }
          sm100::umma_commit(&S->b_empty[rb.i]);
          sm100::umma_commit(&S->acc_full[racc.i]);
          rb.next();
          racc.next();
        }
        sm100::umma_commit(&S->a_empty[ra.i]);
        ra.next();
      }
    }
  } else if (warp >= 4) {  // ------------------------------------------ epilogue
    // Decision value dec (minimized): R = S - kept for squared-sum (argmax E ==
    // argmin R by Parseval), -E for abs-sum.  Ties keep the lower block.
    const int ew = warp - 4, grp = ew >> 2, q = warp & 3;
    const int row = 32 * q + lane;
    const uint32_t lane_base = tmem + (static_cast<uint32_t>(32 * q) << 16);
    Ring racc;
    // per-signal inputs of the NEXT tile are loaded while this tile computes
    // (their global-memory latency would otherwise sit on every tile's path)
    // (raw values: converting here would wait for the load)
    auto preload = [&](int64_t tt, int& es_, double& prev_) {
      const int64_t jj = tt * M + row;
      es_ = 0;
      prev_ = ABS ? -INFINITY : INFINITY;
      if (tt < ntiles && jj < m) {
        es_ = escale[jj];
        if (accumulate) prev_ = ABS ? __ldcg(score + jj) : __ldcg(residual + jj);
      }
    };
    // one block's decision inputs from its 64 TMEM columns: the signal norm sq,
    // discarded energy r, kept energy e and decision value dec (unscaled)
    auto eval_block = [&](uint32_t taddr, int b, int es, float& sq, float& r, float& e,
                      float& dec) {
      float v[64];
      sm100::tmem_ld64(taddr, v);
      float t8[8];
#pragma unroll
      for (int a = 0; a < 8; ++a) {
        float acc = 0.0f;
#pragma unroll
        for (int i = 0; i < 8; ++i) acc = fmaf(v[8 * a + i], v[8 * a + i], acc);
        t8[a] = acc;
      }
      sq = ((t8[0] + t8[1]) + (t8[2] + t8[3])) + ((t8[4] + t8[5]) + (t8[6] + t8[7]));
#pragma unroll
      for (int i = 0; i < 64; ++i) v[i] = ABS ? fabsf(v[i]) : v[i] * v[i];
      // squared-sum: the discarded energy R is summed from the values the
      // network drops (+ the tail of the top-G list beyond k): no S - kept cancellation
      float dropped = 0.0f;
      if constexpr (ABS) topk::top_of_64<G>(v);
      else if (ksel == G) dropped = topk::top_of_64_dropped<G, false>(v);  // order unused
      else dropped = topk::top_of_64_dropped<G>(v);
      float kept = 0.0f;
      e = 0.0f;
#pragma unroll
      for (int i = 0; i < G; ++i) {
        if (i < ksel) {
          kept += ABS ? v[i] * v[i] : v[i];
          e += v[i];
        } else if (!ABS) {
          dropped += v[i];
        }
      }
      // unscale by 2^-(e_s + f_b), exact
      const float u = exp2f(static_cast<float>(-(es + fscale[b])));
      const float u2 = u * u;
      sq *= u2;
      kept *= u2;
      e *= ABS ? u : u2;
      r = ABS ? sq - kept : dropped * u2;
      dec = ABS ? -e : r;
    };
    if (nblk == 1) {
      // a single block (represent #1's appended block): the two groups take
      // alternate tiles — accumulator stage g holds this group's tiles — so no
      // epilogue warp idles and no cross-group combine is needed
      int es_next;
      double prev_next;
      const int64_t tstep = 2 * static_cast<int64_t>(gridDim.x);
      preload(blockIdx.x + grp * gridDim.x, es_next, prev_next);
      uint32_t phg = 0;
      for (int64_t t = blockIdx.x + grp * gridDim.x; t < ntiles; t += tstep) {
        const int64_t j = t * M + row;
        const bool valid = j < m;
        const int es = es_next;
        const double prev_pre = prev_next;
        preload(t + tstep, es_next, prev_next);
        sm100::mbar_wait(&S->acc_full[grp], phg);
        phg ^= 1u;
        sm100::tc_fence_after();
        float sq, r, e, dec;
        eval_block(lane_base + grp * 256, b0, es, sq, r, e, dec);
        sm100::tc_fence_before();
        __syncwarp();
        if (lane == 0) sm100::mbar_arrive(&S->acc_empty[grp]);
        if (!valid) continue;
        const float dc = coef_err(sq);
        const int nd = P - ksel;
        auto err = [&](float dv) -> float {
          return ABS ? (ksel * dc + 1e-6f * fabsf(dv)) : resid_err(dv, sq, dc, nd);
        };
        if (accumulate) {
          const float prev = ABS ? -static_cast<float>(prev_pre) : static_cast<float>(prev_pre);
          const bool flag = fabsf(dec - prev) <= err(dec) + err(prev);
          // a flagged signal keeps its incoming exact winner / score: the float64
          // re-decision compares the new block against them (first maximum wins)
          if (dec < prev && !flag) {
            best[j] = b0;
            score[j] = ABS ? e : static_cast<double>(sq) - r;
            residual[j] = r;
          }
          if (flag) {
            const int ix = atomicAdd(nflag, 1);
            flags[ix] = static_cast<int32_t>(j);
            if (cand) cand[ix] = accum_cand(__ldcg(best + j), b0, b1);
          }
        } else {
          best[j] = b0;
          score[j] = ABS ? e : static_cast<double>(sq) - r;
          residual[j] = r;
        }
      }
    } else {
    int es_next;
    double prev_next;
    preload(blockIdx.x, es_next, prev_next);
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
      const int64_t j = t * M + row;
      const bool valid = j < m;
      const int es = es_next;
      const double prev_pre = prev_next;
      preload(t + gridDim.x, es_next, prev_next);
      float d1 = INFINITY, d2 = INFINITY, rb = 0.0f, eb = 0.0f, snorm = 0.0f;
      int bb = -1;
      // decision values are kept per block (shared memory) so that the flagged
      // signals' candidate masks can be formed against the final best
      for (int c = 0; c < nchunks; ++c) {
        const int nb = min(CHUNK, nblk - c * CHUNK);
        sm100::mbar_wait(&S->acc_full[racc.i], racc.ph);
        sm100::tc_fence_after();
#pragma unroll 1
        for (int h = 0; h < 2; ++h) {
          const int jb = 2 * grp + h;
          if (jb >= nb) break;
          const int b = b0 + c * CHUNK + jb;
          float sq, r, e, dec;
          eval_block(lane_base + racc.i * 256 + jb * 64, b, es, sq, r, e, dec);
          if (dec < d1) {
            d2 = d1;
            d1 = dec;
            bb = b;
            rb = r;
            eb = e;
          } else if (dec < d2) {
            d2 = dec;
          }
          snorm = sq;
          if (cand) {
            if (nblk <= 32) S->x_dec.f[b - b0][row] = dec;
            else if (b - b0 < 64) S->x_dec.h[b - b0][row] = __float2half_ru(dec);
          }
        }
        sm100::tc_fence_before();
        __syncwarp();
        if (lane == 0) sm100::mbar_arrive(&S->acc_empty[racc.i]);
        racc.next();
      }
      // combine the two epilogue groups (same signals, different blocks)
      if (grp == 1) {
        S->x_r1[row] = d1;
        S->x_r2[row] = d2;
        S->x_b1[row] = bb;
        S->x_s[row] = snorm;
        S->x_rb[row] = rb;
        S->x_eb[row] = eb;
      }
      asm volatile("bar.sync 1, %0;" ::"r"(32 * EPI_WARPS));
      if (grp == 0 && valid) {
        const int cb = S->x_b1[row];
        if (bb < 0) snorm = S->x_s[row];
        if (cb >= 0) {
          const float c1 = S->x_r1[row], c2 = S->x_r2[row];
          if (bb < 0 || c1 < d1 || (c1 == d1 && cb < bb)) {
            d2 = fminf(d1, c2);
            d1 = c1;
            bb = cb;
            rb = S->x_rb[row];
            eb = S->x_eb[row];
          } else {
            d2 = fminf(d2, c1);
          }
        }
        const float dc = coef_err(snorm);
        const int nd = P - ksel;
        auto err = [&](float dec) -> float {
          return ABS ? (ksel * dc + 1e-6f * fabsf(dec)) : resid_err(dec, snorm, dc, nd);
        };
        bool flag;
        if (accumulate) {  // incoming winner covers blocks < b0 and keeps ties
          const float prev = ABS ? -static_cast<float>(prev_pre) : static_cast<float>(prev_pre);
          flag = fabsf(d1 - prev) <= err(d1) + err(prev);
          // flagged: keep the incoming exact winner / score for the float64 re-decision
          if (d1 < prev && !flag) {
            best[j] = bb;
            score[j] = ABS ? eb : static_cast<double>(snorm) - rb;
            residual[j] = rb;
          }
        } else {
          flag = d2 != INFINITY && fabsf(d2 - d1) <= err(d1) + err(d2);
          best[j] = bb;
          score[j] = ABS ? eb : static_cast<double>(snorm) - rb;
          residual[j] = rb;
        }
        if (flag) {
          const int ix = atomicAdd(nflag, 1);
          flags[ix] = static_cast<int32_t>(j);
          if (cand && accumulate) {
            // incremental pass: the incoming winner and the appended blocks, all
            // re-evaluated by the same float64 kernel (exact ties -> lower block)
            cand[ix] = accum_cand(__ldcg(best + j), b0, b1);
          } else if (cand) {
            // candidate blocks: within the certificate's tolerance of the final best
            // (1 % slack on the bound; the fp16 decision values were rounded up,
            // and 2^-10 of |dv| more covers a downward rounding of dv)
            uint64_t cmask = 0ull;
            const float lim = d1 + 1.01f * err(d1);
            if (nblk <= 32) {
              for (int jb = 0; jb < nblk; ++jb) {
                const float dv = S->x_dec.f[jb][row];
                if (dv <= lim + 1.01f * err(dv)) cmask |= 1ull << jb;
              }
            } else {
              for (int jb = 0; jb < nblk; ++jb) {
                const float h = __half2float(S->x_dec.h[jb][row]);
                // fp16 spacing: 2^-10 relative, 2^-24 absolute near zero; an
                // out-of-range value (inf) is always a candidate
                const float slack = fabsf(h) * 9.765625e-4f + 6.0e-8f;
                if (!isfinite(h) || h - slack <= lim + 1.01f * err(h) + slack) cmask |= 1ull << jb;
              }
            }
            cand[ix] = cmask;
          }
        }
      }
      asm volatile("bar.sync 1, %0;" ::"r"(32 * EPI_WARPS));
    }
    }  // nblk > 1
  }
  __syncthreads();
  if (warp == 2) sm100::tmem_dealloc(tmem, 512);
}

// ---------------------------------------------------------------------------
// operand preparation: scale to [16, 32) by a power of two, split into fp16
// hi + lo, store 128-B rows pre-swizzled.
template <typename TY>
__global__ void k_split_signals(const TY* __restrict__ y, int64_t m, int64_t m_pad, __half* yh,
                                __half* yl, int16_t* escale) {
  // one warp per signal row (64 values, 2 per lane)
  const int64_t j = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (j >= m_pad) return;
  double a = 0.0, b = 0.0;
  if (j < m) {
    a = static_cast<double>(y[j * P + 2 * lane]);
    b = static_cast<double>(y[j * P + 2 * lane + 1]);
  }
  double mx = fmax(fabs(a), fabs(b));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  int e = 0;
  if (mx > 0.0) {
    int ex;
    frexp(mx, &ex);  // mx = f * 2^ex, f in [0.5, 1)
    e = 5 - ex;      // mx * 2^e in [16, 32)
    e = max(-120, min(120, e));
  }
  const double sa = ldexp(a, e), sb = ldexp(b, e);
  const __half ha = __double2half(sa), hb = __double2half(sb);
  const __half la = __double2half(sa - static_cast<double>(__half2float(ha)));
  const __half lb = __double2half(sb - static_cast<double>(__half2float(hb)));
  const uint32_t off = sm100::sw128_offset(static_cast<uint32_t>(j & 7), lane * 4);
  unsigned char* rh = reinterpret_cast<unsigned char*>(yh) + (j >> 3) * 1024;
  unsigned char* rl = reinterpret_cast<unsigned char*>(yl) + (j >> 3) * 1024;
  *reinterpret_cast<__half2*>(rh + off) = __halves2half2(ha, hb);
  *reinterpret_cast<__half2*>(rl + off) = __halves2half2(la, lb);
  if (lane == 0) escale[j] = static_cast<int16_t>(e);
}

// blocks Q_b (row-major [k][i], float64) -> atom rows [b][i][k] split/scaled
__global__ void k_split_blocks(const double* __restrict__ Q, int K, __half* qh, __half* ql,
                               int16_t* fscale) {
  const int b = blockIdx.x;
  __shared__ double red[32];
  const double* q = Q + static_cast<int64_t>(b) * P * P;
  double mx = 0.0;
  for (int e = threadIdx.x; e < P * P; e += blockDim.x) mx = fmax(mx, fabs(q[e]));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  mx = 0.0;
  for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) mx = fmax(mx, red[w]);
  int f = 0;
  if (mx > 0.0) {
    int ex;
    frexp(mx, &ex);
    f = max(-120, min(120, 5 - ex));
  }
  for (int e = threadIdx.x; e < P * P; e += blockDim.x) {
    const int i = e / P, k = e % P;  // atom i, coordinate k
    const double s = ldexp(q[k * P + i], f);
    const __half h = __double2half(s);
    const __half l = __double2half(s - static_cast<double>(__half2float(h)));
    const uint32_t row = static_cast<uint32_t>(b * P + i);
    const uint32_t off = sm100::sw128_offset(row & 7u, k * 2);
    const int64_t base = static_cast<int64_t>(row >> 3) * 1024;
    *reinterpret_cast<__half*>(reinterpret_cast<unsigned char*>(qh) + base + off) = h;
    *reinterpret_cast<__half*>(reinterpret_cast<unsigned char*>(ql) + base + off) = l;
  }
  if (threadIdx.x == 0) fscale[b] = static_cast<int16_t>(f);
}

template <int G, bool ABS>
int launch_energy(const __half* yh, const __half* yl, const int16_t* es, int64_t m,
                  const __half* qh, const __half* ql, const int16_t* fs, int b0, int b1, int ksel,
                  int accumulate, int32_t* best, double* score, double* residual,
                  int32_t* flags, int32_t* nflag, uint64_t* cand, cudaStream_t st) {
  auto kern = k_energy_tc<G, ABS>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       static_cast<int>(SMEM_BYTES));
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t ntiles = ceil_div(m, M);
  const int grid = static_cast<int>(ntiles < sms ? ntiles : sms);
  kern<<<grid, THREADS, SMEM_BYTES, st>>>(yh, yl, es, m, qh, ql, fs, b0, b1, ksel, accumulate,
                                          best, score, residual, flags, nflag, cand);
  return check_launch("k_energy_tc");
}

}  // namespace tc
}  // namespace sbo

using namespace sbo;

extern "C" int64_t sbo_tc_padded_rows(int64_t m) { return ceil_div(m, tc::M) * tc::M; }

extern "C" int sbo_tc_split_signals(const void* y, int dtype, int64_t m, int p, void* yhv,
                                    void* ylv, int16_t* escale, void* stream) {
  __half* yh = static_cast<__half*>(yhv);
  __half* yl = static_cast<__half*>(ylv);
  if (p == 256)
    return tc256_split_signals(y, dtype, m, sbo_tc_padded_rows(m), yhv, ylv, escale,
                               as_stream(stream));
  if (p != tc::P) return fail(SBO_EINVAL, "the tensor-core path needs p = 64 or 256");
  const int64_t mp = sbo_tc_padded_rows(m);
  if (mp == 0) return SBO_OK;
  const unsigned grid = static_cast<unsigned>(ceil_div(mp * 32, 256));
  if (dtype == SBO_F32)
    tc::k_split_signals<float><<<grid, 256, 0, as_stream(stream)>>>(
        static_cast<const float*>(y), m, mp, yh, yl, escale);
  else
    tc::k_split_signals<double><<<grid, 256, 0, as_stream(stream)>>>(
        static_cast<const double*>(y), m, mp, yh, yl, escale);
  return check_launch("k_split_signals");
}

extern "C" int sbo_tc_split_blocks(const double* Q, int K, int p, void* qhv, void* qlv,
                                   int16_t* fscale, void* stream) {
  __half* qh = static_cast<__half*>(qhv);
  __half* ql = static_cast<__half*>(qlv);
  if (p == 256) return tc256_split_blocks(Q, K, qhv, qlv, fscale, as_stream(stream));
  if (p != tc::P) return fail(SBO_EINVAL, "the tensor-core path needs p = 64 or 256");
  if (K < 1) return SBO_OK;
  tc::k_split_blocks<<<K, 256, 0, as_stream(stream)>>>(Q, K, qh, ql, fscale);
  return check_launch("k_split_blocks");
}

extern "C" int sbo_tc_energy(const void* yhv, const void* ylv, const int16_t* escale,
                             int64_t m, const void* qhv, const void* qlv,
                             const int16_t* fscale, int b0, int b1, int s0, int kind,
                             int accumulate, int32_t* best, double* score, double* residual,
                             int32_t* flags, int32_t* nflag, uint64_t* cand, void* stream) {
  const __half* yh = static_cast<const __half*>(yhv);
  const __half* yl = static_cast<const __half*>(ylv);
  const __half* qh = static_cast<const __half*>(qhv);
  const __half* ql = static_cast<const __half*>(qlv);
  if (s0 < 1) return fail(SBO_EINVAL, "s0 must be at least 1");
  if (b0 < 0 || b1 <= b0 || (!accumulate && b0 != 0))
    return fail(SBO_EINVAL, "bad block range for the energy pass");
  if (cand && b1 > 64) return fail(SBO_EINVAL, "candidate masks cover at most 64 blocks");
  if (m == 0) return SBO_OK;
  const int k = s0 < tc::P ? s0 : tc::P;
  cudaStream_t st = as_stream(stream);
  const bool abs = kind == SBO_KIND_ABS_SUM;
#define SBO_TC_CASE(GG)                                                                       \
  if (k <= GG)                                                                                \
    return abs ? tc::launch_energy<GG, true>(yh, yl, escale, m, qh, ql, fscale, b0, b1, k,   \
                                             accumulate, best, score, residual, flags, nflag, \
                                             cand, st)                                        \
               : tc::launch_energy<GG, false>(yh, yl, escale, m, qh, ql, fscale, b0, b1, k,  \
                                              accumulate, best, score, residual, flags,       \
                                              nflag, cand, st);
  // k <= 8 shares the 8-wide network: the top-8 list holds the top-k (kept)
  // and the rest (dropped); the narrower networks need twice as many merges
  // (G = 4: 9.0 vs 3.8 ms for a 16-block pass at m = 2^22, profiles/r02e_*)
  SBO_TC_CASE(8)
  SBO_TC_CASE(16)
  SBO_TC_CASE(32)
  SBO_TC_CASE(64)
#undef SBO_TC_CASE
  return fail(SBO_EINVAL, "unsupported s0");
}
