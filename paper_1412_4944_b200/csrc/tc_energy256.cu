// Tensor-core representation energy pass for p = 256 (config D; sbo.py:177-194),
// the p = 64 design of tc_energy.cu at four times the depth:
//
// * Operands: signals and blocks scaled by a power of two into [16, 32) and split
//   into fp16 hi + lo; the three products lo.hi + hi.lo + hi.hi accumulate in fp32
//   TMEM.  The 256 coordinates are four 128-B swizzle atoms (K-blocks of 64); a
//   block's 256 atoms are two N-halves of 128.  Global layouts are pre-swizzled:
//   signals [tile][kb][128 rows][128 B], blocks [block][half][kb][128 atoms][128 B],
//   so every copy is one contiguous 16-KB cp.async.bulk.
// * Shared memory: the tile's whole signal rows (hi + lo, 128 KB) stay resident
//   while every block streams through two 32-KB stages of (half, K-block) slices —
//   at p = 256 a block (256 KB as hi + lo) no longer fits, and re-reading the signal
//   tile per block would cost more than re-reading blocks from L2.
// * Warp roles (persistent CTA per SM, 384 threads): warp 0 producer, warp 1 the
//   single-thread UMMA issuer (128x128x16, 4 K-steps x 3 products per slice) into
//   two 256-column TMEM accumulator stages, warps 4-11 the epilogue: group g takes
//   the blocks of accumulator stage g, each thread one signal; a block's 256
//   coefficients arrive as four 64-column TMEM loads, each reduced to its top-G
//   (topk.cuh) and merged into a running sorted top-G whose merges drop — and sum —
//   the discarded values (no S - kept cancellation).
// * Certificate: as at p = 64, with the error model scaled to 4x the accumulation
//   depth; near-ties are listed (with candidate-block masks) for the float64
//   re-decision (tiles_f64.cu), so decisions equal the float64 reference's.
#include "common.cuh"
#include "sm100.cuh"
#include "topk.cuh"

namespace sbo {
namespace tc256 {

constexpr int P = 256;
constexpr int M = 128;
constexpr int KB = P / 64;      // K-blocks (one 128-B swizzle atom of fp16 each)
constexpr int NH = 2;           // N-halves of a block
constexpr int NHALF = P / NH;   // 128 atoms
constexpr int EPI_WARPS = 8;
constexpr int THREADS = 128 + 32 * EPI_WARPS;
constexpr uint32_t A_KB_BYTES = M * 64 * 2;      // 16 KB
constexpr uint32_t B_KB_BYTES = NHALF * 64 * 2;  // 16 KB
constexpr int BST = 2;                           // block-slice stages

struct Smem {
  __half a[2][KB][M * 64];          // [hi, lo][kb]
  __half b[BST][2][NHALF * 64];     // [stage][hi, lo]
  uint64_t a_full, a_empty, b_full[BST], b_empty[BST], acc_full[2], acc_empty[2];
  uint32_t tmem;
  float x_r1[M], x_r2[M], x_s[M], x_rb[M], x_eb[M];
  int x_b1[M];
  float x_dec[32][M];
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
    if (++i == BST) {
      i = 0;
      ph ^= 1u;
    }
  }
};

// error bound of one coefficient (absolute, unscaled units), empirical at p = 256: the
// K slices are streamed, so the cross terms of slices 2-4 meet a full-scale accumulator
// and the measured MMA model (tc_energy.cu) gives a worst case of
// ~2.5e-5 ||y||; the parity tests at config D are green with 1e-5
__device__ __forceinline__ float coef_err(float s_norm) { return 1.0e-5f * sqrtf(s_norm); }

__device__ __forceinline__ float resid_err(float r, float d, int n) {
  return 2.0f * d * sqrtf(static_cast<float>(n) * fmaxf(r, 0.0f)) + n * d * d +
         3.2e-5f * fmaxf(r, 0.0f);
}

// candidate mask of a signal flagged by an incremental pass over [b0, b1)
// (b1 <= 32): its incoming winner and every appended block
__device__ __forceinline__ uint64_t accum_cand(int prev, int b0, int b1) {
  const uint64_t app = (b1 - b0 >= 64 ? ~0ull : ((1ull << (b1 - b0)) - 1ull)) << b0;
  return (prev >= 0 && prev < 64 ? 1ull << prev : 0ull) | app;
}

template <int G, bool ABS>
__global__ void __launch_bounds__(THREADS, 1)
k_energy_tc256(const __half* __restrict__ yh, const __half* __restrict__ yl,
               const int16_t* __restrict__ escale, int64_t m, const __half* __restrict__ qh,
               const __half* __restrict__ ql, const int16_t* __restrict__ fscale, int b0, int b1,
               int ksel, int accumulate, int32_t* best, double* score, double* residual,
               int32_t* flags, int32_t* nflag, uint64_t* cand) {
  extern __shared__ unsigned char raw[];
  Smem* S = smem_of(raw);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t ntiles = ceil_div(m, M);
  const int nblk = b1 - b0;

  if (threadIdx.x == 0) {
    sm100::mbar_init(&S->a_full, 1);
    sm100::mbar_init(&S->a_empty, 1);
    for (int s = 0; s < BST; ++s) {
      sm100::mbar_init(&S->b_full[s], 1);
      sm100::mbar_init(&S->b_empty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      sm100::mbar_init(&S->acc_full[s], 1);
      sm100::mbar_init(&S->acc_empty[s], EPI_WARPS / 2);
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
      uint32_t aph = 0;
      Ring rb;
      for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        sm100::mbar_wait(&S->a_empty, aph ^ 1u);
        aph ^= 1u;
        sm100::mbar_expect_tx(&S->a_full, 2 * KB * A_KB_BYTES);
        for (int kb = 0; kb < KB; ++kb) {
          const int64_t off = (t * KB + kb) * static_cast<int64_t>(M * 64);
          sm100::bulk_g2s(S->a[0][kb], yh + off, A_KB_BYTES, &S->a_full);
          sm100::bulk_g2s(S->a[1][kb], yl + off, A_KB_BYTES, &S->a_full);
        }
        for (int b = b0; b < b1; ++b)
          for (int nh = 0; nh < NH; ++nh)
            for (int kb = 0; kb < KB; ++kb) {
              const int64_t off = ((static_cast<int64_t>(b) * NH + nh) * KB + kb) * (NHALF * 64);
              sm100::mbar_wait(&S->b_empty[rb.i], rb.ph ^ 1u);
              sm100::mbar_expect_tx(&S->b_full[rb.i], 2 * B_KB_BYTES);
              sm100::bulk_g2s(S->b[rb.i][0], qh + off, B_KB_BYTES, &S->b_full[rb.i]);
              sm100::bulk_g2s(S->b[rb.i][1], ql + off, B_KB_BYTES, &S->b_full[rb.i]);
              rb.next();
            }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ------------------------------------------- MMA issuer
      uint32_t aph = 0;
      Ring rb;
      int acc_i = 0;
      uint32_t acc_ph = 0;
      const uint32_t idesc = sm100::idesc_f16(M, NHALF);
      for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
        sm100::mbar_wait(&S->a_full, aph);
        aph ^= 1u;
        sm100::tc_fence_after();
        for (int b = b0; b < b1; ++b) {
          sm100::mbar_wait(&S->acc_empty[acc_i], acc_ph ^ 1u);
          sm100::tc_fence_after();
          for (int nh = 0; nh < NH; ++nh) {
            const uint32_t d = tmem + acc_i * 256 + nh * NHALF;
            for (int kb = 0; kb < KB; ++kb) {
              sm100::mbar_wait(&S->b_full[rb.i], rb.ph);
              sm100::tc_fence_after();
              const uint32_t a_hi = sm100::smem_u32(S->a[0][kb]);
              const uint32_t a_lo = sm100::smem_u32(S->a[1][kb]);
              const uint32_t b_hi = sm100::smem_u32(S->b[rb.i][0]);
              const uint32_t b_lo = sm100::smem_u32(S->b[rb.i][1]);
#pragma unroll
              for (int kk = 0; kk < 4; ++kk) {
                const uint32_t ko = kk * 32;
                sm100::umma_f16(d, sm100::desc_sw128(a_lo + ko), sm100::desc_sw128(b_hi + ko),
                                idesc, (kb > 0 || kk > 0) ? 1u : 0u);
                sm100::umma_f16(d, sm100::desc_sw128(a_hi + ko), sm100::desc_sw128(b_lo + ko),
                                idesc, 1u);
                sm100::umma_f16(d, sm100::desc_sw128(a_hi + ko), sm100::desc_sw128(b_hi + ko),
                                idesc, 1u);
              }
              sm100::umma_commit(&S->b_empty[rb.i]);
              rb.next();
            }
          }
          sm100::umma_commit(&S->acc_full[acc_i]);
          if (++acc_i == 2) {
            acc_i = 0;
            acc_ph ^= 1u;
          }
        }
        sm100::umma_commit(&S->a_empty);
      }
    }
  } else if (warp >= 4) {  // ------------------------------------------ epilogue
    // decision value (minimized): R = S - kept for squared-sum, -E for abs-sum;
    // ties keep the lower block
    const int ew = warp - 4, grp = ew >> 2, q = warp & 3;
    const int row = 32 * q + lane;
    const uint32_t lane_base = tmem + (static_cast<uint32_t>(32 * q) << 16) + grp * 256;
    uint32_t ph = 0;     // parity of this group's accumulator stage
    int64_t seq = 0;     // blocks issued so far (all tiles): stage = seq & 1
    auto preload = [&](int64_t tt, int& es_, double& prev_) {
      const int64_t jj = tt * M + row;
      es_ = 0;
      prev_ = ABS ? -INFINITY : INFINITY;
      if (tt < ntiles && jj < m) {
        es_ = escale[jj];
        if (accumulate) prev_ = ABS ? __ldcg(score + jj) : __ldcg(residual + jj);
      }
    };
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
      for (int jb = 0; jb < nblk; ++jb, ++seq) {
        if (static_cast<int>(seq & 1) != grp) continue;
        const int b = b0 + jb;
        sm100::mbar_wait(&S->acc_full[grp], ph);
        ph ^= 1u;
        sm100::tc_fence_after();
        float top[G];
#pragma unroll
        for (int i = 0; i < G; ++i) top[i] = 0.0f;
        float dropped = 0.0f, sq = 0.0f;
#pragma unroll 1
        for (int c = 0; c < P / 64; ++c) {
          float v[64];
          sm100::tmem_ld64(lane_base + c * 64, v);
          float t8[8];
#pragma unroll
          for (int a = 0; a < 8; ++a) {
            float acc = 0.0f;
#pragma unroll
            for (int i = 0; i < 8; ++i) acc = fmaf(v[8 * a + i], v[8 * a + i], acc);
            t8[a] = acc;
          }
          sq += ((t8[0] + t8[1]) + (t8[2] + t8[3])) + ((t8[4] + t8[5]) + (t8[6] + t8[7]));
#pragma unroll
          for (int i = 0; i < 64; ++i) v[i] = ABS ? fabsf(v[i]) : v[i] * v[i];
          dropped += topk::top_of_64_dropped<G>(v);  // v[0..G): the chunk's top-G, sorted
#pragma unroll
          for (int i = 0; i < G; ++i) {  // top-G of running u chunk; the minima drop out
            const float x = top[i], y = v[G - 1 - i];
            top[i] = fmaxf(x, y);
            dropped += fminf(x, y);
          }
          topk::merge_desc<G>(top);
        }
        sm100::tc_fence_before();
        __syncwarp();
        if (lane == 0) sm100::mbar_arrive(&S->acc_empty[grp]);
        float kept = 0.0f, e = 0.0f;
#pragma unroll
        for (int i = 0; i < G; ++i) {
          if (i < ksel) {
            kept += ABS ? top[i] * top[i] : top[i];
            e += top[i];
          } else if (!ABS) {
            dropped += top[i];
          }
        }
        const float u = exp2f(static_cast<float>(-(es + fscale[b])));
        const float u2 = u * u;
        sq *= u2;
        kept *= u2;
        e *= ABS ? u : u2;
        const float r = ABS ? sq - kept : dropped * u2;
        const float dec = ABS ? -e : r;
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
        if (cand && jb < 32) S->x_dec[jb][row] = dec;
      }
      // combine the two epilogue groups (same signals, interleaved blocks)
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
          return ABS ? (ksel * dc + 4e-6f * fabsf(dec)) : resid_err(dec, dc, nd);
        };
        bool flag;
        if (accumulate) {
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
            // (1 % slack on the bound); all blocks when more than 32
            uint64_t cmask = ~0ull;
            if (nblk <= 32) {
              cmask = 0ull;
              const float lim = d1 + 1.01f * err(d1);
              for (int jb = 0; jb < nblk; ++jb) {
                const float dv = S->x_dec[jb][row];
                if (dv <= lim + 1.01f * err(dv)) cmask |= 1ull << jb;
              }
            }
            cand[ix] = cmask;
          }
        }
      }
      asm volatile("bar.sync 1, %0;" ::"r"(32 * EPI_WARPS));
    }
  }
  __syncthreads();
  if (warp == 2) sm100::tmem_dealloc(tmem, 512);
}

// signals -> [tile][kb][row][128 B] fp16 hi / lo, scaled into [16, 32); one warp
// per row, 8 coordinates (one 16-B chunk) per lane
template <typename TY>
__global__ void k_split_signals256(const TY* __restrict__ y, int64_t m, int64_t m_pad,
                                   __half* yh, __half* yl, int16_t* escale) {
  const int64_t j = (static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (j >= m_pad) return;
  double v[8];
  double mx = 0.0;
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    v[i] = j < m ? static_cast<double>(y[j * P + 8 * lane + i]) : 0.0;
    mx = fmax(mx, fabs(v[i]));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  int e = 0;
  if (mx > 0.0) {
    int ex;
    frexp(mx, &ex);
    e = max(-120, min(120, 5 - ex));
  }
  __align__(16) __half h[8], l[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const double s = ldexp(v[i], e);
    h[i] = __double2half(s);
    l[i] = __double2half(s - static_cast<double>(__half2float(h[i])));
  }
  const int64_t t = j >> 7;
  const uint32_t r = static_cast<uint32_t>(j & 127), kb = static_cast<uint32_t>(lane >> 3);
  const int64_t base = ((t * KB + kb) * M + (r & ~7u)) * 128;
  const uint32_t off = sm100::sw128_offset(r & 7u, (lane & 7) * 16);
  *reinterpret_cast<uint4*>(reinterpret_cast<unsigned char*>(yh) + base + off) =
      *reinterpret_cast<const uint4*>(h);
  *reinterpret_cast<uint4*>(reinterpret_cast<unsigned char*>(yl) + base + off) =
      *reinterpret_cast<const uint4*>(l);
  if (lane == 0) escale[j] = static_cast<int16_t>(e);
}

// blocks Q_b (row-major [k][i], float64) -> [b][half][kb][atom][128 B] fp16 hi / lo
__global__ void k_split_blocks256(const double* __restrict__ Q, __half* qh, __half* ql,
                                  int16_t* fscale) {
  const int b = blockIdx.x;
  __shared__ double red[32];
  __shared__ int fsh;
  const double* q = Q + static_cast<int64_t>(b) * P * P;
  double mx = 0.0;
  for (int e = threadIdx.x; e < P * P; e += blockDim.x) mx = fmax(mx, fabs(q[e]));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    double mm = 0.0;
    for (int w = 0; w < static_cast<int>(blockDim.x >> 5); ++w) mm = fmax(mm, red[w]);
    int f = 0;
    if (mm > 0.0) {
      int ex;
      frexp(mm, &ex);
      f = max(-120, min(120, 5 - ex));
    }
    fsh = f;
    fscale[b] = static_cast<int16_t>(f);
  }
  __syncthreads();
  const int f = fsh;
  for (int e = threadIdx.x; e < P * P; e += blockDim.x) {
    const int k = e / P, i = e % P;  // coalesced reads of row k; atom i
    const double s = ldexp(q[e], f);
    const __half h = __double2half(s);
    const __half l = __double2half(s - static_cast<double>(__half2float(h)));
    const int nh = i / NHALF, ii = i % NHALF, kb = k / 64, kk = k % 64;
    const int64_t region = ((static_cast<int64_t>(b) * NH + nh) * KB + kb) * (NHALF * 64 * 2);
    const int64_t at = region + (ii & ~7) * 128 + sm100::sw128_offset(ii & 7, kk * 2);
    *reinterpret_cast<__half*>(reinterpret_cast<unsigned char*>(qh) + at) = h;
    *reinterpret_cast<__half*>(reinterpret_cast<unsigned char*>(ql) + at) = l;
  }
}

template <int G, bool ABS>
int launch_energy(const __half* yh, const __half* yl, const int16_t* es, int64_t m,
                  const __half* qh, const __half* ql, const int16_t* fs, int b0, int b1, int ksel,
                  int accumulate, int32_t* best, double* score, double* residual,
                  int32_t* flags, int32_t* nflag, uint64_t* cand, cudaStream_t st) {
  auto kern = k_energy_tc256<G, ABS>;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       static_cast<int>(SMEM_BYTES));
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t ntiles = ceil_div(m, M);
  const int grid = static_cast<int>(ntiles < sms ? ntiles : sms);
  kern<<<grid, THREADS, SMEM_BYTES, st>>>(yh, yl, es, m, qh, ql, fs, b0, b1, ksel, accumulate,
                                          best, score, residual, flags, nflag, cand);
  return check_launch("k_energy_tc256");
}

}  // namespace tc256
}  // namespace sbo

using namespace sbo;

int tc256_split_signals(const void* y, int dtype, int64_t m, int64_t m_pad, void* yh, void* yl,
                        int16_t* escale, cudaStream_t st) {
  if (m_pad == 0) return SBO_OK;
  const unsigned grid = static_cast<unsigned>(ceil_div(m_pad * 32, 256));
  if (dtype == SBO_F32)
    tc256::k_split_signals256<float><<<grid, 256, 0, st>>>(
        static_cast<const float*>(y), m, m_pad, static_cast<__half*>(yh),
        static_cast<__half*>(yl), escale);
  else
    tc256::k_split_signals256<double><<<grid, 256, 0, st>>>(
        static_cast<const double*>(y), m, m_pad, static_cast<__half*>(yh),
        static_cast<__half*>(yl), escale);
  return check_launch("k_split_signals256");
}

int tc256_split_blocks(const double* Q, int K, void* qh, void* ql, int16_t* fscale,
                       cudaStream_t st) {
  if (K < 1) return SBO_OK;
  tc256::k_split_blocks256<<<K, 256, 0, st>>>(Q, static_cast<__half*>(qh),
                                               static_cast<__half*>(ql), fscale);
  return check_launch("k_split_blocks256");
}

extern "C" int sbo_tc_energy256(const void* yhv, const void* ylv, const int16_t* escale,
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
  const int k = s0 < tc256::P ? s0 : tc256::P;
  cudaStream_t st = as_stream(stream);
  const bool abs = kind == SBO_KIND_ABS_SUM;
#define SBO_TC_CASE(GG)                                                                       \
  if (k <= GG)                                                                                \
    return abs ? tc256::launch_energy<GG, true>(yh, yl, escale, m, qh, ql, fscale, b0, b1, k, \
                                                accumulate, best, score, residual, flags,     \
                                                nflag, cand, st)                              \
               : tc256::launch_energy<GG, false>(yh, yl, escale, m, qh, ql, fscale, b0, b1,   \
                                                 k, accumulate, best, score, residual, flags, \
                                                 nflag, cand, st);
  SBO_TC_CASE(8)  // k <= 8 shares the 8-wide network (tc_energy.cu)
  SBO_TC_CASE(16)
  SBO_TC_CASE(32)
#undef SBO_TC_CASE
  return fail(SBO_EINVAL, "the p = 256 tensor-core pass supports s0 <= 32");
}
