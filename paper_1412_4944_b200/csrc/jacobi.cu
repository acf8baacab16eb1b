// Batched one-sided (Hestenes) Jacobi in float64, one CTA per p x p matrix.
//
//  * sbo_polar:      Q_b = U V^T of P_b  (linalg.py:68-78 procrustes_polar; the
//                    reference calls LAPACK gesdd, linalg.py:52) + the
//                    orthonormality guard of onb.py:119-124.
//  * sbo_init_block: eigenvectors of the Gram matrix of the worst set, i.e. the
//                    left singular vectors of ysub (onb.py:79-95 init_onb), with
//                    descending order and canonical signs (linalg.py:32-37) and
//                    the seeded Gram–Schmidt completion (onb.py:98-116).
//
// Columns of the working matrix A (and of the rotation accumulator V) are
// stored contiguously (column-major).  A round-robin tournament gives p/2
// disjoint column pairs per step; each pair is handled by g = 256/(p/2) lanes
// (capped at a warp) that reduce alpha = |a_i|^2, beta = |a_j|^2, gamma = a_i.a_j
// with shuffles and apply the Rutishauser rotation.  A sweep without a rotation
// (|gamma| <= tol sqrt(alpha beta) everywhere) ends the iteration.
#include <cfloat>
#include <cstdlib>

#include <cooperative_groups.h>

#include "common.cuh"
#include "sm100.cuh"

namespace sbo {

constexpr int kJacobiThreads = 256;
constexpr int kMaxSweeps = 60;

// A pair is rotated whenever |gamma| > eps sqrt(alpha beta) (so the result is as
// orthogonal as float64 allows); a sweep only counts as "still moving" when some
// pair exceeded 4 sqrt(rows) eps — the rounding floor of the computed gamma.
__device__ __forceinline__ double jacobi_rot_tol() { return DBL_EPSILON; }
__device__ __forceinline__ double jacobi_conv_tol(int rows) {
  return 4.0 * sqrt(static_cast<double>(rows < 4 ? 4 : rows)) * DBL_EPSILON;
}

// Rotation of one column pair: t = tan(theta) in fp32 from power-of-two-scaled
// inputs (no overflow, no float64 division chain), then c, s normalized in
// float64 so c^2 + s^2 = 1 to rounding and V stays orthogonal; an fp32-accurate
// angle only leaves ~1e-7 gamma for the next sweep.
__device__ __forceinline__ void rotation(double al, double be, double ga, double& c, double& s) {
  const double d = be - al, gg = 2.0 * ga;
  // exact power-of-two scale 2^-e from the exponent bits of max(|d|, |gg|)
  // (both finite, gg != 0 here): a handful of integer ops instead of frexp/ldexp
  const int hi = __double2hiint(fmax(fabs(d), fabs(gg)));
  const int e = ((hi >> 20) & 0x7ff) - 1023;
  const double scale = __hiloint2double((1023 - e) << 20, 0);
  const float df = static_cast<float>(d * scale);
  const float gf = static_cast<float>(gg * scale);
  const float tf = copysignf(1.0f, df) * gf / (fabsf(df) + sqrtf(fmaf(df, df, gf * gf)));
  const double t = static_cast<double>(tf);
  c = rsqrt(fma(t, t, 1.0));
  s = c * t;
}

// The same rotation with approximate fp32 MUFU square root / reciprocal for the
// angle (a few ulp, like the fp32 angle itself) and c = (1 + t^2)^-1/2 from the
// float64 MUFU estimate refined by two Newton steps (to rounding, so c^2 + s^2 = 1
// as before): a shorter dependent chain than the IEEE sqrt / div / rsqrt paths.
__device__ __forceinline__ void rotation_fast(double al, double be, double ga, double& c,
                                              double& s) {
  const double d = be - al, gg = 2.0 * ga;
  const int hi = __double2hiint(fmax(fabs(d), fabs(gg)));
  const int e = ((hi >> 20) & 0x7ff) - 1023;
  const double scale = __hiloint2double((1023 - e) << 20, 0);
  const float df = static_cast<float>(d * scale);
  const float gf = static_cast<float>(gg * scale);
  const float h2 = fmaf(df, df, gf * gf);
  const float h = h2 * rsqrtf(h2);
  const float tf = copysignf(1.0f, df) * __fdividef(gf, fabsf(df) + h);
  const double t = static_cast<double>(tf);
  const double x = fma(t, t, 1.0);
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
#pragma unroll
  for (int it = 0; it < 2; ++it) {
    const double r = fma(-x * y, y, 1.0);
    y = fma(0.5 * y, r, y);
  }
  c = y;
  s = c * t;
}

// p = 64 specialization: 32 column pairs per step.  A half-warp (16 lanes) owns a
// pair, so each shared-memory access reads 16 consecutive rows of ONE column —
// conflict-free whatever the columns (8 lanes per pair put 4 columns of equal
// bank alignment in a warp's wavefront); every thread handles pairs q and
// q + 16 (rows lg + 16u), which also gives two independent chains.  The
// round-robin schedule advances incrementally.
template <int NT>
__device__ __forceinline__ int jacobi_sweeps64(double* A, double* V, int* flag) {
  static_assert(NT == 256 || NT == 512, "256 threads: 2 pairs each; 512: 1 pair each");
  constexpr int N = 64, NP = NT == 256 ? 2 : 1;
  const int tid = threadIdx.x, q = tid >> 4, lg = tid & 15;
  const double tol2 = DBL_EPSILON * DBL_EPSILON;
  const double conv = 4.0 * 8.0 * DBL_EPSILON, conv2 = conv * conv;
  for (int sweep = 0; sweep < kMaxSweeps; ++sweep) {
    if (tid == 0) *flag = 0;
    __syncthreads();
    // step 0 of the tournament for pairs q and (256 threads) q + 16
    int i0 = q, j0 = q == 0 ? N - 1 : N - 1 - q;
    int i1 = q + 16, j1 = N - 1 - (q + 16);
    for (int step = 0; step < N - 1; ++step) {
      double* ai[2] = {A + i0 * N + lg, A + i1 * N + lg};
      double* aj[2] = {A + j0 * N + lg, A + j1 * N + lg};
      double x[2][4], y[2][4], al[2], be[2], ga[2];
#pragma unroll
      for (int h = 0; h < NP; ++h) {
        al[h] = be[h] = ga[h] = 0.0;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          x[h][u] = ai[h][16 * u];
          y[h][u] = aj[h][16 * u];
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          al[h] = fma(x[h][u], x[h][u], al[h]);
          be[h] = fma(y[h][u], y[h][u], be[h]);
          ga[h] = fma(x[h][u], y[h][u], ga[h]);
        }
      }
#pragma unroll
      for (int o = 8; o > 0; o >>= 1) {
#pragma unroll
        for (int h = 0; h < NP; ++h) {
          al[h] += __shfl_xor_sync(0xffffffffu, al[h], o);
          be[h] += __shfl_xor_sync(0xffffffffu, be[h], o);
          ga[h] += __shfl_xor_sync(0xffffffffu, ga[h], o);
        }
      }
#pragma unroll
      for (int h = 0; h < NP; ++h) {
        const double g2 = ga[h] * ga[h], ab = al[h] * be[h];
        if (al[h] > 0.0 && be[h] > 0.0 && g2 > tol2 * ab) {
          double c, sn;
          rotation(al[h], be[h], ga[h], c, sn);
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            ai[h][16 * u] = c * x[h][u] - sn * y[h][u];
            aj[h][16 * u] = sn * x[h][u] + c * y[h][u];
          }
          if (V) {  // V == nullptr: only the orthogonalised columns are wanted
            double* vi = V + (h ? i1 : i0) * N + lg;
            double* vj = V + (h ? j1 : j0) * N + lg;
            double vx[4], vy[4];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              vx[u] = vi[16 * u];
              vy[u] = vj[16 * u];
            }
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              vi[16 * u] = c * vx[u] - sn * vy[u];
              vj[16 * u] = sn * vx[u] + c * vy[u];
            }
          }
          if (lg == 0 && g2 > conv2 * ab) *flag = 1;
        }
      }
      __syncthreads();
      // next step: i, j advance by one modulo 63 (slot 0 keeps j = 63)
      i0 = (i0 == N - 2) ? 0 : i0 + 1;
      if (q != 0) j0 = (j0 == N - 2) ? 0 : j0 + 1;
      i1 = (i1 == N - 2) ? 0 : i1 + 1;
      j1 = (j1 == N - 2) ? 0 : j1 + 1;
    }
    if (*flag == 0) return sweep + 1;
    __syncthreads();
  }
  return -1;
}

// p = 64 sweeps without V on LP lanes per column pair (32 LP threads, the
// CTA's first warps; the rest wait at the final __syncthreads).  The one-CTA
// init is issue-bound with 16 lanes per pair: 16 warps x ~185 instructions per
// tournament step on 4 schedulers.  With LP = 4 one warp per scheduler carries 8
// pairs of 16 rows each, so a step costs its dependency chain instead.  Lane lg
// of pair q reads rows LP ((u + q) mod R) + lg (a rotation of the row blocks per
// pair), so the 32 / LP pairs of a warp hit distinct banks whatever the columns.
// Same rotations, schedule and tolerances as jacobi_sweeps64.  Returns the
// sweep count (or -1) to every thread of the CTA.
template <int LP>
__device__ __noinline__ int jacobi_sweeps64_lp(double* A, int* flag, int* result_smem,
                                               bool fast) {
  constexpr int N = 64, R = N / LP, NT = 32 * LP, PPW = 32 / LP;
  static_assert(LP == 4 || LP == 8, "4 or 8 lanes per pair");
  const int tid = threadIdx.x;
  if (tid < NT) {
    const int q = tid / LP, lg = tid % LP, qw = q % PPW;
    const double tol2 = DBL_EPSILON * DBL_EPSILON;
    const double conv = 4.0 * 8.0 * DBL_EPSILON, conv2 = conv * conv;
    int result = -1;
    int roff[R];
#pragma unroll
    for (int u = 0; u < R; ++u) roff[u] = LP * ((u + qw) % R) + lg;
    for (int sweep = 0; sweep < kMaxSweeps; ++sweep) {
      if (tid == 0) *flag = 0;
      asm volatile("bar.sync 1, %0;" ::"r"(NT) : "memory");
      int i = q, j = q == 0 ? N - 1 : N - 1 - q;
      for (int step = 0; step < N - 1; ++step) {
        double* ai = A + i * N;
        double* aj = A + j * N;
        double x[R], y[R];
#pragma unroll
        for (int u = 0; u < R; ++u) {
          x[u] = ai[roff[u]];
          y[u] = aj[roff[u]];
        }
        // two accumulator chains per sum (half the dependent DFMA depth)
        double al0 = 0.0, al1 = 0.0, be0 = 0.0, be1 = 0.0, ga0 = 0.0, ga1 = 0.0;
#pragma unroll
        for (int u = 0; u < R; u += 2) {
          al0 = fma(x[u], x[u], al0);
          be0 = fma(y[u], y[u], be0);
          ga0 = fma(x[u], y[u], ga0);
          al1 = fma(x[u + 1], x[u + 1], al1);
          be1 = fma(y[u + 1], y[u + 1], be1);
          ga1 = fma(x[u + 1], y[u + 1], ga1);
        }
        double al = al0 + al1, be = be0 + be1, ga = ga0 + ga1;
#pragma unroll
        for (int o = LP / 2; o > 0; o >>= 1) {
          al += __shfl_xor_sync(0xffffffffu, al, o);
          be += __shfl_xor_sync(0xffffffffu, be, o);
          ga += __shfl_xor_sync(0xffffffffu, ga, o);
        }
        const double g2 = ga * ga, ab = al * be;
        if (al > 0.0 && be > 0.0 && g2 > tol2 * ab) {
          double c, sn;
          if (fast) rotation_fast(al, be, ga, c, sn);
          else rotation(al, be, ga, c, sn);
#pragma unroll
          for (int u = 0; u < R; ++u) {
            ai[roff[u]] = c * x[u] - sn * y[u];
            aj[roff[u]] = sn * x[u] + c * y[u];
          }
          if (lg == 0 && g2 > conv2 * ab) *flag = 1;
        }
        asm volatile("bar.sync 1, %0;" ::"r"(NT) : "memory");
        // next step: i, j advance by one modulo 63 (slot 0 keeps j = 63)
        i = (i == N - 2) ? 0 : i + 1;
        if (q != 0) j = (j == N - 2) ? 0 : j + 1;
      }
      if (*reinterpret_cast<volatile int*>(flag) == 0) {
        result = sweep + 1;
        break;
      }
      asm volatile("bar.sync 1, %0;" ::"r"(NT) : "memory");  // flag read before reset
    }
    if (tid == 0) *result_smem = result;
  }
  __syncthreads();
  return *reinterpret_cast<volatile int*>(result_smem);
}

// Runs the sweeps on A (p x p, col-major) accumulating V.  Returns the sweep
// count, or -1 when kMaxSweeps is exhausted.  All threads of the CTA call it.
__device__ __forceinline__ int jacobi_sweeps(double* A, double* V, int rows, int p, int* flag) {
  if (rows == 64 && p == 64 && blockDim.x == 256) return jacobi_sweeps64<256>(A, V, flag);
  if (rows == 64 && p == 64 && blockDim.x == 512) return jacobi_sweeps64<512>(A, V, flag);
  const int n = p + (p & 1);
  const int npairs = n >> 1;
  int g = 32;
  while (g > 1 && npairs * g > kJacobiThreads) g >>= 1;
  const int per_round = kJacobiThreads / g;  // pairs handled concurrently
  const int tid = threadIdx.x;
  const int lg = tid & (g - 1);
  const double tol = jacobi_rot_tol(), conv = jacobi_conv_tol(rows);
  for (int sweep = 0; sweep < kMaxSweeps; ++sweep) {
    if (tid == 0) *flag = 0;
    __syncthreads();
    for (int step = 0; step < n - 1; ++step) {
      for (int q0 = 0; q0 < npairs; q0 += per_round) {
        const int q = q0 + tid / g;
        int i = -1, j = -1;
        if (q < npairs) {
          if (q == 0) {
            i = step;
            j = n - 1;
          } else {
            i = (step + q) % (n - 1);
            j = (step - q + n - 1) % (n - 1);
          }
          if (i >= p || j >= p) i = j = -1;
        }
        double al = 0.0, be = 0.0, ga = 0.0;
        if (i >= 0) {
          const double* ai = A + static_cast<int64_t>(i) * rows;
          const double* aj = A + static_cast<int64_t>(j) * rows;
          for (int r = lg; r < rows; r += g) {
            const double x = ai[r], y = aj[r];
            al = fma(x, x, al);
            be = fma(y, y, be);
            ga = fma(x, y, ga);
          }
        }
        for (int o = g >> 1; o > 0; o >>= 1) {
          al += __shfl_xor_sync(0xffffffffu, al, o);
          be += __shfl_xor_sync(0xffffffffu, be, o);
          ga += __shfl_xor_sync(0xffffffffu, ga, o);
        }
        const double g2 = ga * ga, ab = al * be;
        if (i >= 0 && al > 0.0 && be > 0.0 && g2 > tol * tol * ab) {
          // Rotation angle t = tan(theta) in fp32 from power-of-two-scaled inputs
          // (no overflow, no float64 division chain); c, s are then normalized in
          // float64 so c^2 + s^2 = 1 to rounding and V stays orthogonal.  An
          // fp32-accurate angle only leaves ~1e-7 gamma for the next sweep.
          const double d = be - al, gg = 2.0 * ga;
          int ex;
          frexp(fmax(fabs(d), fabs(gg)), &ex);
          const float df = static_cast<float>(ldexp(d, -ex));
          const float gf = static_cast<float>(ldexp(gg, -ex));
          const float tf = copysignf(1.0f, df) * gf / (fabsf(df) + sqrtf(fmaf(df, df, gf * gf)));
          const double t = static_cast<double>(tf);
          const double c = rsqrt(fma(t, t, 1.0));
          const double s = c * t;
          double* ai = A + static_cast<int64_t>(i) * rows;
          double* aj = A + static_cast<int64_t>(j) * rows;
          double* vi = V + static_cast<int64_t>(i) * p;
          double* vj = V + static_cast<int64_t>(j) * p;
          for (int r = lg; r < rows; r += g) {
            const double x = ai[r], y = aj[r];
            ai[r] = c * x - s * y;
            aj[r] = s * x + c * y;
          }
          for (int r = lg; r < p; r += g) {
            const double u = vi[r], w = vj[r];
            vi[r] = c * u - s * w;
            vj[r] = s * u + c * w;
          }
          if (lg == 0 && g2 > conv * conv * ab) *flag = 1;
        }
      }
      __syncthreads();
    }
    if (*flag == 0) return sweep + 1;
    __syncthreads();
  }
  return -1;
}

// norms of the columns of A -> sig[j]; descending order with index tie-break -> ord
__device__ __forceinline__ void column_order(const double* A, int rows, int p, double* sig, int* ord,
                             bool sqrt_norm) {
  for (int j = threadIdx.x; j < p; j += blockDim.x) {
    const double* a = A + static_cast<int64_t>(j) * rows;
    double acc = 0.0;
    for (int r = 0; r < rows; ++r) acc = fma(a[r], a[r], acc);
    sig[j] = sqrt_norm ? sqrt(acc) : acc;
  }
  __syncthreads();
  for (int j = threadIdx.x; j < p; j += blockDim.x) {
    int rank = 0;
    for (int l = 0; l < p; ++l) rank += (sig[l] > sig[j]) || (sig[l] == sig[j] && l < j);
    ord[rank] = j;
  }
  __syncthreads();
}

// orthonormality defect of a row-major p x p matrix (CTA-wide, deterministic)
template <int NT = kJacobiThreads>
__device__ __forceinline__ double defect_of(const double* Q, int p, double* red) {
  double acc = 0.0;
  for (int e = threadIdx.x; e < p * p; e += blockDim.x) {
    const int a = e / p, b = e % p;
    double g = 0.0;
    for (int k = 0; k < p; ++k) g = fma(Q[k * p + a], Q[k * p + b], g);
    g -= (a == b) ? 1.0 : 0.0;
    acc = fma(g, g, acc);
  }
  return sqrt(block_sum<NT>(acc, red));
}

// ---------------------------------------------------------------------------
struct JacobiSmem {
  double red[32];
  int flag;
  int count;
};

constexpr int kStNsFallback = 4;  // internal: Newton-Schulz handed the matrix to Jacobi
constexpr int kNsMaxIter = 48;

// ---------------------------------------------------------------------------
// Polar factor of a 64 x 64 P by the scaled Newton-Schulz iteration
//   X_0 = P / ||P||_F,  X_{k+1} = X_k (1.5 a_k I - 0.5 a_k^3 X_k^T X_k),
// a_k = sqrt(3 / (1 + l_k + l_k^2)), l_{k+1} = a_k l_k (3 - a_k^2 l_k^2) / 2, l_0 = 1e-6
// (Chen & Chow scaling for singular values in [l_k, 1]).  Every iteration is two
// dense 64^3 float64 GEMMs in shared memory — no sequential sweep steps — and it
// converges to the same orthogonal factor U V^T the SVD gives (~1e-12 at
// cond 1e5).  Stops when ||X^T X - I||_F < 1e-13; matrices that do not converge
// (rank deficient: the polar factor is then not unique) are flagged for the
// Jacobi kernel, which completes the null space.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void dmma64(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__global__ void __launch_bounds__(kJacobiThreads) k_polar_ns(const double* __restrict__ P,
                                                             const int64_t* __restrict__ counts,
                                                             double* Q, int32_t* status) {
  constexpr int N = 64, LD = 68;  // padded rows: conflict-free DMMA fragment loads
  const int b = blockIdx.x;
  __shared__ double red[32];
  extern __shared__ __align__(16) unsigned char dyn[];
  double* X = reinterpret_cast<double*>(dyn);  // [r][c]
  double* Y = X + N * LD;                      // next iterate
  double* A = Y + N * LD;                      // polynomial factor
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t4 = lane & 3;
  if (counts && counts[b] == 0) {
    if (tid == 0) status[b] = SBO_ST_SKIPPED;
    return;
  }
  const double* Pb = P + static_cast<int64_t>(b) * N * N;
  double nrm = 0.0;
  for (int e = tid; e < N * N; e += kJacobiThreads) {
    const double v = Pb[e];
    X[(e >> 6) * LD + (e & 63)] = v;
    nrm = fma(v, v, nrm);
  }
  nrm = sqrt(block_sum<kJacobiThreads>(nrm, red));
  if (!(nrm > 0.0)) {
    if (tid == 0) status[b] = kStNsFallback;
    return;
  }
  const double inv = 1.0 / nrm;
  for (int e = tid; e < N * N; e += kJacobiThreads) X[(e >> 6) * LD + (e & 63)] *= inv;
  __syncthreads();
  // lower bound for sigma_min / ||P||_F (image-patch P: ~7e-6); an overestimate only
  // slows the smallest singular values to plain Newton-Schulz speed
  double l = 1e-6;
  int it = 0;
  bool done = false;
  const int row = 8 * warp + g;  // this thread's output row in both GEMMs
  for (; it < kNsMaxIter; ++it) {
    // G = X^T X on DMMA: warp w owns rows [8w, 8w+8) x 64
    double acc[8][2];
#pragma unroll
    for (int n = 0; n < 8; ++n) acc[n][0] = acc[n][1] = 0.0;
#pragma unroll 4
    for (int r0 = 0; r0 < N; r0 += 4) {
      const double* xr = X + (r0 + t4) * LD;
      const double a = xr[8 * warp + g];
#pragma unroll
      for (int n = 0; n < 8; ++n) dmma64(acc[n][0], acc[n][1], a, xr[8 * n + g]);
    }
    double dev = 0.0;
#pragma unroll
    for (int n = 0; n < 8; ++n)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const double d = acc[n][h] - ((row == 8 * n + 2 * t4 + h) ? 1.0 : 0.0);
        dev = fma(d, d, dev);
      }
    dev = sqrt(block_sum<kJacobiThreads>(dev, red));
    if (dev < 1e-13) {
      done = true;
      break;
    }
    const double al = l < 0.99 ? sqrt(3.0 / (1.0 + l + l * l)) : 1.0;
    const double c1 = 1.5 * al, c3 = -0.5 * al * al * al;
#pragma unroll
    for (int n = 0; n < 8; ++n) {
      const int col = 8 * n + 2 * t4;
      *reinterpret_cast<double2*>(A + row * LD + col) =
          make_double2(c3 * acc[n][0] + (row == col ? c1 : 0.0),
                       c3 * acc[n][1] + (row == col + 1 ? c1 : 0.0));
    }
    l = fmin(1.0, al * l * (3.0 - al * al * l * l) * 0.5);
    __syncthreads();
    // Y = X A on DMMA
#pragma unroll
    for (int n = 0; n < 8; ++n) acc[n][0] = acc[n][1] = 0.0;
    const double* xa = X + row * LD + t4;
#pragma unroll 4
    for (int k0 = 0; k0 < N; k0 += 4) {
      const double a = xa[k0];
      const double* ab = A + (k0 + t4) * LD + g;
#pragma unroll
      for (int n = 0; n < 8; ++n) dmma64(acc[n][0], acc[n][1], a, ab[8 * n]);
    }
#pragma unroll
    for (int n = 0; n < 8; ++n)
      *reinterpret_cast<double2*>(Y + row * LD + 8 * n + 2 * t4) =
          make_double2(acc[n][0], acc[n][1]);
    __syncthreads();
    double* t = X;
    X = Y;
    Y = t;
  }
  if (!done) {
    if (tid == 0) status[b] = kStNsFallback;
    return;
  }
  double* Qb = Q + static_cast<int64_t>(b) * N * N;
  for (int e = tid; e < N * N; e += kJacobiThreads) Qb[e] = X[(e >> 6) * LD + (e & 63)];
  if (tid == 0) status[b] = SBO_ST_OK | (it << 8) | (1 << 16);  // bit 16: Newton-Schulz
}

// ---------------------------------------------------------------------------
// The same scaled Newton-Schulz iteration spread over a cluster of NC = 4 or 8
// CTAs per matrix (one per SM), exchanging through distributed shared memory.
// CTA r owns the column slice J_r = [W r, W r + W), W = 64 / NC:
//   G rows J_r    = X[:, J_r]^T X                         (local, full X held)
//   A cols J_r    = c1 I + c3 G[J_r, :]^T                 (G symmetric: local)
//   X' cols J_r   = X A[:, J_r]                           (local)
// and pushes its X' slice into every CTA's next-X buffer with one bulk copy per
// peer, completing transaction bytes on the receiver's mbarrier: one all-gather per
// iteration, no cluster barrier (a receiver's "full" wait of iteration k also
// proves every peer has finished reading the buffer it will overwrite in k+1,
// since peers push only after their last read of it).  The convergence test of
// X_k (the deviation ||X_k^T X_k - I||_F, a sum of per-CTA partials pushed with
// the slice) is read after the wait; X_{k+1} is computed speculatively
// meanwhile, so a converged X_k is still in the other buffer.  All CTAs take identical decisions
// (same partial sums in the same order), so the cluster leaves the loop together.
// ---------------------------------------------------------------------------

// DSMEM helpers: shared::cluster addresses and cluster-scope release/acquire
// (generic stores would make the barrier fence at GPU scope)
__device__ __forceinline__ uint32_t cluster_addr(const void* local, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;"
               : "=r"(r)
               : "r"(static_cast<uint32_t>(__cvta_generic_to_shared(local))), "r"(rank));
  return r;
}
__device__ __forceinline__ void cluster_barrier() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// X is held slice-major: Xs[q][k][c] = X[k][W q + c] with a W + 4 double row stride
// (conflict-free DMMA fragments), so a CTA's slice is one contiguous block
// that a single cp.async.bulk shared::cta -> shared::cluster copy delivers to a
// peer (completing on the peer's mbarrier).  The slice's padding column W of
// row 0 carries the CTA's deviation partial.

__device__ __forceinline__ void bulk_s2cluster(uint32_t dst, const void* src, uint32_t bytes,
                                               uint32_t mbar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
      ::"r"(dst), "r"(static_cast<uint32_t>(__cvta_generic_to_shared(src))), "r"(bytes), "r"(mbar)
      : "memory");
}

template <int NC>
__global__ void __cluster_dims__(NC, 1, 1) __launch_bounds__(kJacobiThreads)
    k_polar_ns_cluster(const double* __restrict__ P, const int64_t* __restrict__ counts,
                       double* Q, int32_t* status, double l0) {
  // slice row stride: slice columns + 4 (conflict-free fragments)
  constexpr int N = 64, W = N / NC, SL = W + 4, SZ = 64 * SL;
  constexpr int A2 = W / 8;  // 8-column tiles per slice
  static_assert(W % 8 == 0 && (SL % 16 == 4 || SL % 16 == 12), "slice layout");
  const int r = static_cast<int>(blockIdx.x % NC);  // == %cluster_ctarank for 1-D clusters
  const int b = blockIdx.x / NC;
  __shared__ double red[32];
  __shared__ __align__(8) uint64_t full[2];
  extern __shared__ __align__(128) unsigned char dyn_ns[];
  double* X0 = reinterpret_cast<double*>(dyn_ns);  // buffer u, slice q: X0 + (u * NC + q) * SZ
  constexpr int AL = SL;
  double* As = X0 + 2 * NC * SZ;                // A[:, J_r] as As[j][i] (stride AL)
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t4 = lane & 3;
  if (counts && counts[b] == 0) {
    if (tid == 0 && r == 0) status[b] = SBO_ST_SKIPPED;
    return;
  }
  auto at = [&](int u, int k, int c) -> double* {  // &X_u[k][c]
    return X0 + (u * NC + c / W) * SZ + k * SL + (c % W);
  };
  const double* Pb = P + static_cast<int64_t>(b) * N * N;
  double nrm = 0.0;
  {  // all 16 loads in flight before the first store (one global latency, not 16)
    constexpr int PER = N * N / kJacobiThreads;
    double v[PER];
#pragma unroll
    for (int u = 0; u < PER; ++u) v[u] = __ldg(Pb + tid + u * kJacobiThreads);
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int e = tid + u * kJacobiThreads;
      *at(0, e >> 6, e & 63) = v[u];
      nrm = fma(v[u], v[u], nrm);
    }
  }
  nrm = sqrt(block_sum<kJacobiThreads>(nrm, red));
  if (!(nrm > 0.0)) {
    if (tid == 0 && r == 0) status[b] = kStNsFallback;
    return;
  }
  const double inv = 1.0 / nrm;
  for (int e = tid; e < N * N; e += kJacobiThreads) *at(0, e >> 6, e & 63) *= inv;
  if (tid == 0) {
    sm100::mbar_init(&full[0], 1);
    sm100::mbar_init(&full[1], 1);
    sm100::fence_barrier_init();
  }
  // peers in the cluster must be running (barriers initialised) before their
  // shared memory is written
  cluster_barrier();
  constexpr uint32_t kTx = (NC - 1) * SZ * sizeof(double);  // bytes received per iteration
  uint32_t phases = 0u;  // bit u: parity of full[u]
  double l = l0;
  int it = 0, cur = 0;
  bool done = false;
  for (; it < kNsMaxIter; ++it) {
    const double* Xr = X0 + (cur * NC + r) * SZ;                    // this CTA's slice
    const double* Xw = X0 + (cur * NC + (8 * warp) / W) * SZ + (8 * warp) % W;  // columns 8 warp ..
    // G[16r + 8a + g][8 warp + 2 t4 + h] = sum_k X[k][16r + 8a + g] X[k][8 warp + 2 t4 + h]
    // K split in two halves with separate accumulators: chains of 8 DMMAs, not 16
    double gg[A2][2], gh[A2][2];
#pragma unroll
    for (int a2 = 0; a2 < A2; ++a2) gg[a2][0] = gg[a2][1] = gh[a2][0] = gh[a2][1] = 0.0;
#pragma unroll 4
    for (int k0 = 0; k0 < N / 2; k0 += 4) {
      const double bv = Xw[(k0 + t4) * SL + g], bw = Xw[(k0 + N / 2 + t4) * SL + g];
#pragma unroll
      for (int a2 = 0; a2 < A2; ++a2) {
        dmma64(gg[a2][0], gg[a2][1], Xr[(k0 + t4) * SL + 8 * a2 + g], bv);
        dmma64(gh[a2][0], gh[a2][1], Xr[(k0 + N / 2 + t4) * SL + 8 * a2 + g], bw);
      }
    }
#pragma unroll
    for (int a2 = 0; a2 < A2; ++a2) {
      gg[a2][0] += gh[a2][0];
      gg[a2][1] += gh[a2][1];
    }
    const int gj = 8 * warp + 2 * t4;
    double dsum = 0.0;
    const double al = l < 0.99 ? sqrt(3.0 / (1.0 + l + l * l)) : 1.0;
    const double c1 = 1.5 * al, c3 = -0.5 * al * al * al;
#pragma unroll
    for (int a2 = 0; a2 < A2; ++a2) {
      const int gi = W * r + 8 * a2 + g;
      const double d0 = gg[a2][0] - (gi == gj ? 1.0 : 0.0);
      const double d1 = gg[a2][1] - (gi == gj + 1 ? 1.0 : 0.0);
      dsum = fma(d0, d0, fma(d1, d1, dsum));
      // A[j][16r + i] = c1 [j == 16r + i] + c3 G[16r + i][j]
      As[gj * AL + 8 * a2 + g] = c3 * gg[a2][0] + (gi == gj ? c1 : 0.0);
      As[(gj + 1) * AL + 8 * a2 + g] = c3 * gg[a2][1] + (gi == gj + 1 ? c1 : 0.0);
    }
    const double part = block_sum<kJacobiThreads>(dsum, red);  // (syncs: As complete)
    l = fmin(1.0, al * l * (3.0 - al * al * l * l) * 0.5);
    // X'[8 warp + g][16r + 8a + 2 t4 + h] = sum_j X[8 warp + g][j] A[j][16r + 8a + 2 t4 + h]
    double yy[A2][2], yh[A2][2];
#pragma unroll
    for (int a2 = 0; a2 < A2; ++a2) yy[a2][0] = yy[a2][1] = yh[a2][0] = yh[a2][1] = 0.0;
#pragma unroll 4
    for (int k0 = 0; k0 < N / 2; k0 += 4) {
      const double av = *at(cur, 8 * warp + g, k0 + t4);
      const double aw = *at(cur, 8 * warp + g, k0 + N / 2 + t4);
#pragma unroll
      for (int a2 = 0; a2 < A2; ++a2) {
        dmma64(yy[a2][0], yy[a2][1], av, As[(k0 + t4) * AL + 8 * a2 + g]);
        dmma64(yh[a2][0], yh[a2][1], aw, As[(k0 + N / 2 + t4) * AL + 8 * a2 + g]);
      }
    }
#pragma unroll
    for (int a2 = 0; a2 < A2; ++a2) {
      yy[a2][0] += yh[a2][0];
      yy[a2][1] += yh[a2][1];
    }
    const int nxt = cur ^ 1;
    double* mine = X0 + (nxt * NC + r) * SZ;
#pragma unroll
    for (int a2 = 0; a2 < A2; ++a2)
      *reinterpret_cast<double2*>(mine + (8 * warp + g) * SL + 8 * a2 + 2 * t4) =
          make_double2(yy[a2][0], yy[a2][1]);
    if (tid == 0) mine[W] = part;
    // generic-proxy writes -> visible to the bulk-copy (async) proxy
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (tid == 0) {
      sm100::mbar_expect_tx(&full[nxt], kTx);
#pragma unroll 1
      for (int q = 1; q < NC; ++q) {
        const uint32_t peer = static_cast<uint32_t>((r + q) % NC);
        bulk_s2cluster(cluster_addr(mine, peer), mine, SZ * sizeof(double),
                       cluster_addr(&full[nxt], peer));
      }
    }
    sm100::mbar_wait(&full[nxt], (phases >> nxt) & 1u);
    phases ^= 1u << nxt;
    double dev = 0.0;
#pragma unroll
    for (int q = 0; q < NC; ++q) dev += X0[(nxt * NC + q) * SZ + W];
    if (sqrt(dev) < 1e-13) {
      done = true;
      break;
    }
    cur = nxt;
  }
  if (!done) {
    if (tid == 0 && r == 0) status[b] = kStNsFallback;
    return;
  }
  double* Qb = Q + static_cast<int64_t>(b) * N * N;
  for (int e = tid; e < W * N; e += kJacobiThreads) {
    const int row = W * r + (e >> 6), col = e & 63;
    Qb[row * N + col] = *at(cur, row, col);
  }
  if (tid == 0 && r == 0) status[b] = SBO_ST_OK | (it << 8) | (1 << 16);  // bit 16: Newton-Schulz
}

template <bool SMEM>
__global__ void __launch_bounds__(kJacobiThreads) k_polar(const double* __restrict__ P, int p,
                                                          const int64_t* __restrict__ counts,
                                                          double* Q, double* Vio,
                                                          double* sigma_out, int32_t* status,
                                                          double* ws, int only_fallback) {
  const int b = blockIdx.x;
  const int64_t pp = static_cast<int64_t>(p) * p;
  __shared__ JacobiSmem S;
  extern __shared__ __align__(16) unsigned char dyn[];
  // after the Newton-Schulz pass, only the matrices it handed back are solved here
  if (only_fallback && (status[b] & 0xFF) != kStNsFallback) return;
  if (counts && counts[b] == 0) {
    if (threadIdx.x == 0 && status) status[b] = SBO_ST_SKIPPED;
    return;
  }
  double* A;
  double* V;
  double* sig;
  int* ord;
  if constexpr (SMEM) {  // compile-time: shared accesses compile to LDS/STS
    A = reinterpret_cast<double*>(dyn);
    V = A + pp;
    sig = V + pp;
    ord = reinterpret_cast<int*>(sig + p);
  } else {
    A = ws + b * (2 * pp + 2 * p);
    V = A + pp;
    sig = V + pp;
    ord = reinterpret_cast<int*>(sig + p);
  }
  const double* Pb = P + b * pp;
  double* Vb = Vio ? Vio + b * pp : nullptr;
  if (Vb) {
    // warm start: A = P V_prev (columns nearly orthogonal when P moved little
    // since the previous round), V = V_prev; V_prev is column-major
    for (int64_t e = threadIdx.x; e < pp; e += blockDim.x) V[e] = Vb[e];
    __syncthreads();
    for (int64_t e = threadIdx.x; e < pp; e += blockDim.x) {
      const int j = static_cast<int>(e / p), r = static_cast<int>(e % p);
      const double* pr = Pb + static_cast<int64_t>(r) * p;
      const double* vj = V + static_cast<int64_t>(j) * p;
      double acc = 0.0;
      for (int c = 0; c < p; ++c) acc = fma(pr[c], vj[c], acc);
      A[e] = acc;
    }
  } else {
    // cold start: A = P in column-major (a_j = column j of P); V = I
    for (int64_t e = threadIdx.x; e < pp; e += blockDim.x) {
      const int r = static_cast<int>(e / p), c = static_cast<int>(e % p);
      A[static_cast<int64_t>(c) * p + r] = Pb[e];
      V[static_cast<int64_t>(c) * p + r] = (r == c) ? 1.0 : 0.0;
    }
  }
  __syncthreads();
  const int sweeps = jacobi_sweeps(A, V, p, p, &S.flag);
  if (Vb)
    for (int64_t e = threadIdx.x; e < pp; e += blockDim.x) Vb[e] = V[e];
  column_order(A, p, p, sig, ord, true);
  const double smax = sig[ord[0]];
  const double null_tol = smax * 64.0 * DBL_EPSILON;
  // U_j = a_j / sigma_j in place; null directions completed deterministically
  for (int64_t e = threadIdx.x; e < pp; e += blockDim.x) {
    const int j = static_cast<int>(e / p);
    if (sig[j] > null_tol) A[e] /= sig[j];
  }
  __syncthreads();
  for (int rnk = 0; rnk < p; ++rnk) {
    const int j = ord[rnk];
    if (sig[j] > null_tol) continue;
    double* u = A + static_cast<int64_t>(j) * p;
    for (int cand = 0; cand < p; ++cand) {
      for (int r = threadIdx.x; r < p; r += blockDim.x) u[r] = (r == cand) ? 1.0 : 0.0;
      __syncthreads();
      for (int pass = 0; pass < 2; ++pass) {
        for (int l = 0; l < p; ++l) {
          const int jl = ord[l];
          if (jl == j || (sig[jl] <= null_tol && l > rnk)) continue;
          const double* w = A + static_cast<int64_t>(jl) * p;
          double d = 0.0;
          for (int r = threadIdx.x; r < p; r += blockDim.x) d = fma(w[r], u[r], d);
          d = block_sum<kJacobiThreads>(d, S.red);
          for (int r = threadIdx.x; r < p; r += blockDim.x) u[r] -= d * w[r];
          __syncthreads();
        }
      }
      double nn = 0.0;
      for (int r = threadIdx.x; r < p; r += blockDim.x) nn = fma(u[r], u[r], nn);
      nn = sqrt(block_sum<kJacobiThreads>(nn, S.red));
      if (nn > 1e-3) {
        for (int r = threadIdx.x; r < p; r += blockDim.x) u[r] /= nn;
        __syncthreads();
        break;
      }
    }
  }
  __syncthreads();
  // Q[k][i] = sum_j U[k][j] V[i][j]
  double* Qb = Q + b * pp;
  for (int64_t e = threadIdx.x; e < pp; e += blockDim.x) {
    const int k = static_cast<int>(e / p), i = static_cast<int>(e % p);
    double acc = 0.0;
    for (int j = 0; j < p; ++j)
      acc = fma(A[static_cast<int64_t>(j) * p + k], V[static_cast<int64_t>(j) * p + i], acc);
    Qb[e] = acc;
  }
  if (sigma_out)
    for (int r = threadIdx.x; r < p; r += blockDim.x) sigma_out[b * p + r] = sig[ord[r]];
  __syncthreads();
  const double d = defect_of(Qb, p, S.red);
  if (threadIdx.x == 0 && status) {  // low byte: status, bits 8..15: sweeps used
    const int code = sweeps < 0 ? SBO_ST_NOCONV : (!(d <= 1e-8) ? SBO_ST_DEFECT : SBO_ST_OK);
    status[b] = code | ((sweeps < 0 ? kMaxSweeps : sweeps) << 8);
  }
}

// Eigenvectors of a 64 x 64 symmetric PSD G (the worst set's Gram matrix) by
// Drmac-Veselic preconditioning: pivoted Cholesky P^T G P = R^T R (largest
// remaining diagonal first), then one-sided Jacobi on the columns of X = R^T,
// which converges in a few sweeps from this start; X V = U Sigma gives
// R^T R = U Sigma^2 U^T, so G's eigenvectors are P U (rows permuted back) with
// eigenvalues sigma_j^2.  Columns whose sigma is negligible come out zero (the
// caller's rank test drops them and completes the basis).  512 threads.
// Out: V col-major eigenvectors (unordered), lam[j] = sigma_j^2.  Returns sweeps.
__device__ int init_eig64_precond(const double* __restrict__ G, double* A, double* V,
                                  double* W, double* lam, int* perm, int* flag, int lp) {
  constexpr int N = 64, LDW = 65;
  const int tid = threadIdx.x;
  __shared__ int piv;
  __shared__ double dmax0;
  // W = G (row-major, stride 65), perm = identity
  for (int e = tid; e < N * N; e += 512) W[(e >> 6) * LDW + (e & 63)] = G[e];
  if (tid < N) perm[tid] = tid;
  __syncthreads();
  int rank = N;
  for (int k = 0; k < N; ++k) {
    if (tid < 32) {  // pivot: largest remaining diagonal, lowest index on ties
      double best = -1.0;
      int bi = k;
      for (int i = k + tid; i < N; i += 32) {
        const double d = W[i * LDW + i];
        if (d > best) {
          best = d;
          bi = i;
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (ob > best || (ob == best && oi < bi)) {
          best = ob;
          bi = oi;
        }
      }
      if (tid == 0) {
        piv = bi;
        if (k == 0) dmax0 = best;
      }
    }
    __syncthreads();
    const int j = piv;
    if (j != k) {  // symmetric swap of rows / columns k and j, and of the permutation
      for (int c = tid; c < N; c += 512) {
        const double t = W[k * LDW + c];
        W[k * LDW + c] = W[j * LDW + c];
        W[j * LDW + c] = t;
      }
      __syncthreads();
      for (int r = tid; r < N; r += 512) {
        const double t = W[r * LDW + k];
        W[r * LDW + k] = W[r * LDW + j];
        W[r * LDW + j] = t;
      }
      if (tid == 0) {
        const int t = perm[k];
        perm[k] = perm[j];
        perm[j] = t;
      }
      __syncthreads();
    }
    const double d = W[k * LDW + k];
    if (!(d > 64.0 * DBL_EPSILON * dmax0) || !(d > 0.0)) {  // the rest is numerically zero
      rank = k;
      break;
    }
    const double rkk = sqrt(d);
    // row k of R: R[k][k] = sqrt(d), R[k][c] = W[k][c] / R[k][k] (c > k)
    for (int c = tid; c < N; c += 512) W[k * LDW + c] = c < k ? 0.0 : (c == k ? rkk : W[k * LDW + c] / rkk);
    __syncthreads();
    // Schur complement of the trailing block
    for (int e = tid; e < N * N; e += 512) {
      const int r = e >> 6, c = e & 63;
      if (r > k && c > k) W[r * LDW + c] = fma(-W[k * LDW + r], W[k * LDW + c], W[r * LDW + c]);
    }
    __syncthreads();
  }
  // X = R^T as A col-major: column j of A = row j of R (rows >= rank are zero)
  for (int e = tid; e < N * N; e += 512) {
    const int j = e >> 6, r = e & 63;
    A[e] = (j < rank && r >= j) ? W[j * LDW + r] : 0.0;
  }
  __syncthreads();
  __shared__ int sweeps_smem;
  const bool fast = lp > 0;  // lp < 0: the same lanes with the IEEE rotation (A/B)
  const int lpa = lp < 0 ? -lp : lp;
  const int sweeps = lpa == 4   ? jacobi_sweeps64_lp<4>(A, flag, &sweeps_smem, fast)
                     : lpa == 8 ? jacobi_sweeps64_lp<8>(A, flag, &sweeps_smem, fast)
                                : jacobi_sweeps64<512>(A, nullptr, flag);
  // sigma_j = ||A_j||; eigenvector j of G = P (A_j / sigma_j)
  if (tid < N) {
    double ss = 0.0;
    for (int r = 0; r < N; ++r) ss = fma(A[tid * N + r], A[tid * N + r], ss);
    lam[tid] = ss;
  }
  __syncthreads();
  for (int e = tid; e < N * N; e += 512) {
    const int j = e >> 6, r = e & 63;
    const double sg = sqrt(lam[j]);
    V[j * N + perm[r]] = sg > 0.0 ? A[e] / sg : 0.0;
  }
  __syncthreads();
  return sweeps;
}

// A = G (col-major), V = I: the Jacobi starting point (one CTA per column)
__global__ void k_fill_gram(const double* __restrict__ G, int p, double* A, double* V) {
  const int c = blockIdx.x;
  for (int r = threadIdx.x; r < p; r += blockDim.x) {
    A[static_cast<int64_t>(c) * p + r] = G[static_cast<int64_t>(r) * p + c];
    V[static_cast<int64_t>(c) * p + r] = r == c ? 1.0 : 0.0;
  }
}

// ---------------------------------------------------------------------------
// One-sided Jacobi for 64 < p <= 256 over the whole GPU: a cooperative grid whose
// warps take the p/2 column pairs of each tournament step (columns in global
// memory, L2-resident), with a grid-wide barrier between steps.  Same rotations,
// tolerances and ordering as jacobi_sweeps; A = G, V = I on entry (col-major).
// The sweep count (or -1) is written to *sweeps_out.
__global__ void __launch_bounds__(256) k_jacobi_grid(double* A, double* V, int rows, int p,
                                                     int* flag, int* sweeps_out) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  const int lane = threadIdx.x & 31;
  const int wg = static_cast<int>(blockIdx.x) * 8 + (threadIdx.x >> 5);
  const int nw = static_cast<int>(gridDim.x) * 8;
  const int n = p + (p & 1), npairs = n >> 1;
  const double tol = jacobi_rot_tol(), conv = jacobi_conv_tol(rows);
  int result = -1;
  for (int sweep = 0; sweep < kMaxSweeps; ++sweep) {
    if (grid.thread_rank() == 0) *flag = 0;
    grid.sync();
    for (int step = 0; step < n - 1; ++step) {
      for (int q = wg; q < npairs; q += nw) {
        int i, j;
        if (q == 0) {
          i = step;
          j = n - 1;
        } else {
          i = (step + q) % (n - 1);
          j = (step - q + n - 1) % (n - 1);
        }
        if (i >= p || j >= p) continue;
        double* ai = A + static_cast<int64_t>(i) * rows;
        double* aj = A + static_cast<int64_t>(j) * rows;
        double al = 0.0, be = 0.0, ga = 0.0;
        for (int r = lane; r < rows; r += 32) {
          const double x = ai[r], y = aj[r];
          al = fma(x, x, al);
          be = fma(y, y, be);
          ga = fma(x, y, ga);
        }
        al = warp_sum(al);
        be = warp_sum(be);
        ga = warp_sum(ga);
        const double g2 = ga * ga, ab = al * be;
        if (al > 0.0 && be > 0.0 && g2 > tol * tol * ab) {
          double c, sn;
          rotation(al, be, ga, c, sn);
          for (int r = lane; r < rows; r += 32) {
            const double x = ai[r], y = aj[r];
            ai[r] = c * x - sn * y;
            aj[r] = sn * x + c * y;
          }
          double* vi = V + static_cast<int64_t>(i) * p;
          double* vj = V + static_cast<int64_t>(j) * p;
          for (int r = lane; r < p; r += 32) {
            const double x = vi[r], y = vj[r];
            vi[r] = c * x - sn * y;
            vj[r] = sn * x + c * y;
          }
          if (lane == 0 && g2 > conv * conv * ab) atomicExch(flag, 1);
        }
      }
      grid.sync();
    }
    const int moving = *reinterpret_cast<volatile int*>(flag);
    grid.sync();  // everyone has read the flag before it is reset
    if (!moving) {
      result = sweep + 1;
      break;
    }
  }
  if (grid.thread_rank() == 0) *sweeps_out = result;
}

// ---------------------------------------------------------------------------
template <bool SMEM, int NT>
__global__ void __launch_bounds__(NT) k_init_block(
    const double* __restrict__ G, int p, int64_t ncols, const double* __restrict__ draws,
    int ndraws, double* Q, int32_t* rank_out, int32_t* status, double* ws, int use_smem,
    const int* presolved_sweeps, int lp) {
  const int64_t pp = static_cast<int64_t>(p) * p;
  __shared__ JacobiSmem S;
  extern __shared__ __align__(16) unsigned char dyn[];
  double *A, *V, *lam, *U;
  int* ord;
  double* base;
  if constexpr (SMEM) base = reinterpret_cast<double*>(dyn);
  else base = ws;
  A = base;
  V = A + pp;
  U = V + pp;
  lam = U + pp;
  ord = reinterpret_cast<int*>(lam + p);
  int sweeps;
  bool lam_ready = false;
  if constexpr (SMEM && NT == 512) {
    if (p == 64 && !presolved_sweeps) {
      __shared__ int permv[64];
      sweeps = init_eig64_precond(G, A, V, U, lam, permv, &S.flag, lp);
      lam_ready = true;
    }
  }
  if (lam_ready) {
    // eigenvalues ready: descending order with index tie-break
    for (int j = threadIdx.x; j < p; j += blockDim.x) {
      int rk = 0;
      for (int l = 0; l < p; ++l) rk += (lam[l] > lam[j]) || (lam[l] == lam[j] && l < j);
      ord[rk] = j;
    }
    __syncthreads();
  } else if (presolved_sweeps) {  // A, V already rotated by k_jacobi_grid
    sweeps = *presolved_sweeps;
  } else {
    for (int64_t e = threadIdx.x; e < pp; e += blockDim.x) {
      const int r = static_cast<int>(e / p), c = static_cast<int>(e % p);
      A[static_cast<int64_t>(c) * p + r] = G[e];
      V[static_cast<int64_t>(c) * p + r] = (r == c) ? 1.0 : 0.0;
    }
    __syncthreads();
    sweeps = jacobi_sweeps(A, V, p, p, &S.flag);
  }
  if (!lam_ready) column_order(A, p, p, lam, ord, true);  // |G v_j| = lambda_j
  const double l0 = lam[ord[0]];
  // kept directions: sqrt(l) > 1e-12 sqrt(l0) and above the Gram floor; at most ncols
  if (threadIdx.x == 0) {
    int r = 0;
    if (l0 > 0.0) {
      const int cap = static_cast<int>(ncols < p ? ncols : p);
      while (r < cap) {
        const double l = lam[ord[r]];
        if (!(sqrt(l) > 1e-12 * sqrt(l0)) || !(l > 64.0 * DBL_EPSILON * l0)) break;
        ++r;
      }
    }
    S.count = r;
  }
  __syncthreads();
  const int rank = S.count;
  // copy kept eigenvectors (descending) into U with canonical signs
  for (int c = threadIdx.x; c < rank; c += blockDim.x) {
    const double* v = V + static_cast<int64_t>(ord[c]) * p;
    int piv = 0;
    double best = -1.0;
    for (int r = 0; r < p; ++r)
      if (fabs(v[r]) > best) {
        best = fabs(v[r]);
        piv = r;
      }
    const double sgn = v[piv] < 0.0 ? -1.0 : 1.0;
    double* u = U + static_cast<int64_t>(c) * p;
    for (int r = 0; r < p; ++r) u[r] = sgn * v[r];
  }
  __syncthreads();
  // seeded completion: twice-projected Gram–Schmidt on the draws, in order
  int have = rank, d = 0;
  bool ran_out = false;
  while (have < p) {
    if (d >= ndraws) {
      ran_out = true;
      break;
    }
    double* u = U + static_cast<int64_t>(have) * p;
    for (int r = threadIdx.x; r < p; r += blockDim.x) u[r] = draws[static_cast<int64_t>(d) * p + r];
    __syncthreads();
    ++d;
    for (int pass = 0; pass < 2; ++pass) {
      for (int l = 0; l < have; ++l) {
        const double* w = U + static_cast<int64_t>(l) * p;
        double dd = 0.0;
        for (int r = threadIdx.x; r < p; r += blockDim.x) dd = fma(w[r], u[r], dd);
        dd = block_sum<NT>(dd, S.red);
        for (int r = threadIdx.x; r < p; r += blockDim.x) u[r] -= dd * w[r];
        __syncthreads();
      }
    }
    double nn = 0.0;
    for (int r = threadIdx.x; r < p; r += blockDim.x) nn = fma(u[r], u[r], nn);
    nn = sqrt(block_sum<NT>(nn, S.red));
    if (nn < 1e-8) continue;
    for (int r = threadIdx.x; r < p; r += blockDim.x) u[r] /= nn;
    __syncthreads();
    ++have;
  }
  // Q[k][i] = U column i, row k
  for (int64_t e = threadIdx.x; e < pp; e += blockDim.x) {
    const int k = static_cast<int>(e / p), i = static_cast<int>(e % p);
    Q[e] = U[static_cast<int64_t>(i) * p + k];
  }
  __syncthreads();
  const double df = defect_of<NT>(Q, p, S.red);
  if (threadIdx.x == 0) {
    if (rank_out) {
      rank_out[0] = rank;
      rank_out[1] = d;  // completion draws consumed
    }
    if (status)
      *status = ((sweeps < 0 || ran_out) ? SBO_ST_NOCONV : (!(df <= 1e-8) ? SBO_ST_DEFECT : SBO_ST_OK)) |
                ((sweeps < 0 ? kMaxSweeps : sweeps) << 8);
  }
}

}  // namespace sbo

using namespace sbo;

namespace {
size_t polar_smem_bytes(int p) {
  const size_t pp = static_cast<size_t>(p) * p;
  return sizeof(double) * (2 * pp + 2 * p);
}
size_t init_smem_bytes(int p) {
  const size_t pp = static_cast<size_t>(p) * p;
  return sizeof(double) * (3 * pp + 2 * p);
}
constexpr size_t kSmemBudget = 200 * 1024;
}  // namespace

extern "C" size_t sbo_polar_ns_big_workspace_bytes(int K, int p);
int sbo_polar_ns_big(const double* P, int K, int p, const int64_t* counts, double* Q,
                     int32_t* status, void* ws, size_t ws_bytes, void* stream);

extern "C" size_t sbo_polar_workspace_bytes(int K, int p) {
  const size_t jac = static_cast<size_t>(K) * polar_smem_bytes(p) + 64;
  const size_t ns = p > 64 ? sbo_polar_ns_big_workspace_bytes(K, p) : 0;
  return jac > ns ? jac : ns;
}

extern "C" int sbo_polar(const double* P, int K, int p, const int64_t* counts, double* Q,
                         double* V, double* sigma, int32_t* status, void* ws, size_t ws_bytes,
                         void* stream) {
  if (K < 1 || p < 1 || p > kPMax) return fail(SBO_EINVAL, "bad polar shape");
  const bool smem = polar_smem_bytes(p) <= kSmemBudget;
  if (!smem && ws_bytes < sbo_polar_workspace_bytes(K, p))
    return fail(SBO_EINVAL, "polar workspace too small");
  const size_t dyn = smem ? polar_smem_bytes(p) : 0;
  // p = 64: Newton-Schulz first; Jacobi only for the matrices it hands back
  static const bool force_jacobi = getenv("SBO_POLAR_JACOBI") != nullptr;
  const bool ns = p == 64 && status && !sigma && !force_jacobi;
  const bool ns_big = p > 64 && status && !sigma && !force_jacobi;
  if (ns_big) {  // batched DMMA Newton-Schulz; Jacobi below for what it hands back
    if (int rc = sbo_polar_ns_big(P, K, p, counts, Q, status, ws, ws_bytes, stream)) return rc;
  }
  if (ns) {
    static const bool single = getenv("SBO_POLAR_SINGLE_CTA") != nullptr;
    if (single) {
      const size_t nsb = sizeof(double) * 3 * 64 * 68;
      cudaFuncSetAttribute(k_polar_ns, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(nsb));
      k_polar_ns<<<K, kJacobiThreads, nsb, as_stream(stream)>>>(P, counts, Q, status);
      if (int rc = check_launch("k_polar_ns")) return rc;
    } else {
      // > half of an SM's shared memory: one CTA per SM, so the 8 CTAs of a
      // cluster run on 8 SMs (they would otherwise pack 3 to an SM)
      const size_t nsb = 120 * 1024;
      cudaFuncSetAttribute(k_polar_ns_cluster<4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(nsb));
      cudaFuncSetAttribute(k_polar_ns_cluster<8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(nsb));
      // 8-CTA clusters (half the DMMA work per SM per iteration) when all K of them
      // are co-resident; otherwise 4 (a second wave would cost more than it saves).
      // SBO_NS_CLUSTER = 4 or 8 forces the size.
      static const int max8 = [nsb] {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(8, 1, 1);
        cfg.blockDim = dim3(kJacobiThreads, 1, 1);
        cfg.dynamicSmemBytes = nsb;
        int n = 0;
        if (cudaOccupancyMaxActiveClusters(&n, k_polar_ns_cluster<8>, &cfg) != cudaSuccess) {
          cudaGetLastError();
          n = 0;
        }
        return n;
      }();
      static const int force = [] {
        const char* e = std::getenv("SBO_NS_CLUSTER");
        return e ? std::atoi(e) : 0;
      }();
      const bool c8 = force == 8 || (force != 4 && K <= max8);
      // Chen-Chow lower bound l0 for sigma_min(P) / ||P||_F: on the benchmark's patch
      // data the P matrices have ratios ~1e-5 .. 1e-4, where l0 = 1e-5 converges in
      // 17 iterations (1e-6: 19; 1e-4: 19-20; 1e-3: 23).  A ratio below l0 only
      // costs iterations (1e-6 with l0 = 1e-5: 23), never accuracy: the stop test
      // is on ||X^T X - I||.  SBO_NS_L0 overrides it.
      static const double l0 = [] {
        const char* e = std::getenv("SBO_NS_L0");
        return e ? std::atof(e) : 1e-5;
      }();
      if (c8)
        k_polar_ns_cluster<8><<<K * 8, kJacobiThreads, nsb, as_stream(stream)>>>(P, counts, Q,
                                                                               status, l0);
      else
        k_polar_ns_cluster<4><<<K * 4, kJacobiThreads, nsb, as_stream(stream)>>>(P, counts, Q,
                                                                               status, l0);
      if (int rc = check_launch("k_polar_ns_cluster")) return rc;
    }
  }
  if (smem) {
    cudaFuncSetAttribute(k_polar<true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(dyn));
    k_polar<true><<<K, kJacobiThreads, dyn, as_stream(stream)>>>(
        P, p, counts, Q, V, sigma, status, static_cast<double*>(ws), ns ? 1 : 0);
  } else {
    k_polar<false><<<K, kJacobiThreads, 0, as_stream(stream)>>>(
        P, p, counts, Q, V, sigma, status, static_cast<double*>(ws), ns_big ? 1 : 0);
  }
  return check_launch("k_polar");
}

extern "C" size_t sbo_init_workspace_bytes(int p) { return init_smem_bytes(p) + 64; }  // + 2 ints

extern "C" int sbo_init_block(const double* G, int p, int64_t ncols, const double* draws,
                              int ndraws, double* Q, int32_t* rank, int32_t* status, void* ws,
                              size_t ws_bytes, void* stream) {
  if (p < 1 || p > kPMax) return fail(SBO_EINVAL, "bad init shape");
  const bool smem = init_smem_bytes(p) <= kSmemBudget;
  if (!smem && ws_bytes < sbo_init_workspace_bytes(p))
    return fail(SBO_EINVAL, "init workspace too small");
  const size_t dyn = smem ? init_smem_bytes(p) : 0;
  if (smem) {
    if (p == 64) {  // 512 threads: one column pair per half-warp (jacobi_sweeps64)
      cudaFuncSetAttribute(k_init_block<true, 512>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           static_cast<int>(dyn));
      // lanes per Jacobi column pair (jacobi_sweeps64_lp); SBO_INIT_LP = 16 selects
      // the 512-thread jacobi_sweeps64 (A/B)
      static const int lp = [] {
        const char* e = std::getenv("SBO_INIT_LP");
        return e ? std::atoi(e) : 8;
      }();
      k_init_block<true, 512><<<1, 512, dyn, as_stream(stream)>>>(
          G, p, ncols, draws, ndraws, Q, rank, status, static_cast<double*>(ws), 1, nullptr, lp);
    } else {
      cudaFuncSetAttribute(k_init_block<true, kJacobiThreads>,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, static_cast<int>(dyn));
      k_init_block<true, kJacobiThreads><<<1, kJacobiThreads, dyn, as_stream(stream)>>>(
          G, p, ncols, draws, ndraws, Q, rank, status, static_cast<double*>(ws), 1, nullptr, 16);
    }
  } else {
    // large p: the sweeps on a cooperative grid, then the single-CTA finish
    double* A = static_cast<double*>(ws);
    double* V = A + static_cast<int64_t>(p) * p;
    int* aux = reinterpret_cast<int*>(static_cast<char*>(ws) + init_smem_bytes(p));
    k_fill_gram<<<p, 256, 0, as_stream(stream)>>>(G, p, A, V);
    int* flag = aux;
    int* sweeps = aux + 1;
    int rows = p, pp_ = p;
    void* args[] = {&A, &V, &rows, &pp_, &flag, &sweeps};
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const int blocks = (p / 2 + 7) / 8 < sms ? (p / 2 + 7) / 8 : sms;
    SBO_CHECK_CUDA(cudaLaunchCooperativeKernel(reinterpret_cast<void*>(k_jacobi_grid), blocks,
                                               256, args, 0, as_stream(stream)));
    k_init_block<false, kJacobiThreads><<<1, kJacobiThreads, 0, as_stream(stream)>>>(
        G, p, ncols, draws, ndraws, Q, rank, status, static_cast<double*>(ws), 0, sweeps, 16);
  }
  return check_launch("k_init_block");
}

// ---------------------------------------------------------------------------
// Thin SVD of a rows x cols matrix (rows >= cols), linalg.py:40-65: one-sided
// Jacobi on the columns, singular values descending (index tie-break), U
// columns with their largest-|entry| nonnegative (linalg.py:32-37), V matched.
// Directions with sigma <= 64 eps sigma_max get a deterministic orthonormal
// completion (the reference accepts whatever orthogonal factor its SVD yields
// for them, SPEC linalg-core design decisions).  Global-memory workspace.
// Outputs are row-major: U[rows][cols], V[cols][cols], S[cols].
__global__ void __launch_bounds__(kJacobiThreads) k_svd(const double* __restrict__ M, int rows,
                                                        int cols, double* U, double* S,
                                                        double* Vout, int32_t* status,
                                                        double* ws) {
  __shared__ JacobiSmem Sm;
  const int64_t rc = static_cast<int64_t>(rows) * cols;
  double* A = ws;                 // cols columns of length rows
  double* V = A + rc;             // cols x cols, column-major
  double* sig = V + static_cast<int64_t>(cols) * cols;
  int* ord = reinterpret_cast<int*>(sig + cols);
  for (int64_t e = threadIdx.x; e < rc; e += blockDim.x) {
    const int r = static_cast<int>(e / cols), c = static_cast<int>(e % cols);
    A[static_cast<int64_t>(c) * rows + r] = M[e];
  }
  for (int64_t e = threadIdx.x; e < static_cast<int64_t>(cols) * cols; e += blockDim.x)
    V[e] = (e / cols == e % cols) ? 1.0 : 0.0;
  __syncthreads();
  const int sweeps = jacobi_sweeps(A, V, rows, cols, &Sm.flag);
  column_order(A, rows, cols, sig, ord, true);
  const double smax = sig[ord[0]];
  const double null_tol = smax * 64.0 * DBL_EPSILON;
  for (int64_t e = threadIdx.x; e < rc; e += blockDim.x) {
    const int j = static_cast<int>(e / rows);
    if (sig[j] > null_tol) A[e] /= sig[j];
  }
  __syncthreads();
  for (int rnk = 0; rnk < cols; ++rnk) {
    const int j = ord[rnk];
    if (sig[j] > null_tol) continue;
    double* u = A + static_cast<int64_t>(j) * rows;
    for (int cand = 0; cand < rows; ++cand) {
      for (int r = threadIdx.x; r < rows; r += blockDim.x) u[r] = (r == cand) ? 1.0 : 0.0;
      __syncthreads();
      for (int pass = 0; pass < 2; ++pass) {
        for (int l = 0; l < cols; ++l) {
          const int jl = ord[l];
          if (jl == j || (sig[jl] <= null_tol && l > rnk)) continue;
          const double* w = A + static_cast<int64_t>(jl) * rows;
          double d = 0.0;
          for (int r = threadIdx.x; r < rows; r += blockDim.x) d = fma(w[r], u[r], d);
          d = block_sum<kJacobiThreads>(d, Sm.red);
          for (int r = threadIdx.x; r < rows; r += blockDim.x) u[r] -= d * w[r];
          __syncthreads();
        }
      }
      double nn = 0.0;
      for (int r = threadIdx.x; r < rows; r += blockDim.x) nn = fma(u[r], u[r], nn);
      nn = sqrt(block_sum<kJacobiThreads>(nn, Sm.red));
      if (nn > 1e-3) {
        for (int r = threadIdx.x; r < rows; r += blockDim.x) u[r] /= nn;
        __syncthreads();
        break;
      }
    }
  }
  __syncthreads();
  // canonical signs, sorted output
  for (int c = threadIdx.x; c < cols; c += blockDim.x) {
    const int j = ord[c];
    const double* u = A + static_cast<int64_t>(j) * rows;
    int piv = 0;
    double best = -1.0;
    for (int r = 0; r < rows; ++r)
      if (fabs(u[r]) > best) {
        best = fabs(u[r]);
        piv = r;
      }
    const double sgn = u[piv] < 0.0 ? -1.0 : 1.0;
    for (int r = 0; r < rows; ++r) U[static_cast<int64_t>(r) * cols + c] = sgn * u[r];
    const double* v = V + static_cast<int64_t>(j) * cols;
    for (int r = 0; r < cols; ++r) Vout[static_cast<int64_t>(r) * cols + c] = sgn * v[r];
    S[c] = sig[j];
  }
  if (threadIdx.x == 0 && status) *status = sweeps < 0 ? SBO_ST_NOCONV : SBO_ST_OK;
}

extern "C" size_t sbo_svd_workspace_bytes(int rows, int cols) {
  return sizeof(double) * (static_cast<size_t>(rows) * cols + static_cast<size_t>(cols) * cols +
                           2 * static_cast<size_t>(cols)) + 64;
}

extern "C" int sbo_svd(const double* M, int rows, int cols, double* U, double* S, double* V,
                       int32_t* status, void* ws, size_t ws_bytes, void* stream) {
  if (rows < 1 || cols < 1 || cols > rows) return fail(SBO_EINVAL, "sbo_svd needs rows >= cols >= 1");
  if (ws_bytes < sbo_svd_workspace_bytes(rows, cols)) return fail(SBO_EINVAL, "svd workspace too small");
  k_svd<<<1, kJacobiThreads, 0, as_stream(stream)>>>(M, rows, cols, U, S, V, status,
                                                     static_cast<double*>(ws));
  return check_launch("k_svd");
}
