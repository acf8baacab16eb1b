// Polar factors of p x p matrices for 64 < p <= 256 (linalg.py:68-78, config D: p =
// 256) by the same scaled Newton-Schulz iteration as the p = 64 cluster kernel,
//   X_0 = P / ||P||_F,  X_{k+1} = X_k (c1_k I + c3_k X_k^T X_k),
// with every product a batched float64 tensor-core (DMMA) GEMM over all matrices:
// one CTA per 64 x 64 output tile and matrix, K in 64-wide chunks staged in shared
// memory.  The first GEMM's epilogue forms A = c1 I + c3 G directly and the tile's
// part of ||G - I||_F^2; a check kernel sums the parts in a fixed order and retires
// the converged matrices (their later launches return at once).  Matrices are padded
// to a multiple of 64 with zeros, which the iteration keeps at zero.  Matrices that
// do not converge go to the one-sided Jacobi kernel, as for p = 64.
#include <cfloat>
#include <cstdlib>

#include "common.cuh"

namespace sbo {
namespace pbig {

constexpr int T = 64;
constexpr int LDS = 68;  // shared row stride (doubles): conflict-free DMMA fragments
constexpr int kMaxIter = 40;

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// X_0 = P / ||P||_F (zero padded to PP x PP); one CTA per matrix
__global__ void __launch_bounds__(256) k_ns_init(const double* __restrict__ P, int p, int PP,
                                                 const int64_t* __restrict__ counts, double* X,
                                                 int* done, int* final_buf, int32_t* status) {
  const int b = blockIdx.x;
  __shared__ double red[32];
  const double* Pb = P + static_cast<int64_t>(b) * p * p;
  double* Xb = X + static_cast<int64_t>(b) * PP * PP;
  if (counts && counts[b] == 0) {
    if (threadIdx.x == 0) {
      done[b] = 2;  // skipped
      status[b] = SBO_ST_SKIPPED;
    }
    return;
  }
  double s = 0.0;
  for (int e = threadIdx.x; e < p * p; e += 256) s = fma(Pb[e], Pb[e], s);
  const double nrm = sqrt(block_sum<256>(s, red));
  const double inv = nrm > 0.0 ? 1.0 / nrm : 0.0;
  for (int e = threadIdx.x; e < PP * PP; e += 256) {
    const int r = e / PP, c = e % PP;
    Xb[e] = (r < p && c < p) ? Pb[r * p + c] * inv : 0.0;
  }
  if (threadIdx.x == 0) {
    done[b] = nrm > 0.0 ? 0 : 3;  // 3: not converged (zero matrix) -> Jacobi
    final_buf[b] = 0;
  }
}

// C = op(A) B per matrix, TT x TT tile per CTA (TT = 64: 8 warps; TT = 32 for
// small batches: 4 warps, four times the CTAs of one matrix).  EPI = 1:
// C = c1 I + c3 (A^T B) and the tile's sum of (G - I)^2 over the valid p x p
// region into part[b][tile].
template <bool TRANS_A, int EPI, int TT>
__global__ void __launch_bounds__(TT * 4) k_ns_gemm(const double* __restrict__ A,
                                                   const double* __restrict__ B, double* C,
                                                   int p, int PP, const int* __restrict__ done,
                                                   double c1, double c3, double* part) {
  constexpr int NT = TT * 4, NF = TT / 8;  // threads; 8-column fragments per warp
  const int b = blockIdx.y;
  if (done[b]) return;
  extern __shared__ __align__(16) unsigned char dyn[];
  double* sA = reinterpret_cast<double*>(dyn);  // [i][k], stride LDS
  double* sB = sA + T * LDS;                      // [k][j], stride LDS
  __shared__ double red[32];
  const int nt = PP / TT;
  const int ti = blockIdx.x / nt, tj = blockIdx.x % nt;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t4 = lane & 3;
  const int64_t off = static_cast<int64_t>(b) * PP * PP;
  const double* Ab = A + off;
  const double* Bb = B + off;
  double acc[NF][2];
#pragma unroll
  for (int n = 0; n < NF; ++n) acc[n][0] = acc[n][1] = 0.0;
  for (int kc = 0; kc < PP; kc += T) {
    __syncthreads();
    for (int e = tid; e < TT * T; e += NT) {
      if (TRANS_A) {  // op(A)[i][k] = A[k][i]
        const int r = e / TT, c = e % TT;
        sA[c * LDS + r] = Ab[static_cast<int64_t>(kc + r) * PP + ti * TT + c];
      } else {
        const int r = e >> 6, c = e & 63;
        sA[r * LDS + c] = Ab[static_cast<int64_t>(ti * TT + r) * PP + kc + c];
      }
      const int rb = e / TT, cb = e % TT;
      sB[rb * LDS + cb] = Bb[static_cast<int64_t>(kc + rb) * PP + tj * TT + cb];
    }
    __syncthreads();
    const double* ya = sA + (8 * warp + g) * LDS + t4;
#pragma unroll 4
    for (int k0 = 0; k0 < T; k0 += 4) {
      const double a = ya[k0];
      const double* bb = sB + (k0 + t4) * LDS + g;
#pragma unroll
      for (int n = 0; n < NF; ++n) dmma(acc[n][0], acc[n][1], a, bb[8 * n]);
    }
  }
  const int row = ti * TT + 8 * warp + g;
  double dsum = 0.0;
#pragma unroll
  for (int n = 0; n < NF; ++n) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int col = tj * TT + 8 * n + 2 * t4 + h;
      double v = acc[n][h];
      if (EPI == 1) {
        const double delta = row == col ? 1.0 : 0.0;
        if (row < p && col < p) dsum = fma(v - delta, v - delta, dsum);
        v = c3 * v + c1 * delta;
      }
      acc[n][h] = v;
    }
    *reinterpret_cast<double2*>(C + off + static_cast<int64_t>(row) * PP + tj * TT + 8 * n +
                                2 * t4) = make_double2(acc[n][0], acc[n][1]);
  }
  if (EPI == 1) {
    dsum = block_sum<NT>(dsum, red);
    if (tid == 0) part[static_cast<int64_t>(b) * nt * nt + blockIdx.x] = dsum;
  }
}

// The 64 x 64 tile GEMM with its K chunks (32 wide) double-buffered by cp.async:
// the next chunk streams from L2 while the current one runs on DMMA.  op(A) for
// TRANS_A is staged untransposed ([k][i], rows of A) and read transposed.
// Strides keep every fragment read at the 2-wavefront minimum.
constexpr int KC = 32, LDA_N = KC + 4, LDA_T = T + 8, LDB = T + 8;
constexpr int STAGE_DBL = (T * LDA_N > KC * LDA_T ? T * LDA_N : KC * LDA_T) + KC * LDB;
constexpr size_t PIPE_SMEM = 2 * STAGE_DBL * sizeof(double);

__device__ __forceinline__ void cp16(double* dst, const double* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                   static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
               "l"(src));
}

template <bool TRANS_A, int EPI>
__global__ void __launch_bounds__(256) k_ns_gemm_pipe(const double* __restrict__ A,
                                                      const double* __restrict__ B, double* C,
                                                      int p, int PP, const int* __restrict__ done,
                                                      double c1, double c3, double* part) {
  const int b = blockIdx.y;
  if (done[b]) return;
  extern __shared__ __align__(16) unsigned char dyn[];
  double* stage[2] = {reinterpret_cast<double*>(dyn),
                      reinterpret_cast<double*>(dyn) + STAGE_DBL};
  __shared__ double red[32];
  const int nt = PP / T;
  const int ti = blockIdx.x / nt, tj = blockIdx.x % nt;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t4 = lane & 3;
  const int64_t off = static_cast<int64_t>(b) * PP * PP;
  const double* Ab = A + off;
  const double* Bb = B + off;
  constexpr int A_DBL = T * LDA_N > KC * LDA_T ? T * LDA_N : KC * LDA_T;
  auto issue = [&](int kc, double* st) {
    double* sA = st;
    double* sB = st + A_DBL;
    // 1024 16-B pieces per operand, 4 per thread
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int e = tid + 256 * u;
      if (TRANS_A) {  // rows k = kc .. kc + 31 of A, columns ti*T .. + 63
        const int r = e >> 5, c = 2 * (e & 31);
        cp16(sA + r * LDA_T + c, Ab + static_cast<int64_t>(kc + r) * PP + ti * T + c);
      } else {        // rows i = ti*T .. + 63 of A, columns kc .. kc + 31
        const int r = e >> 4, c = 2 * (e & 15);
        cp16(sA + r * LDA_N + c, Ab + static_cast<int64_t>(ti * T + r) * PP + kc + c);
      }
      const int rb = e >> 5, cb = 2 * (e & 31);
      cp16(sB + rb * LDB + cb, Bb + static_cast<int64_t>(kc + rb) * PP + tj * T + cb);
    }
    asm volatile("cp.async.commit_group;");
  };
  double acc[8][2];
#pragma unroll
  for (int n = 0; n < 8; ++n) acc[n][0] = acc[n][1] = 0.0;
  const int nk = PP / KC;
  issue(0, stage[0]);
  for (int c = 0; c < nk; ++c) {
    if (c + 1 < nk) {
      issue((c + 1) * KC, stage[(c + 1) & 1]);
      asm volatile("cp.async.wait_group 1;" ::: "memory");
    } else {
      asm volatile("cp.async.wait_group 0;" ::: "memory");
    }
    __syncthreads();
    const double* sA = stage[c & 1];
    const double* sB = sA + A_DBL;
#pragma unroll
    for (int k0 = 0; k0 < KC; k0 += 4) {
      const double a = TRANS_A ? sA[(k0 + t4) * LDA_T + 8 * warp + g]
                               : sA[(8 * warp + g) * LDA_N + k0 + t4];
      const double* bb = sB + (k0 + t4) * LDB + g;
#pragma unroll
      for (int n = 0; n < 8; ++n) dmma(acc[n][0], acc[n][1], a, bb[8 * n]);
    }
    __syncthreads();  // the stage is refilled two chunks later
  }
  const int row = ti * T + 8 * warp + g;
  double dsum = 0.0;
#pragma unroll
  for (int n = 0; n < 8; ++n) {
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int col = tj * T + 8 * n + 2 * t4 + h;
      double v = acc[n][h];
      if (EPI == 1) {
        const double delta = row == col ? 1.0 : 0.0;
        if (row < p && col < p) dsum = fma(v - delta, v - delta, dsum);
        v = c3 * v + c1 * delta;
      }
      acc[n][h] = v;
    }
    *reinterpret_cast<double2*>(C + off + static_cast<int64_t>(row) * PP + tj * T + 8 * n +
                                2 * t4) = make_double2(acc[n][0], acc[n][1]);
  }
  if (EPI == 1) {
    dsum = block_sum<256>(dsum, red);
    if (tid == 0) part[static_cast<int64_t>(b) * nt * nt + blockIdx.x] = dsum;
  }
}

// retire converged matrices: ||X_k^T X_k - I||_F < tol (parts summed in tile order)
__global__ void k_ns_check(const double* __restrict__ part, int ntile2, int K, int cur, int it,
                           int* done, int* final_buf, int* iters) {
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= K || done[b]) return;
  double s = 0.0;
  for (int t = 0; t < ntile2; ++t) s += part[static_cast<int64_t>(b) * ntile2 + t];
  if (sqrt(s) < 1e-13) {
    done[b] = 1;
    final_buf[b] = cur;
    iters[b] = it;
  }
}

__global__ void __launch_bounds__(256) k_ns_finish(const double* __restrict__ X0,
                                                   const double* __restrict__ X1, int p, int PP,
                                                   const int* done, const int* final_buf,
                                                   const int* iters, double* Q,
                                                   int32_t* status) {
  const int b = blockIdx.x;
  if (done[b] == 2) return;  // skipped (empty block): status already set
  if (done[b] != 1) {
    if (threadIdx.x == 0) status[b] = 4;  // kStNsFallback: the Jacobi kernel solves it
    return;
  }
  const double* X = (final_buf[b] ? X1 : X0) + static_cast<int64_t>(b) * PP * PP;
  double* Qb = Q + static_cast<int64_t>(b) * p * p;
  for (int e = threadIdx.x; e < p * p; e += 256) Qb[e] = X[(e / p) * PP + e % p];
  if (threadIdx.x == 0) status[b] = SBO_ST_OK | (iters[b] << 8) | (1 << 16);
}

}  // namespace pbig
}  // namespace sbo

using namespace sbo;

// workspace: 3 PP x PP buffers, the tile parts and 3 ints per matrix
extern "C" size_t sbo_polar_ns_big_workspace_bytes(int K, int p) {
  const int64_t PP = ceil_div(p, pbig::T) * pbig::T, nt = PP / 32;  // parts of 32-tiles
  return static_cast<size_t>(K) * (3 * PP * PP + nt * nt) * sizeof(double) +
         static_cast<size_t>(K) * 3 * sizeof(int) + 256;
}

int sbo_polar_ns_big(const double* P, int K, int p, const int64_t* counts, double* Q,
                     int32_t* status, void* ws, size_t ws_bytes, void* stream) {
  if (ws_bytes < sbo_polar_ns_big_workspace_bytes(K, p)) return fail(SBO_EINVAL, "polar workspace too small");
  cudaStream_t st = as_stream(stream);
  const int PP = static_cast<int>(ceil_div(p, pbig::T) * pbig::T), nt = PP / pbig::T;
  const int64_t mat = static_cast<int64_t>(PP) * PP;
  double* X[2] = {static_cast<double*>(ws), static_cast<double*>(ws) + K * mat};
  double* Am = X[1] + K * mat;
  double* part = Am + K * mat;
  int* done = reinterpret_cast<int*>(part + static_cast<int64_t>(K) * (PP / 32) * (PP / 32));
  int* final_buf = done + K;
  int* iters = final_buf + K;
  pbig::k_ns_init<<<K, 256, 0, st>>>(P, p, PP, counts, X[0], done, final_buf, status);
  // small batches (the new block's rounds): 32 x 32 tiles, 4x the CTAs
  const bool small = K <= 4;
  const int TT = small ? 32 : pbig::T, ntt = PP / TT;
  const dim3 grid(static_cast<unsigned>(ntt * ntt), static_cast<unsigned>(K));
  // larger batches: the cp.async-pipelined 64 x 64 GEMM
  const int smem = small ? static_cast<int>(2 * pbig::T * pbig::LDS * sizeof(double))
                         : static_cast<int>(pbig::PIPE_SMEM);
  auto g1 = small ? pbig::k_ns_gemm<true, 1, 32> : pbig::k_ns_gemm_pipe<true, 1>;
  auto g0 = small ? pbig::k_ns_gemm<false, 0, 32> : pbig::k_ns_gemm_pipe<false, 0>;
  cudaFuncSetAttribute(g1, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  cudaFuncSetAttribute(g0, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  // lower bound of sigma_min / ||P||_F for the scaling (a ratio below it only costs
  // iterations, never accuracy: the stop test is on ||X^T X - I||)
  static const double l0 = [] {
    const char* e = std::getenv("SBO_NS_L0_BIG");
    return e ? std::atof(e) : 1e-6;
  }();
  double l = l0;
  int cur = 0;
  for (int it = 0; it < pbig::kMaxIter; ++it) {
    const double al = l < 0.99 ? sqrt(3.0 / (1.0 + l + l * l)) : 1.0;
    const double c1 = 1.5 * al, c3 = -0.5 * al * al * al;
    g1<<<grid, TT * 4, smem, st>>>(X[cur], X[cur], Am, p, PP, done, c1, c3, part);
    pbig::k_ns_check<<<(K + 127) / 128, 128, 0, st>>>(part, ntt * ntt, K, cur, it, done,
                                                        final_buf, iters);
    g0<<<grid, TT * 4, smem, st>>>(X[cur], Am, X[cur ^ 1], p, PP, done, 0.0, 0.0, nullptr);
    l = fmin(1.0, al * l * (3.0 - al * al * l * l) * 0.5);
    cur ^= 1;
  }
  pbig::k_ns_finish<<<K, 256, 0, st>>>(X[0], X[1], p, PP, done, final_buf, iters, Q, status);
  return check_launch("polar_ns_big");
}
