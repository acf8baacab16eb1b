// Shared helpers of the sm_100a SBO kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>

#include "sbo_b200.h"

namespace sbo {

constexpr int kPMax = 256;      // largest supported signal dimension
constexpr int kTile = 64;       // signals per CTA tile of the float64 kernels
constexpr int kThreads = 256;   // threads per CTA of the float64 tile kernels

void set_error(const std::string& msg);

}  // namespace sbo

// round64.cu: Gram partials of a member list on DMMA (p <= 64)
// p = 256 tensor-core operand preparation (tc_energy256.cu)
int tc256_split_signals(const void* y, int dtype, int64_t m, int64_t m_pad, void* yh, void* yl,
                        int16_t* escale, cudaStream_t st);
int tc256_split_blocks(const double* Q, int K, void* qh, void* ql, int16_t* fscale,
                       cudaStream_t st);
int sbo_gram_partials64(const void* y, int dtype, int p, const int32_t* members,
                        const int64_t* seg_lo, const int64_t* seg_hi, const int32_t* nseg,
                        int64_t max_seg, double* partial, void* stream);

namespace sbo {
int fail(int code, const std::string& msg);
int check_launch(const char* what);

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

__host__ __device__ inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }
__host__ __device__ inline int64_t min64(int64_t a, int64_t b) { return a < b ? a : b; }

// order-preserving map of a nonnegative double to its bit pattern (residual keys)
__device__ __forceinline__ uint64_t key_of(double x) {
  return x > 0.0 ? static_cast<uint64_t>(__double_as_longlong(x)) : 0ull;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

__device__ __forceinline__ int warp_sum_int(int v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// deterministic CTA-wide sum (fixed tree), result valid in every thread
template <int NT>
__device__ double block_sum(double v, double* red) {
  v = warp_sum(v);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  double t = 0.0;
  if (w == 0) {
    t = (l < NT / 32) ? red[l] : 0.0;
    t = warp_sum(t);
    if (l == 0) red[0] = t;
  }
  __syncthreads();
  t = red[0];
  __syncthreads();
  return t;
}

}  // namespace sbo

#define SBO_CHECK_CUDA(expr)                                                         \
  do {                                                                               \
    cudaError_t _e = (expr);                                                         \
    if (_e != cudaSuccess)                                                           \
      return ::sbo::fail(SBO_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(_e)); \
  } while (0)
