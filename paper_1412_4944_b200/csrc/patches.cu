// Device-side signal ingestion: random square patches of a
// grayscale grid vectorized into signal rows — data.py:182-208 (extract_patches)
// after its corner draws, which stay on the host (numpy PCG64, bit-identical).
//
// Patch j's entry k = c*e + r (column-major vectorization, data.py:203-204) is
// grid[(row_j + r) * ld + col_j + c] / 255 in float64 (data.py:205).  Unit range:
// one thread per (patch, patch row) — e contiguous grid bytes in, e stores that
// a warp's lanes fill as 32-B runs; an 8-bit grid goes through a 256-entry
// table of k/255 in shared memory (no float64 division per element).  The
// dc-removed variant (data.py:206-207): one warp per patch subtracting the patch
// mean computed exactly as numpy's float64 add.reduce over a contiguous axis:
// pairwise summation (blocks of <= 128 with 8 interleaved accumulators, halving
// above that, plain accumulation below 8), then a true division by e^2 — so the
// rows are bit-identical to the reference's columns.  Output rows are float64,
// or float32 (the benchmark's float32-rounded signals; round-to-nearest of the
// float64 value).  The grid (4 MB for a 2048^2 8-bit scene) stays in L2.
#include "common.cuh"

namespace sbo {

enum { GRID_U8 = 0, GRID_F64 = 1 };
enum { NORM_UNIT = 0, NORM_UNIT_DC = 1 };

// numpy's pairwise_sum (umath loops_utils.h.src) over a[0 .. n)
__device__ double np_pairwise_sum(const double* a, int n) {
  if (n < 8) {
    double res = 0.0;
    for (int i = 0; i < n; ++i) res += a[i];
    return res;
  }
  if (n <= 128) {
    double r[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = a[j];
    int i = 8;
    for (; i < n - (n % 8); i += 8)
#pragma unroll
      for (int j = 0; j < 8; ++j) r[j] += a[i + j];
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; ++i) res += a[i];
    return res;
  }
  int n2 = n / 2;
  n2 -= n2 % 8;
  return np_pairwise_sum(a, n2) + np_pairwise_sum(a + n2, n - n2);
}

constexpr int kPatchWarps = 8;
constexpr int kMaxPatchElems = 1024;  // e <= 32

template <typename TG, typename TO>
__global__ void __launch_bounds__(256) k_patches_unit(
    const TG* __restrict__ grid, int64_t ld, int e, const int32_t* __restrict__ rows,
    const int32_t* __restrict__ cols, int64_t count, TO* __restrict__ out) {
  __shared__ TO lut[256];  // k/255 rounded to the output type
  if constexpr (sizeof(TG) == 1) {
    lut[threadIdx.x] = static_cast<TO>(static_cast<double>(threadIdx.x) / 255.0);
    __syncthreads();
  }
  const int64_t total = count * e, n = static_cast<int64_t>(e) * e;
  const bool small = total < (int64_t(1) << 32);
  for (int64_t t = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; t < total;
       t += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int64_t j;
    int r;
    if (small) {
      const unsigned tu = static_cast<unsigned>(t), ju = tu / static_cast<unsigned>(e);
      j = ju;
      r = static_cast<int>(tu - ju * static_cast<unsigned>(e));
    } else {
      j = t / e;
      r = static_cast<int>(t - j * e);
    }
    const TG* src = grid + static_cast<int64_t>(rows[j] + r) * ld + cols[j];
    TO* o = out + j * n + r;
    if constexpr (sizeof(TG) == 1) {
      // the patch row in aligned 4-byte words (<= 9 for e <= 32), realigned by
      // funnel shifts: 3 loads instead of 8 for e = 8 (the loads, one L1
      // wavefront per lane, are what bounds this kernel)
      const uintptr_t ad = reinterpret_cast<uintptr_t>(src);
      const uint32_t* wp = reinterpret_cast<const uint32_t*>(ad & ~uintptr_t(3));
      const int sh = static_cast<int>(ad & 3u) * 8, nw = (static_cast<int>(ad & 3u) + e + 3) >> 2;
      uint32_t wv[9];
#pragma unroll
      for (int i = 0; i < 9; ++i) wv[i] = i < nw ? __ldg(wp + i) : 0u;
#pragma unroll
      for (int i = 0; i < 8; ++i) wv[i] = __funnelshift_r(wv[i], wv[i + 1], sh);
#pragma unroll
      for (int c = 0; c < 32; ++c)
        if (c < e) o[c * e] = lut[(wv[c >> 2] >> (8 * (c & 3))) & 0xffu];
    } else {
      for (int c = 0; c < e; ++c) o[c * e] = static_cast<TO>(static_cast<double>(src[c]) / 255.0);
    }
  }
}

template <typename TG, typename TO>
__global__ void __launch_bounds__(32 * kPatchWarps) k_extract_patches(
    const TG* __restrict__ grid, int64_t ld, int e, const int32_t* __restrict__ rows,
    const int32_t* __restrict__ cols, int64_t count, int norm, TO* __restrict__ out) {
  extern __shared__ double sv[];  // [warp][n] (dc-removed only)
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int n = e * e;
  double* buf = sv + static_cast<int64_t>(warp) * n;
  for (int64_t j = static_cast<int64_t>(blockIdx.x) * kPatchWarps + warp; j < count;
       j += static_cast<int64_t>(gridDim.x) * kPatchWarps) {
    const TG* g0 = grid + static_cast<int64_t>(rows[j]) * ld + cols[j];
    TO* o = out + j * n;
    for (int k = lane; k < n; k += 32) {
      const int c = k / e, r = k - c * e;
      buf[k] = static_cast<double>(g0[static_cast<int64_t>(r) * ld + c]) / 255.0;
    }
    __syncwarp();
    double mean = 0.0;
    if (lane == 0) mean = np_pairwise_sum(buf, n) / static_cast<double>(n);
    mean = __shfl_sync(0xffffffffu, mean, 0);
    for (int k = lane; k < n; k += 32) o[k] = static_cast<TO>(buf[k] - mean);
    __syncwarp();
  }
}

template <typename TG, typename TO>
int launch_extract(const void* grid, int64_t ld, int e, const int32_t* rows, const int32_t* cols,
                   int64_t count, int norm, void* out, cudaStream_t st) {
  if (norm == NORM_UNIT) {
    int64_t blocks = ceil_div(count * e, 256);
    if (blocks > 148 * 32) blocks = 148 * 32;
    k_patches_unit<TG, TO><<<static_cast<unsigned>(blocks), 256, 0, st>>>(
        static_cast<const TG*>(grid), ld, e, rows, cols, count, static_cast<TO*>(out));
    return check_launch("k_patches_unit");
  }
  const size_t smem = sizeof(double) * kPatchWarps * e * e;
  if (smem > 48 * 1024)
    cudaFuncSetAttribute(k_extract_patches<TG, TO>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         static_cast<int>(smem));
  int64_t blocks = ceil_div(count, kPatchWarps);
  if (blocks > 148 * 64) blocks = 148 * 64;
  k_extract_patches<TG, TO><<<static_cast<unsigned>(blocks), 32 * kPatchWarps, smem, st>>>(
      static_cast<const TG*>(grid), ld, e, rows, cols, count, norm, static_cast<TO*>(out));
  return check_launch("k_extract_patches");
}

}  // namespace sbo

using namespace sbo;

extern "C" int sbo_extract_patches(const void* grid, int grid_dtype, int64_t h, int64_t w,
                                   int64_t ld, int edge, const int32_t* rows,
                                   const int32_t* cols, int64_t count, int normalization,
                                   int out_dtype, void* out, void* stream) {
  if (grid_dtype != GRID_U8 && grid_dtype != GRID_F64) return fail(SBO_EINVAL, "bad grid dtype");
  if (out_dtype != SBO_F32 && out_dtype != SBO_F64) return fail(SBO_EINVAL, "bad output dtype");
  if (normalization != NORM_UNIT && normalization != NORM_UNIT_DC)
    return fail(SBO_EINVAL, "bad normalization");
  if (edge < 1 || edge * edge > kMaxPatchElems) return fail(SBO_EINVAL, "patch edge must be in [1, 32]");
  if (h < edge || w < edge) return fail(SBO_EINVAL, "grid is smaller than a patch");
  if (ld < w) return fail(SBO_EINVAL, "grid row stride is smaller than its width");
  if (count < 0) return fail(SBO_EINVAL, "count must be non-negative");
  if (count == 0) return SBO_OK;
  const cudaStream_t st = as_stream(stream);
  if (grid_dtype == GRID_U8)
    return out_dtype == SBO_F32
               ? launch_extract<uint8_t, float>(grid, ld, edge, rows, cols, count, normalization, out, st)
               : launch_extract<uint8_t, double>(grid, ld, edge, rows, cols, count, normalization, out, st);
  return out_dtype == SBO_F32
             ? launch_extract<double, float>(grid, ld, edge, rows, cols, count, normalization, out, st)
             : launch_extract<double, double>(grid, ld, edge, rows, cols, count, normalization, out, st);
}
