// Streaming persistence of codes: the float64 payloads of
// the ODM1 records store.py:99-115 (save_sbo_codes) writes, produced on the device
// for a signal range so the host only streams bytes to the file.
//
// The records are column-major (data.py:232-237, tobytes(order="F")):
//   0: block as float64, 1 x m        3: energy, 1 x m
//   1: indices as float64, k x m      4: residual_sq, 1 x m
//   2: values, k x m
// so signal j's k entries of records 1 / 2 are contiguous; the device code keeps
// them as k rows of stride ld (int16 indices, float64 values).  Records 3 and 4
// are the device arrays themselves (no kernel); 0, 1, 2 are converted here.  One
// thread per output element, reads of the k-row layout coalesced along j.
#include "common.cuh"

namespace sbo {

__global__ void k_pack_block(const int32_t* __restrict__ block, int64_t n, double* __restrict__ out) {
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x)
    out[i] = static_cast<double>(block[i]);
}

// out[(j - j0) * k + t] = src[t * ld + j]: a 32-signal x k tile through shared memory
template <typename TS>
__global__ void __launch_bounds__(256) k_pack_rows(const TS* __restrict__ src, int64_t ld, int k,
                                                   int64_t j0, int64_t n, double* __restrict__ out) {
  __shared__ double tile[64 * 33];
  const int64_t jb = j0 + static_cast<int64_t>(blockIdx.x) * 32;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  for (int t0 = 0; t0 < k; t0 += 64) {
    const int kt = k - t0 < 64 ? k - t0 : 64;
    for (int t = w; t < kt; t += 8) {  // coalesced along j
      const int64_t j = jb + lane;
      tile[t * 33 + lane] = j < j0 + n ? static_cast<double>(src[(t0 + t) * ld + j]) : 0.0;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < 32 * kt; e += 256) {  // coalesced along the output
      const int s = e / kt, t = e - s * kt;
      const int64_t j = jb + s;
      if (j < j0 + n) out[(j - j0) * k + t0 + t] = tile[t * 33 + s];
    }
    __syncthreads();
  }
}

}  // namespace sbo

using namespace sbo;

extern "C" int sbo_codes_pack(int record, const int32_t* block, const int16_t* indices,
                              const double* values, int64_t ld, int k, int64_t j0, int64_t n,
                              double* out, void* stream) {
  if (n < 0 || j0 < 0) return fail(SBO_EINVAL, "bad signal range");
  if (k < 1 && (record == 1 || record == 2)) return fail(SBO_EINVAL, "k must be at least 1");
  if (n == 0) return SBO_OK;
  const cudaStream_t st = as_stream(stream);
  switch (record) {
    case 0: {
      int64_t g = ceil_div(n, 256);
      k_pack_block<<<static_cast<unsigned>(g < 148 * 16 ? g : 148 * 16), 256, 0, st>>>(block + j0, n, out);
      return check_launch("k_pack_block");
    }
    case 1:
      k_pack_rows<int16_t><<<static_cast<unsigned>(ceil_div(n, 32)), 256, 0, st>>>(indices, ld, k, j0, n, out);
      return check_launch("k_pack_rows<idx>");
    case 2:
      k_pack_rows<double><<<static_cast<unsigned>(ceil_div(n, 32)), 256, 0, st>>>(values, ld, k, j0, n, out);
      return check_launch("k_pack_rows<val>");
    default:
      return fail(SBO_EINVAL, "record must be 0 (block), 1 (indices) or 2 (values)");
  }
}
