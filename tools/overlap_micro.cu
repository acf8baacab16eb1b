// Do tcgen05 kind::i8 MMAs (issued by one thread) and DMMA (mma.sync f64 in the
// other warps) share the tensor pipe on B200?  Times each alone and both together
// in one CTA per SM (the shape of a hybrid round kernel: int8 Ozaki projection on
// tcgen05, float64 outer product on DMMA).
#include <cstdio>

#include "sm100.cuh"

using namespace sbo;

constexpr int M = 128, N = 64, KT = 128;

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
__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// mode bit 0: tcgen05 MMAs (thread 0), bit 1: DMMA loops (warps 1..7)
__global__ void __launch_bounds__(256, 1) k_mix(int mode, int umma_reps, int dmma_reps,
                                                double* out) {
  extern __shared__ unsigned char raw[];
  const uint32_t base = sm100::smem_u32(raw);
  int8_t* sa = reinterpret_cast<int8_t*>(raw + ((1024u - (base & 1023u)) & 1023u));
  int8_t* sb = sa + M * KT;
  __shared__ uint64_t done;
  __shared__ uint32_t slot;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  for (int e = tid; e < (M + N) * KT; e += 256) sa[e] = static_cast<int8_t>(e * 7);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (tid == 0) {
    sm100::mbar_init(&done, 1);
    sm100::fence_barrier_init();
  }
  if (warp == 0) sm100::tmem_alloc(&slot, 512);
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem = slot;
  double acc = 0.0;
  if (tid == 0 && (mode & 1)) {
    const uint32_t a0 = sm100::smem_u32(sa), b0 = sm100::smem_u32(sb), id = idesc_i8(M, N);
    for (int r = 0; r < umma_reps; ++r)
#pragma unroll
      for (int kk = 0; kk < 4; ++kk)
        umma_i8(tmem + (r & 7) * N, sm100::desc_sw128(a0 + kk * 32),
                sm100::desc_sw128(b0 + kk * 32), id, kk > 0 ? 1u : 0u);
    sm100::umma_commit(&done);
  }
  if (warp >= 1 && (mode & 2)) {
    double c[8][2];
    for (int n = 0; n < 8; ++n) c[n][0] = c[n][1] = 0.0;
    const double a = 1.0 + lane * 1e-3, b = 1.0 - lane * 1e-3;
    for (int r = 0; r < dmma_reps; ++r)
#pragma unroll
      for (int n = 0; n < 8; ++n) dmma(c[n][0], c[n][1], a, b);
    for (int n = 0; n < 8; ++n) acc += c[n][0] + c[n][1];
  }
  if (mode & 1) sm100::mbar_wait(&done, 0);
  if (acc == 12345.0) out[0] = acc;
  sm100::tc_fence_before();
  __syncthreads();
  if (warp == 0) sm100::tmem_dealloc(tmem, 512);
}

int main() {
  double* d;
  cudaMalloc(&d, 64);
  const int smem = (M + N) * KT + 1024;
  cudaFuncSetAttribute(k_mix, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  const int ur = 20000, dr = 20000;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float t[4] = {0, 0, 0, 0};
  for (int pass = 0; pass < 2; ++pass)
    for (int mode = 1; mode <= 3; ++mode) {
      cudaEventRecord(e0);
      k_mix<<<148, 256, smem>>>(mode, ur, dr, d);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&t[mode], e0, e1);
    }
  const double uops = 2.0 * M * N * KT * ur * 148, dflop = 2.0 * 8 * 8 * 4 * 8 * dr * 7 * 148;
  printf("tcgen05 i8 128x64x32 alone: %.2f ms (%.0f TOPS)\n", t[1], uops / (t[1] * 1e-3) / 1e12);
  printf("DMMA (7 warps) alone:       %.2f ms (%.1f TFLOP/s)\n", t[2], dflop / (t[2] * 1e-3) / 1e12);
  printf("both together:              %.2f ms (sum of the two alone: %.2f ms)\n", t[3], t[1] + t[2]);
  return 0;
}
