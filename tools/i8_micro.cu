// tcgen05 kind::i8 on B200: exactness of the int32 accumulation and throughput of
// 128x256x32 UMMAs from 128-B-swizzled shared tiles (the building block of an
// int8 Ozaki float64 projection).  One CTA per SM.
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "sm100.cuh"

using namespace sbo;

constexpr int M = 128, N = 256, KT = 128;  // K per tile: one 128-B swizzle atom of int8

__host__ __device__ constexpr uint32_t idesc_i8(int m, int n) {
  // D = s32 (2 << 4), A = B = s8 (1 << 7, 1 << 10), K-major, N >> 3 at 17, M >> 4 at 24
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

__global__ void __launch_bounds__(128, 1) k_i8(const int8_t* A, const int8_t* B, int reps,
                                               int32_t* out) {
  extern __shared__ unsigned char raw[];
  const uint32_t base = sm100::smem_u32(raw);
  int8_t* sa = reinterpret_cast<int8_t*>(raw + ((1024u - (base & 1023u)) & 1023u));
  int8_t* sb = sa + M * KT;
  __shared__ uint64_t done;
  __shared__ uint32_t tmem_slot;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int e = tid; e < M * KT; e += 128) {
    const int r = e / KT, k = e % KT;
    sa[(r >> 3) * 1024 + sm100::sw128_offset(r & 7, k)] = A[e];
  }
  for (int e = tid; e < N * KT; e += 128) {
    const int r = e / KT, k = e % KT;
    sb[(r >> 3) * 1024 + sm100::sw128_offset(r & 7, k)] = B[e];
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (tid == 0) {
    sm100::mbar_init(&done, 1);
    sm100::fence_barrier_init();
  }
  if (warp == 0) sm100::tmem_alloc(&tmem_slot, 256);
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem = tmem_slot;
  if (tid == 0) {
    const uint32_t a0 = sm100::smem_u32(sa), b0 = sm100::smem_u32(sb);
    const uint32_t id = idesc_i8(M, N);
    for (int r = 0; r < reps; ++r)
#pragma unroll
      for (int kk = 0; kk < KT / 32; ++kk)
        umma_i8(tmem, sm100::desc_sw128(a0 + kk * 32), sm100::desc_sw128(b0 + kk * 32), id,
                (r > 0 || kk > 0) ? 1u : 0u);
    sm100::umma_commit(&done);
  }
  sm100::mbar_wait(&done, 0);
  sm100::tc_fence_after();
  if (blockIdx.x == 0) {
    for (int c = 0; c < N; c += 64) {
      float v[64];
      sm100::tmem_ld64(tmem + (static_cast<uint32_t>(32 * warp) << 16) + c, v);
      for (int i = 0; i < 64; ++i) out[(32 * warp + (tid & 31)) * N + c + i] = __float_as_int(v[i]);
    }
  }
  sm100::tc_fence_before();
  __syncthreads();
  if (warp == 0) sm100::tmem_dealloc(tmem, 256);
}

int main() {
  std::vector<int8_t> A(M * KT), B(N * KT);
  srand(7);
  for (auto& x : A) x = static_cast<int8_t>(rand() % 255 - 127);
  for (auto& x : B) x = static_cast<int8_t>(rand() % 255 - 127);
  int8_t *dA, *dB;
  int32_t* dO;
  cudaMalloc(&dA, A.size());
  cudaMalloc(&dB, B.size());
  cudaMalloc(&dO, M * N * 4);
  cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice);
  // exactness: reps = 8 -> |sum| <= 8 * 128 * 127^2 < 2^31
  const int reps_chk = 8;
  const int smem = M * KT + N * KT + 1024;
  cudaFuncSetAttribute(k_i8, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k_i8<<<1, 128, smem>>>(dA, dB, reps_chk, dO);
  std::vector<int32_t> O(M * N);
  cudaError_t err = cudaMemcpy(O.data(), dO, O.size() * 4, cudaMemcpyDeviceToHost);
  if (err != cudaSuccess) {
    printf("error %s\n", cudaGetErrorString(err));
    return 1;
  }
  long bad = 0;
  for (int i = 0; i < M; ++i)
    for (int j = 0; j < N; ++j) {
      long s = 0;
      for (int k = 0; k < KT; ++k) s += static_cast<long>(A[i * KT + k]) * B[j * KT + k];
      if (static_cast<long>(O[i * N + j]) != s * reps_chk) ++bad;
    }
  printf("exactness: %ld of %d int32 accumulators differ from the CPU sum\n", bad, M * N);
  // throughput
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int reps = 20000;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k_i8<<<sms, 128, smem>>>(dA, dB, 100, dO);
  cudaEventRecord(e0);
  k_i8<<<sms, 128, smem>>>(dA, dB, reps, dO);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double ops = 2.0 * M * N * KT * reps * static_cast<double>(sms);
  printf("kind::i8 128x256x32 UMMAs: %.1f TOPS dense (%d SMs, %d x %d MMAs, %.2f ms)\n",
         ops / (ms * 1e-3) / 1e12, sms, reps, KT / 32, ms);
  return 0;
}
