// Micro test: tcgen05.mma kind::i8 with an MN-major B operand (the signal-major
// digit rows of sbo_y_digits used as B = Y^T without a transpose).  B is stored
// as 5 digit planes of [128 K rows][64 B] (N = 64 dims per plane), 64-B swizzle
// (16-B chunk ^= (row >> 1) & 3), planes 8 KB apart: an N-stack of planes
// a0..a1 is one MN-major operand with LBO = 8 KB (stride between 64-element
// MN atoms) and SBO = 512 B (stride between 8-row K groups).  A is K-major SW128
// (M = 128 rows of K = 128).  Every N-stack start plane 0..4 and lengths 1..4 are
// checked against a CPU sum; also reports the MMA rate.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 \
//        -Ipaper_1412_4944_b200/csrc -Iinclude tools/mn_micro.cu -o tools/mn_micro
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "sm100.cuh"

using namespace sbo;

constexpr int M = 128, KT = 128, NP = 5, PN = 64;  // K = signals, 5 planes of 64 dims
constexpr int A_BYTES = M * KT;                     // SW128 K-major, 16 KB
constexpr int PLANE = KT * PN;                      // 8 KB

__host__ __device__ constexpr uint32_t idesc_i8(int m, int n, bool b_mn) {
  return (2u << 4) | (1u << 7) | (1u << 10) | (b_mn ? (1u << 16) : 0u) |
         (static_cast<uint32_t>(n >> 3) << 17) | (static_cast<uint32_t>(m >> 4) << 24);
}
__device__ __forceinline__ void umma_i8(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc,
                                        uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(acc));
}
// MN-major, 64-B swizzle: LBO = stride between MN atoms, SBO = stride between
// 8-row K groups (both in 16-B units)
__device__ __forceinline__ uint64_t desc_mn_sw64(uint32_t addr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((addr >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32;
  d |= static_cast<uint64_t>(1) << 46;
  d |= static_cast<uint64_t>(4) << 61;  // SWIZZLE_64B
  return d;
}
__host__ __device__ inline uint32_t sw64_off(int row, int byte) {
  return row * 64u + ((((byte >> 4) ^ ((row >> 1) & 3)) << 4) | (byte & 15));
}

// out[which][128][N]: D for N-stack (a0, len) combos
__global__ void k_mn(const int8_t* ga, const int8_t* gb, int a0, int len, int reps,
                     int32_t* out) {
  extern __shared__ unsigned char raw[];
  const uint32_t base = sm100::smem_u32(raw);
  unsigned char* s = raw + ((1024u - (base & 1023u)) & 1023u);
  int8_t* sa = reinterpret_cast<int8_t*>(s);
  int8_t* sb = sa + A_BYTES;
  __shared__ uint64_t done;
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x, warp = tid >> 5;
  // A: row m, K byte k -> SW128
  for (int e = tid; e < M * KT; e += 128) {
    const int m = e / KT, k = e % KT;
    sa[(m >> 3) * 1024 + sm100::sw128_offset(m & 7, k)] = ga[e];
  }
  // B: gb[k][a][d] (signal-major digit rows) -> plane a, row k, byte d (SW64)
  for (int e = tid; e < KT * NP * PN; e += 128) {
    const int k = e / (NP * PN), a = (e / PN) % NP, d = e % PN;
    sb[a * PLANE + sw64_off(k, d)] = gb[e];
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (tid == 0) {
    sm100::mbar_init(&done, 1);
    sm100::fence_barrier_init();
  }
  if (warp == 0) sm100::tmem_alloc(&tslot, 256);
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem = tslot;
  const int n = len * PN;
  if (tid == 0) {
    const uint32_t ab = sm100::smem_u32(sa), bb = sm100::smem_u32(sb) + a0 * PLANE;
    for (int r = 0; r < reps; ++r)
      for (int kk = 0; kk < KT / 32; ++kk)
        umma_i8(tmem, sm100::desc_sw128(ab + kk * 32),
                desc_mn_sw64(bb + kk * 32 * 64, PLANE, 512), idesc_i8(M, n, true),
                (r > 0 || kk > 0) ? 1u : 0u);
    sm100::umma_commit(&done);
  }
  __syncwarp();
  sm100::mbar_wait(&done, 0);
  sm100::tc_fence_after();
  for (int c0 = 0; c0 < n; c0 += 8) {
    uint32_t v[8];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]),
                   "=r"(v[6]), "=r"(v[7])
                 : "r"(tmem + (static_cast<uint32_t>(32 * warp) << 16) + c0));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    if (out)
      for (int j = 0; j < 8; ++j) out[tid * 256 + c0 + j] = static_cast<int32_t>(v[j]);
  }
  sm100::tc_fence_before();
  __syncthreads();
  if (warp == 0) sm100::tmem_dealloc(tmem, 256);
}

int main() {
  std::vector<int8_t> A(M * KT), B(KT * NP * PN);
  srand(11);
  for (auto& x : A) x = static_cast<int8_t>(rand() % 255 - 127);
  for (auto& x : B) x = static_cast<int8_t>(rand() % 255 - 127);
  int8_t *dA, *dB;
  int32_t* dO;
  cudaMalloc(&dA, A.size());
  cudaMalloc(&dB, B.size());
  cudaMalloc(&dO, M * 256 * 4);
  cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice);
  const int smem = A_BYTES + NP * PLANE + 2048;
  cudaFuncSetAttribute(k_mn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  long total_bad = 0;
  for (int a0 = 0; a0 < NP; ++a0)
    for (int len = 1; len <= 4 && a0 + len <= NP; ++len) {
      cudaMemset(dO, 0, M * 256 * 4);
      k_mn<<<1, 128, smem>>>(dA, dB, a0, len, 1, dO);
      std::vector<int32_t> O(M * 256);
      cudaError_t err = cudaMemcpy(O.data(), dO, O.size() * 4, cudaMemcpyDeviceToHost);
      if (err != cudaSuccess) {
        printf("a0=%d len=%d: CUDA error %s\n", a0, len, cudaGetErrorString(err));
        return 1;
      }
      long bad = 0;
      for (int m = 0; m < M; ++m)
        for (int j = 0; j < len * PN; ++j) {
          const int a = a0 + j / PN, d = j % PN;
          long s = 0;
          for (int k = 0; k < KT; ++k)
            s += static_cast<long>(A[m * KT + k]) * B[(k * NP + a) * PN + d];
          if (O[m * 256 + j] != s) ++bad;
        }
      printf("N-stack planes %d..%d (N = %d): %ld of %d differ\n", a0, a0 + len - 1, len * PN,
             bad, M * len * PN);
      total_bad += bad;
    }
  printf("MN-major SW64 int8 B: %s\n", total_bad ? "MISMATCH" : "exact");
  // rate of the N = 256 shape from MN-major B
  int sms = 148;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int reps = 20000;
  k_mn<<<sms, 128, smem>>>(dA, dB, 0, 4, 100, nullptr);
  cudaEventRecord(e0);
  k_mn<<<sms, 128, smem>>>(dA, dB, 0, 4, reps, nullptr);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  printf("128x256x32 MN-major B: %.1f TOPS (%.2f ms)\n",
         2.0 * M * 256 * KT * reps * static_cast<double>(sms) / (ms * 1e-3) / 1e12, ms);
  return 0;
}
