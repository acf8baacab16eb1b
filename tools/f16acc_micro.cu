// How tcgen05.mma kind::f16 accumulates into fp32 TMEM on B200: the premise of the
// energy pass's certificate (coef_err in tc_energy.cu).
// 128 test rows (A) x 64 columns (B), K = 64 = 4 MMAs of K = 16, fp16 operands.
// Every result is compared with the exact dot product (__float128 on the host) and
// with model E: each MMA adds its 16 exact products to the accumulator with ONE
// round-to-nearest to fp32, and model Z: the same with one truncation toward zero.  Rows 0-7 are crafted cases (sub-ulp addends before and
// after a large one, cancellation); rows 8-127 are random mixed-magnitude vectors.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include <cuda_fp16.h>

#include "sm100.cuh"

using namespace sbo;

constexpr int M = 128, N = 64, KT = 64;  // KT fp16 = one 128-B swizzle row

__global__ void __launch_bounds__(128, 1) k_f16(const __half* A, const __half* B, float* out) {
  extern __shared__ unsigned char raw[];
  const uint32_t base = sm100::smem_u32(raw);
  unsigned char* sa = raw + ((1024u - (base & 1023u)) & 1023u);
  unsigned char* sb = sa + M * KT * 2;
  __shared__ uint64_t done;
  __shared__ uint32_t tmem_slot;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int e = tid; e < M * KT; e += 128) {
    const int r = e / KT, k = e % KT;
    *reinterpret_cast<__half*>(sa + (r >> 3) * 1024 + sm100::sw128_offset(r & 7, 2 * k)) = A[e];
  }
  for (int e = tid; e < N * KT; e += 128) {
    const int r = e / KT, k = e % KT;
    *reinterpret_cast<__half*>(sb + (r >> 3) * 1024 + sm100::sw128_offset(r & 7, 2 * k)) = B[e];
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (tid == 0) {
    sm100::mbar_init(&done, 1);
    sm100::fence_barrier_init();
  }
  if (warp == 0) sm100::tmem_alloc(&tmem_slot, 64);
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem = tmem_slot;
  if (tid == 0) {
    const uint32_t a0 = sm100::smem_u32(sa), b0 = sm100::smem_u32(sb);
    const uint32_t id = sm100::idesc_f16(M, N);
#pragma unroll
    for (int kk = 0; kk < KT / 16; ++kk)
      sm100::umma_f16(tmem, sm100::desc_sw128(a0 + kk * 32), sm100::desc_sw128(b0 + kk * 32), id,
                      kk > 0 ? 1u : 0u);
    sm100::umma_commit(&done);
  }
  sm100::mbar_wait(&done, 0);
  sm100::tc_fence_after();
  float v[64];
  sm100::tmem_ld64(tmem + (static_cast<uint32_t>(32 * warp) << 16), v);
  for (int i = 0; i < 64; ++i) out[(32 * warp + (tid & 31)) * N + i] = v[i];
  sm100::tc_fence_before();
  __syncthreads();
  if (warp == 0) sm100::tmem_dealloc(tmem, 64);
}

static float h2f(__half h) { return __half2float(h); }

// __float128 -> float rounded toward zero
static float to_f32_rz(__float128 x) {
  float f = static_cast<float>(x);
  const __float128 af = f < 0 ? -static_cast<__float128>(f) : static_cast<__float128>(f);
  const __float128 ax = x < 0 ? -x : x;
  if (af > ax) f = std::nextafter(f, 0.0f);
  return f;
}

// model A(F, trunc_acc): the 16 products (and the accumulator when trunc_acc) are
// aligned to the largest addend's exponent, each truncated toward zero to F bits
// below that leading bit, summed exactly, and the total truncated toward zero to fp32
static float mma_model(float acc, const __float128* p, int F, bool trunc_acc) {
  int emax = -100000;
  auto upd = [&](__float128 v) {
    if (v != 0) {
      int e;
      std::frexp(static_cast<double>(v), &e);
      if (e > emax) emax = e;
    }
  };
  upd(static_cast<__float128>(acc));
  for (int k = 0; k < 16; ++k) upd(p[k]);
  if (emax == -100000) return 0.0f;
  const __float128 q = static_cast<__float128>(std::ldexp(1.0, emax - F));
  auto tr = [&](__float128 v) {
    __float128 n = v / q;
    long long t = static_cast<long long>(n);  // toward zero
    return static_cast<__float128>(t) * q;
  };
  __float128 s = trunc_acc ? tr(static_cast<__float128>(acc)) : static_cast<__float128>(acc);
  for (int k = 0; k < 16; ++k) s += tr(p[k]);
  return to_f32_rz(s);
}

int main(int argc, char** argv) {
  std::vector<__half> A(M * KT), B(N * KT);
  srand(argc > 1 ? std::atoi(argv[1]) : 11);
  auto rnd_mixed = [] {
    // +-(1 + f) 2^e, e in [-12, 0], 10-bit f: exact fp16 normals
    const int e = -(rand() % 13);
    const float f = 1.0f + static_cast<float>(rand() % 1024) / 1024.0f;
    return __float2half(((rand() & 1) ? -1.0f : 1.0f) * std::ldexp(f, e));
  };
  for (auto& x : A) x = rnd_mixed();
  for (auto& x : B) x = rnd_mixed();
  // column 0: B row 0 = all ones, so A row r . B row 0 = sum of A row r
  for (int k = 0; k < KT; ++k) B[k] = __float2half(1.0f);
  const __half tiny = __float2half(std::ldexp(1.0f, -24));  // fp16 subnormal 2^-24
  for (int r = 0; r < 8; ++r)
    for (int k = 0; k < KT; ++k) A[r * KT + k] = __float2half(0.0f);
  // 0: 1, then 15 x 2^-24 in the same MMA (sub-half-ulp addends after a large one)
  A[0] = __float2half(1.0f);
  for (int k = 1; k < 16; ++k) A[0 * KT + k] = tiny;
  // 1: the same, the large addend last
  for (int k = 0; k < 15; ++k) A[1 * KT + k] = tiny;
  A[1 * KT + 15] = __float2half(1.0f);
  // 2: 1 in the first MMA, 16 x 2^-24 in the second
  A[2 * KT] = __float2half(1.0f);
  for (int k = 16; k < 32; ++k) A[2 * KT + k] = tiny;
  // 3: cancellation: 1, -1, 2^-24 in one MMA
  A[3 * KT] = __float2half(1.0f);
  A[3 * KT + 1] = __float2half(-1.0f);
  A[3 * KT + 2] = tiny;
  // 4: 65504, -65504, 1
  A[4 * KT] = __float2half(65504.0f);
  A[4 * KT + 1] = __float2half(-65504.0f);
  A[4 * KT + 2] = __float2half(1.0f);
  // 5: one 2^-24 addend after 1 (a quarter-ulp in fp32 at 1)
  A[5 * KT] = __float2half(1.0f);
  A[5 * KT + 1] = tiny;
  // 6: 3 x 2^-24 after 1 (0.75 ulp)
  A[6 * KT] = __float2half(1.0f);
  for (int k = 1; k < 4; ++k) A[6 * KT + k] = tiny;
  // 7: alternating +-(1 + 2^-10) with a small remainder per MMA
  for (int k = 0; k < KT; ++k)
    A[7 * KT + k] = __float2half((k & 1 ? -1.0f : 1.0f) * (1.0f + std::ldexp(1.0f, -10)) +
                                 (k % 16 == 15 ? std::ldexp(1.0f, -20) : 0.0f));
  __half *dA, *dB;
  float* dO;
  cudaMalloc(&dA, A.size() * 2);
  cudaMalloc(&dB, B.size() * 2);
  cudaMalloc(&dO, M * N * 4);
  cudaMemcpy(dA, A.data(), A.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 2, cudaMemcpyHostToDevice);
  const int smem = (M + N) * KT * 2 + 1024;
  cudaFuncSetAttribute(k_f16, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k_f16<<<1, 128, smem>>>(dA, dB, dO);
  std::vector<float> O(M * N);
  if (cudaMemcpy(O.data(), dO, O.size() * 4, cudaMemcpyDeviceToHost) != cudaSuccess) {
    printf("error %s\n", cudaGetErrorString(cudaGetLastError()));
    return 1;
  }
  // raw dump for offline model fitting: A (M x KT fp16 bits), B (N x KT), D (M x N fp32)
  if (FILE* f = std::fopen(argc > 2 ? argv[2] : "gpurun_out/f16acc.bin", "wb")) {
    std::fwrite(A.data(), 2, A.size(), f);
    std::fwrite(B.data(), 2, B.size(), f);
    std::fwrite(O.data(), 4, O.size(), f);
    std::fclose(f);
  }
  long match_e = 0, match_z = 0, total = 0;
  constexpr int NF = 10;  // F = 23 .. 32
  long match_a[NF][2] = {};
  double worst_rel = 0.0;  // |got - exact| / (2^-23 sum |p|)
  for (int r = 0; r < M; ++r)
    for (int c = 0; c < N; ++c) {
      __float128 exact = 0, absum = 0;
      float acc_e = 0.0f;  // model E
      float acc_z = 0.0f;  // model Z: the same sum, truncated toward zero
      float acc_a[NF][2] = {};
      for (int kk = 0; kk < KT / 16; ++kk) {
        __float128 s16 = 0, pk[16];
        for (int k = 16 * kk; k < 16 * kk + 16; ++k) {
          const __float128 p = static_cast<__float128>(h2f(A[r * KT + k])) * h2f(B[c * KT + k]);
          pk[k - 16 * kk] = p;
          s16 += p;
          absum += p < 0 ? -p : p;
        }
        for (int f = 0; f < NF; ++f)
          for (int t = 0; t < 2; ++t) acc_a[f][t] = mma_model(acc_a[f][t], pk, 23 + f, t == 1);
        exact += s16;
        acc_e = static_cast<float>(static_cast<__float128>(acc_e) + s16);
        acc_z = to_f32_rz(static_cast<__float128>(acc_z) + s16);
      }
      const float got = O[r * N + c];
      ++total;
      if (got == acc_e) ++match_e;
      if (got == acc_z) ++match_z;
      for (int f = 0; f < NF; ++f)
        for (int t = 0; t < 2; ++t) match_a[f][t] += got == acc_a[f][t];
      const double err = std::fabs(static_cast<double>(static_cast<__float128>(got) - exact));
      const double rel = absum > 0 ? err / (std::ldexp(1.0, -23) * static_cast<double>(absum)) : 0.0;
      if (r >= 8 && rel > worst_rel) worst_rel = rel;
      if (r < 8 && c == 0)
        printf("case %d: got %.10e  exact %.10e  model-E %.10e  model-Z %.10e  %s\n", r, got,
               static_cast<double>(exact), acc_e, acc_z, got == acc_z ? "= model Z" : "!= model Z");
    }
  printf("model E (exact 16-product sum, one RN per MMA) reproduces %ld of %ld results\n", match_e,
         total);
  printf("model Z (exact 16-product sum, one truncation toward zero per MMA) reproduces %ld of %ld\n",
         match_z, total);
  for (int f = 0; f < NF; ++f)
    printf("model A(F = %d): aligned addends truncated to F bits below the largest: %ld (acc exact), %ld (acc truncated too)\n",
           23 + f, match_a[f][0], match_a[f][1]);
  printf("random rows: max |got - exact| = %.3f x 2^-23 sum|p| over 4 MMAs\n", worst_rel);
  return 0;
}
