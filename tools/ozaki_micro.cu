// Int8 Ozaki projection on tcgen05 (item 1): C = Y Q for a
// tile of 128 float32 signal rows and one 64 x 64 float64 block, with
//   y rows in fixed point (per-row power-of-two scale) as 5 signed 7-bit digits,
//   Q columns (per-column scale) as 8 digits,
// every digit pair of weight level i + j <= 7 accumulated exactly in int32 TMEM
// (8 level accumulators x 64 columns = 512), recombined in float64.  Checks the
// result against a long-double reference and times the MMA stage.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "sm100.cuh"

using namespace sbo;

constexpr int M = 128, P = 64, DY = 5, DQ = 8, LV = 8;

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
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, int32_t* v) {
  uint32_t* r = reinterpret_cast<uint32_t*>(v);
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
        "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
        "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
        "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
        "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

// smem tiles: A digit i: 128 rows x 128 B (K = 64 used, the rest zero); B digit j:
// 64 atom rows x 128 B.  Both 128-B swizzled, 1024-B aligned.
constexpr int A_BYTES = M * 128, B_BYTES = P * 128;

__global__ void __launch_bounds__(128, 1) k_ozaki(const int8_t* ga, const int8_t* gb,
                                                  const int* ey, const int* eq, int reps,
                                                  double* C) {
  extern __shared__ unsigned char raw[];
  const uint32_t base = sm100::smem_u32(raw);
  unsigned char* s = raw + ((1024u - (base & 1023u)) & 1023u);
  int8_t* sa = reinterpret_cast<int8_t*>(s);
  int8_t* sb = sa + DY * A_BYTES;
  __shared__ uint64_t done;
  __shared__ uint32_t tslot;
  const int tid = threadIdx.x, warp = tid >> 5;
  for (int e = tid; e < DY * A_BYTES / 16; e += 128)
    reinterpret_cast<int4*>(sa)[e] = reinterpret_cast<const int4*>(ga)[e];
  for (int e = tid; e < DQ * B_BYTES / 16; e += 128)
    reinterpret_cast<int4*>(sb)[e] = reinterpret_cast<const int4*>(gb)[e];
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (tid == 0) {
    sm100::mbar_init(&done, 1);
    sm100::fence_barrier_init();
  }
  if (warp == 0) sm100::tmem_alloc(&tslot, 512);
  sm100::tc_fence_before();
  __syncthreads();
  sm100::tc_fence_after();
  const uint32_t tmem = tslot;
  if (tid == 0) {
    const uint32_t id = idesc_i8(M, P);
    for (int r = 0; r < reps; ++r) {
      uint32_t started = 0u;  // bit L: level L written this repetition
      for (int i = 0; i < DY; ++i)
        for (int j = 0; j + i < LV && j < DQ; ++j) {
          const int L = i + j;
          const uint32_t a0 = sm100::smem_u32(sa + i * A_BYTES), b0 = sm100::smem_u32(sb + j * B_BYTES);
#pragma unroll
          for (int kk = 0; kk < 2; ++kk) {  // K = 64 as two K = 32 steps
            umma_i8(tmem + L * P, sm100::desc_sw128(a0 + kk * 32), sm100::desc_sw128(b0 + kk * 32),
                    id, ((started >> L) & 1u) || kk > 0 ? 1u : 0u);
          }
          started |= 1u << L;
        }
    }
    sm100::umma_commit(&done);
  }
  sm100::mbar_wait(&done, 0);
  sm100::tc_fence_after();
  // recombine: c = 2^-(ey + eq) sum_L 2^(-7 L) acc_L (exact int32 -> double)
  const int row = 32 * warp + (tid & 31);
  const uint32_t lane = tmem + (static_cast<uint32_t>(32 * warp) << 16);
  for (int h = 0; h < 2; ++h) {
    double c[32];
#pragma unroll
    for (int a = 0; a < 32; ++a) c[a] = 0.0;
    for (int L = LV - 1; L >= 0; --L) {  // small levels first
      int32_t v[32];
      tmem_ld32(lane + L * P + 32 * h, v);
      const double w = ldexp(1.0, -7 * L);
#pragma unroll
      for (int a = 0; a < 32; ++a) c[a] = fma(static_cast<double>(v[a]), w, c[a]);
    }
#pragma unroll
    for (int a = 0; a < 32; ++a)
      C[row * P + 32 * h + a] = ldexp(c[a], -(ey[row] + eq[32 * h + a]));
  }
  sm100::tc_fence_before();
  __syncthreads();
  if (warp == 0) sm100::tmem_dealloc(tmem, 512);
}

// signed base-128 digits of x (|x| < 2^7 after scaling): truncation keeps every
// digit in [-127, 127]; each step is exact in float64
static void digits(double x, int n, int8_t* d) {
  for (int t = 0; t < n; ++t) {
    const double q = std::trunc(x);
    d[t] = static_cast<int8_t>(q);
    x = (x - q) * 128.0;
  }
}

int main(int argc, char** argv) {
  const bool gauss = argc > 1;
  srand(3);
  std::vector<float> Y(M * P);
  for (auto& v : Y) {
    if (gauss) {
      double u1 = (rand() + 1.0) / (RAND_MAX + 2.0), u2 = (rand() + 1.0) / (RAND_MAX + 2.0);
      v = static_cast<float>(std::sqrt(-2 * std::log(u1)) * std::cos(6.283185307179586 * u2));
    } else {
      v = static_cast<float>((rand() % 256) / 255.0);  // unit-range patch values
    }
  }
  // a random orthogonal Q by modified Gram-Schmidt (columns)
  std::vector<double> Q(P * P);
  for (auto& v : Q) v = (rand() / (double)RAND_MAX) - 0.5;
  for (int c = 0; c < P; ++c) {
    for (int d = 0; d < c; ++d) {
      double dot = 0;
      for (int k = 0; k < P; ++k) dot += Q[k * P + c] * Q[k * P + d];
      for (int k = 0; k < P; ++k) Q[k * P + c] -= dot * Q[k * P + d];
    }
    double n = 0;
    for (int k = 0; k < P; ++k) n += Q[k * P + c] * Q[k * P + c];
    n = std::sqrt(n);
    for (int k = 0; k < P; ++k) Q[k * P + c] /= n;
  }
  // slices in the swizzled smem layout
  std::vector<int8_t> ga(DY * A_BYTES, 0), gb(DQ * B_BYTES, 0);
  std::vector<int> ey(M), eq(P);
  for (int r = 0; r < M; ++r) {
    double mx = 0;
    for (int k = 0; k < P; ++k) mx = std::fmax(mx, std::fabs(Y[r * P + k]));
    int e = 0;
    if (mx > 0) std::frexp(mx, &e);
    ey[r] = 7 - e;  // mx * 2^ey in [64, 128)
    for (int k = 0; k < P; ++k) {
      int8_t d[DY];
      digits(std::ldexp(static_cast<double>(Y[r * P + k]), ey[r]), DY, d);
      for (int t = 0; t < DY; ++t)
        ga[t * A_BYTES + (r >> 3) * 1024 + sm100::sw128_offset(r & 7, k)] = d[t];
    }
  }
  for (int i = 0; i < P; ++i) {
    double mx = 0;
    for (int k = 0; k < P; ++k) mx = std::fmax(mx, std::fabs(Q[k * P + i]));
    int e = 0;
    std::frexp(mx, &e);
    eq[i] = 7 - e;
    for (int k = 0; k < P; ++k) {
      int8_t d[DQ];
      digits(std::ldexp(Q[k * P + i], eq[i]), DQ, d);
      for (int t = 0; t < DQ; ++t)
        gb[t * B_BYTES + (i >> 3) * 1024 + sm100::sw128_offset(i & 7, k)] = d[t];
    }
  }
  int8_t *dA, *dB;
  int *dey, *deq;
  double* dC;
  cudaMalloc(&dA, ga.size());
  cudaMalloc(&dB, gb.size());
  cudaMalloc(&dey, M * 4);
  cudaMalloc(&deq, P * 4);
  cudaMalloc(&dC, M * P * 8);
  cudaMemcpy(dA, ga.data(), ga.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(dB, gb.data(), gb.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(dey, ey.data(), M * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(deq, eq.data(), P * 4, cudaMemcpyHostToDevice);
  const int smem = DY * A_BYTES + DQ * B_BYTES + 1024;
  cudaFuncSetAttribute(k_ozaki, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  k_ozaki<<<1, 128, smem>>>(dA, dB, dey, deq, 1, dC);
  std::vector<double> C(M * P);
  const cudaError_t err = cudaMemcpy(C.data(), dC, C.size() * 8, cudaMemcpyDeviceToHost);
  if (err != cudaSuccess) {
    printf("error: %s\n", cudaGetErrorString(err));
    return 1;
  }
  double worst = 0, worst_d = 0;
  for (int r = 0; r < M; ++r) {
    long double yn = 0;
    for (int k = 0; k < P; ++k) yn += (long double)Y[r * P + k] * Y[r * P + k];
    for (int i = 0; i < P; ++i) {
      long double ref = 0;
      double dref = 0;
      for (int k = 0; k < P; ++k) {
        ref += (long double)Y[r * P + k] * Q[k * P + i];
        dref = std::fma(static_cast<double>(Y[r * P + k]), Q[k * P + i], dref);
      }
      const double nrm = std::sqrt(static_cast<double>(yn)) + 1e-300;
      worst = std::fmax(worst, std::fabs(static_cast<double>(C[r * P + i] - ref)) / nrm);
      worst_d = std::fmax(worst_d, std::fabs(static_cast<double>(dref - ref)) / nrm);
    }
  }
  printf("%s rows: max |C - exact| / ||y||: ozaki %.3g, float64 fma loop %.3g\n",
         gauss ? "gaussian" : "unit-range", worst, worst_d);
  // MMA-stage throughput: 148 CTAs, many repetitions of the 30-pair set
  const int reps = 4000;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  k_ozaki<<<148, 128, smem>>>(dA, dB, dey, deq, 10, dC);
  cudaEventRecord(e0);
  k_ozaki<<<148, 128, smem>>>(dA, dB, dey, deq, reps, dC);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double tiles = 148.0 * reps;
  printf("MMA stage: %.2f ns per 128-signal tile per SM (%.0f cycles at 1.9 GHz); a float64 "
         "projection equivalent of %.1f TFLOP/s (2 x 128 x 64 x 64 per tile)\n",
         ms * 1e6 / reps, ms * 1e-3 / reps * 1.9e9,
         2.0 * M * P * P * tiles / (ms * 1e-3) / 1e12);
  return 0;
}
