// Microbenchmark: DFMA / FFMA dependent latency and peak throughput on this GPU.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o fp64_micro tools/fp64_micro.cu
#include <cstdio>
#include <cuda_runtime.h>

template <typename T>
__global__ void latency(T* out, long long* cycles, int n) {
  T a = out[0], b = out[1], c = out[2];
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) {
    a = fma(a, b, c);
    a = fma(a, b, c);
    a = fma(a, b, c);
    a = fma(a, b, c);
  }
  long long t1 = clock64();
  out[3] = a;
  cycles[0] = t1 - t0;
}

template <typename T>
__global__ void throughput(T* out, int n) {
  T a[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) a[j] = out[j] + threadIdx.x;
  const T b = out[8], c = out[9];
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) a[j] = fma(a[j], b, c);
  }
  T s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += a[j];
  if (s == T(12345.678)) out[10] = s;
}

__global__ void shfl_lat(double* out, long long* cycles, int n) {
  double a = out[threadIdx.x];
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) a += __shfl_xor_sync(0xffffffffu, a, 1);
  long long t1 = clock64();
  out[threadIdx.x] = a;
  if (threadIdx.x == 0) cycles[0] = t1 - t0;
}

__global__ void lds_lat(double* out, long long* cycles, int n) {
  __shared__ int idx[256];
  idx[threadIdx.x] = (threadIdx.x + 1) & 255;
  __syncthreads();
  int j = threadIdx.x;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) j = idx[j];
  long long t1 = clock64();
  out[threadIdx.x] = j;
  if (threadIdx.x == 0) cycles[0] = t1 - t0;
}

__global__ void bar_lat(double* out, long long* cycles, int n) {
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) __syncthreads();
  long long t1 = clock64();
  if (threadIdx.x == 0) cycles[0] = t1 - t0;
}

int dmma_main();
int main() {
  dmma_main();
  double* d;
  float* f;
  long long* cyc;
  cudaMalloc(&d, 1 << 20);
  cudaMalloc(&f, 1 << 20);
  cudaMalloc(&cyc, 64);
  cudaMemset(d, 0, 1 << 20);
  cudaMemset(f, 0, 1 << 20);
  long long h;
  const int n = 1 << 14;
  latency<double><<<1, 1>>>(d, cyc, n);
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("DFMA dependent latency: %.2f cycles\n", double(h) / (4.0 * n));
  latency<float><<<1, 1>>>(f, cyc, n);
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("FFMA dependent latency: %.2f cycles\n", double(h) / (4.0 * n));
  shfl_lat<<<1, 32>>>(d, cyc, n);
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("SHFL(f64)+DADD dependent latency: %.2f cycles\n", double(h) / n);
  lds_lat<<<1, 256>>>(d, cyc, n);
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("LDS dependent latency: %.2f cycles\n", double(h) / n);
  bar_lat<<<1, 256>>>(d, cyc, n);
  cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("__syncthreads (8 warps): %.2f cycles\n", double(h) / n);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int m = 1 << 12;
  for (int pass = 0; pass < 2; ++pass) {
    cudaEventRecord(a);
    throughput<double><<<sms * 4, 256>>>(d, m);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    if (pass) printf("FP64 FMA throughput: %.1f TFLOP/s\n", 2.0 * 8 * m * sms * 4 * 256 / (ms * 1e9));
    cudaEventRecord(a);
    throughput<float><<<sms * 4, 256>>>(f, m);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    if (pass) printf("FP32 FMA throughput: %.1f TFLOP/s\n", 2.0 * 8 * m * sms * 4 * 256 / (ms * 1e9));
  }
  return 0;
}

// DMMA m8n8k4 f64 throughput (register-resident operands, 4 independent chains per warp)
__global__ void dmma_tp(double* out, int n) {
  double a = out[threadIdx.x & 7] + 1.0, b = out[(threadIdx.x + 3) & 7] + 1.0;
  double c[4][2] = {{0, 0}, {0, 0}, {0, 0}, {0, 0}};
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int j = 0; j < 4; ++j)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[j][0]), "+d"(c[j][1]) : "d"(a), "d"(b));
  }
  double s = 0;
  for (int j = 0; j < 4; ++j) s += c[j][0] + c[j][1];
  if (s == 12345.678) out[11] = s;
}

int dmma_main() {
  double* d;
  cudaMalloc(&d, 1 << 20);
  cudaMemset(d, 0, 1 << 20);
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const int m = 1 << 12;
  for (int warps = 4; warps <= 16; warps *= 2) {
    for (int pass = 0; pass < 2; ++pass) {
      cudaEventRecord(a);
      dmma_tp<<<sms * 2, 32 * warps>>>(d, m);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (pass)
        printf("DMMA m8n8k4 (%d warps/CTA, 2 CTA/SM): %.1f TFLOP/s\n", warps,
               2.0 * 256 * 4 * m * sms * 2 * warps / (ms * 1e9));
    }
  }
  return 0;
}
