// Throughput of integer max/min (IMNMX / VIMNMX) vs FMNMX on B200.
#include <cstdio>
__global__ void k_f(float* out, int n) {
  float a[8];
  for (int i = 0; i < 8; ++i) a[i] = out[threadIdx.x % 7 + i];
  for (int it = 0; it < n; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fmaxf(a[i], a[(i + 3) & 7]);
  float s = 0; for (int i = 0; i < 8; ++i) s += a[i];
  if (s == 1234.5f) out[0] = s;
}
__global__ void k_i(int* out, int n) {
  int a[8];
  for (int i = 0; i < 8; ++i) a[i] = out[threadIdx.x % 7 + i];
  for (int it = 0; it < n; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = max(a[i], a[(i + 3) & 7]);
  int s = 0; for (int i = 0; i < 8; ++i) s += a[i];
  if (s == 12345) out[0] = s;
}
int main() {
  float* d; cudaMalloc(&d, 4096); cudaMemset(d, 0, 4096);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int n = 1 << 14, grid = 148 * 8, blk = 256;
  float ms;
  for (int pass = 0; pass < 2; ++pass) {
    cudaEventRecord(a); k_f<<<grid, blk>>>(d, n); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    if (pass) printf("FMNMX: %.1f per clk per SM (1.9 GHz)\n", 8.0 * n * grid * blk / (ms * 1e-3) / 148 / 1.9e9);
    cudaEventRecord(a); k_i<<<grid, blk>>>((int*)d, n); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    if (pass) printf("IMNMX: %.1f per clk per SM\n", 8.0 * n * grid * blk / (ms * 1e-3) / 148 / 1.9e9);
  }
  return 0;
}
