// Throughput of the float32 -> float64 conversion (F2F.F64.F32) vs DFMA on B200,
// and of the two mixed (the sparse outer product's inner loop shape).
#include <cstdio>

__global__ void k_cvt(float* out, int n) {
  float a[8]; double s[8];
  for (int i = 0; i < 8; ++i) { a[i] = out[threadIdx.x % 7 + i]; s[i] = 0.0; }
  for (int it = 0; it < n; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) { s[i] += (double)a[i]; a[i] = __int_as_float(__float_as_int(a[i]) ^ it); }
  }
  double t = 0; for (int i = 0; i < 8; ++i) t += s[i];
  if (t == 1234.5) out[0] = (float)t;
}
__global__ void k_dfma(double* out, int n) {
  double a[8], b = out[1];
  for (int i = 0; i < 8; ++i) a[i] = out[threadIdx.x % 7 + i];
  for (int it = 0; it < n; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fma(a[i], b, a[(i + 3) & 7]);
  double t = 0; for (int i = 0; i < 8; ++i) t += a[i];
  if (t == 1234.5) out[0] = t;
}
__global__ void k_iadd(int* out, int n) {
  int a[8];
  for (int i = 0; i < 8; ++i) a[i] = out[threadIdx.x % 7 + i];
  for (int it = 0; it < n; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = a[i] ^ (a[(i + 3) & 7] + it);
  int t = 0; for (int i = 0; i < 8; ++i) t += a[i];
  if (t == 12345) out[0] = t;
}
int main() {
  float* d; cudaMalloc(&d, 1 << 16); cudaMemset(d, 0, 1 << 16);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int n = 1 << 13, grid = 148 * 8, blk = 256;
  float ms;
  for (int pass = 0; pass < 2; ++pass) {
    cudaEventRecord(a); k_cvt<<<grid, blk>>>(d, n); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    if (pass) printf("F2F.F64.F32 (+DADD+LOP): %.1f G conversions/s = %.1f per clk per SM at 1.9 GHz\n",
                     8.0 * n * grid * blk / (ms * 1e6), 8.0 * n * grid * blk / (ms * 1e-3) / 148 / 1.9e9);
    cudaEventRecord(a); k_dfma<<<grid, blk>>>((double*)d, n); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    if (pass) printf("DFMA: %.1f G/s = %.1f per clk per SM\n", 8.0 * n * grid * blk / (ms * 1e6),
                     8.0 * n * grid * blk / (ms * 1e-3) / 148 / 1.9e9);
    cudaEventRecord(a); k_iadd<<<grid, blk>>>((int*)d, n); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    if (pass) printf("IADD+LOP pairs: %.1f G/s = %.1f per clk per SM\n", 8.0 * n * grid * blk / (ms * 1e6),
                     8.0 * n * grid * blk / (ms * 1e-3) / 148 / 1.9e9);
  }
  return 0;
}
