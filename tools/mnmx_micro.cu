// Throughput of FMNMX vs HMNMX2 and whether they share a pipe (B200).
#include <cstdio>
#include <cuda_fp16.h>

__global__ void k_f(float* out, int n) {
  float a[8];
  for (int i = 0; i < 8; ++i) a[i] = out[threadIdx.x % 7 + i];
  for (int it = 0; it < n; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fmaxf(a[i], a[(i + 3) & 7]) ;
  float s = 0; for (int i = 0; i < 8; ++i) s += a[i];
  if (s == 1234.5f) out[0] = s;
}
__global__ void k_h(__half2* out, int n) {
  __half2 a[8];
  for (int i = 0; i < 8; ++i) a[i] = out[threadIdx.x % 7 + i];
  for (int it = 0; it < n; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = __hmax2(a[i], a[(i + 3) & 7]);
  __half2 s = a[0]; for (int i = 1; i < 8; ++i) s = __hadd2(s, a[i]);
  if (__low2float(s) == 1234.5f) out[0] = s;
}
__global__ void k_fh(float* out, __half2* outh, int n) {
  float a[8]; __half2 b[8];
  for (int i = 0; i < 8; ++i) { a[i] = out[threadIdx.x % 7 + i]; b[i] = outh[threadIdx.x % 7 + i]; }
  for (int it = 0; it < n; ++it)
#pragma unroll
    for (int i = 0; i < 8; ++i) { a[i] = fmaxf(a[i], a[(i + 3) & 7]); b[i] = __hmax2(b[i], b[(i + 3) & 7]); }
  float s = 0; for (int i = 0; i < 8; ++i) s += a[i] + __low2float(b[i]);
  if (s == 1234.5f) out[0] = s;
}
int main() {
  float* d; __half2* h;
  cudaMalloc(&d, 4096); cudaMalloc(&h, 4096); cudaMemset(d, 0, 4096); cudaMemset(h, 0, 4096);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int n = 1 << 14, grid = 148 * 8, blk = 256;
  float ms;
  for (int pass = 0; pass < 2; ++pass) {
    cudaEventRecord(a); k_f<<<grid, blk>>>(d, n); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    if (pass) printf("FMNMX: %.1f G ops/s\n", 8.0 * n * grid * blk / (ms * 1e6));
    cudaEventRecord(a); k_h<<<grid, blk>>>(h, n); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    if (pass) printf("HMNMX2: %.1f G instr/s\n", 8.0 * n * grid * blk / (ms * 1e6));
    cudaEventRecord(a); k_fh<<<grid, blk>>>(d, h, n); cudaEventRecord(b); cudaEventSynchronize(b);
    cudaEventElapsedTime(&ms, a, b);
    if (pass) printf("FMNMX+HMNMX2 interleaved: %.1f G instr/s (both counted)\n", 16.0 * n * grid * blk / (ms * 1e6));
  }
  return 0;
}
