// Kernel-to-kernel gap inside a CUDA graph on B200, with and without programmatic
// dependent launch (PDL): a chain of N tiny dependent kernels (148 CTAs each).
#include <cstdio>

__global__ void k_step(int* x, int pdl) {
  if (pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
  if (threadIdx.x == 0) atomicAdd(x + blockIdx.x, 1);
}

int main() {
  int* x;
  cudaMalloc(&x, 148 * 4);
  cudaMemset(x, 0, 148 * 4);
  cudaStream_t s;
  cudaStreamCreate(&s);
  const int N = 200;
  for (int pdl = 0; pdl < 2; ++pdl) {
    cudaGraph_t g;
    cudaGraphExec_t ge;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
    for (int i = 0; i < N; ++i) {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(148);
      cfg.blockDim = dim3(128);
      cfg.stream = s;
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[0].val.programmaticStreamSerializationAllowed = 1;
      cfg.attrs = at;
      cfg.numAttrs = pdl ? 1 : 0;
      cudaLaunchKernelEx(&cfg, k_step, x, pdl);
    }
    cudaStreamEndCapture(s, &g);
    cudaGraphInstantiate(&ge, g, 0);
    cudaGraphLaunch(ge, s);
    cudaStreamSynchronize(s);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0, s);
    for (int r = 0; r < 10; ++r) cudaGraphLaunch(ge, s);
    cudaEventRecord(e1, s);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("%s: %.2f us per dependent kernel in a graph\n", pdl ? "PDL" : "plain", ms * 1e3 / (10 * N));
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
