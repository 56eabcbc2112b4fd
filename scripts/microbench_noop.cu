// Cost of early-exit ("no-op") kernel launches inside a CUDA graph, with and
// without programmatic dependent launch (sizing the gated fallback of Step 1(a)).
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_work(float* p, int n) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) p[i] = p[i] * 1.0001f + 1.f;
}
__global__ void k_noop(const int* flag) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  if (*flag == 0) return;
}
int main() {
  float* p; int* flag;
  cudaMalloc(&p, 1 << 24); cudaMalloc(&flag, 4); cudaMemset(flag, 0, 4);
  cudaStream_t st; cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
  for (int pdl = 0; pdl < 2; ++pdl) {
    for (int nnoop : {0, 1, 5, 10, 20}) {
      cudaLaunchAttribute at[1];
      at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
      at[0].val.programmaticStreamSerializationAllowed = pdl;
      auto launch = [&](auto kern, unsigned grid, auto... args) {
        cudaLaunchConfig_t c = {};
        c.gridDim = grid; c.blockDim = 256; c.stream = st; c.attrs = at; c.numAttrs = 1;
        cudaLaunchKernelEx(&c, kern, args...);
      };
      cudaGraph_t g; cudaGraphExec_t ge;
      cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
      for (int rep = 0; rep < 4; ++rep) {
        launch(k_work, 148u * 4, p, 1 << 20);
        for (int i = 0; i < nnoop; ++i) launch(k_noop, 148u * 4, (const int*)flag);
      }
      cudaStreamEndCapture(st, &g);
      cudaGraphInstantiate(&ge, g, 0);
      for (int i = 0; i < 20; ++i) cudaGraphLaunch(ge, st);
      cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
      cudaEventRecord(a, st);
      for (int i = 0; i < 200; ++i) cudaGraphLaunch(ge, st);
      cudaEventRecord(b, st); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      printf("{\"pdl\": %d, \"noops_per_work\": %d, \"us_per_graph\": %.2f, \"us_per_noop_est\": null}\n", pdl, nnoop, ms * 1000 / 200);
    }
  }
  return 0;
}
