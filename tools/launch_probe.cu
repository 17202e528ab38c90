// Floor of a chain of dependent kernels on one stream: plain launches,
// PDL launches, and a CUDA graph of each; 148x256 CTAs that each read one
// value the previous kernel wrote and write one value.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_chain(double* buf, int i, int pdl) {
  if (pdl) asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  if (pdl) asm volatile("griddepcontrol.wait;" ::: "memory");
  int t = blockIdx.x * blockDim.x + threadIdx.x;
  double v = buf[(t + i) % (148 * 256)];
  buf[t] = v * 1.0000001 + 1e-9;
}

int main() {
  double* buf;
  cudaMalloc(&buf, 148 * 256 * 8);
  cudaMemset(buf, 0, 148 * 256 * 8);
  cudaStream_t st;
  cudaStreamCreate(&st);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int N = 200;
  for (int pdl = 0; pdl < 2; ++pdl) {
    for (int graph = 0; graph < 2; ++graph) {
      auto enqueue = [&]() {
        for (int i = 0; i < N; ++i) {
          cudaLaunchConfig_t cfg = {};
          cfg.gridDim = dim3(148);
          cfg.blockDim = dim3(256);
          cfg.stream = st;
          cudaLaunchAttribute at[1];
          at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
          at[0].val.programmaticStreamSerializationAllowed = pdl;
          cfg.attrs = at;
          cfg.numAttrs = 1;
          cudaLaunchKernelEx(&cfg, k_chain, buf, i, pdl);
        }
      };
      cudaGraphExec_t ge = nullptr;
      if (graph) {
        cudaGraph_t g;
        cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
        enqueue();
        cudaStreamEndCapture(st, &g);
        cudaGraphInstantiate(&ge, g, 0);
      }
      for (int rep = 0; rep < 3; ++rep) {
        cudaEventRecord(e0, st);
        if (graph) cudaGraphLaunch(ge, st); else enqueue();
        cudaEventRecord(e1, st);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        if (rep == 2) printf("pdl=%d graph=%d: %.2f us per dependent kernel\n", pdl, graph, 1e3 * ms / N);
      }
    }
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
}
