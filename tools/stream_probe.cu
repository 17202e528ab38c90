// Bandwidth probe for the panel streaming pattern (no gathers / epilogues):
// each thread owns two rows of a [C][TR] column-major tile and accumulates
// M[col] * x[col] with x in shared memory.  Prints GB/s for tile heights,
// batch sizes and column counts, next to a plain float4 copy-read.
#include <cstdio>
#include <cuda_runtime.h>
#include "../paper_2306_02526_b200/csrc/stream.cuh"

using namespace hpsb;

template <int U>
__global__ void probe(const double* __restrict__ base, int C, int TR, double* out) {
  extern __shared__ double xs[];
  for (int i = threadIdx.x; i < C; i += blockDim.x) xs[i] = 1.0 + 1e-3 * i;
  __syncthreads();
  const double2* M = reinterpret_cast<const double2*>(base + (size_t)blockIdx.x * C * TR) + threadIdx.x;
  double acc0[1] = {0.0}, acc1[1] = {0.0};
  double2 A[U];
  if (C >= U) load_batch<U>(A, M, TR / 2, 0);
  stream_cols<1, U>(A, M, TR / 2, 0, C, xs, 0, 0, 0, acc0, acc1);
  if (acc0[0] + acc1[0] == 12345.0) out[0] = acc0[0];
}

__global__ void readall(const double2* __restrict__ p, size_t n, double* out) {
  double s = 0;
  for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
    double2 v = __ldcs(p + i);
    s += v.x + v.y;
  }
  if (s == 12345.0) out[0] = s;
}

int main() {
  const size_t bytes = 1ull << 30;
  double* buf;
  double* out;
  cudaMalloc(&buf, bytes);
  cudaMalloc(&out, 8);
  cudaMemset(buf, 0, bytes);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms;
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0);
    readall<<<148 * 8, 256>>>((const double2*)buf, bytes / 16, out);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("read-all float4x2: %.0f GB/s\n", bytes / ms / 1e6);
  }
  int TRs[] = {64, 128, 256, 512};
  int Cs[] = {16, 32, 64, 128, 256, 1024};
  for (int TR : TRs)
    for (int C : Cs) {
      size_t tile = (size_t)C * TR * 8;
      int nt = (int)(bytes / tile);
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        probe<8><<<nt, TR / 2, C * 8>>>(buf, C, TR, out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        if (rep) printf("TR=%3d C=%4d U=8 blocks=%7d: %.0f GB/s\n", TR, C, nt, (double)nt * tile / ms / 1e6);
      }
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(e0);
        probe<4><<<nt, TR / 2, C * 8>>>(buf, C, TR, out);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        if (rep) printf("TR=%3d C=%4d U=4 blocks=%7d: %.0f GB/s\n", TR, C, nt, (double)nt * tile / ms / 1e6);
      }
    }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
