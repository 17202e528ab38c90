// DMMA (mma.sync m8n8k4 f64) throughput vs warps per SM and independent
// accumulators per warp.
#include <cstdio>
#include <cuda_runtime.h>

template <int CH>
__global__ void dmma_loop(double* out, int iters) {
  double acc[CH][2];
  for (int j = 0; j < CH; ++j) { acc[j][0] = 0; acc[j][1] = 0; }
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-6;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < CH; ++j)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(acc[j][0]), "+d"(acc[j][1]) : "d"(a), "d"(b));
  }
  double s = 0;
  for (int j = 0; j < CH; ++j) s += acc[j][0] + acc[j][1];
  if (s == 12345.0) out[0] = s;
}

template <int CH>
void run(double* d, int warps_per_sm) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int iters = 4096 / CH * 8;
  int threads = 32 * (warps_per_sm < 8 ? warps_per_sm : 8);
  int blocks = 148 * (warps_per_sm * 32 / threads);
  for (int rep = 0; rep < 2; ++rep) {
    cudaEventRecord(e0);
    dmma_loop<CH><<<blocks, threads>>>(d, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 8 * 8 * 4 * CH * (double)iters * blocks * (threads / 32);
    if (rep) printf("warps/SM=%2d chains/warp=%2d: %.2f TFLOP/s\n", warps_per_sm, CH, fl / ms / 1e9);
  }
}

int main() {
  double* d;
  cudaMalloc(&d, 8);
  for (int w : {4, 8, 16, 32}) {
    run<4>(d, w);
    run<8>(d, w);
    run<16>(d, w);
    run<32>(d, w);
  }
  return 0;
}
