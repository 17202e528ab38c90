// FP64 throughput probe on B200: DFMA (CUDA cores) and DMMA (mma.sync
// m8n8k4 f64 tensor path).  Prints TFLOP/s for each; used to state the FP64
// roofline denominator (MEASURED_PEAKS.json has no FP64 entry).
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_loop(double* out, int iters) {
  double a[8];
  for (int i = 0; i < 8; ++i) a[i] = threadIdx.x * 1e-3 + i;
  const double b = 1.0000001, c = 1e-9;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fma(a[i], b, c);
  }
  double s = 0;
  for (int i = 0; i < 8; ++i) s += a[i];
  if (s == 12345.0) out[0] = s;
}

__global__ void dmma_loop(double* out, int iters) {
  double acc[4][2];
  for (int j = 0; j < 4; ++j) { acc[j][0] = 0; acc[j][1] = 0; }
  double a = threadIdx.x * 1e-3, b = 1.0 + threadIdx.x * 1e-6;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 4; ++j)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(acc[j][0]), "+d"(acc[j][1]) : "d"(a), "d"(b));
  }
  double s = 0;
  for (int j = 0; j < 4; ++j) s += acc[j][0] + acc[j][1];
  if (s == 12345.0) out[0] = s;
}

int main() {
  double* d;
  cudaMalloc(&d, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 20000;
  for (int rep = 0; rep < 2; ++rep) {
    int blocks = sms * 8, threads = 256;
    cudaEventRecord(e0);
    dfma_loop<<<blocks, threads>>>(d, iters);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    double fl = 2.0 * 8 * iters * (double)blocks * threads;
    printf("DFMA: %.2f TFLOP/s (%.3f ms)\n", fl / ms / 1e9, ms);
    cudaEventRecord(e0);
    dmma_loop<<<blocks, threads>>>(d, iters / 4);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    double fm = 2.0 * 8 * 8 * 4 * 4 * (iters / 4) * (double)blocks * (threads / 32);
    printf("DMMA m8n8k4: %.2f TFLOP/s (%.3f ms)\n", fm / ms / 1e9, ms);
  }
  printf("err: %s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
