// Common helpers for the hpstep-b200 CUDA library (sm_100a).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>

#include <atomic>
#include <utility>
#include <string>

namespace hpsb {

constexpr int kNumSMs = 148;  // B200

// thread-local last error, surfaced through hps_last_error()
void set_error(const char* fmt, ...);
void set_error_node(long long node);

#define HPSB_CUDA(expr)                                                        \
  do {                                                                         \
    cudaError_t _e = (expr);                                                   \
    if (_e != cudaSuccess) {                                                   \
      ::hpsb::set_error("%s:%d: %s -> %s", __FILE__, __LINE__, #expr,          \
                        cudaGetErrorString(_e));                               \
      return -2;                                                               \
    }                                                                          \
  } while (0)

// kernel launches issued by this library (hps_launch_count); every launch
// site is followed by HPSB_LAUNCH_CHECK
extern std::atomic<long long> g_launches;

#define HPSB_LAUNCH_CHECK()                                                    \
  do {                                                                         \
    ::hpsb::g_launches.fetch_add(1, std::memory_order_relaxed);                \
    cudaError_t _e = cudaGetLastError();                                       \
    if (_e != cudaSuccess) {                                                   \
      ::hpsb::set_error("%s:%d: launch failed: %s", __FILE__, __LINE__,         \
                        cudaGetErrorString(_e));                               \
      return -2;                                                               \
    }                                                                          \
  } while (0)

__host__ __device__ inline long long cdiv(long long a, long long b) { return (a + b - 1) / b; }

// ---------------------------------------------------------------------------
// Programmatic dependent launch (sm_90+): the solve is a chain of ~30
// dependent kernels on one stream.  Every kernel of the chain triggers its
// dependents on entry and waits for its predecessor (griddepcontrol.wait)
// only before touching vectors; loads of the immutable operators may be
// issued before the wait, so a kernel's launch, prologue and first operator
// batch overlap the tail of the previous one.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }

// release / acquire counters (the CUTLASS semaphore pattern): a CTA's writes,
// ordered before one thread by a barrier, are published by that thread's
// release atomic; the consumer's acquire load plus a barrier orders its reads
// after them.  Cheaper than __threadfence (MEMBAR.SC + an L1 invalidate).
__device__ __forceinline__ unsigned atom_add_acq_rel(unsigned* p, unsigned v) {
  unsigned old;
  asm volatile("atom.add.acq_rel.gpu.global.u32 %0, [%1], %2;" : "=r"(old) : "l"(p), "r"(v) : "memory");
  return old;
}
__device__ __forceinline__ void red_add_release(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

bool pdl_enabled();  // HPSB_NO_PDL=1 disables

// Per-kernel CUDA-event timing (hps_ktimer_enable): while on, every launch
// through launch_pdl / launch_plain on a stream that is not being captured is
// bracketed by two events on its stream; hps_ktimer_collect sums the elapsed
// times per kernel.  The events serialise the PDL overlap of neighbouring
// kernels, so this is a measurement pass, not the timed one.
extern std::atomic<int> g_ktimer_on;
cudaEvent_t ktimer_begin(cudaStream_t st);           // nullptr unless timing this launch
void ktimer_end(cudaEvent_t a, const void* fn, cudaStream_t st);

template <typename... KArgs, typename... Args>
cudaError_t launch_kernel(bool pdl, void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                          Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl && pdl_enabled() ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaEvent_t ev = g_ktimer_on.load(std::memory_order_relaxed) ? ktimer_begin(st) : nullptr;
  cudaError_t e = cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
  if (ev) ktimer_end(ev, (const void*)kern, st);
  return e;
}

template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                       Args&&... args) {
  return launch_kernel(true, kern, grid, block, smem, st, std::forward<Args>(args)...);
}

// no programmatic dependency (a kernel that reads its predecessor's output
// from its first instruction)
template <typename... KArgs, typename... Args>
cudaError_t launch_plain(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                         Args&&... args) {
  return launch_kernel(false, kern, grid, block, smem, st, std::forward<Args>(args)...);
}

// ---------------------------------------------------------------------------
// Batched FP64 GEMM:  C[b] = alpha * op(A[b]) * op(B[b]) + beta * D[b]
// row-major operands; op(X) = X or X^T.  D may alias C (beta applied to D).
// Any stride may be 0 (broadcast one matrix over the batch).
// ---------------------------------------------------------------------------
struct GemmArgs {
  int M, N, K;
  double alpha, beta;
  const double* A; long long lda, sA; int tA;
  const double* B; long long ldb, sB; int tB;
  const double* D; long long ldd, sD;
  double* C; long long ldc, sC;
  int batch;
};
int gemm(const GemmArgs& g, cudaStream_t st);
// A * Bt^T on the FP64 tensor pipe when aligned (mma_gemm.cu), else gemm()
int gemm_nt(const GemmArgs& g, cudaStream_t st);

}  // namespace hpsb
