// FP64 tensor-core (DMMA, mma.sync m8n8k4 f64) batched "NT" GEMM for the
// leaf passes of the solve:
//     C[b] = alpha * A[b] * Bt[b]^T + beta * D[b]
// A (M x K) and Bt (N x K) row-major with K contiguous, which is how every
// leaf product of the solve is posed (solver.py:221-228, 269-272):
//     W = G_int * Ainv^T,  H = W * D_bi^T,  U_int = U_bnd * S_leaf^T + W.
// sm_100a has no tcgen05 f64 kind; the FP64 tensor path is the legacy DMMA
// pipe (measured 37 TFLOP/s, the same as DFMA on B200), used here because
// warp-level register blocking (a 32x32 warp tile = 4x4 DMMA tiles, 8
// fragment loads per 16 MMAs) keeps shared-memory traffic far below the
// DFMA register-tile kernel's.  Operands stream through a 2-stage cp.async
// (LDGSTS) pipeline; fragment rows are padded to 20 doubles so the 8x4
// fragment gathers hit every bank pair exactly twice.
#include "hps_common.cuh"

namespace hpsb {

namespace {

constexpr int BK = 16;
constexpr int SROW = BK + 4;  // padded smem row (doubles)

__device__ __forceinline__ void cp16(void* smem, const void* gmem, bool valid) {
  unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  int n = valid ? 16 : 0;  // src-size 0 zero-fills
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(n));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

template <int WM, int WN>
__global__ void __launch_bounds__(WM* WN * 32) k_mma_nt(GemmArgs g, int tilesM, int tilesN) {
  constexpr int BM = WM * 32, BN = WN * 32, NT = WM * WN * 32;
  extern __shared__ double sm[];
  double* As = sm;                        // [2][BM][SROW]
  double* Bs = sm + 2 * BM * SROW;        // [2][BN][SROW]
  const int tiles = tilesM * tilesN;
  const int b = blockIdx.x / tiles, t = blockIdx.x % tiles;
  const int m0 = (t / tilesN) * BM, n0 = (t % tilesN) * BN;
  const double* __restrict__ A = g.A + (long long)b * g.sA;
  const double* __restrict__ B = g.B + (long long)b * g.sB;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp / WN, wn = warp % WN;
  const int nk = (g.K + BK - 1) / BK;
  pdl_trigger();
  pdl_wait();

  auto issue = [&](int kt, int buf) {
    const int k0 = kt * BK;
    for (int e = tid; e < BM * BK / 2; e += NT) {
      const int r = e / (BK / 2), c = 2 * (e % (BK / 2));
      const int gm = m0 + r, gk = k0 + c;
      const bool ok = gm < g.M && gk < g.K;
      cp16(As + (buf * BM + r) * SROW + c, ok ? A + (long long)gm * g.lda + gk : A, ok);
    }
    for (int e = tid; e < BN * BK / 2; e += NT) {
      const int r = e / (BK / 2), c = 2 * (e % (BK / 2));
      const int gn = n0 + r, gk = k0 + c;
      const bool ok = gn < g.N && gk < g.K;
      cp16(Bs + (buf * BN + r) * SROW + c, ok ? B + (long long)gn * g.ldb + gk : B, ok);
    }
    cp_commit();
  };

  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) { acc[i][j][0] = 0.0; acc[i][j][1] = 0.0; }

  issue(0, 0);
  for (int kt = 0; kt < nk; ++kt) {
    const int buf = kt & 1;
    if (kt + 1 < nk) {
      issue(kt + 1, buf ^ 1);
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    __syncthreads();
    const double* Ab = As + (buf * BM + wm * 32 + (lane >> 2)) * SROW + (lane & 3);
    const double* Bb = Bs + (buf * BN + wn * 32 + (lane >> 2)) * SROW + (lane & 3);
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double af[4], bf[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) af[i] = Ab[i * 8 * SROW + kk];
#pragma unroll
      for (int j = 0; j < 4; ++j) bf[j] = Bb[j * 8 * SROW + kk];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
    __syncthreads();
  }

  double* C = g.C + (long long)b * g.sC;
  const double* D = g.D ? g.D + (long long)b * g.sD : nullptr;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int gm = m0 + wm * 32 + i * 8 + (lane >> 2);
    if (gm >= g.M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int gn = n0 + wn * 32 + j * 8 + 2 * (lane & 3) + h;
        if (gn >= g.N) continue;
        double v = g.alpha * acc[i][j][h];
        if (D && g.beta != 0.0) v = fma(g.beta, D[(long long)gm * g.ldd + gn], v);
        C[(long long)gm * g.ldc + gn] = v;
      }
    }
  }
}

template <int WM, int WN>
int launch_nt(const GemmArgs& g, cudaStream_t st) {
  constexpr int BM = WM * 32, BN = WN * 32;
  const size_t smem = (size_t)2 * (BM + BN) * SROW * 8;
  static bool attr = false;
  if (!attr) {
    HPSB_CUDA(cudaFuncSetAttribute(k_mma_nt<WM, WN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr = true;
  }
  int tm = (int)cdiv(g.M, BM), tn = (int)cdiv(g.N, BN);
  long long blocks = (long long)tm * tn * g.batch;
  if (blocks > 0x7fffffffLL) { set_error("gemm grid too large"); return -1; }
  HPSB_CUDA(launch_pdl(k_mma_nt<WM, WN>, dim3((unsigned)blocks), dim3(WM * WN * 32), smem, st, g, tm, tn));
  HPSB_LAUNCH_CHECK();
  return 0;
}

}  // namespace

// Tensor-core path when the operands allow 16-byte cp.async (even K and
// leading dimensions, 16-byte aligned bases); otherwise the DFMA kernel.
int gemm_nt(const GemmArgs& g, cudaStream_t st) {
  if (g.M <= 0 || g.N <= 0 || g.batch <= 0) return 0;
  const bool vec = g.tA == 0 && g.tB == 1 && (g.K % 2 == 0) && (g.lda % 2 == 0) && (g.ldb % 2 == 0) &&
                   ((uintptr_t)g.A % 16 == 0) && ((uintptr_t)g.B % 16 == 0) &&
                   (g.batch == 1 || ((g.sA % 2 == 0) && (g.sB % 2 == 0)));
  if (!vec) return gemm(g, st);
  if (g.N <= 32) return launch_nt<8, 1>(g, st);
  return launch_nt<4, 2>(g, st);
}

}  // namespace hpsb
