// Batched FP64 GEMM with DFMA register tiling (sm_100a).
//
// FP64 has no tcgen05 kind on sm_100a (ptxas rejects .kind::f64) and B200's
// DFMA and DMMA peaks are the same, so the build/shared-leaf GEMMs use a
// classic shared-memory tiled DFMA kernel: 64x64 CTA tile, K-slab 16,
// 256 threads with a 4x4 register tile each, register-staged double buffer.
#include "hps_common.cuh"

namespace hpsb {

namespace {

constexpr int BM = 64, BN = 64, BK = 16, NT = 256;

template <int TA, int TB>
__global__ void __launch_bounds__(NT) k_gemm(GemmArgs g, int tilesM, int tilesN) {
  __shared__ double As[2][BK][BM + 2];
  __shared__ double Bs[2][BK][BN + 2];
  const int tiles = tilesM * tilesN;
  const long long bid = blockIdx.x;
  const int b = (int)(bid / tiles);
  const int t = (int)(bid % tiles);
  const int m0 = (t / tilesN) * BM, n0 = (t % tilesN) * BN;
  const double* __restrict__ A = g.A + (long long)b * g.sA;
  const double* __restrict__ B = g.B + (long long)b * g.sB;
  const int tid = threadIdx.x, tx = tid & 15, ty = tid >> 4;
  pdl_trigger();
  pdl_wait();

  double ra[4], rb[4];
  auto loadA = [&](int k0) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      int e = tid + NT * i;
      int m, k;
      if (TA) { k = e / BM; m = e % BM; } else { m = e / BK; k = e % BK; }
      int gm = m0 + m, gk = k0 + k;
      double v = 0.0;
      if (gm < g.M && gk < g.K) v = TA ? A[(long long)gk * g.lda + gm] : A[(long long)gm * g.lda + gk];
      ra[i] = v;
    }
  };
  auto loadB = [&](int k0) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      int e = tid + NT * i;
      int n, k;
      if (TB) { n = e / BK; k = e % BK; } else { k = e / BN; n = e % BN; }
      int gn = n0 + n, gk = k0 + k;
      double v = 0.0;
      if (gn < g.N && gk < g.K) v = TB ? B[(long long)gn * g.ldb + gk] : B[(long long)gk * g.ldb + gn];
      rb[i] = v;
    }
  };
  auto storeAB = [&](int buf) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      int e = tid + NT * i;
      int m, k;
      if (TA) { k = e / BM; m = e % BM; } else { m = e / BK; k = e % BK; }
      As[buf][k][m] = ra[i];
      int n, kk;
      if (TB) { n = e / BK; kk = e % BK; } else { kk = e / BN; n = e % BN; }
      Bs[buf][kk][n] = rb[i];
    }
  };

  double acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = 0.0;

  const int nk = (g.K + BK - 1) / BK;
  loadA(0); loadB(0);
  storeAB(0);
  __syncthreads();
  for (int kt = 0; kt < nk; ++kt) {
    const int buf = kt & 1;
    if (kt + 1 < nk) { loadA((kt + 1) * BK); loadB((kt + 1) * BK); }
#pragma unroll
    for (int k = 0; k < BK; ++k) {
      double a[4], bb[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[buf][k][ty + 16 * i];
#pragma unroll
      for (int j = 0; j < 4; ++j) bb[j] = Bs[buf][k][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], bb[j], acc[i][j]);
    }
    if (kt + 1 < nk) {
      storeAB(buf ^ 1);
    }
    __syncthreads();
  }

  double* C = g.C + (long long)b * g.sC;
  const double* D = g.D ? g.D + (long long)b * g.sD : nullptr;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    int gm = m0 + ty + 16 * i;
    if (gm >= g.M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      int gn = n0 + tx + 16 * j;
      if (gn >= g.N) continue;
      double v = g.alpha * acc[i][j];
      if (D && g.beta != 0.0) v = fma(g.beta, D[(long long)gm * g.ldd + gn], v);
      C[(long long)gm * g.ldc + gn] = v;
    }
  }
}

}  // namespace

int gemm(const GemmArgs& g, cudaStream_t st) {
  if (g.M <= 0 || g.N <= 0 || g.batch <= 0) return 0;
  int tm = (int)cdiv(g.M, BM), tn = (int)cdiv(g.N, BN);
  long long blocks = (long long)tm * tn * g.batch;
  if (blocks > 0x7fffffffLL) { set_error("gemm grid too large"); return -1; }
  dim3 grid((unsigned)blocks);
  if (g.tA) {
    if (g.tB) HPSB_CUDA(launch_pdl(k_gemm<1, 1>, grid, dim3(NT), 0, st, g, tm, tn));
    else HPSB_CUDA(launch_pdl(k_gemm<1, 0>, grid, dim3(NT), 0, st, g, tm, tn));
  } else {
    if (g.tB) HPSB_CUDA(launch_pdl(k_gemm<0, 1>, grid, dim3(NT), 0, st, g, tm, tn));
    else HPSB_CUDA(launch_pdl(k_gemm<0, 0>, grid, dim3(NT), 0, st, g, tm, tn));
  }
  HPSB_LAUNCH_CHECK();
  return 0;
}

}  // namespace hpsb
