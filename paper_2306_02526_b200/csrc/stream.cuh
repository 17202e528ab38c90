// Column-streaming core shared by the level and subtree GEMV kernels.
//
// A thread owns two adjacent rows of a column-major panel tile (one 16-byte
// load per column) and accumulates acc{0,1}[kk] += M[col].{x,y} * x[kk][col]
// with x in shared memory.  Two register batches of U columns alternate
// without copies (a copy would force a wait on the in-flight loads), so one
// batch is always in flight while the other is consumed.
#pragma once

#include "hps_common.cuh"

namespace hpsb {

template <int U>
__device__ __forceinline__ void load_batch(double2 (&m)[U], const double2* __restrict__ M, int cs, int col) {
#pragma unroll
  for (int u = 0; u < U; ++u) m[u] = __ldcs(M + (size_t)(col + u) * cs);
}

template <int KM, int U>
__device__ __forceinline__ void fma_batch(const double2 (&m)[U], const double* xs, int oa, int ob, int XS, int col,
                                          double (&acc0)[KM], double (&acc1)[KM]) {
#pragma unroll
  for (int u = 0; u < U; ++u)
#pragma unroll
    for (int kk = 0; kk < KM; ++kk) {
      acc0[kk] = fma(m[u].x, xs[oa + kk * XS + col + u], acc0[kk]);
      acc1[kk] = fma(m[u].y, xs[ob + kk * XS + col + u], acc1[kk]);
    }
}

// A must already hold columns [c0, c0+U) when (c1 - c0) >= U.
template <int KM, int U>
__device__ __forceinline__ void stream_cols(double2 (&A)[U], const double2* __restrict__ M, int cs, int c0, int c1,
                                            const double* xs, int oa, int ob, int XS, double (&acc0)[KM],
                                            double (&acc1)[KM]) {
  double2 B[U];
  const int nfull = (c1 - c0) / U;
  int b = 0;
  for (; b + 1 < nfull; b += 2) {
    load_batch<U>(B, M, cs, c0 + (b + 1) * U);
    fma_batch<KM, U>(A, xs, oa, ob, XS, c0 + b * U, acc0, acc1);
    if (b + 2 < nfull) load_batch<U>(A, M, cs, c0 + (b + 2) * U);
    fma_batch<KM, U>(B, xs, oa, ob, XS, c0 + (b + 1) * U, acc0, acc1);
  }
  if (b < nfull) fma_batch<KM, U>(A, xs, oa, ob, XS, c0 + b * U, acc0, acc1);
  for (int col = c0 + nfull * U; col < c1; ++col) {
    const double2 m = __ldcs(M + (size_t)col * cs);
#pragma unroll
    for (int kk = 0; kk < KM; ++kk) {
      acc0[kk] = fma(m.x, xs[oa + kk * XS + col], acc0[kk]);
      acc1[kk] = fma(m.y, xs[ob + kk * XS + col], acc1[kk]);
    }
  }
}

// Both rows of the thread apply to ONE input vector x (a shared operator:
// the row pair belongs to one node): x is read two columns at a time
// (16-byte shared loads; x 16-byte aligned), operator addresses advance by a
// pointer increment.  Columns [0, n) of x and of the panel starting at M.
__device__ __forceinline__ void stream_pairs(const double2* __restrict__ M, int cs, int n, const double* x,
                                             double& acc0, double& acc1) {
  constexpr int U = 4;
  const double2* p = M;
  double2 A[U], B[U];
  auto ld = [&](double2 (&m)[U]) {
#pragma unroll
    for (int u = 0; u < U; ++u) { m[u] = __ldcs(p); p += cs; }
  };
  auto fma4 = [&](const double2 (&m)[U], int col) {
#pragma unroll
    for (int u = 0; u < U; u += 2) {
      const double2 xv = *reinterpret_cast<const double2*>(x + col + u);
      acc0 = fma(m[u].x, xv.x, acc0);
      acc1 = fma(m[u].y, xv.x, acc1);
      acc0 = fma(m[u + 1].x, xv.y, acc0);
      acc1 = fma(m[u + 1].y, xv.y, acc1);
    }
  };
  const int nfull = n / U;
  if (nfull > 0) ld(A);
  int b = 0;
  for (; b + 1 < nfull; b += 2) {
    ld(B);
    fma4(A, b * U);
    if (b + 2 < nfull) ld(A);
    fma4(B, (b + 1) * U);
  }
  if (b < nfull) fma4(A, b * U);
  for (int col = nfull * U; col < n; ++col) {
    const double2 m = __ldcs(p);
    p += cs;
    acc0 = fma(m.x, x[col], acc0);
    acc1 = fma(m.y, x[col], acc1);
  }
}

// NB input vectors at x + j * XS (16-byte aligned rows, XS even) share one
// operator (row pair of a one-node panel): acc{0,1}[j] += M[col].{x,y} x[j][col]
// over columns [0, n).  A must already hold columns [0, U) when n >= U.
template <int NB, int U>
__device__ __forceinline__ void stream_pairs_nb(double2 (&A)[U], const double2* __restrict__ M, int cs, int n,
                                                const double* x, int XS, double (&acc0)[NB], double (&acc1)[NB]) {
  static_assert(U % 2 == 0, "column pairs");
  const int nfull = n / U;
  const double2* p = M + (size_t)(nfull > 0 ? U : 0) * cs;
  double2 B[U];
  auto ld = [&](double2 (&m)[U]) {
#pragma unroll
    for (int u = 0; u < U; ++u) { m[u] = __ldcs(p); p += cs; }
  };
  auto fma4 = [&](const double2 (&m)[U], int col) {
#pragma unroll
    for (int u = 0; u < U; u += 2)
#pragma unroll
      for (int j = 0; j < NB; ++j) {
        const double2 xv = *reinterpret_cast<const double2*>(x + j * XS + col + u);
        acc0[j] = fma(m[u].x, xv.x, acc0[j]);
        acc1[j] = fma(m[u].y, xv.x, acc1[j]);
        acc0[j] = fma(m[u + 1].x, xv.y, acc0[j]);
        acc1[j] = fma(m[u + 1].y, xv.y, acc1[j]);
      }
  };
  int b = 0;
  for (; b + 1 < nfull; b += 2) {
    ld(B);
    fma4(A, b * U);
    if (b + 2 < nfull) ld(A);
    fma4(B, (b + 1) * U);
  }
  if (b < nfull) fma4(A, b * U);
  for (int col = nfull * U; col < n; ++col) {
    const double2 m = __ldcs(p);
    p += cs;
#pragma unroll
    for (int j = 0; j < NB; ++j) {
      acc0[j] = fma(m.x, x[j * XS + col], acc0[j]);
      acc1[j] = fma(m.y, x[j * XS + col], acc1[j]);
    }
  }
}

}  // namespace hpsb
