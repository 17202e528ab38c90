// One-time HPS build on the device (solver.py:53-158).
//
//  leaf:  A_ii = sigma I + dtg A_ii, A_ib = dtg A_ib  (operators.py:252-274)
//         Ainv = A_ii^-1 (pivoted Gauss-Jordan), S = -Ainv A_ib, T = D_bi S + D_bb
//  merge: X33 = Ta33 - Tb33, Xinv = X33^-1, S = Xinv [-Ta31 | Tb32],
//         Tstack = [Ta13; Tb23], T = blkdiag(Ta11, Tb22) + Tstack S
//
// The singularity policy of linalg.py:17,36-42 (min|pivot| <= 1e-13 max|pivot|
// of the partial-pivoting elimination) is evaluated on the Gauss-Jordan
// pivots, which coincide with the LU pivots (the sub-diagonal part of the
// elimination is the same); the host reports the first failing node.
#include "hps_plan.cuh"

namespace hpsb {

namespace {

// ---------------------------------------------------------------------------
// leaf collocation blocks
// ---------------------------------------------------------------------------
__global__ void k_leaf_assemble(int Lc, int ni, int nb, const double* __restrict__ cv,
                                int has_c1, int has_c2, int has_c,
                                const double* __restrict__ D2x, const double* __restrict__ D2y,
                                const double* __restrict__ D1x, const double* __restrict__ D1y,
                                double sigma, double dtg, double* __restrict__ Aii,
                                double* __restrict__ Aib) {
  const int m = ni + nb;
  long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (e >= (long long)Lc * ni * m) return;
  int l = (int)(e / ((long long)ni * m));
  int r = (int)(e % ((long long)ni * m));
  int i = r / m, j = r % m;
  const double* v = cv + (long long)l * 5 * ni;
  double c11 = v[i], c22 = v[ni + i], c1 = v[2 * ni + i], c2 = v[3 * ni + i], c0 = v[4 * ni + i];
  long long o = (long long)i * m + j;
  // rows = -c11 D2x - c22 D2y (+ c1 D1x) (+ c2 D1y) (+ diag c), no contraction
  double t = __dmul_rn(-c11, D2x[o]);
  t = __dsub_rn(t, __dmul_rn(c22, D2y[o]));
  if (has_c1) t = __dadd_rn(t, __dmul_rn(c1, D1x[o]));
  if (has_c2) t = __dadd_rn(t, __dmul_rn(c2, D1y[o]));
  if (has_c && j == i) t = __dadd_rn(t, c0);
  if (j < ni) {
    double d = (j == i) ? sigma : 0.0;
    Aii[(long long)l * ni * ni + (long long)i * ni + j] = __dadd_rn(d, __dmul_rn(dtg, t));
  } else {
    Aib[(long long)l * ni * nb + (long long)i * nb + (j - ni)] = __dmul_rn(dtg, t);
  }
}

// ---------------------------------------------------------------------------
// Gauss-Jordan inversion with partial pivoting, one CTA per matrix (n <= 128)
// in: A (n x n, ld n), out: X (n x n, ld ldx); stats[b] = (min|piv|, max|piv|)
// ---------------------------------------------------------------------------
constexpr int GJ_SMALL = 128;

__global__ void __launch_bounds__(512) k_gj_small(int n, const double* __restrict__ A, long long sA,
                                                   double* __restrict__ X, int ldx, long long sX,
                                                   double* __restrict__ stats) {
  extern __shared__ double sm[];
  double* M = sm;               // n x n
  double* fcol = sm + n * n;    // n
  int* piv = (int*)(fcol + n);  // n
  __shared__ int s_p;
  __shared__ double s_pmin, s_pmax;
  __shared__ double s_bv[32];
  __shared__ int s_bi[32];
  const int b = blockIdx.x, tid = threadIdx.x, nt = blockDim.x;
  const double* Ab = A + (long long)b * sA;
  for (int e = tid; e < n * n; e += nt) M[e] = Ab[e];
  if (tid == 0) { s_pmin = INFINITY; s_pmax = 0.0; }
  __syncthreads();
  for (int j = 0; j < n; ++j) {
    // argmax |M[i][j]|, i >= j, first index on ties
    double bv = -1.0; int bi = n;
    for (int i = j + tid; i < n; i += nt) {
      double a = fabs(M[i * n + j]);
      if (a > bv) { bv = a; bi = i; }
    }
    for (int off = 16; off > 0; off >>= 1) {
      double ov = __shfl_xor_sync(0xffffffffu, bv, off);
      int oi = __shfl_xor_sync(0xffffffffu, bi, off);
      if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
    }
    if ((tid & 31) == 0) { s_bv[tid >> 5] = bv; s_bi[tid >> 5] = bi; }
    __syncthreads();
    if (tid == 0) {
      double v = s_bv[0]; int ii = s_bi[0];
      for (int w = 1; w < nt / 32; ++w)
        if (s_bv[w] > v || (s_bv[w] == v && s_bi[w] < ii)) { v = s_bv[w]; ii = s_bi[w]; }
      s_p = ii;
      piv[j] = ii;
      s_pmin = fmin(s_pmin, v);
      s_pmax = fmax(s_pmax, v);
    }
    __syncthreads();
    const int p = s_p;
    if (p != j)
      for (int c = tid; c < n; c += nt) {
        double t = M[j * n + c]; M[j * n + c] = M[p * n + c]; M[p * n + c] = t;
      }
    __syncthreads();
    const double pv = M[j * n + j];
    __syncthreads();
    for (int c = tid; c < n; c += nt) M[j * n + c] = (c == j) ? 1.0 / pv : M[j * n + c] / pv;
    for (int i = tid; i < n; i += nt) fcol[i] = M[i * n + j];
    __syncthreads();
    for (int e = tid; e < n * n; e += nt) {
      int i = e / n, c = e % n;
      if (i == j) continue;
      double f = fcol[i];
      M[e] = (c == j) ? -f * M[j * n + j] : M[e] - f * M[j * n + c];
    }
    __syncthreads();
  }
  // undo the row interchanges as column interchanges, last first
  for (int j = n - 1; j >= 0; --j) {
    int p = piv[j];
    if (p != j)
      for (int i = tid; i < n; i += nt) {
        double t = M[i * n + j]; M[i * n + j] = M[i * n + p]; M[i * n + p] = t;
      }
    __syncthreads();
  }
  double* Xb = X + (long long)b * sX;
  for (int e = tid; e < n * n; e += nt) Xb[(long long)(e / n) * ldx + e % n] = M[e];
  if (tid == 0) { stats[2 * b] = s_pmin; stats[2 * b + 1] = s_pmax; }
}

// ---------------------------------------------------------------------------
// Large matrices: one grid-wide launch per elimination step, ping-pong
// buffers so the pivot row is read unmodified by every CTA; each CTA also
// publishes its candidate for the next pivot column.
// ---------------------------------------------------------------------------
constexpr int GJ_RB = 16;  // rows per CTA

struct Cand { double v; int i; int pad; };

__global__ void k_gj_cand0(int n, const double* __restrict__ A, long long sA, Cand* cand, int nrb) {
  const int rb = blockIdx.x, b = blockIdx.y, tid = threadIdx.x;
  const double* Ab = A + (long long)b * sA;
  double bv = -1.0; int bi = n;
  for (int i = rb * GJ_RB + tid; i < min(n, (rb + 1) * GJ_RB); i += blockDim.x) {
    double a = fabs(Ab[(long long)i * n]);
    if (a > bv) { bv = a; bi = i; }
  }
  for (int off = 16; off > 0; off >>= 1) {
    double ov = __shfl_xor_sync(0xffffffffu, bv, off);
    int oi = __shfl_xor_sync(0xffffffffu, bi, off);
    if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
  }
  if (tid == 0) cand[(long long)b * nrb + rb] = Cand{bv, bi, 0};
}

__global__ void __launch_bounds__(256) k_gj_step(int n, int j, const double* __restrict__ Ain,
                                                  double* __restrict__ Aout, long long sA,
                                                  const Cand* __restrict__ cin, Cand* __restrict__ cout,
                                                  int nrb, int* __restrict__ piv,
                                                  double* __restrict__ stats) {
  __shared__ double s_bv[8];
  __shared__ int s_bi[8];
  __shared__ int s_p;
  const int rb = blockIdx.x, b = blockIdx.y, tid = threadIdx.x, nt = blockDim.x;
  const double* Ai = Ain + (long long)b * sA;
  double* Ao = Aout + (long long)b * sA;
  // pivot: reduce the candidates published by the previous step
  {
    double bv = -1.0; int bi = n;
    for (int t = tid; t < nrb; t += nt) {
      Cand c = cin[(long long)b * nrb + t];
      if (c.v > bv || (c.v == bv && c.i < bi)) { bv = c.v; bi = c.i; }
    }
    for (int off = 16; off > 0; off >>= 1) {
      double ov = __shfl_xor_sync(0xffffffffu, bv, off);
      int oi = __shfl_xor_sync(0xffffffffu, bi, off);
      if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
    }
    if ((tid & 31) == 0) { s_bv[tid >> 5] = bv; s_bi[tid >> 5] = bi; }
    __syncthreads();
    if (tid == 0) {
      double v = s_bv[0]; int ii = s_bi[0];
      for (int w = 1; w < nt / 32; ++w)
        if (s_bv[w] > v || (s_bv[w] == v && s_bi[w] < ii)) { v = s_bv[w]; ii = s_bi[w]; }
      s_p = ii;
      if (rb == 0) {
        piv[(long long)b * n + j] = ii;
        double* st = stats + 2 * b;
        st[0] = (j == 0) ? v : fmin(st[0], v);
        st[1] = (j == 0) ? v : fmax(st[1], v);
      }
    }
    __syncthreads();
  }
  const int p = s_p;
  const double pv = Ai[(long long)p * n + j];
  const double inv = 1.0 / pv;
  double bv = -1.0; int bi = n;
  const int r0 = rb * GJ_RB, r1 = min(n, r0 + GJ_RB);
  for (int i = r0; i < r1; ++i) {
    const int src = (i == j) ? p : ((i == p) ? j : i);
    const double* rs = Ai + (long long)src * n;
    const double* rp = Ai + (long long)p * n;
    double* ro = Ao + (long long)i * n;
    if (i == j) {
      for (int c = tid; c < n; c += nt) {
        double v = (c == j) ? inv : rp[c] / pv;
        ro[c] = v;
      }
    } else {
      const double f = rs[j];
      for (int c = tid; c < n; c += nt) {
        double v = (c == j) ? -f * inv : rs[c] - f * (rp[c] / pv);
        ro[c] = v;
        if (c == j + 1 && i >= j + 1) {
          double a = fabs(v);
          if (a > bv || (a == bv && i < bi)) { bv = a; bi = i; }
        }
      }
    }
  }
  // publish the candidate for column j+1 (the thread owning column j+1 holds it)
  for (int off = 16; off > 0; off >>= 1) {
    double ov = __shfl_xor_sync(0xffffffffu, bv, off);
    int oi = __shfl_xor_sync(0xffffffffu, bi, off);
    if (ov > bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
  }
  __syncthreads();
  if ((tid & 31) == 0) { s_bv[tid >> 5] = bv; s_bi[tid >> 5] = bi; }
  __syncthreads();
  if (tid == 0 && j + 1 < n) {
    double v = s_bv[0]; int ii = s_bi[0];
    for (int w = 1; w < nt / 32; ++w)
      if (s_bv[w] > v || (s_bv[w] == v && s_bi[w] < ii)) { v = s_bv[w]; ii = s_bi[w]; }
    cout[(long long)b * nrb + rb] = Cand{v, ii, 0};
  }
}

__global__ void k_gj_unscramble(int n, const double* __restrict__ A, long long sA, const int* __restrict__ piv,
                                double* __restrict__ X, int ldx, long long sX) {
  extern __shared__ int pos[];
  const int b = blockIdx.y, tid = threadIdx.x;
  if (tid == 0) {
    for (int c = 0; c < n; ++c) pos[c] = c;
    const int* pb = piv + (long long)b * n;
    for (int j = n - 1; j >= 0; --j) {
      int p = pb[j];
      int t = pos[j]; pos[j] = pos[p]; pos[p] = t;
    }
  }
  __syncthreads();
  const double* Ab = A + (long long)b * sA;
  double* Xb = X + (long long)b * sX;
  for (int i = blockIdx.x; i < n; i += gridDim.x)
    for (int c = tid; c < n; c += blockDim.x) Xb[(long long)i * ldx + c] = Ab[(long long)i * n + pos[c]];
}

// ---------------------------------------------------------------------------
// merge assembly from the children's DtN maps (tree-uniform index maps)
// ---------------------------------------------------------------------------
__global__ void k_merge_gather(int c, int n3, int n1a, int n2b, int nbc, const double* __restrict__ Tc,
                               long long sTc, const int* __restrict__ i1a, const int* __restrict__ i3a,
                               const int* __restrict__ i2b, const int* __restrict__ i3b,
                               double* __restrict__ X33, double* __restrict__ R, double* __restrict__ Tst,
                               int ld3, double* __restrict__ Tnew) {
  const int n12 = n1a + n2b;
  const long long per = (long long)n3 * n3 + (long long)n3 * n12 + (long long)n12 * n3 +
                        (Tnew ? (long long)n12 * n12 : 0);
  long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (e >= per * c) return;
  const int node = (int)(e / per);
  long long r = e % per;
  const double* Ta = Tc + (2LL * node) * sTc;
  const double* Tb = Tc + (2LL * node + 1) * sTc;
  if (r < (long long)n3 * n3) {
    int a = (int)(r / n3), bb = (int)(r % n3);
    X33[(long long)node * n3 * n3 + r] = Ta[(long long)i3a[a] * nbc + i3a[bb]] - Tb[(long long)i3b[a] * nbc + i3b[bb]];
    return;
  }
  r -= (long long)n3 * n3;
  if (r < (long long)n3 * n12) {
    int a = (int)(r / n12), bb = (int)(r % n12);
    double v = (bb < n1a) ? -Ta[(long long)i3a[a] * nbc + i1a[bb]] : Tb[(long long)i3b[a] * nbc + i2b[bb - n1a]];
    R[(long long)node * n3 * n12 + r] = v;
    return;
  }
  r -= (long long)n3 * n12;
  if (r < (long long)n12 * n3) {
    int a = (int)(r / n3), bb = (int)(r % n3);
    double v = (a < n1a) ? Ta[(long long)i1a[a] * nbc + i3a[bb]] : Tb[(long long)i2b[a - n1a] * nbc + i3b[bb]];
    Tst[(long long)node * n12 * ld3 + (long long)a * ld3 + bb] = v;
    return;
  }
  r -= (long long)n12 * n3;
  int a = (int)(r / n12), bb = (int)(r % n12);
  double v = 0.0;
  if (a < n1a && bb < n1a) v = Ta[(long long)i1a[a] * nbc + i1a[bb]];
  else if (a >= n1a && bb >= n1a) v = Tb[(long long)i2b[a - n1a] * nbc + i2b[bb - n1a]];
  Tnew[(long long)node * n12 * n12 + r] = v;
}

__global__ void k_broadcast(long long n, int copies, const double* __restrict__ src, double* __restrict__ dst) {
  long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  long long tot = n * (copies - 1);
  for (; e < tot; e += (long long)gridDim.x * blockDim.x) dst[n + e] = src[e % n];
}

}  // namespace

// ---------------------------------------------------------------------------
// host-side helpers
// ---------------------------------------------------------------------------

// Invert `batch` n x n matrices (ld n, stride n*n) into X (ld ldx, stride sX).
// stats (device, 2*batch) receives (min|pivot|, max|pivot|).
int gj_invert(int n, int batch, double* A, double* X, int ldx, long long sX, double* stats,
              cudaStream_t st) {
  if (n <= 0 || batch <= 0) return 0;
  if (n <= GJ_SMALL) {
    size_t smem = (size_t)n * n * 8 + (size_t)n * 8 + (size_t)n * 4 + 16;
    static bool set = false;
    if (!set) {
      HPSB_CUDA(cudaFuncSetAttribute(k_gj_small, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
      set = true;
    }
    int nt = n * n >= 4096 ? 512 : 256;
    k_gj_small<<<batch, nt, smem, st>>>(n, A, (long long)n * n, X, ldx, sX, stats);
    HPSB_LAUNCH_CHECK();
    return 0;
  }
  const long long sA = (long long)n * n;
  const int nrb = (int)cdiv(n, GJ_RB);
  double* B = nullptr;
  Cand* cand = nullptr;
  int* piv = nullptr;
  HPSB_CUDA(cudaMallocAsync(&B, (size_t)sA * batch * 8, st));
  HPSB_CUDA(cudaMallocAsync(&cand, (size_t)2 * nrb * batch * sizeof(Cand), st));
  HPSB_CUDA(cudaMallocAsync(&piv, (size_t)n * batch * sizeof(int), st));
  Cand* c0 = cand;
  Cand* c1 = cand + (long long)nrb * batch;
  k_gj_cand0<<<dim3(nrb, batch), 32, 0, st>>>(n, A, sA, c0, nrb);
  HPSB_LAUNCH_CHECK();
  double* cur = A;
  double* nxt = B;
  for (int j = 0; j < n; ++j) {
    k_gj_step<<<dim3(nrb, batch), 256, 0, st>>>(n, j, cur, nxt, sA, (j & 1) ? c1 : c0, (j & 1) ? c0 : c1,
                                                nrb, piv, stats);
    double* t = cur; cur = nxt; nxt = t;
  }
  g_launches.fetch_add(n - 1, std::memory_order_relaxed);  // n step launches, one check
  HPSB_LAUNCH_CHECK();
  k_gj_unscramble<<<dim3(min(n, 1024), batch), 256, (size_t)n * 4, st>>>(n, cur, sA, piv, X, ldx, sX);
  HPSB_LAUNCH_CHECK();
  HPSB_CUDA(cudaFreeAsync(B, st));
  HPSB_CUDA(cudaFreeAsync(cand, st));
  HPSB_CUDA(cudaFreeAsync(piv, st));
  return 0;
}

int leaf_assemble(int Lc, int ni, int nb, const double* cv, int has_c1, int has_c2, int has_c,
                  const double* D2x, const double* D2y, const double* D1x, const double* D1y,
                  double sigma, double dtg, double* Aii, double* Aib, cudaStream_t st) {
  long long n = (long long)Lc * ni * (ni + nb);
  k_leaf_assemble<<<(unsigned)cdiv(n, 256), 256, 0, st>>>(Lc, ni, nb, cv, has_c1, has_c2, has_c, D2x, D2y,
                                                          D1x, D1y, sigma, dtg, Aii, Aib);
  HPSB_LAUNCH_CHECK();
  return 0;
}

int merge_gather(int c, int n3, int n1a, int n2b, int nbc, const double* Tc, long long sTc,
                 const int* i1a, const int* i3a, const int* i2b, const int* i3b, double* X33, double* R,
                 double* Tst, int ld3, double* Tnew, cudaStream_t st) {
  const int n12 = n1a + n2b;
  long long per = (long long)n3 * n3 + 2LL * n3 * n12 + (Tnew ? (long long)n12 * n12 : 0);
  long long n = per * c;
  k_merge_gather<<<(unsigned)cdiv(n, 256), 256, 0, st>>>(c, n3, n1a, n2b, nbc, Tc, sTc, i1a, i3a, i2b, i3b,
                                                         X33, R, Tst, ld3, Tnew);
  HPSB_LAUNCH_CHECK();
  return 0;
}

int broadcast_copies(long long n, int copies, double* base, cudaStream_t st) {
  if (copies <= 1) return 0;
  long long tot = n * (copies - 1);
  unsigned blocks = (unsigned)std::min<long long>(cdiv(tot, 256), 148LL * 64);
  k_broadcast<<<blocks, 256, 0, st>>>(n, copies, base, base);
  HPSB_LAUNCH_CHECK();
  return 0;
}

}  // namespace hpsb
