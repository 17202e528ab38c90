// Tensor-product ("fast diagonalisation") leaf solve for constant coefficients.
//
// With constant coefficients the interior collocation block is a Kronecker
// sum (operators.py:252-269 with x-major interior order):
//     A_ii = Ax (x) I + I (x) Ay + s I,   Ax = dtg(-c11 d2x + c1 d1x)_int,
//                                         Ay = dtg(-c22 d2y + c2 d1y)_int,
//                                         s  = sigma + dtg c,
// so with Ax = Vx Lx Vx^-1, Ay = Vy Ly Vy^-1 (real spectra, checked on the
// host) the leaf particular solution w = A_ii^-1 r of solver.py:221-223 is
//     W = Vx [ (Vx^-1 R Vy^-T) ./ (lx_a + ly_b + s) ] Vy^T     (R, W: q x q)
// -- 8 q^3 flops per leaf instead of the dense inverse's 2 q^4 -- and the
// leaf's outgoing flux h = D_bi w (solver.py:228) reads one grid line per
// boundary point (2 q^2 flops instead of 8 q^3).  Results agree with the
// LU-based reference to round-off times cond(V) (checked by the parity tests).
//
// One CTA works on LB leaves at a time (persistent over leaf groups); the
// four q x q products run from shared memory, one output per thread-slot.
#include <stdlib.h>

#include "hps_plan.cuh"

namespace hpsb {

namespace {

constexpr int NT = 256;

constexpr int kFdTerms = 12;  // FD_UP_T: terms of the body load

struct FdArgs {
  int L, k, nw;
  const double* g; long long ld_g;   // body load rows (leaf l interior at l*ni); null = zero
  double* WH; long long ld_wh;       // FD_UP_WH: [w | h] rows of nw = ni + nb per leaf
  double* H; long long ld_h;         // FD_UP_H: h rows of nb per leaf
  const int* lbg;                    // FD_DOWN: leaf boundary DOF ids (L x nb, first leaf of the range)
  const double* u; long long ld_u;   // FD_DOWN: solution rows (boundary values read through lbg)
  double* uint; long long ld_uint;   // FD_DOWN: interior output (leaf l at l*ni)
  double* lu; long long ld_lu;       // FD_DOWN, optional: L u at the interiors (the stage history)
  double lu_sigma, lu_inv_dtg;       // FD_DOWN with lu: inv_dtg != 0 -> L u = (sigma u_int - r) / dtg from the
                                     // solved interior equation instead of two more leaf-grid products
  unsigned long long* guard;         // ... and max |u| over the leaves' grids (bits, NaN sticky)
  int nterm; const double* tv[kFdTerms]; const double* tdc;  // FD_UP_T: body load = sum_t tdc[t] tv[t] ...
  long long tld[kFdTerms];                                   // (rhs row strides of the terms, 0 = shared row)
  double* rout; long long ld_rout;                           // ... written here (leaf l interior at l*ni)
  // FD_UP_H, optional: the solve's Dirichlet data u[ids[i]] = fb[i] (solver.py:259-260), written by the
  // CTAs after the dependency wait (the up sweep never reads u) -- one launch fewer per solve
  int nbd; const int* bids; const double* fb; long long ld_f; double* ubnd; long long ld_ubnd;
  const double* mats;                // Vxi, VyiT, Vx, VyT, den (q x q each), flux rows ex0, ex1, ey0, ey1,
                                     // then the interior-boundary couplings bx0, bx1, by0, by1 (q each),
                                     // then Mx = c11 d2x - c1 d1x, My = c22 d2y - c2 d1y (16 x 16, zero
                                     // padded) and c: L u = Mx G + G My^T - c G on the leaf grid G
};

// modes of the tensor-core kernel
// FD_LU: L u at the interiors of a given state (interiors from a.uint, boundary
// values through lbg), the stage history of an explicit stage
// FD_UP_T: FD_UP_H with the body load formed from terms (sum_t c_t v_t, the
// stage combination) and written out for the downward sweep
enum FdMode { FD_UP_WH = 0, FD_UP_H = 1, FD_DOWN = 2, FD_LU = 3, FD_UP_T = 4 };

template <int Q>
__global__ void __launch_bounds__(NT) k_leaf_fd(FdArgs a) {
  constexpr int QS = Q + 1, QQ = Q * QS, NI = Q * Q, NB = 4 * Q, P = Q + 2;
  constexpr int LB = Q >= 12 ? 8 : 16;  // leaves per group (static smem < 48 KB)
  __shared__ double M[5][QQ];
  __shared__ double E[4][Q];
  __shared__ double B0[LB][QQ], B1[LB][QQ];
  const int tid = threadIdx.x, kk = blockIdx.y;
  pdl_trigger();
  for (int e = tid; e < 5 * NI; e += NT) M[e / NI][(e % NI) / Q * QS + e % Q] = a.mats[e];
  for (int e = tid; e < 4 * Q; e += NT) E[e / Q][e % Q] = a.mats[5 * NI + e];
  pdl_wait();
  const double* g = a.g + kk * a.ld_g;
  double* wh = a.WH + kk * a.ld_wh;
  for (int l0 = blockIdx.x * LB; l0 < a.L; l0 += gridDim.x * LB) {
    const int nl = min(LB, a.L - l0);
    __syncthreads();
    for (int e = tid; e < nl * NI; e += NT) B0[e / NI][(e % NI) / Q * QS + e % Q] = g[(long long)l0 * NI + e];
    __syncthreads();
    // B1 = Vx^-1 B0
    for (int e = tid; e < nl * NI; e += NT) {
      const int l = e / NI, i = (e % NI) / Q, j = e % Q;
      double s = 0.0;
#pragma unroll
      for (int t = 0; t < Q; ++t) s = fma(M[0][i * QS + t], B0[l][t * QS + j], s);
      B1[l][i * QS + j] = s;
    }
    __syncthreads();
    // B0 = (B1 Vy^-T) ./ den
    for (int e = tid; e < nl * NI; e += NT) {
      const int l = e / NI, i = (e % NI) / Q, j = e % Q;
      double s = 0.0;
#pragma unroll
      for (int t = 0; t < Q; ++t) s = fma(B1[l][i * QS + t], M[1][t * QS + j], s);
      B0[l][i * QS + j] = s * M[4][i * QS + j];
    }
    __syncthreads();
    // B1 = Vx B0
    for (int e = tid; e < nl * NI; e += NT) {
      const int l = e / NI, i = (e % NI) / Q, j = e % Q;
      double s = 0.0;
#pragma unroll
      for (int t = 0; t < Q; ++t) s = fma(M[2][i * QS + t], B0[l][t * QS + j], s);
      B1[l][i * QS + j] = s;
    }
    __syncthreads();
    // w = B1 Vy^T  ->  B0 and the w part of the output rows
    for (int e = tid; e < nl * NI; e += NT) {
      const int l = e / NI, i = (e % NI) / Q, j = e % Q;
      double s = 0.0;
#pragma unroll
      for (int t = 0; t < Q; ++t) s = fma(B1[l][i * QS + t], M[3][t * QS + j], s);
      B0[l][i * QS + j] = s;
      wh[(long long)(l0 + l) * a.nw + i * Q + j] = s;
    }
    __syncthreads();
    // h = D_bi w: normal derivative along the grid line through each boundary point
    for (int e = tid; e < nl * NB; e += NT) {
      const int l = e / NB, b = e % NB;
      double s = 0.0;
      if (b < Q || b >= 3 * Q) {  // east (xi = 0) / west (xi = p-1): d/dx along row yi
        const int yi = (b < Q ? b : b - 3 * Q);
        const double* r = E[b < Q ? 0 : 1];
#pragma unroll
        for (int t = 0; t < Q; ++t) s = fma(r[t], B0[l][t * QS + yi], s);
      } else {                    // north / south interleaved: d/dy along column xi
        const int jj = b - Q, xi = jj / 2;
        const double* r = E[(jj & 1) ? 3 : 2];
#pragma unroll
        for (int t = 0; t < Q; ++t) s = fma(r[t], B0[l][xi * QS + t], s);
      }
      wh[(long long)(l0 + l) * a.nw + NI + b] = s;
    }
  }
  (void)P;
}

// DMMA variant: one warp per leaf, the q x q blocks zero-padded to 16 x 16 so
// each of the four products is 2 x 2 output tiles x 4 k-steps of
// mma.sync.m8n8k4.f64.  The four constant matrices and 1/den live in
// registers as MMA fragments for the whole kernel; the leaf's blocks move
// through two per-warp shared buffers whose strides make every fragment load
// conflict-free (B-operand reads use stride 24, A-operand reads stride 20).
constexpr int SB = 24, SA = 20;

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// FD_DOWN is the leaf half of the downward sweep without storing w:
//     u_int = A_ii^-1 (r - A_ib u_b)   (= S_leaf u_b + w, solver.py:269-276)
// where A_ib u_b at interior point (x, y) couples only the four boundary
// points on its grid lines: bx0[x] u(0,y) + bx1[x] u(p-1,y) + by0[y] u(x,0)
// + by1[y] u(x,p-1).
// Constant operands live in shared memory (one copy per CTA) in strides that
// make every fragment load conflict-free: A-type (row-indexed by the lane's
// group) stride CSA = 20, B-type stride CSB = 24.
constexpr int CSA = 20, CSB = 24;
constexpr int kFdCst = 5 * 16 * CSA + 2 * 16 * CSB + 8 * CSA + 16 * 8;  // Vxi, Vx, Mx, My, 1/den | VyiT, VyT |
                                                                        // flux projections (FD_UP_H)

template <int Q, int MODE>
__global__ void __launch_bounds__(256, 2) k_leaf_fd_mma(FdArgs a) {
  constexpr bool DOWNLIKE = MODE == FD_DOWN || MODE == FD_LU;   // leaf grid + boundary values
  constexpr bool UPH = MODE == FD_UP_H || MODE == FD_UP_T;       // fluxes only on the way up
  constexpr int NI = Q * Q, NB = 4 * Q, UBS = 4 * Q + 8;
  // k-steps of 4 that cover the q (leaf solve) / p (stage history) columns:
  // the zero padding beyond them is never multiplied
  constexpr int KS = (Q + 3) / 4, KSL = (Q + 2 + 3) / 4;
  extern __shared__ double sm[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double* bufB = sm + warp * (16 * (SB + SA) + UBS);   // stride SB
  double* bufA = bufB + 16 * SB;                       // stride SA
  double* ub = bufA + 16 * SA;                         // FD_DOWN: the leaf's boundary values
  double* cst = sm + 8 * (16 * (SB + SA) + UBS);       // flux rows + couplings (8q), shared by the CTA
  double* cm = cst + 8 * Q + 1;                        // constant matrices (kFdCst)
  double* cVxi = cm;
  double* cVx = cVxi + 16 * CSA;
  double* cMx = cVx + 16 * CSA;
  double* cMy = cMx + 16 * CSA;
  double* cR = cMy + 16 * CSA;
  double* cVyit = cR + 16 * CSA;
  double* cVyt = cVyit + 16 * CSB;
  double* cAew = cVyt + 16 * CSB;                      // FD_UP_H: rows Vx^T e_east, Vx^T e_west (A type, 8 rows)
  double* cBns = cAew + 8 * CSA;                       // FD_UP_H: cols Vy^T e_n0, Vy^T e_n1 (B type, 16 x 8)
  for (int e = threadIdx.x; e < 8 * Q; e += 256) cst[e] = a.mats[5 * NI + e];
  if (threadIdx.x == 0) cst[8 * Q] = DOWNLIKE ? a.mats[5 * NI + 8 * Q + 512] : 0.0;  // c
  for (int e = threadIdx.x; e < 256; e += 256) {
    const int r = e >> 4, c = e & 15;
    auto mat = [&](int m) -> double { return (r < Q && c < Q) ? a.mats[m * NI + r * Q + c] : 0.0; };
    cVxi[r * CSA + c] = mat(0);
    cVyit[r * CSB + c] = mat(1);
    cVx[r * CSA + c] = mat(2);
    cVyt[r * CSB + c] = mat(3);
    cR[r * CSA + c] = mat(4);
    if (DOWNLIKE) {
      cMx[r * CSA + c] = a.mats[5 * NI + 8 * Q + e];
      cMy[r * CSA + c] = a.mats[5 * NI + 8 * Q + 256 + e];
    }
  }
  if (MODE == FD_DOWN) {
    __syncthreads();
    // coupling constants in the padding (see the staging of the leaf below)
    for (int e = threadIdx.x; e < 64; e += 256) {
      const int j = e >> 4, r = e & 15;
      if (r >= Q) continue;
      const double* bc = a.mats + 5 * NI + 4 * Q + j * Q;
      double v = 0.0;
      if (j < 2) {
        for (int t = 0; t < Q; ++t) v = fma(cVxi[r * CSA + t], bc[t], v);
        cVxi[r * CSA + Q + j] = -v;
      } else {
        for (int t = 0; t < Q; ++t) v = fma(bc[t], cVyit[t * CSB + r], v);
        cVyit[(Q + j - 2) * CSB + r] = -v;
      }
    }
  }
  if (UPH) {
    __syncthreads();
    // the fluxes of w = Vx T2 Vy^T need only projections of T2:
    //   east / west (d/dx rows E0, E1):  h[y] = sum_r (a^T T2)[r] Vy[y][r],  a = Vx^T E
    //   north / south (d/dy rows E2, E3): h[x] = sum_s Vx[x][s] (T2 b)[s],   b = Vy^T E
    for (int e = threadIdx.x; e < 8 * CSA + 16 * 8; e += 256) {
      double v = 0.0;
      if (e < 8 * CSA) {
        const int r = e / CSA, c = e % CSA;
        if (r < 2 && c < Q)
          for (int t = 0; t < Q; ++t) v = fma(a.mats[5 * NI + r * Q + t], cVx[t * CSA + c], v);
        cAew[e] = v;
      } else {
        const int f = e - 8 * CSA, r = f >> 3, n = f & 7;
        if (n < 2 && r < Q)
          for (int t = 0; t < Q; ++t) v = fma(a.mats[5 * NI + (2 + n) * Q + t], cVyt[r * CSB + t], v);
        cBns[f] = v;
      }
    }
  }
  const double* Mx = cMx;                              // FD_DOWN with L u: [x][s]
  const double* My = cMy;                              // [y][s]
  double gmax = 0.0;
  const int gr = lane >> 2, gc = lane & 3;
  pdl_trigger();
  const double* E = cst;
  // FD_UP_H: the first two products' constant fragments in registers (the
  // kernel is bound by shared-memory traffic; it has registers to spare)
  double rVxi[2][KS], rVyit[2][KS];
  if (MODE == FD_UP_H) {
#pragma unroll
    for (int i = 0; i < 2; ++i)
#pragma unroll
      for (int k = 0; k < KS; ++k) {
        rVxi[i][k] = cVxi[(i * 8 + gr) * CSA + k * 4 + gc];
        rVyit[i][k] = cVyit[(k * 4 + gc) * CSB + i * 8 + gr];
      }
  }
  for (int e = lane; e < 16 * (SB + SA); e += 32) bufB[e] = 0.0;  // zero padding stays zero
  __syncthreads();
  pdl_wait();
  // rhs rows kk of this CTA: the constant staging above is paid once for all of them
  for (int kk = blockIdx.y; kk < a.k; kk += gridDim.y) {
  if (UPH && a.nbd > 0) {
    for (int i = blockIdx.x * 256 + threadIdx.x; i < a.nbd; i += gridDim.x * 256)
      a.ubnd[kk * a.ld_ubnd + a.bids[i]] = a.fb[kk * a.ld_f + i];
  }
  const double* g = a.g ? a.g + kk * a.ld_g : nullptr;
  // FD_DOWN: 16-byte stores of u_int pairs (every leaf block starts at an even offset when Q is even)
  const bool vec = MODE == FD_DOWN && Q % 2 == 0 &&
                   (reinterpret_cast<uintptr_t>(a.uint + (long long)kk * a.ld_uint) & 15) == 0;
  const bool vec_lu = MODE == FD_DOWN && Q % 2 == 0 && a.lu &&
                      (reinterpret_cast<uintptr_t>(a.lu + (long long)kk * a.ld_lu) & 15) == 0 &&
                      (reinterpret_cast<uintptr_t>(g) & 15) == 0;
  const int nwarps = gridDim.x * 8;
  constexpr int NR = (NI + 31) / 32;  // body-load values per lane
  constexpr int NU = (NB + 31) / 32;  // boundary values per lane (FD_DOWN)
  double nxt[NR];                     // next leaf's body load, prefetched during this leaf
  double nub[DOWNLIKE ? NU : 1];
  // FD_UP_T: the stage combination in term order (the fma order of k_combine).
  // The first two terms of the NEXT leaf are issued before this leaf's products
  // (fetch) and stay in flight across them; finish() sums them and streams the
  // remaining terms two loads at a time, then writes the formed load out
  double va[MODE == FD_UP_T ? NR : 1], vb[MODE == FD_UP_T ? NR : 1];
  auto ldt = [&](double* v, int t, int leaf) {
    const double* src = a.tv[t] + kk * a.tld[t] + (long long)leaf * NI;
#pragma unroll
    for (int i = 0; i < NR; ++i) {
      const int e = lane + 32 * i;
      v[i] = (leaf < a.L && e < NI) ? __ldcs(src + e) : 0.0;
    }
  };
  auto finish = [&](int leaf) {
#pragma unroll
    for (int i = 0; i < NR; ++i) nxt[i] = 0.0;
    for (int t = 0; t < a.nterm; t += 2) {
      const double c0 = __ldg(a.tdc + t);
#pragma unroll
      for (int i = 0; i < NR; ++i) nxt[i] = fma(c0, va[i], nxt[i]);
      if (t + 1 >= a.nterm) break;
      if (t + 2 < a.nterm) ldt(va, t + 2, leaf);
      const double c1 = __ldg(a.tdc + t + 1);
#pragma unroll
      for (int i = 0; i < NR; ++i) nxt[i] = fma(c1, vb[i], nxt[i]);
      if (t + 3 < a.nterm) ldt(vb, t + 3, leaf);
    }
    double* ro = a.rout + kk * a.ld_rout + (long long)leaf * NI;
#pragma unroll
    for (int i = 0; i < NR; ++i) {
      const int e = lane + 32 * i;
      if (e < NI) ro[e] = nxt[i];
    }
  };
  auto fetch = [&](int leaf) {
    if (MODE == FD_UP_T) {
      ldt(va, 0, leaf);
      if (a.nterm > 1) ldt(vb, 1, leaf);
      return;
    }
#pragma unroll
    for (int i = 0; i < NR; ++i) {
      const int e = lane + 32 * i;
      nxt[i] = (g && leaf < a.L && e < NI) ? g[(long long)leaf * NI + e] : 0.0;
    }
    if (DOWNLIKE) {
      const double* u = a.u + kk * a.ld_u;
#pragma unroll
      for (int i = 0; i < NU; ++i) {
        const int b = lane + 32 * i;
        nub[i] = (leaf < a.L && b < NB) ? u[a.lbg[(long long)leaf * NB + b]] : 0.0;
      }
    }
  };
  fetch(blockIdx.x * 8 + warp);
  for (int l = blockIdx.x * 8 + warp; l < a.L; l += nwarps) {
    if (MODE == FD_UP_T) finish(l);
    if (MODE == FD_LU) {
#pragma unroll
      for (int i = 0; i < NU; ++i) {
        const int b = lane + 32 * i;
        if (b < NB) ub[b] = nub[i];
      }
    }
    if (MODE == FD_DOWN) {
      // R = r - A_ib u_b without forming it: the boundary values ride in the
      // zero padding of the 16 x 16 tile -- east / west rows q, q + 1 meet the
      // constant columns -Vx^-1 bx0, -Vx^-1 bx1 of the first product's A
      // operand, north / south columns q, q + 1 pass through it (Vx^-1 u_S,
      // Vx^-1 u_N) and meet the constant rows -by0 Vy^-T, -by1 Vy^-T of the
      // second product's B operand: T2 = Vx^-1 (r - A_ib u_b) Vy^-T with no
      // extra products (q + 2 <= 16) and no per-element coupling sums
      const bool need_ub = a.lu && a.lu_inv_dtg == 0.0;  // the leaf-grid L u reads the ring from ub
#pragma unroll
      for (int i = 0; i < NU; ++i) {
        const int b = lane + 32 * i;
        if (b < NB) {
          int x, y;
          if (b < Q) { x = Q; y = b; }
          else if (b >= 3 * Q) { x = Q + 1; y = b - 3 * Q; }
          else { x = (b - Q) >> 1; y = Q + ((b - Q) & 1); }
          bufB[x * SB + y] = nub[i];
          if (need_ub) ub[b] = nub[i];
          const double av = fabs(nub[i]);
          if (a.guard) gmax = (av > gmax || av != av) ? av : gmax;
        }
      }
      int x = lane / Q, y = lane % Q;  // grid point of element lane + 32 i, advanced incrementally
#pragma unroll
      for (int i = 0; i < NR; ++i) {
        if (x < Q) bufB[x * SB + y] = nxt[i];
        x += 32 / Q;
        y += 32 % Q;
        if (y >= Q) { y -= Q; ++x; }
      }
    } else {
      int x = lane / Q, y = lane % Q;
#pragma unroll
      for (int i = 0; i < NR; ++i) {
        if (x < Q) bufB[x * SB + y] = nxt[i];
        x += 32 / Q;
        y += 32 % Q;
        if (y >= Q) { y -= Q; ++x; }
      }
    }
    fetch(l + nwarps);
    __syncwarp();
    double acc[2][2][2];
    auto clear = [&]() {
#pragma unroll
      for (int mi = 0; mi < 2; ++mi)
#pragma unroll
        for (int nj = 0; nj < 2; ++nj) { acc[mi][nj][0] = 0.0; acc[mi][nj][1] = 0.0; }
    };
    auto store = [&](double* buf, int ld) {
#pragma unroll
      for (int mi = 0; mi < 2; ++mi)
#pragma unroll
        for (int nj = 0; nj < 2; ++nj)
          *reinterpret_cast<double2*>(buf + (mi * 8 + gr) * ld + nj * 8 + 2 * gc) =
              make_double2(acc[mi][nj][0], acc[mi][nj][1]);
    };
    if (MODE != FD_LU) {
    // T1 = Vx^-1 R  (B operand from bufB)
    constexpr int KS1 = MODE == FD_DOWN ? KSL : KS;  // FD_DOWN: q + 2 columns (the boundary values)
    clear();
#pragma unroll
    for (int k = 0; k < KS1; ++k) {
      double b0 = bufB[(k * 4 + gc) * SB + gr], b1 = bufB[(k * 4 + gc) * SB + 8 + gr];
#pragma unroll
      for (int mi = 0; mi < 2; ++mi) {
        const double am = MODE == FD_UP_H ? rVxi[mi][k] : cVxi[(mi * 8 + gr) * CSA + k * 4 + gc];
        dmma(acc[mi][0][0], acc[mi][0][1], am, b0);
        dmma(acc[mi][1][0], acc[mi][1][1], am, b1);
      }
    }
    store(bufA, SA);
    __syncwarp();
    // T2 = (T1 Vy^-T) .* rden  (A operand from bufA)
    clear();
#pragma unroll
    for (int k = 0; k < KS1; ++k) {
      double a0 = bufA[gr * SA + k * 4 + gc], a1 = bufA[(8 + gr) * SA + k * 4 + gc];
#pragma unroll
      for (int nj = 0; nj < 2; ++nj) {
        const double bm = MODE == FD_UP_H ? rVyit[nj][k] : cVyit[(k * 4 + gc) * CSB + nj * 8 + gr];
        dmma(acc[0][nj][0], acc[0][nj][1], a0, bm);
        dmma(acc[1][nj][0], acc[1][nj][1], a1, bm);
      }
    }
#pragma unroll
    for (int mi = 0; mi < 2; ++mi)
#pragma unroll
      for (int nj = 0; nj < 2; ++nj)
#pragma unroll
        for (int h = 0; h < 2; ++h) acc[mi][nj][h] *= cR[(mi * 8 + gr) * CSA + nj * 8 + 2 * gc + h];
    store(bufB, SB);
    __syncwarp();
    if (UPH) {
      // fluxes of w = Vx T2 Vy^T without forming w, as line sums (as DMMA
      // products they would pad 2 useful rows / columns to 8):
      //   east / west:   pe_r = a_r^T T2 (a_r = Vx^T e_r),  h_r[y] = sum_s pe_r[s] Vy[y][s]
      //   north / south: qn_n = T2 b_n   (b_n = Vy^T e_n),  h_n[x] = sum_s Vx[x][s] qn_n[s]
      // lanes 0..q-1 take the east / west rows (column y of T2, conflict-free
      // in bufB), lanes 16..16+q-1 the north / south ones (row x of T2 read
      // as column x of its transpose, stored to bufA from the accumulators)
#pragma unroll
      for (int mi = 0; mi < 2; ++mi)
#pragma unroll
        for (int nj = 0; nj < 2; ++nj)
#pragma unroll
          for (int h = 0; h < 2; ++h) bufA[(nj * 8 + 2 * gc + h) * SA + mi * 8 + gr] = acc[mi][nj][h];
      __syncwarp();
      const int li = lane & 15;
      const bool ew = lane < 16;
      double p0 = 0.0, p1 = 0.0;
      if (li < Q) {
        if (ew) {
#pragma unroll
          for (int x = 0; x < Q; ++x) {
            const double t = bufB[x * SB + li];
            p0 = fma(cAew[x], t, p0);
            p1 = fma(cAew[CSA + x], t, p1);
          }
        } else {
#pragma unroll
          for (int y = 0; y < Q; ++y) {
            const double t = bufA[y * SA + li];
            p0 = fma(cBns[y * 8], t, p0);
            p1 = fma(cBns[y * 8 + 1], t, p1);
          }
        }
      }
      __syncwarp();
      double* pq = bufA + 16 * SA;  // the warp's ub scratch (4q + 8): pe_0, pe_1, qn_0, qn_1 (q each)
      if (li < Q) {
        pq[(ew ? 0 : 2 * Q) + li] = p0;
        pq[(ew ? Q : 3 * Q) + li] = p1;
      }
      __syncwarp();
      double* out = a.H + kk * a.ld_h + (long long)l * NB;
      if (li < Q) {
        double h0 = 0.0, h1 = 0.0;
        if (ew) {
#pragma unroll
          for (int s2 = 0; s2 < Q; ++s2) {
            const double v = cVyt[s2 * CSB + li];
            h0 = fma(pq[s2], v, h0);
            h1 = fma(pq[Q + s2], v, h1);
          }
          out[li] = h0;
          out[3 * Q + li] = h1;
        } else {
#pragma unroll
          for (int s2 = 0; s2 < Q; ++s2) {
            const double v = cVx[li * CSA + s2];
            h0 = fma(v, pq[2 * Q + s2], h0);
            h1 = fma(v, pq[3 * Q + s2], h1);
          }
          out[Q + 2 * li] = h0;
          out[Q + 2 * li + 1] = h1;
        }
      }
      __syncwarp();
      continue;
    }
    // T3 = Vx T2  (B operand from bufB)
    clear();
#pragma unroll
    for (int k = 0; k < KS; ++k) {
      double b0 = bufB[(k * 4 + gc) * SB + gr], b1 = bufB[(k * 4 + gc) * SB + 8 + gr];
#pragma unroll
      for (int mi = 0; mi < 2; ++mi) {
        const double am = cVx[(mi * 8 + gr) * CSA + k * 4 + gc];
        dmma(acc[mi][0][0], acc[mi][0][1], am, b0);
        dmma(acc[mi][1][0], acc[mi][1][1], am, b1);
      }
    }
    store(bufA, SA);
    __syncwarp();
    // FD_DOWN with the stage history from the solved interior equation: r in
    // the fragment layout, in flight during the last product (an L1 / L2 hit)
    const bool lu_res = MODE == FD_DOWN && a.lu && a.lu_inv_dtg != 0.0;
    double2 rf[2][2];
    if (MODE == FD_DOWN && lu_res) {
      const double* rr = g ? g + (long long)l * NI : nullptr;
#pragma unroll
      for (int mi = 0; mi < 2; ++mi)
#pragma unroll
        for (int nj = 0; nj < 2; ++nj) {
          const int x = mi * 8 + gr, y = nj * 8 + 2 * gc;
          rf[mi][nj] = make_double2(0.0, 0.0);
          if (rr && x < Q && y < Q) {
            if (vec_lu && y + 1 < Q) {
              rf[mi][nj] = *reinterpret_cast<const double2*>(rr + x * Q + y);
            } else {
              rf[mi][nj].x = rr[x * Q + y];
              if (y + 1 < Q) rf[mi][nj].y = rr[x * Q + y + 1];
            }
          }
        }
    }
    // W = T3 Vy^T  (A operand from bufA)
    clear();
#pragma unroll
    for (int k = 0; k < KS; ++k) {
      double a0 = bufA[gr * SA + k * 4 + gc], a1 = bufA[(8 + gr) * SA + k * 4 + gc];
#pragma unroll
      for (int nj = 0; nj < 2; ++nj) {
        const double bm = cVyt[(k * 4 + gc) * CSB + nj * 8 + gr];
        dmma(acc[0][nj][0], acc[0][nj][1], a0, bm);
        dmma(acc[1][nj][0], acc[1][nj][1], a1, bm);
      }
    }
    if (MODE == FD_DOWN) {
      // u_int straight from the accumulator fragments: row x = mi * 8 + gr, columns y, y + 1
      double* out = a.uint + kk * a.ld_uint + (long long)l * NI;
#pragma unroll
      for (int mi = 0; mi < 2; ++mi)
#pragma unroll
        for (int nj = 0; nj < 2; ++nj) {
          const int x = mi * 8 + gr, y = nj * 8 + 2 * gc;
          if (x < Q && y < Q) {
            if (vec && y + 1 < Q) {
              *reinterpret_cast<double2*>(out + x * Q + y) = make_double2(acc[mi][nj][0], acc[mi][nj][1]);
            } else {
              out[x * Q + y] = acc[mi][nj][0];
              if (y + 1 < Q) out[x * Q + y + 1] = acc[mi][nj][1];
            }
          }
        }
      if (lu_res) {
        // the interior rows of the leaf system just solved read
        //   sigma u_int - dtg (L u)_int = r   (A = sigma I - dtg L, operators.py:252-269),
        // so the stage history L u_i (timestep.py:259-261) is (sigma u_int - r) / dtg to the
        // solve's residual (~1e-15 relative)
        double* lo = a.lu + kk * a.ld_lu + (long long)l * NI;
#pragma unroll
        for (int mi = 0; mi < 2; ++mi)
#pragma unroll
          for (int nj = 0; nj < 2; ++nj) {
            const int x = mi * 8 + gr, y = nj * 8 + 2 * gc;
            if (x < Q && y < Q) {
              const double l0 = (a.lu_sigma * acc[mi][nj][0] - rf[mi][nj].x) * a.lu_inv_dtg;
              const double l1 = (a.lu_sigma * acc[mi][nj][1] - rf[mi][nj].y) * a.lu_inv_dtg;
              if (vec_lu && y + 1 < Q) {
                *reinterpret_cast<double2*>(lo + x * Q + y) = make_double2(l0, l1);
              } else {
                lo[x * Q + y] = l0;
                if (y + 1 < Q) lo[x * Q + y + 1] = l1;
              }
            }
          }
      }
      if (!a.lu || lu_res) {
        if (a.guard) {  // max |u| over the leaf's grid: interior fragments and boundary values
#pragma unroll
          for (int mi = 0; mi < 2; ++mi)
#pragma unroll
            for (int nj = 0; nj < 2; ++nj)
#pragma unroll
              for (int h = 0; h < 2; ++h) {
                const int x = mi * 8 + gr, y = nj * 8 + 2 * gc + h;
                const double av = (x < Q && y < Q) ? fabs(acc[mi][nj][h]) : 0.0;
                gmax = (av > gmax || av != av) ? av : gmax;
              }
        }
        __syncwarp();
        continue;
      }
    } else {
      store(bufB, SB);
      __syncwarp();
      double* out = MODE == FD_UP_WH ? a.WH + kk * a.ld_wh + (long long)l * a.nw
                                     : a.H + kk * a.ld_h + (long long)l * NB - NI;  // h at out[NI + b]
      if (MODE == FD_UP_WH)
        for (int e = lane; e < NI; e += 32) out[e] = bufB[(e / Q) * SB + e % Q];
      // h = D_bi w along the grid line of each boundary point
      for (int b = lane; b < NB; b += 32) {
        double s = 0.0;
        if (b < Q || b >= 3 * Q) {
          const int yi = b < Q ? b : b - 3 * Q;
          const double* rr = E + (b < Q ? 0 : Q);
#pragma unroll
          for (int t = 0; t < Q; ++t) s = fma(rr[t], bufB[t * SB + yi], s);
        } else {
          const int jj = b - Q, xi = jj / 2;
          const double* rr = E + ((jj & 1) ? 3 : 2) * Q;
#pragma unroll
          for (int t = 0; t < Q; ++t) s = fma(rr[t], bufB[xi * SB + t], s);
        }
        out[NI + b] = s;
      }
      __syncwarp();
      continue;
    }
    }  // MODE != FD_LU
    // FD_DOWN with the stage history (u_int in the accumulator fragments), FD_LU
    // (the interior staged in bufB): the leaf grid G (p x p in 16 x 16) in bufA
    // (stride SA), read as the B operand of Mx G and the A operand of G My^T.
    // Interior and boundary ring are written here; the four corners and (for
    // p < 16) the padding keep finite values from the products / the initial
    // zeroing, and only reach outputs that are discarded (every interior
    // output's sums run along one grid line).
    __syncwarp();
    if (MODE == FD_LU) {
      for (int e = lane; e < NI; e += 32) {
        const int x = e / Q, y = e - x * Q;
        const double v = bufB[x * SB + y];
        bufA[(x + 1) * SA + y + 1] = v;
        const double av = fabs(v);
        gmax = (av > gmax || av != av) ? av : gmax;
      }
    } else {
#pragma unroll
      for (int mi = 0; mi < 2; ++mi)
#pragma unroll
        for (int nj = 0; nj < 2; ++nj)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            const int x = mi * 8 + gr, y = nj * 8 + 2 * gc + h;
            if (x < Q && y < Q) {
              const double v = acc[mi][nj][h];
              bufA[(x + 1) * SA + y + 1] = v;
              const double av = fabs(v);
              gmax = (av > gmax || av != av) ? av : gmax;
            }
          }
    }
    for (int b = lane; b < NB; b += 32) {  // boundary order: east y, north / south by x, west y
      int x, y;
      if (b < Q) { x = 0; y = b + 1; }
      else if (b >= 3 * Q) { x = Q + 1; y = b - 3 * Q + 1; }
      else { x = (b - Q) / 2 + 1; y = ((b - Q) & 1) ? Q + 1 : 0; }
      const double v = ub[b];
      bufA[x * SA + y] = v;
      const double av = fabs(v);
      gmax = (av > gmax || av != av) ? av : gmax;
    }
    __syncwarp();
    clear();
#pragma unroll
    for (int k = 0; k < KSL; ++k) {  // Mx G (SA = 4 mod 16: conflict-free as a B operand too)
      const double b0 = bufA[(k * 4 + gc) * SA + gr], b1 = bufA[(k * 4 + gc) * SA + 8 + gr];
#pragma unroll
      for (int mi = 0; mi < 2; ++mi) {
        const double am = Mx[(mi * 8 + gr) * CSA + k * 4 + gc];
        dmma(acc[mi][0][0], acc[mi][0][1], am, b0);
        dmma(acc[mi][1][0], acc[mi][1][1], am, b1);
      }
    }
#pragma unroll
    for (int k = 0; k < KSL; ++k) {  // + G My^T
      const double a0 = bufA[gr * SA + k * 4 + gc], a1 = bufA[(8 + gr) * SA + k * 4 + gc];
#pragma unroll
      for (int nj = 0; nj < 2; ++nj) {
        const double bm = My[(nj * 8 + gr) * CSA + k * 4 + gc];
        dmma(acc[0][nj][0], acc[0][nj][1], a0, bm);
        dmma(acc[1][nj][0], acc[1][nj][1], a1, bm);
      }
    }
    double* lo = a.lu + kk * a.ld_lu + (long long)l * NI;
    const double c0 = cst[8 * Q];
#pragma unroll
    for (int mi = 0; mi < 2; ++mi)
#pragma unroll
      for (int nj = 0; nj < 2; ++nj)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int x = mi * 8 + gr, y = nj * 8 + 2 * gc + h;
          if (x >= 1 && x <= Q && y >= 1 && y <= Q)
            lo[(x - 1) * Q + (y - 1)] = acc[mi][nj][h] - c0 * bufA[x * SA + y];
        }
    __syncwarp();
  }
  }  // rhs rows
  if (DOWNLIKE && a.guard) {  // max |u| over the staged grids (NaN sorts above inf)
    unsigned long long bits = __double_as_longlong(gmax);
    for (int off = 16; off > 0; off >>= 1) {
      const unsigned long long o = __shfl_xor_sync(0xffffffffu, bits, off);
      bits = o > bits ? o : bits;
    }
    if (lane == 0 && bits && bits > __ldcg(a.guard)) atomicMax(a.guard, bits);
  }
}

}  // namespace

template <int MODE>
static int launch_fd_mma(const Plan& P, const FdArgs& a, int nleaf, int k, cudaStream_t st) {
  const size_t smem = ((size_t)8 * (16 * (SB + SA) + 4 * P.q + 8) + 8 * P.q + 1 + kFdCst) * 8;
  const unsigned warps = (unsigned)std::min<long long>(cdiv(nleaf, 8), (long long)kNumSMs * 2);  // one wave
  dim3 g2(warps, (unsigned)std::min(k, 8));  // each CTA loops over rhs rows blockIdx.y + 8 i
#define HPSB_FD2(QQ)                                                                                   \
  if (P.q == QQ) {                                                                                     \
    static bool attr = false;                                                                          \
    if (!attr) {                                                                                       \
      HPSB_CUDA(cudaFuncSetAttribute(k_leaf_fd_mma<QQ, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                     (int)smem));                                                       \
      attr = true;                                                                                     \
    }                                                                                                  \
    HPSB_CUDA(launch_pdl(k_leaf_fd_mma<QQ, MODE>, g2, dim3(256), smem, st, a));                        \
    HPSB_LAUNCH_CHECK();                                                                               \
    return 0;                                                                                          \
  }
  HPSB_FD2(4) HPSB_FD2(5) HPSB_FD2(6) HPSB_FD2(7) HPSB_FD2(8) HPSB_FD2(9) HPSB_FD2(10) HPSB_FD2(11) HPSB_FD2(12)
  HPSB_FD2(13) HPSB_FD2(14)
#undef HPSB_FD2
  set_error("leaf_fd: no kernel for q = %d", P.q);
  return -1;
}

bool leaf_fd_down_enabled() { return !getenv("HPSB_FD_SIMT") && !getenv("HPSB_NO_FD_DOWN"); }

int leaf_fd_up_h(const Ops& ops, int k, int nleaf, const double* g, long long ld_g, double* H, long long ld_h,
                 cudaStream_t st, int nbd, const int* bids, const double* fb, long long ld_f, double* u,
                 long long ld_u) {
  if (nleaf <= 0) return 0;
  FdArgs a{};
  a.L = nleaf; a.k = k; a.g = g; a.ld_g = ld_g; a.H = H; a.ld_h = ld_h; a.mats = ops.fd;
  a.nbd = nbd; a.bids = bids; a.fb = fb; a.ld_f = ld_f; a.ubnd = u; a.ld_ubnd = ld_u;
  return launch_fd_mma<FD_UP_H>(*ops.plan, a, nleaf, k, st);
}

int leaf_fd_down(const Ops& ops, int k, int nleaf, const double* g, long long ld_g, const int* lbg, const double* u,
                 long long ld_u, double* uint, long long ld_uint, double* lu, long long ld_lu, double* guard,
                 cudaStream_t st) {
  if (nleaf <= 0) return 0;
  FdArgs a{};
  a.L = nleaf; a.k = k; a.g = g; a.ld_g = ld_g; a.lbg = lbg; a.u = u; a.ld_u = ld_u;
  a.uint = uint; a.ld_uint = ld_uint; a.mats = ops.fd;
  a.lu = lu; a.ld_lu = ld_lu; a.guard = reinterpret_cast<unsigned long long*>(guard);
  static const bool lu_products = getenv("HPSB_LU_PRODUCTS") != nullptr;
  if (lu && !lu_products && ops.dtg != 0.0) { a.lu_sigma = ops.sigma; a.lu_inv_dtg = 1.0 / ops.dtg; }
  return launch_fd_mma<FD_DOWN>(*ops.plan, a, nleaf, k, st);
}

int leaf_fd_lu(const Ops& ops, int k, int nleaf, const int* lbg, const double* u, long long ld_u, const double* uint,
               double* lu, long long ld_lu, double* guard, cudaStream_t st) {
  if (nleaf <= 0) return 0;
  FdArgs a{};
  a.L = nleaf; a.k = k; a.g = uint; a.ld_g = ld_u; a.lbg = lbg; a.u = u; a.ld_u = ld_u; a.mats = ops.fd;
  a.lu = lu; a.ld_lu = ld_lu; a.guard = reinterpret_cast<unsigned long long*>(guard);
  return launch_fd_mma<FD_LU>(*ops.plan, a, nleaf, k, st);
}

int leaf_fd_up_terms(const Ops& ops, int k, int nleaf, int nterm, const double* const* tv, const long long* tld,
                     const double* tdc, double* rout, long long ld_rout, double* H, long long ld_h, cudaStream_t st,
                     int nbd, const int* bids, const double* fb, long long ld_f, double* u, long long ld_u) {
  if (nleaf <= 0) return 0;
  if (nterm <= 0 || nterm > kFdTerms) { set_error("leaf_fd_up_terms: %d terms (1..%d)", nterm, kFdTerms); return -1; }
  FdArgs a{};
  a.L = nleaf; a.k = k; a.H = H; a.ld_h = ld_h; a.mats = ops.fd;
  a.nterm = nterm; a.tdc = tdc; a.rout = rout; a.ld_rout = ld_rout;
  for (int t = 0; t < nterm; ++t) { a.tv[t] = tv[t]; a.tld[t] = tld ? tld[t] : 0; }
  a.nbd = nbd; a.bids = bids; a.fb = fb; a.ld_f = ld_f; a.ubnd = u; a.ld_ubnd = ld_u;
  return launch_fd_mma<FD_UP_T>(*ops.plan, a, nleaf, k, st);
}

int leaf_fd(const Ops& ops, int k, int nleaf, const double* g, long long ld_g, double* WH, long long ld_wh,
            cudaStream_t st) {
  const Plan& P = *ops.plan;
  if (nleaf <= 0) return 0;
  FdArgs a{};
  a.L = nleaf; a.k = k; a.nw = P.ni + P.nb;
  a.g = g; a.ld_g = ld_g; a.WH = WH; a.ld_wh = ld_wh; a.mats = ops.fd;
  const unsigned groups = (unsigned)std::min<long long>(cdiv(nleaf, 8), (long long)kNumSMs * 4);
  dim3 grid(groups, (unsigned)k);
  if (!getenv("HPSB_FD_SIMT")) return launch_fd_mma<FD_UP_WH>(P, a, nleaf, k, st);  // tensor-core variant
#define HPSB_FD(QQ) \
  if (P.q == QQ) { HPSB_CUDA(launch_pdl(k_leaf_fd<QQ>, grid, dim3(NT), 0, st, a)); HPSB_LAUNCH_CHECK(); return 0; }
  HPSB_FD(4) HPSB_FD(5) HPSB_FD(6) HPSB_FD(7) HPSB_FD(8) HPSB_FD(9) HPSB_FD(10) HPSB_FD(11) HPSB_FD(12) HPSB_FD(13)
  HPSB_FD(14)
#undef HPSB_FD
  set_error("leaf_fd: no kernel for q = %d", P.q);
  return -1;
}

// every leaf order p = q + 2 from 6 to 16 (the leaf grid fits one 16 x 16 DMMA tile)
bool leaf_fd_supported(int q) { return q >= 4 && q <= 14; }

}  // namespace hpsb
