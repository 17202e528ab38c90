// Stage right-hand-side kernels of the IMEX ARK stepper (sm_100a, FP64).
//
//   k_leaf_eval : leaf-local spectral evaluations of a grid vector, the
//                 tensor-product form of the reference's dense leaf products
//                 (operators.py:276-336):
//                   L u  = c11 u_xx + c22 u_yy - c1 u_x - c2 u_y - c u
//                   grad = (u_x, u_y)
//                   flux jump = sign * D_bnd u  (edge points only)
//                 Every leaf's p x p grid (corners unused) is staged in shared
//                 memory from the global vector (interiors are one contiguous
//                 run per leaf, edges are gathered through leaf_bnd_gidx);
//                 derivative rows are p-term sums along grid lines, with the
//                 edge-local (p-2)-node rows for tangential derivatives at edge
//                 points (operators.py:192-213).  Interface values are the mean
//                 of the two abutting leaves (operators.py:339-346): the
//                 interior is written directly, edge points accumulate w*value
//                 with w = 1/multiplicity (exact for multiplicity 1 or 2, and
//                 order independent for two addends).
//                 The kernel also folds a max|u| / non-finite reduction over
//                 every value it stages (the divergence guard of
//                 timestep.py:198-203).
//   k_combine   : out = sum_m c_m v_m over a DOF range (the ARK stage
//                 combinations, timestep.py:255-257 and 263-264).
//   k_maxabs    : guard reduction of a vector.
#include "../../include/hpstep_b200.h"
#include "hps_plan.cuh"

namespace hpsb {

struct Disc {
  const Plan* P = nullptr;
  int p = 0, q = 0, ni = 0, nb = 0, m = 0, L = 0;
  int Lc = 1;                     // coefficient sample sets (1 = constant)
  int has_c1 = 0, has_c2 = 0, has_c = 0;
  double cc[5] = {0, 0, 0, 0, 0};  // constant coefficients (Lc == 1)
  double* coef = nullptr;         // Lc x 5 x m (device) when Lc > 1
  double* mats = nullptr;         // d1x d2x d1y d2y (p*p each) ex1 ex2 ey1 ey2 (q*q each)
  signed char* sign = nullptr;    // L x nb leaf_bnd_sign (device)
  std::vector<void*> allocs;
};

namespace {

constexpr int NT = 256;

struct EvalArgs {
  int k;
  const double* u; long long ld_u;
  int L, p, q, ni, nb, m, lpb;
  long long N;
  long long ioff;                   // first interior DOF of the leaf range (lbg / sign / coef start there)
  const int* lbg;                   // L x nb
  const signed char* sign;          // L x nb
  const double* mats;
  int Lc; const double* coef; double cc[5]; int has_c1, has_c2, has_c;
  // outputs (nullptr = not requested), all row stride ld_o
  double* lu_int;                   // L u at interior points only (no averaging)
  double* lu;                       // L u at every DOF, interface-averaged
  double* ux; double* uy;           // gradient, interface-averaged
  double* jump;                     // signed flux jumps at edge points
  long long ld_o;
  unsigned long long* guard;        // max |u| bits (nullptr = off)
};

// running max |v| that keeps NaN sticky (fmax would drop it)
__device__ __forceinline__ void gacc(double& g, double v) {
  double av = fabs(v);
  g = (av > g || av != av) ? av : g;
}

// block-wide max |v| then one atomic per block, skipped when the running
// maximum already covers it (thousands of blocks would otherwise serialise
// on one address)
__device__ __forceinline__ void guard_max(unsigned long long* slot, double v) {
  __shared__ unsigned long long s_w[32];  // up to 1024 threads
  // |v| as an unsigned bit pattern orders like the value; NaN sorts above inf
  unsigned long long b = __double_as_longlong(fabs(v));
  for (int off = 16; off > 0; off >>= 1) {
    unsigned long long o = __shfl_xor_sync(0xffffffffu, b, off);
    b = o > b ? o : b;
  }
  if ((threadIdx.x & 31) == 0) s_w[threadIdx.x >> 5] = b;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) b = s_w[w] > b ? s_w[w] : b;
    if (b && b > __ldcg(slot)) atomicMax(slot, b);
  }
}

// local edge index e -> grid (xi, yi): east (xi = 0), north/south interleaved,
// west (xi = p-1); reference tree.py:236-243 / operators.py:172-178
__device__ __forceinline__ void edge_xy(int e, int p, int q, int& xi, int& yi) {
  if (e < q) { xi = 0; yi = e + 1; }
  else if (e < 3 * q) { int j = e - q; xi = j / 2 + 1; yi = (j & 1) ? p - 1 : 0; }
  else { xi = p - 1; yi = e - 3 * q + 1; }
}

__global__ void __launch_bounds__(NT) k_leaf_eval(EvalArgs a) {
  extern __shared__ double sm[];
  // row strides padded to odd lengths: lanes walking different rows of a
  // matrix / grid at the same column hit different banks
  const int p = a.p, q = a.q, PS = (p + 1) | 1, QS = (q + 1) | 1;
  const int pp = p * PS, qq = q * QS;
  double* d1x = sm;
  double* d2x = d1x + pp;
  double* d1y = d2x + pp;
  double* d2y = d1y + pp;
  double* ex1 = d2y + pp;
  double* ex2 = ex1 + qq;
  double* ey1 = ex2 + qq;
  double* ey2 = ey1 + qq;
  double* U = ey2 + qq;  // lpb x p x PS
  const int tid = threadIdx.x;
  for (int e = tid; e < 4 * p * p; e += NT) {
    int mtx = e / (p * p), r = e % (p * p);
    sm[mtx * pp + (r / p) * PS + r % p] = a.mats[e];
  }
  for (int e = tid; e < 4 * q * q; e += NT) {
    int mtx = e / (q * q), r = e % (q * q);
    ex1[mtx * qq + (r / q) * QS + r % q] = a.mats[4 * p * p + e];
  }
  const int kk = blockIdx.y;
  const double* u = a.u + kk * a.ld_u;
  double gmax = 0.0;
  const bool want_all = a.lu || a.ux || a.uy;
  const int npts = want_all ? a.m : (a.lu_int ? a.ni : 0);
  const long long ob = kk * a.ld_o;
  // persistent over leaf groups: the stencil matrices are staged once per CTA
  for (int l0 = blockIdx.x * a.lpb; l0 < a.L; l0 += gridDim.x * a.lpb) {
  const int nl = min(a.lpb, a.L - l0);
  __syncthreads();
  // interior: one contiguous run of nl*ni values
  for (int e = tid; e < nl * a.ni; e += NT) {
    int ll = e / a.ni, i = e % a.ni;
    double v = u[a.ioff + (long long)l0 * a.ni + e];
    U[ll * pp + (i / q + 1) * PS + (i % q + 1)] = v;
    gacc(gmax, v);
  }
  for (int e = tid; e < nl * a.nb; e += NT) {
    int ll = e / a.nb, j = e % a.nb, xi, yi;
    edge_xy(j, p, q, xi, yi);
    double v = u[a.lbg[(long long)(l0 + ll) * a.nb + j]];
    U[ll * pp + xi * PS + yi] = v;
    gacc(gmax, v);
  }
  __syncthreads();

  for (int e = tid; e < nl * npts; e += NT) {
    const int ll = e / npts, t = e % npts, l = l0 + ll;
    int xi, yi;
    const bool inner = t < a.ni;
    if (inner) { xi = t / q + 1; yi = t % q + 1; }
    else edge_xy(t - a.ni, p, q, xi, yi);
    const double* G = U + ll * pp;
    const bool vert = !inner && (xi == 0 || xi == p - 1);
    const bool horz = !inner && !vert;
    double ux = 0.0, uxx = 0.0, uy = 0.0, uyy = 0.0;
    if (horz) {  // tangential x on north/south edges: edge-local rows
      const double* r1 = ex1 + (xi - 1) * QS;
      const double* r2 = ex2 + (xi - 1) * QS;
      for (int s = 0; s < q; ++s) {
        double v = G[(s + 1) * PS + yi];
        ux = fma(r1[s], v, ux);
        uxx = fma(r2[s], v, uxx);
      }
    } else {
      const double* r1 = d1x + xi * PS;
      const double* r2 = d2x + xi * PS;
      for (int s = 0; s < p; ++s) {
        double v = G[s * PS + yi];
        ux = fma(r1[s], v, ux);
        uxx = fma(r2[s], v, uxx);
      }
    }
    if (vert) {  // tangential y on east/west edges
      const double* r1 = ey1 + (yi - 1) * QS;
      const double* r2 = ey2 + (yi - 1) * QS;
      for (int s = 0; s < q; ++s) {
        double v = G[xi * PS + s + 1];
        uy = fma(r1[s], v, uy);
        uyy = fma(r2[s], v, uyy);
      }
    } else {
      const double* r1 = d1y + yi * PS;
      const double* r2 = d2y + yi * PS;
      for (int s = 0; s < p; ++s) {
        double v = G[xi * PS + s];
        uy = fma(r1[s], v, uy);
        uyy = fma(r2[s], v, uyy);
      }
    }
    double lop = 0.0;
    if (a.lu || (a.lu_int && inner)) {
      double c11, c22, c1, c2, c0;
      if (a.Lc == 1) { c11 = a.cc[0]; c22 = a.cc[1]; c1 = a.cc[2]; c2 = a.cc[3]; c0 = a.cc[4]; }
      else {
        const double* cv = a.coef + (long long)l * 5 * a.m;
        c11 = cv[t]; c22 = cv[a.m + t]; c1 = cv[2 * a.m + t]; c2 = cv[3 * a.m + t]; c0 = cv[4 * a.m + t];
      }
      // operators.py:292-300, in the same association, without contraction
      lop = __dmul_rn(c11, uxx);
      lop = __dadd_rn(lop, __dmul_rn(c22, uyy));
      if (a.has_c1) lop = __dsub_rn(lop, __dmul_rn(c1, ux));
      if (a.has_c2) lop = __dsub_rn(lop, __dmul_rn(c2, uy));
      if (a.has_c) lop = __dsub_rn(lop, __dmul_rn(c0, G[xi * PS + yi]));
    }
    if (inner) {
      const long long gi = (long long)l * a.ni + t;
      if (a.lu_int) a.lu_int[ob + gi] = lop;
      if (a.lu) a.lu[ob + a.ioff + gi] = lop;
      if (a.ux) a.ux[ob + a.ioff + gi] = ux;
      if (a.uy) a.uy[ob + a.ioff + gi] = uy;
    } else {
      const int j = t - a.ni;
      const long long gi = a.lbg[(long long)l * a.nb + j];
      const double w = a.sign[(long long)l * a.nb + j] ? 0.5 : 1.0;
      if (a.lu) atomicAdd(a.lu + ob + gi, w * lop);
      if (a.ux) atomicAdd(a.ux + ob + gi, w * ux);
      if (a.uy) atomicAdd(a.uy + ob + gi, w * uy);
    }
  }
  if (a.jump) {
    // flux rows: normal derivative from the full tensor line (operators.py:188-190)
    for (int e = tid; e < nl * a.nb; e += NT) {
      const int ll = e / a.nb, j = e % a.nb, l = l0 + ll;
      const signed char sg = a.sign[(long long)l * a.nb + j];
      if (!sg) continue;
      int xi, yi;
      edge_xy(j, p, q, xi, yi);
      const double* G = U + ll * pp;
      double v = 0.0;
      if (xi == 0 || xi == p - 1) {
        const double* r = d1x + xi * PS;
        for (int s = 0; s < p; ++s) v = fma(r[s], G[s * PS + yi], v);
      } else {
        const double* r = d1y + yi * PS;
        for (int s = 0; s < p; ++s) v = fma(r[s], G[xi * PS + s], v);
      }
      atomicAdd(a.jump + ob + a.lbg[(long long)l * a.nb + j], sg > 0 ? v : -v);
    }
  }
  }  // leaf groups
  if (a.guard) guard_max(a.guard, gmax);
}

// Interior-only L u (the stage history, timestep.py:253-261): thread <->
// fixed interior point of the CTA's leaf slot, its derivative rows held in
// registers across the persistent leaf loop, so the inner loops read only
// the staged grid values from shared memory.
template <int P, bool G1>
__global__ void __launch_bounds__(NT) k_leaf_lop_int(EvalArgs a) {
  extern __shared__ double U[];  // lpb x P x PS
  pdl_trigger();
  constexpr int Q = P - 2, NI = Q * Q, PS = (P + 1) | 1, PP = P * PS, NB = 4 * Q;
  constexpr int LANES = NT / NI;  // threads sharing one interior point (over leaves)
  const int tid = threadIdx.x, lpb = a.lpb;
  const int kk = blockIdx.y;
  const double* u = a.u + kk * a.ld_u;
  const long long ob = kk * a.ld_o;
  const bool active = tid < LANES * NI;
  const int t = tid % NI, lane0 = tid / NI, xi = t / Q + 1, yi = t % Q + 1;
  double rxx[P], ryy[P], rx[G1 ? P : 1], ry[G1 ? P : 1];
  const double* mats = a.mats;
#pragma unroll
  for (int s = 0; s < P; ++s) {
    if (G1) rx[s] = mats[xi * P + s];
    rxx[s] = mats[P * P + xi * P + s];
    if (G1) ry[s] = mats[2 * P * P + yi * P + s];
    ryy[s] = mats[3 * P * P + yi * P + s];
  }
  double gmax = 0.0;
  // the next leaf group's values are loaded into registers while the current
  // group is computed from shared memory (lpb must equal LPB, set by the host)
  constexpr int LPB = 2048 / (P * P), KI = (LPB * NI + NT - 1) / NT, KB = (LPB * NB + NT - 1) / NT;
  double pi[KI], pb[KB];
  auto fetch = [&](int l0) {
    const int nl = min(LPB, a.L - l0);
#pragma unroll
    for (int i = 0; i < KI; ++i) {
      const int e = tid + i * NT;
      pi[i] = e < nl * NI ? u[a.ioff + (long long)l0 * NI + e] : 0.0;
    }
#pragma unroll
    for (int i = 0; i < KB; ++i) {
      const int e = tid + i * NT;
      pb[i] = e < nl * NB ? u[a.lbg[(long long)l0 * NB + e]] : 0.0;
    }
  };
  const int step = gridDim.x * LPB;
  int l0 = blockIdx.x * LPB;
  pdl_wait();  // the vector below is produced by the previous kernel
  if (l0 < a.L) fetch(l0);
  for (; l0 < a.L; l0 += step) {
    const int nl = min(LPB, a.L - l0);
    __syncthreads();  // the previous group is consumed
#pragma unroll
    for (int i = 0; i < KI; ++i) {
      const int e = tid + i * NT;
      if (e < nl * NI) {
        const int l2 = e / NI, ii = e % NI;
        U[l2 * PP + (ii / Q + 1) * PS + (ii % Q + 1)] = pi[i];
        gacc(gmax, pi[i]);
      }
    }
#pragma unroll
    for (int i = 0; i < KB; ++i) {
      const int e = tid + i * NT;
      if (e < nl * NB) {
        const int l2 = e / NB, j = e % NB;
        int x, y;
        edge_xy(j, P, Q, x, y);
        U[l2 * PP + x * PS + y] = pb[i];
        gacc(gmax, pb[i]);
      }
    }
    __syncthreads();
    if (l0 + step < a.L) fetch(l0 + step);
    if (!active) continue;
    constexpr int PER = (LPB + LANES - 1) / LANES;  // leaf slots per thread and group
#pragma unroll
    for (int it = 0; it < PER; ++it) {
      const int ll = lane0 + it * LANES;
      if (ll >= nl) continue;
      const double* G = U + ll * PP;
      const int l = l0 + ll;
      // variable coefficients: only the fields present, loaded before the line
      // sums so the loads are in flight while they run
      double c11, c22, c1 = 0.0, c2 = 0.0, c0 = 0.0;
      if (a.Lc == 1) { c11 = a.cc[0]; c22 = a.cc[1]; c1 = a.cc[2]; c2 = a.cc[3]; c0 = a.cc[4]; }
      else {
        const double* cv = a.coef + (long long)l * 5 * a.m;
        c11 = __ldcs(cv + t); c22 = __ldcs(cv + a.m + t);
        if (a.has_c1) c1 = __ldcs(cv + 2 * a.m + t);
        if (a.has_c2) c2 = __ldcs(cv + 3 * a.m + t);
        if (a.has_c) c0 = __ldcs(cv + 4 * a.m + t);
      }
      double ux = 0.0, uxx = 0.0, uy = 0.0, uyy = 0.0;
#pragma unroll
      for (int s = 0; s < P; ++s) {
        const double v = G[s * PS + yi];
        uxx = fma(rxx[s], v, uxx);
        if (G1) ux = fma(rx[G1 ? s : 0], v, ux);
      }
#pragma unroll
      for (int s = 0; s < P; ++s) {
        const double v = G[xi * PS + s];
        uyy = fma(ryy[s], v, uyy);
        if (G1) uy = fma(ry[G1 ? s : 0], v, uy);
      }
      double lop = __dmul_rn(c11, uxx);
      lop = __dadd_rn(lop, __dmul_rn(c22, uyy));
      if (a.has_c1) lop = __dsub_rn(lop, __dmul_rn(c1, ux));
      if (a.has_c2) lop = __dsub_rn(lop, __dmul_rn(c2, uy));
      if (a.has_c) lop = __dsub_rn(lop, __dmul_rn(c0, G[xi * PS + yi]));
      a.lu_int[ob + (long long)l * NI + t] = lop;
    }
  }
  if (a.guard) guard_max(a.guard, gmax);
}

// Interface-averaged gradient only (the nonlinear g of timestep.py:192-196):
// thread <-> one grid point of the leaf slot (interior or edge), its two line
// rows held in registers for the whole kernel -- the normal / interior rows
// are the full p-point derivative rows, the tangential rows at edge points
// are the edge-local (p-2)-point rows placed at grid positions 1..p-2 (zeros
// elsewhere, and the grid's unused corners are kept at zero) -- so every
// point is the same two p-term sums.  Interior values are stored, edge values
// accumulate w * value (w = 1/2 on interfaces) as in k_leaf_eval.  The next
// leaf group is loaded into registers while the current one is computed.
// block size: 288 threads for p = 10 / 12 (3 x 96 / 2 x 140 grid points, no
// idle lanes), 256 for p = 16 (252 points); two CTAs per SM
template <int P>
struct GradThreads {
  static constexpr int value = P == 16 ? 256 : 288;
};

template <int P>
__global__ void __launch_bounds__(GradThreads<P>::value, 2) k_leaf_grad(EvalArgs a) {
  constexpr int NT = GradThreads<P>::value;  // a multiple of 32 covering whole grid points
  extern __shared__ double U[];  // LPB x P x PS
  pdl_trigger();
  constexpr int Q = P - 2, NI = Q * Q, NB = 4 * Q, M = NI + NB, PS = (P + 1) | 1, PP = P * PS;
  constexpr int LANES = NT / M > 0 ? NT / M : 1;
  constexpr int LPB = 2048 / (P * P), KI = (LPB * NI + NT - 1) / NT, KB = (LPB * NB + NT - 1) / NT;
  const int tid = threadIdx.x, kk = blockIdx.y;
  const double* u = a.u + kk * a.ld_u;
  const long long ob = kk * a.ld_o;
  const bool active = tid < LANES * M;
  const int t = tid % M, lane0 = tid / M;
  const bool inner = t < NI;
  int xi, yi;
  if (inner) { xi = t / Q + 1; yi = t % Q + 1; }
  else edge_xy(t - NI, P, Q, xi, yi);
  const bool vert = !inner && (xi == 0 || xi == P - 1), horz = !inner && !vert;
  const double* mats = a.mats;
  const double* ex1 = mats + 4 * P * P;
  const double* ey1 = ex1 + 2 * Q * Q;
  double rA[P], rB[P];
#pragma unroll
  for (int s = 0; s < P; ++s) {
    const bool mid = s >= 1 && s <= Q;
    rA[s] = horz ? (mid ? ex1[(xi - 1) * Q + s - 1] : 0.0) : mats[xi * P + s];
    rB[s] = vert ? (mid ? ey1[(yi - 1) * Q + s - 1] : 0.0) : mats[2 * P * P + yi * P + s];
  }
  for (int e = tid; e < LPB * PP; e += NT) U[e] = 0.0;  // corners stay zero
  double gmax = 0.0;
  double pi[KI], pb[KB];
  auto fetch = [&](int l0) {
    const int nl = min(LPB, a.L - l0);
#pragma unroll
    for (int i = 0; i < KI; ++i) {
      const int e = tid + i * NT;
      pi[i] = e < nl * NI ? u[a.ioff + (long long)l0 * NI + e] : 0.0;
    }
#pragma unroll
    for (int i = 0; i < KB; ++i) {
      const int e = tid + i * NT;
      pb[i] = e < nl * NB ? u[a.lbg[(long long)l0 * NB + e]] : 0.0;
    }
  };
  const int step = gridDim.x * LPB;
  int l0 = blockIdx.x * LPB;
  pdl_wait();  // the vector below is produced by the previous kernel
  if (l0 < a.L) fetch(l0);
  for (; l0 < a.L; l0 += step) {
    const int nl = min(LPB, a.L - l0);
    __syncthreads();
#pragma unroll
    for (int i = 0; i < KI; ++i) {
      const int e = tid + i * NT;
      if (e < nl * NI) {
        const int l2 = e / NI, ii = e % NI;
        U[l2 * PP + (ii / Q + 1) * PS + (ii % Q + 1)] = pi[i];
        gacc(gmax, pi[i]);
      }
    }
#pragma unroll
    for (int i = 0; i < KB; ++i) {
      const int e = tid + i * NT;
      if (e < nl * NB) {
        const int l2 = e / NB, j = e % NB;
        int x, y;
        edge_xy(j, P, Q, x, y);
        U[l2 * PP + x * PS + y] = pb[i];
        gacc(gmax, pb[i]);
      }
    }
    __syncthreads();
    if (l0 + step < a.L) fetch(l0 + step);
    if (!active) continue;
    constexpr int PER = (LPB + LANES - 1) / LANES;
#pragma unroll
    for (int it = 0; it < PER; ++it) {
      const int ll = lane0 + it * LANES;
      if (ll >= nl) continue;
      const double* G = U + ll * PP;
      double ux = 0.0, uy = 0.0;
#pragma unroll
      for (int s = 0; s < P; ++s) {
        ux = fma(rA[s], G[s * PS + yi], ux);
        uy = fma(rB[s], G[xi * PS + s], uy);
      }
      const int l = l0 + ll;
      if (inner) {
        const long long gi = ob + a.ioff + (long long)l * NI + t;
        a.ux[gi] = ux;
        a.uy[gi] = uy;
      } else {
        const int j = t - NI;
        const long long gi = ob + a.lbg[(long long)l * NB + j];
        const double w = a.sign[(long long)l * NB + j] ? 0.5 : 1.0;
        atomicAdd(a.ux + gi, w * ux);
        atomicAdd(a.uy + gi, w * uy);
      }
    }
  }
  if (a.guard) guard_max(a.guard, gmax);
}

constexpr int MAXT = 24;
struct CombineArgs {
  int nt, k;
  long long n;                 // DOFs per row
  double c[MAXT];
  const double* v[MAXT];
  long long ld[MAXT];          // row stride of term m (0 = broadcast over rows)
  double* out; long long ld_out;
  unsigned long long* guard;
  const double* dc;            // device coefficient table (graph replay), else c[]
  long long ldc;               // row stride of dc (per-row coefficients; 0 = shared by the rows)
};

__global__ void __launch_bounds__(NT) k_combine(CombineArgs a) {
  pdl_trigger();
  pdl_wait();
  const int kk = blockIdx.y;
  double gmax = 0.0;
  const long long stride = (long long)gridDim.x * NT;
  for (long long e = blockIdx.x * (long long)NT + threadIdx.x; e < a.n; e += stride) {
    double s = 0.0;
    for (int t0 = 0; t0 < a.nt; t0 += 4) {
      double v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = t0 + u < a.nt ? __ldcs(a.v[t0 + u] + kk * a.ld[t0 + u] + e) : 0.0;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (t0 + u >= a.nt) break;
        s = fma(a.dc ? __ldg(a.dc + kk * a.ldc + t0 + u) : a.c[t0 + u], v[u], s);
      }
    }
    a.out[kk * a.ld_out + e] = s;
    gacc(gmax, s);
  }
  if (a.guard) guard_max(a.guard, gmax);
}

// 16-byte variant: every term pointer / row stride and the output 16-byte
// aligned (even offsets), n even; two DOFs per thread and iteration, all
// term loads issued before the sums
__global__ void __launch_bounds__(NT) k_combine2(CombineArgs a) {
  pdl_trigger();
  pdl_wait();
  const int kk = blockIdx.y;
  double gmax = 0.0;
  const long long n2 = a.n / 2, stride = (long long)gridDim.x * NT;
  for (long long e = blockIdx.x * (long long)NT + threadIdx.x; e < n2; e += stride) {
    double2 s = make_double2(0.0, 0.0);
    for (int t0 = 0; t0 < a.nt; t0 += 4) {  // four independent loads in flight, then the fmas in term order
      double2 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u)
        v[u] = t0 + u < a.nt ? __ldcs(reinterpret_cast<const double2*>(a.v[t0 + u] + kk * a.ld[t0 + u]) + e)
                             : make_double2(0.0, 0.0);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (t0 + u >= a.nt) break;
        const double c = a.dc ? __ldg(a.dc + kk * a.ldc + t0 + u) : a.c[t0 + u];
        s.x = fma(c, v[u].x, s.x);
        s.y = fma(c, v[u].y, s.y);
      }
    }
    reinterpret_cast<double2*>(a.out + kk * a.ld_out)[e] = s;
    gacc(gmax, s.x);
    gacc(gmax, s.y);
  }
  if (a.guard) guard_max(a.guard, gmax);
}

// The step's final combination with the Dirichlet overwrite and the guard in
// one pass (timestep.py:263-266): out = sum c v, then fb at the boundary DOFs
// (edge DOFs e >= e0 with ebp[e - e0] >= 0), guard over the final values.
__global__ void __launch_bounds__(NT) k_combine_bnd(CombineArgs a, long long e0, const int* __restrict__ ebp,
                                                    const double* __restrict__ fb, long long ld_f) {
  pdl_trigger();
  pdl_wait();
  const int kk = blockIdx.y;
  double gmax = 0.0;
  const long long stride = (long long)gridDim.x * NT;
  for (long long e = blockIdx.x * (long long)NT + threadIdx.x; e < a.n; e += stride) {
    double s = 0.0;
    const int bp = e >= e0 ? __ldg(ebp + (e - e0)) : -1;
    if (bp >= 0) {
      s = fb[kk * ld_f + bp];
    } else {
      for (int t0 = 0; t0 < a.nt; t0 += 4) {
        double v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) v[u] = t0 + u < a.nt ? __ldcs(a.v[t0 + u] + kk * a.ld[t0 + u] + e) : 0.0;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          if (t0 + u >= a.nt) break;
          s = fma(a.dc ? __ldg(a.dc + kk * a.ldc + t0 + u) : a.c[t0 + u], v[u], s);
        }
      }
    }
    a.out[kk * a.ld_out + e] = s;
    gacc(gmax, s);
  }
  if (a.guard) guard_max(a.guard, gmax);
}

// 16-byte variant of k_combine_bnd (pairs of DOFs; e0 even)
__global__ void __launch_bounds__(NT) k_combine_bnd2(CombineArgs a, long long e0, const int* __restrict__ ebp,
                                                     const double* __restrict__ fb, long long ld_f) {
  pdl_trigger();
  pdl_wait();
  const int kk = blockIdx.y;
  double gmax = 0.0;
  const long long n2 = a.n / 2, stride = (long long)gridDim.x * NT;
  for (long long e = blockIdx.x * (long long)NT + threadIdx.x; e < n2; e += stride) {
    double2 s = make_double2(0.0, 0.0);
    for (int t0 = 0; t0 < a.nt; t0 += 4) {
      double2 v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u)
        v[u] = t0 + u < a.nt ? __ldcs(reinterpret_cast<const double2*>(a.v[t0 + u] + kk * a.ld[t0 + u]) + e)
                             : make_double2(0.0, 0.0);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (t0 + u >= a.nt) break;
        const double c = a.dc ? __ldg(a.dc + kk * a.ldc + t0 + u) : a.c[t0 + u];
        s.x = fma(c, v[u].x, s.x);
        s.y = fma(c, v[u].y, s.y);
      }
    }
    if (2 * e >= e0) {  // edge DOFs: the Dirichlet data where they lie on the domain boundary
      const int2 bp = __ldg(reinterpret_cast<const int2*>(ebp + (2 * e - e0)));
      if (bp.x >= 0) s.x = fb[kk * ld_f + bp.x];
      if (bp.y >= 0) s.y = fb[kk * ld_f + bp.y];
    }
    reinterpret_cast<double2*>(a.out + kk * a.ld_out)[e] = s;
    gacc(gmax, s.x);
    gacc(gmax, s.y);
  }
  if (a.guard) guard_max(a.guard, gmax);
}

bool combine_vec_ok(const CombineArgs& a) {
  if (a.n & 1 || ((uintptr_t)a.out & 15) || (a.ld_out & 1)) return false;
  for (int t = 0; t < a.nt; ++t)
    if (((uintptr_t)a.v[t] & 15) || (a.ld[t] & 1)) return false;
  return true;
}

__global__ void __launch_bounds__(NT) k_maxabs(int k, long long n, const double* x, long long ld,
                                                unsigned long long* guard) {
  pdl_trigger();
  pdl_wait();
  const int kk = blockIdx.y;
  double gmax = 0.0;
  const long long stride = (long long)gridDim.x * NT;
  for (long long e = blockIdx.x * (long long)NT + threadIdx.x; e < n; e += stride) {
    double v = x[kk * ld + e];
    gacc(gmax, v);
  }
  guard_max(guard, gmax);
}

__global__ void k_bnd_put(int k, int nbd, const int* __restrict__ ids, const double* __restrict__ fb,
                          long long ld_f, double* __restrict__ u, long long ld_u) {
  pdl_trigger();
  pdl_wait();
  long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (e >= (long long)k * nbd) return;
  int kk = (int)(e / nbd), i = (int)(e % nbd);
  u[kk * ld_u + ids[i]] = fb[kk * ld_f + i];
}

bool grad_enabled() {
  static const bool on = [] {
    const char* e = getenv("HPSB_NO_GRAD");
    return !(e && e[0] == '1');
  }();
  return on;
}

unsigned stream_blocks(long long n) {
  long long b = cdiv(n, (long long)NT * 4);
  long long cap = (long long)kNumSMs * 8;
  return (unsigned)std::max<long long>(1, std::min(b, cap));
}

}  // namespace

}  // namespace hpsb

using namespace hpsb;

struct hps_disc { Disc D; };

extern "C" {

int hps_disc_create(const hps_plan* pv, const hps_disc_desc* d, hps_disc** out) {
  *out = nullptr;
  if (!pv || !d) { set_error("hps_disc_create: null argument"); return HPS_ERR_ARG; }
  const Plan& P = pv->P;
  hps_disc* h = new hps_disc();
  Disc& D = h->D;
  D.P = &P;
  D.p = P.p; D.q = P.q; D.ni = P.ni; D.nb = P.nb; D.m = P.ni + P.nb; D.L = P.L;
  D.Lc = d->Lc; D.has_c1 = d->has_c1; D.has_c2 = d->has_c2; D.has_c = d->has_c;
  const int p = D.p, q = D.q;
  const size_t nm = 4 * (size_t)p * p + 4 * (size_t)q * q;
  auto fail = [&](const char* what) {
    set_error("hps_disc_create: %s", what);
    for (void* x : D.allocs) cudaFree(x);
    delete h;
    return HPS_ERR_CUDA;
  };
  std::vector<double> mats(nm);
  const double* src[8] = {d->d1x, d->d2x, d->d1y, d->d2y, d->ex1, d->ex2, d->ey1, d->ey2};
  size_t o = 0;
  for (int i = 0; i < 8; ++i) {
    size_t cnt = i < 4 ? (size_t)p * p : (size_t)q * q;
    memcpy(mats.data() + o, src[i], cnt * 8);
    o += cnt;
  }
  if (cudaMalloc(&D.mats, nm * 8) != cudaSuccess) return fail("out of device memory");
  D.allocs.push_back(D.mats);
  if (cudaMemcpy(D.mats, mats.data(), nm * 8, cudaMemcpyHostToDevice) != cudaSuccess) return fail("copy");
  if (D.Lc == 1) {
    for (int i = 0; i < 5; ++i) D.cc[i] = d->coef[(size_t)i * D.m];
  } else {
    size_t n = (size_t)D.Lc * 5 * D.m;
    if (cudaMalloc(&D.coef, n * 8) != cudaSuccess) return fail("out of device memory");
    D.allocs.push_back(D.coef);
    if (cudaMemcpy(D.coef, d->coef, n * 8, cudaMemcpyHostToDevice) != cudaSuccess) return fail("copy");
  }
  size_t ns = (size_t)P.L * P.nb;
  if (cudaMalloc(&D.sign, ns) != cudaSuccess) return fail("out of device memory");
  D.allocs.push_back(D.sign);
  if (cudaMemcpy(D.sign, d->leaf_bnd_sign, ns, cudaMemcpyHostToDevice) != cudaSuccess) return fail("copy");
  *out = h;
  return HPS_OK;
}

void hps_disc_destroy(hps_disc* h) {
  if (!h) return;
  for (void* x : h->D.allocs) cudaFree(x);
  delete h;
}

int hps_leaf_eval(const hps_disc* h, int k, const double* u, long long ld_u, double* lu_int, double* lu,
                  double* ux, double* uy, double* jump, long long ld_o, double* guard, void* stream) {
  if (!h) { set_error("hps_leaf_eval: null argument"); return HPS_ERR_ARG; }
  return hps_leaf_eval_range(h, 0, h->D.L, k, u, ld_u, lu_int, lu, ux, uy, jump, ld_o, guard, stream);
}

int hps_leaf_eval_range(const hps_disc* h, int leaf0, int nleaf, int k, const double* u, long long ld_u,
                        double* lu_int, double* lu, double* ux, double* uy, double* jump, long long ld_o,
                        double* guard, void* stream) {
  if (!h || !u) { set_error("hps_leaf_eval: null argument"); return HPS_ERR_ARG; }
  const Disc& D = h->D;
  const Plan& P = *D.P;
  if (leaf0 < 0 || nleaf < 0 || leaf0 + nleaf > P.L) {
    set_error("hps_leaf_eval: leaf range [%d, %d) outside [0, %d)", leaf0, leaf0 + nleaf, P.L);
    return HPS_ERR_ARG;
  }
  if (k <= 0 || nleaf == 0) return HPS_OK;
  cudaStream_t st = (cudaStream_t)stream;
  const long long Lni = (long long)P.L * P.ni;
  // averaged outputs accumulate at edge DOFs; the flux jump is zero off the edges
  for (double* o : {lu, ux, uy}) {
    if (!o) continue;
    for (int kk = 0; kk < k; ++kk)
      HPSB_CUDA(cudaMemsetAsync(o + kk * ld_o + Lni, 0, (size_t)(P.N - Lni) * 8, st));
  }
  if (jump)
    for (int kk = 0; kk < k; ++kk) HPSB_CUDA(cudaMemsetAsync(jump + kk * ld_o, 0, (size_t)P.N * 8, st));
  EvalArgs a{};
  a.k = k; a.u = u; a.ld_u = ld_u;
  a.L = nleaf; a.p = D.p; a.q = D.q; a.ni = D.ni; a.nb = D.nb; a.m = D.m; a.N = P.N;
  a.ioff = (long long)leaf0 * D.ni;
  a.lpb = std::max(1, NT / (D.p * D.p));
  a.lbg = P.leaf_bnd_gidx + (long long)leaf0 * D.nb; a.sign = D.sign + (long long)leaf0 * D.nb; a.mats = D.mats;
  a.Lc = D.Lc; a.coef = D.Lc > 1 ? D.coef + (long long)leaf0 * 5 * D.m : D.coef;
  for (int i = 0; i < 5; ++i) a.cc[i] = D.cc[i];
  a.has_c1 = D.has_c1; a.has_c2 = D.has_c2; a.has_c = D.has_c;
  a.lu_int = lu_int; a.lu = lu; a.ux = ux; a.uy = uy; a.jump = jump; a.ld_o = ld_o;
  a.guard = reinterpret_cast<unsigned long long*>(guard);
  const int PS = (D.p + 1) | 1, QS = (D.q + 1) | 1;
  const int pp = D.p * PS, qq = D.q * QS;
  unsigned groups = (unsigned)cdiv(nleaf, a.lpb);
  dim3 grid(std::min(groups, (unsigned)(kNumSMs * 8)), (unsigned)k);
  const bool int_only = lu_int && !lu && !ux && !uy && !jump;
  if (int_only && (D.p == 10 || D.p == 12 || D.p == 16)) {
    a.lpb = std::max(1, 2048 / (D.p * D.p));  // ~2K staged values per iteration
    groups = (unsigned)cdiv(nleaf, a.lpb);
    grid.x = std::min(groups, (unsigned)(kNumSMs * 8));
    size_t sm2 = (size_t)a.lpb * pp * 8;
    const bool g1 = D.has_c1 || D.has_c2;
#define HPSB_LOP(PP)                                                        \
    if (D.p == PP) {                                                        \
      if (g1) HPSB_CUDA(launch_pdl(k_leaf_lop_int<PP, true>, grid, dim3(NT), sm2, st, a));  \
      else HPSB_CUDA(launch_pdl(k_leaf_lop_int<PP, false>, grid, dim3(NT), sm2, st, a));    \
    }
    HPSB_LOP(10) HPSB_LOP(12) HPSB_LOP(16)
#undef HPSB_LOP
    HPSB_LAUNCH_CHECK();
    return HPS_OK;
  }
  const bool grad_only = ux && uy && !lu && !lu_int && !jump;
  if (grad_only && (D.p == 10 || D.p == 12 || D.p == 16) && grad_enabled()) {
    a.lpb = std::max(1, 2048 / (D.p * D.p));
    groups = (unsigned)cdiv(nleaf, a.lpb);
    grid.x = std::min(groups, (unsigned)(kNumSMs * 8));
    const size_t sm2 = (size_t)a.lpb * pp * 8;
    if (D.p == 10) HPSB_CUDA(launch_pdl(k_leaf_grad<10>, grid, dim3(GradThreads<10>::value), sm2, st, a));
    if (D.p == 12) HPSB_CUDA(launch_pdl(k_leaf_grad<12>, grid, dim3(GradThreads<12>::value), sm2, st, a));
    if (D.p == 16) HPSB_CUDA(launch_pdl(k_leaf_grad<16>, grid, dim3(GradThreads<16>::value), sm2, st, a));
    HPSB_LAUNCH_CHECK();
    return HPS_OK;
  }
  size_t smem = (size_t)(4 * pp + 4 * qq + a.lpb * pp) * 8;
  k_leaf_eval<<<grid, NT, smem, st>>>(a);
  HPSB_LAUNCH_CHECK();
  return HPS_OK;
}

int hps_combine(int k, long long n, int nterms, const double* coefs, const double* const* vecs,
                const long long* lds, double* out, long long ld_out, double* guard, void* stream) {
  if (k <= 0 || n <= 0) return HPS_OK;
  if (nterms < 0 || nterms > MAXT) { set_error("hps_combine: %d terms (max %d)", nterms, MAXT); return HPS_ERR_ARG; }
  CombineArgs a{};
  a.nt = nterms; a.k = k; a.n = n; a.out = out; a.ld_out = ld_out;
  for (int t = 0; t < nterms; ++t) { a.c[t] = coefs[t]; a.v[t] = vecs[t]; a.ld[t] = lds[t]; }
  a.guard = reinterpret_cast<unsigned long long*>(guard);
  if (combine_vec_ok(a)) {
    dim3 grid(stream_blocks(n / 2), (unsigned)k);
    HPSB_CUDA(launch_pdl(k_combine2, grid, dim3(NT), 0, (cudaStream_t)stream, a));
  } else {
    dim3 grid(stream_blocks(n), (unsigned)k);
    HPSB_CUDA(launch_pdl(k_combine, grid, dim3(NT), 0, (cudaStream_t)stream, a));
  }
  HPSB_LAUNCH_CHECK();
  return HPS_OK;
}

int hps_combine_dev(int k, long long n, int nterms, const double* dcoefs, const double* const* vecs,
                    const long long* lds, double* out, long long ld_out, double* guard, void* stream) {
  return hps_combine_dev_rows(k, n, nterms, dcoefs, 0, vecs, lds, out, ld_out, guard, stream);
}

int hps_combine_dev_rows(int k, long long n, int nterms, const double* dcoefs, long long ld_c,
                         const double* const* vecs, const long long* lds, double* out, long long ld_out,
                         double* guard, void* stream) {
  if (k <= 0 || n <= 0) return HPS_OK;
  if (nterms < 0 || nterms > MAXT) { set_error("hps_combine_dev: %d terms (max %d)", nterms, MAXT); return HPS_ERR_ARG; }
  CombineArgs a{};
  a.nt = nterms; a.k = k; a.n = n; a.out = out; a.ld_out = ld_out; a.dc = dcoefs; a.ldc = ld_c;
  for (int t = 0; t < nterms; ++t) { a.v[t] = vecs[t]; a.ld[t] = lds[t]; }
  a.guard = reinterpret_cast<unsigned long long*>(guard);
  if (combine_vec_ok(a)) {
    dim3 grid(stream_blocks(n / 2), (unsigned)k);
    HPSB_CUDA(launch_pdl(k_combine2, grid, dim3(NT), 0, (cudaStream_t)stream, a));
  } else {
    dim3 grid(stream_blocks(n), (unsigned)k);
    HPSB_CUDA(launch_pdl(k_combine, grid, dim3(NT), 0, (cudaStream_t)stream, a));
  }
  HPSB_LAUNCH_CHECK();
  return HPS_OK;
}

int hps_maxabs(int k, long long n, const double* x, long long ld, double* guard, void* stream) {
  if (k <= 0 || n <= 0) return HPS_OK;
  dim3 grid(stream_blocks(n), (unsigned)k);
  HPSB_CUDA(launch_pdl(k_maxabs, grid, dim3(NT), 0, (cudaStream_t)stream, k, n, x, ld,
                       reinterpret_cast<unsigned long long*>(guard)));
  HPSB_LAUNCH_CHECK();
  return HPS_OK;
}

int hps_combine_bnd(const hps_plan* pv, int k, int nterms, const double* coefs, const double* dcoefs,
                    const double* const* vecs, const long long* lds, const double* fb, long long ld_f, double* out,
                    long long ld_out, double* guard, void* stream) {
  if (!pv || !fb || !out || (!coefs && !dcoefs)) { set_error("hps_combine_bnd: null argument"); return HPS_ERR_ARG; }
  const Plan& P = pv->P;
  if (!P.edge_bpos) { set_error("hps_combine_bnd: boundary DOFs outside the edge range"); return HPS_ERR_ARG; }
  if (nterms < 0 || nterms > MAXT) { set_error("hps_combine_bnd: %d terms (max %d)", nterms, MAXT); return HPS_ERR_ARG; }
  if (k <= 0) return HPS_OK;
  CombineArgs a{};
  a.nt = nterms; a.k = k; a.n = P.N; a.out = out; a.ld_out = ld_out; a.dc = dcoefs;
  for (int t = 0; t < nterms; ++t) { if (coefs) a.c[t] = coefs[t]; a.v[t] = vecs[t]; a.ld[t] = lds[t]; }
  a.guard = reinterpret_cast<unsigned long long*>(guard);
  const long long e0 = (long long)P.L * P.ni;
  if (combine_vec_ok(a) && !(e0 & 1) && !((uintptr_t)P.edge_bpos & 7)) {
    dim3 grid(stream_blocks(P.N / 2), (unsigned)k);
    HPSB_CUDA(launch_pdl(k_combine_bnd2, grid, dim3(NT), 0, (cudaStream_t)stream, a, e0, (const int*)P.edge_bpos,
                         fb, ld_f));
  } else {
    dim3 grid(stream_blocks(P.N), (unsigned)k);
    HPSB_CUDA(launch_pdl(k_combine_bnd, grid, dim3(NT), 0, (cudaStream_t)stream, a, e0, (const int*)P.edge_bpos,
                         fb, ld_f));
  }
  HPSB_LAUNCH_CHECK();
  return HPS_OK;
}

int hps_put_boundary(const hps_plan* pv, int k, const double* fb, long long ld_f, double* u,
                     long long ld_u, void* stream) {
  if (!pv) { set_error("hps_put_boundary: null plan"); return HPS_ERR_ARG; }
  const Plan& P = pv->P;
  long long n = (long long)k * P.nbd;
  if (n <= 0) return HPS_OK;
  HPSB_CUDA(launch_pdl(k_bnd_put, dim3((unsigned)cdiv(n, NT)), dim3(NT), 0, (cudaStream_t)stream, k, P.nbd,
                       (const int*)P.boundary_ids, fb, ld_f, u, ld_u));
  HPSB_LAUNCH_CHECK();
  return HPS_OK;
}

}  // extern "C"
