// Fused subtree kernels for the narrow (deep) levels of the HPS solve.
//
// Below level dF every node's operators are small (tens of KB) and the
// levels hold thousands of nodes, so one launch per level and operator family
// is dominated by launch and gather latency rather than bytes.  Here one CTA
// owns the subtree of one level-dF node and walks all of its levels in one
// launch:
//   up   (solver.py:243-256, deepest level first): r3 from the children's
//        fluxes, w3 = X33^-1 r3, h = [ha[i1a]; hb[i2b]] + Tstack w3, with the
//        children's fluxes and w3 kept in shared memory between levels;
//   down (solver.py:258-268, root first): u[j3] = S u[gidx_bnd] + w3, level by
//        level, the CTA reading back the interface values it wrote one level up.
// The operator rows a CTA needs for one level are one contiguous node-aligned
// panel tile (make_panel_nodes), streamed column by column with the same
// two-rows-per-thread, software-pipelined 16-byte loads as level_gemv.cu.
#include <stdlib.h>

#include "hps_plan.cuh"
#include "stream.cuh"

namespace hpsb {

namespace {

constexpr int NT = 256;          // 512 subtree CTAs of 256 threads (64 registers) fit one wave on 148 SMs
constexpr int MAXF = 10;          // fused levels
constexpr int kMaxRows = 2048;    // operator rows of one CTA on one level
constexpr int U = 4;

struct FLevel {
  Panel Up, S;
  const int *i1a, *i3a, *i2b, *i3b, *j3, *gidx;
  int n3, n12, n1a, nbc;
  double* W3;
  long long W3_k;
};

struct SubArgs {
  int nf, dF, k;
  FLevel lv[MAXF];
  double* H_dF; long long H_k;                  // fluxes of the level-dF nodes (dF > 0)
  const double* Hleaf; long long sh, hs;        // leaf fluxes: rhs stride, per-leaf stride
  const double* jump; long long jump_k; double inv_dt;
  double* u; long long u_k; int has_w3;
  int hcap, rcap;                               // shared-memory carve (doubles)
  // subtree-local numbering (Plan::sub_slots)
  const int* slots; long long slot_off[MAXF + 1]; int j3_base[MAXF]; int nslots;
  const int* gidx_root;                         // level-dF gidx_bnd
  int b0;                                       // first subtree of the launch
  int fold;                                     // shared one-rhs apply: two nodes per thread
};

// y(row) = sum_col M[col][row] x[node(row)][col] over the CTA's tile, then
// out(j, row, kk, y) for every valid row; x is [node][KM][C] in shared memory.
// vn > 1: the tile holds ONE node's operator shared by vn nodes (shared
// layout), row pair q = (node q / pairs, pair q % pairs).
// When there are fewer row pairs than threads, G threads share a row pair,
// each streaming a contiguous column block; their partial sums meet in shared
// memory (red, 2*NT*KM doubles) and are added in block order.
// nodes per thread of the shared one-rhs apply
#ifndef HPSB_SUB_NODES
#define HPSB_SUB_NODES 2
#endif
constexpr int SNF = HPSB_SUB_NODES;

// partial-sum space of a CTA (doubles): 2 rows x KM rhs per thread, or 2 rows
// x SNF nodes per (item, column block) in the shared one-rhs apply
constexpr int red_doubles(int KM, bool SH) { return SH && KM == 1 ? 2 * SNF * NT : 2 * NT * KM; }

// Shared operator, one rhs: a thread owns a row pair of the one-node operator
// for SNF nodes, so each 16-byte operator load feeds 2 SNF fmas (the subtree
// levels are bound by the L1 traffic of the operator loads: every CTA re-reads
// the level's tile once per node otherwise).  x rows 16-byte aligned.
template <int NF>
__device__ __forceinline__ void stream_nodes(const double2* __restrict__ M, int cs, int n, const double* x, int XS,
                                             int nv, double (&acc)[2 * NF]) {
  constexpr int SU = 4;
  const double2* p = M;
  double2 A[SU], B[SU];
  int xo[NF];  // node j's x row (nodes past nv read node nv - 1; their sums are discarded)
#pragma unroll
  for (int j = 0; j < NF; ++j) xo[j] = min(j, nv - 1) * XS;
  auto ld = [&](double2 (&m)[SU]) {
#pragma unroll
    for (int u = 0; u < SU; ++u) { m[u] = __ldcs(p); p += cs; }
  };
  auto fma4 = [&](const double2 (&m)[SU], int col) {
#pragma unroll
    for (int u = 0; u < SU; u += 2)
#pragma unroll
      for (int j = 0; j < NF; ++j) {
        const double2 v = *reinterpret_cast<const double2*>(x + xo[j] + col + u);
        acc[2 * j] = fma(m[u].x, v.x, acc[2 * j]);
        acc[2 * j + 1] = fma(m[u].y, v.x, acc[2 * j + 1]);
        acc[2 * j] = fma(m[u + 1].x, v.y, acc[2 * j]);
        acc[2 * j + 1] = fma(m[u + 1].y, v.y, acc[2 * j + 1]);
      }
  };
  const int nfull = n / SU;
  if (nfull > 0) ld(A);
  int b = 0;
  for (; b + 1 < nfull; b += 2) {
    ld(B);
    fma4(A, b * SU);
    if (b + 2 < nfull) ld(A);
    fma4(B, (b + 1) * SU);
  }
  if (b < nfull) fma4(A, b * SU);
  for (int col = nfull * SU; col < n; ++col) {
    const double2 m = __ldcs(p);
    p += cs;
#pragma unroll
    for (int j = 0; j < NF; ++j) {
      acc[2 * j] = fma(m.x, x[xo[j] + col], acc[2 * j]);
      acc[2 * j + 1] = fma(m.y, x[xo[j] + col], acc[2 * j + 1]);
    }
  }
}

template <class Out>
__device__ __forceinline__ void apply_shared(const double2* base, int R, int C, int cs, const double* xs,
                                             int xstride, double* red, Out out, int vn) {
  const int items = cs * ((vn + SNF - 1) / SNF);
  int G = 1;
  while (2 * G * items <= NT && 2 * G * 4 <= C) G *= 2;  // then G * items <= NT
  const int CKg = ((C + G - 1) / G + 1) & ~1;
  const int t = threadIdx.x;
  for (int q = t % items + (t / items >= G ? NT : 0); q < items; q += (G == 1 ? NT : items)) {
    const int g = G == 1 ? 0 : t / items;
    const int c0 = min(C, g * CKg), c1 = min(C, c0 + CKg);
    const int pr = q % cs, j0 = SNF * (q / cs);
    double acc[2 * SNF];
#pragma unroll
    for (int i = 0; i < 2 * SNF; ++i) acc[i] = 0.0;
    stream_nodes<SNF>(base + pr + (size_t)c0 * cs, cs, c1 - c0, xs + j0 * xstride + c0, xstride, vn - j0, acc);
    if (G == 1) {
#pragma unroll
      for (int j = 0; j < SNF; ++j) {
        if (j0 + j >= vn) break;
        if (2 * pr < R) out(j0 + j, 2 * pr, 0, acc[2 * j]);
        if (2 * pr + 1 < R) out(j0 + j, 2 * pr + 1, 0, acc[2 * j + 1]);
      }
    } else {
#pragma unroll
      for (int i = 0; i < 2 * SNF; ++i) red[(g * 2 * SNF + i) * items + q] = acc[i];
    }
  }
  if (G > 1) {
    __syncthreads();
    for (int i = t; i < 2 * SNF * items; i += NT) {
      const int q = i % items, w = i / items, pr = q % cs, node = SNF * (q / cs) + (w >> 1), row = 2 * pr + (w & 1);
      if (node >= vn || row >= R) continue;
      double y = 0.0;
      for (int g = 0; g < G; ++g) y += red[(g * 2 * SNF + w) * items + q];
      out(node, row, 0, y);
    }
    __syncthreads();
  }
}

template <int KM, bool SH, class Out>
__device__ __forceinline__ void tile_apply(const Panel& pn, int tile, const double* xs, int xstride, double* red,
                                           Out out, int vn = 1, int fold = 0) {
  const int R = pn.R, C = pn.C, TR = pn.TR, TS = pn.TS;
  const double2* base = reinterpret_cast<const double2*>(pn.base + (size_t)tile * C * TS);
  const int cs = TS / 2;          // stored row pairs
  if constexpr (SH && KM == 1) {  // (one-node levels too: the second node's sums are discarded)
    apply_shared(base, R, C, cs, xs, xstride, red, out, vn);
    return;
  }
  const int np = cs * vn;         // row pairs to compute
  int G = 1;
  while (2 * G * np <= NT && 2 * G * 4 <= C) G *= 2;
  const int CKg = SH ? (((C + G - 1) / G + 1) & ~1) : (C + G - 1) / G;  // SH: even column blocks (16-byte x loads)
  const int t = threadIdx.x;
  // (node, local row) of stored row r of pair q; valid = r < rows of that node
  auto where = [&](int q, int h, int& j, int& row) -> bool {
    if (vn > 1) {
      j = q / cs;
      row = 2 * (q % cs) + h;
      return row < R;
    }
    const int r = 2 * q + h;
    j = min(r, TR - 1) / R;
    row = r - j * R;
    return r < TR;
  };
  for (int q = t % np + (t / np >= G ? NT : 0); q < np; q += (G == 1 ? NT : np)) {
    const int g = G == 1 ? 0 : t / np;
    const int c0 = g * CKg, c1 = min(C, c0 + CKg);
    int ja, la, jb, lb;
    const bool va = where(q, 0, ja, la), vb = where(q, 1, jb, lb);
    const double2* M = base + (vn > 1 ? q % cs : q);
    double acc0[KM], acc1[KM];
#pragma unroll
    for (int kk = 0; kk < KM; ++kk) { acc0[kk] = 0.0; acc1[kk] = 0.0; }
    const double* xa = xs + ja * KM * xstride + c0;
    if (SH && KM == 1) {
      // shared operator: both rows belong to node ja (= jb); x rows are 16-byte
      // aligned (even strides and offsets, see the kernels' shared-memory carve)
      stream_pairs(M + (size_t)c0 * cs, cs, c1 - c0, xa, acc0[0], acc1[0]);
    } else {
      double2 A[U];
      if (c1 - c0 >= U) load_batch<U>(A, M, cs, c0);
      stream_cols<KM, U>(A, M, cs, c0, c1, xs, ja * KM * xstride, jb * KM * xstride, xstride, acc0, acc1);
    }
    if (G == 1) {
#pragma unroll
      for (int kk = 0; kk < KM; ++kk) {
        if (va) out(ja, la, kk, acc0[kk]);
        if (vb) out(jb, lb, kk, acc1[kk]);
      }
    } else {
#pragma unroll
      for (int kk = 0; kk < KM; ++kk) {
        red[(g * KM + kk) * 2 * np + 2 * q] = acc0[kk];
        red[(g * KM + kk) * 2 * np + 2 * q + 1] = acc1[kk];
      }
    }
  }
  if (G > 1) {
    __syncthreads();
    for (int i = t; i < 2 * np; i += NT) {
      int j, row;
      if (!where(i / 2, i % 2, j, row)) continue;
#pragma unroll
      for (int kk = 0; kk < KM; ++kk) {
        double y = 0.0;
        for (int g = 0; g < G; ++g) y += red[(g * KM + kk) * 2 * np + i];
        out(j, row, kk, y);
      }
    }
    __syncthreads();
  }
}

template <int KM, bool SH = false>
__global__ void __launch_bounds__(NT, KM == 1 ? 4 : 1) k_sub_up(SubArgs a) {
  extern __shared__ double sm[];
  double* Hs = sm;                    // children's fluxes of the current level [child][KM][nbc]
  double* Hn = Hs + KM * a.hcap;      // this level's fluxes [node][KM][n12]
  double* r3s = Hn + KM * a.hcap;     // [node][KM][n3]
  double* red = r3s + KM * a.rcap;    // red_doubles(KM, SH)
  const int b = a.b0 + blockIdx.x, kg0 = blockIdx.y * KM, tid = threadIdx.x;
  pdl_trigger();
  pdl_wait();
  for (int e = a.nf - 1; e >= 0; --e) {
    const FLevel& L = a.lv[e];
    const int npn = 1 << e, node0 = b * npn, n3 = L.n3, n12 = L.n12, nbc = L.nbc, n3s = (n3 + 1) & ~1;
    const bool leafc = e == a.nf - 1;
    auto child = [&](int j, int kk, int which) -> const double* {  // which: 0 = alpha, 1 = beta
      if (leafc) return a.Hleaf + (kg0 + kk) * a.sh + (2LL * (node0 + j) + which) * a.hs;
      return Hs + ((2 * j + which) * KM + kk) * nbc;
    };
    for (int idx = tid; idx < npn * KM * n3; idx += NT) {
      const int col = idx % n3, t2 = idx / n3, kk = t2 % KM, j = t2 / KM, kg = kg0 + kk;
      double v = 0.0;
      if (kg < a.k) {
        v = child(j, kk, 1)[L.i3b[col]] - child(j, kk, 0)[L.i3a[col]];
        if (a.jump) v = v - a.inv_dt * a.jump[kg * a.jump_k + L.j3[(long long)(node0 + j) * n3 + col]];
      }
      r3s[(j * KM + kk) * n3s + col] = v;
    }
    __syncthreads();
    // [w3; h - base] = [X33^-1; Tstack X33^-1] r3 for the subtree's nodes of this level
    tile_apply<KM, SH>(L.Up, L.Up.c == 1 ? 0 : b, r3s, n3s, red, [&](int j, int row, int kk, double y) {
      const int kg = kg0 + kk;
      if (kg >= a.k) return;
      if (row < n3) {
        L.W3[kg * L.W3_k + (long long)(node0 + j) * n3 + row] = y;
        return;
      }
      const int r = row - n3;
      const double base = r < L.n1a ? child(j, kk, 0)[L.i1a[r]] : child(j, kk, 1)[L.i2b[r - L.n1a]];
      const double h = base + y;
      Hn[(j * KM + kk) * n12 + r] = h;
      if (e == 0) a.H_dF[kg * a.H_k + (long long)(node0 + j) * n12 + r] = h;
    }, L.Up.c == 1 ? npn : 1, a.fold);
    __syncthreads();
    if (a.dF + e == 0) break;  // the root's outer flux is never consumed
    double* t = Hs; Hs = Hn; Hn = t;
  }
}

template <int KM, bool SH = false>
__global__ void __launch_bounds__(NT) k_sub_down(SubArgs a) {
  extern __shared__ double sm[];
  double* red = sm;                          // red_doubles(KM, SH)
  double* xs = sm + red_doubles(KM, SH);     // [node][KM][n12]
  const int b = a.b0 + blockIdx.x, kg0 = blockIdx.y * KM, tid = threadIdx.x;
  pdl_trigger();
  pdl_wait();
  for (int e = 0; e < a.nf; ++e) {
    const FLevel& L = a.lv[e];
    const int npn = 1 << e, node0 = b * npn, n3 = L.n3, n12 = L.n12, n12s = (n12 + 1) & ~1;
    if (e > 0) __syncthreads();  // this CTA's writes one level up are visible from here on
    for (int idx = tid; idx < npn * KM * n12; idx += NT) {
      const int col = idx % n12, t2 = idx / n12, kk = t2 % KM, j = t2 / KM, kg = kg0 + kk;
      xs[(j * KM + kk) * n12s + col] = kg < a.k ? a.u[kg * a.u_k + L.gidx[(long long)(node0 + j) * n12 + col]] : 0.0;
    }
    __syncthreads();
    tile_apply<KM, SH>(L.S, L.S.c == 1 ? 0 : b, xs, n12s, red, [&](int j, int row, int kk, double y) {
      const int kg = kg0 + kk;
      if (kg >= a.k) return;
      const long long nd = (long long)(node0 + j) * n3 + row;
      if (a.has_w3) y = y + L.W3[kg * L.W3_k + nd];
      a.u[kg * a.u_k + L.j3[nd]] = y;
    }, L.S.c == 1 ? npn : 1, a.fold);
  }
}

// Down sweep with the subtree's DOFs held in shared memory: the root
// boundary is read from u once, every interface value this CTA produces is
// kept (and written through to u) so lower levels gather from shared memory.
template <int KM, bool SH = false>
__global__ void __launch_bounds__(NT, KM == 1 ? 4 : 1) k_sub_down_local(SubArgs a) {
  extern __shared__ double sm[];
  double* red = sm;                        // red_doubles(KM, SH)
  double* uloc = sm + red_doubles(KM, SH); // [KM][nslots]
  double* xs = uloc + ((KM * a.nslots + 1) & ~1);  // [node][KM][n12 rounded up to even]
  const int b = a.b0 + blockIdx.x, kg0 = blockIdx.y * KM, tid = threadIdx.x, ns = a.nslots;
  pdl_trigger();
  pdl_wait();
  {
    const int n12 = a.lv[0].n12;
    for (int idx = tid; idx < KM * n12; idx += NT) {
      const int kk = idx / n12, col = idx % n12, kg = kg0 + kk;
      uloc[kk * ns + col] = kg < a.k ? a.u[kg * a.u_k + a.gidx_root[(long long)b * n12 + col]] : 0.0;
    }
  }
  for (int e = 0; e < a.nf; ++e) {
    const FLevel& L = a.lv[e];
    const int npn = 1 << e, node0 = b * npn, n3 = L.n3, n12 = L.n12, jb = a.j3_base[e], n12s = (n12 + 1) & ~1;
    const int* sl = a.slots + a.slot_off[e];
    __syncthreads();
    for (int idx = tid; idx < npn * KM * n12; idx += NT) {
      const int col = idx % n12, t2 = idx / n12, kk = t2 % KM, j = t2 / KM;
      xs[(j * KM + kk) * n12s + col] = uloc[kk * ns + sl[j * n12 + col]];
    }
    __syncthreads();
    tile_apply<KM, SH>(L.S, L.S.c == 1 ? 0 : b, xs, n12s, red, [&](int j, int row, int kk, double y) {
      const int kg = kg0 + kk;
      if (kg >= a.k) return;
      const long long nd = (long long)(node0 + j) * n3 + row;
      if (a.has_w3) y = y + L.W3[kg * L.W3_k + nd];
      uloc[kk * ns + jb + j * n3 + row] = y;
      a.u[kg * a.u_k + L.j3[nd]] = y;
    }, L.S.c == 1 ? npn : 1, a.fold);
  }
}

// ---------------------------------------------------------------------------
// Tensor-core subtree levels (shared operators, one rhs).
//
// The SIMT applies above are issue-bound: ~20 instructions per fma go to
// address arithmetic, index gathers and operator loads (ncu: k_sub_up issues
// 40 M warp instructions for 65 M fmas per C2 solve; its time is that
// instruction count over the SMs' issue slots).  Here a level's apply
//     Y[row][node] = sum_c Op[row][c] X[node][c]
// runs as DMMA m8n8k4 tiles, (8 operator rows) x (8 nodes) x (4 columns) per
// instruction:
//  * A fragments from a fragment-ordered copy of the level operator
//    (sub_mma_prepare: tile (m, k) is 32 consecutive doubles in lane order,
//    zero padded to whole 8-row tiles and to k-steps in multiples of 4), so a
//    warp's operator load is one coalesced 256-byte line with no predicates
//    (L1-cached: the CTAs of an SM read the same level tiles);
//  * B fragments from the CTA's staged node vectors (row stride = 4 mod 16
//    doubles: conflict-free), zero padded to 16 columns;
//  * the level's index tables (child-flux offsets, slot maps) staged in
//    shared memory before the dependency wait; the subtree's leaf fluxes
//    staged by one coalesced copy.
// Work units are (row tile, node tile, column split) spread over the warps;
// split partials meet in shared memory and are added in split order, so the
// results are deterministic.  Levels with fewer than 8 nodes in a subtree pad
// the node tile.
constexpr int MW = NT / 32;      // warps per CTA
constexpr int kRedUnits = 16;    // partial 8 x 8 tiles in shared memory
constexpr int kRedMma = kRedUnits * 64;

__device__ __forceinline__ void dmma8(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// staged node-vector stride: = 4 (mod 16) doubles (the 8 x 4 B-fragment reads
// of a warp, node = lane / 4, column = lane % 4, hit distinct banks), with
// room for the zero padding to 16 columns
__host__ __device__ __forceinline__ int mma_xs(int C) { return ((C + 15) & ~15) + 4; }

// Y = Op X^T for one (level, operator): units (m, n, s) over the warps.
// F: fragment-ordered operator (mt x kt4 tiles of 32); xs: [node][XS], vn nodes.
// pre(node, row, ctx) runs before the k-loop of a single-split unit (prefetch of
// epilogue operands), out(node, row, y, ctx) after it.
struct MmaShape { int mt, kt4, ks, kper; };

// UNR: k-loop iterations (4 k-steps each) unrolled, i.e. operator loads in flight: 2 for the
// up sweep's short column chains, 4 for the down sweep's long ones (k_sub_down_mma 39.4 -> 36.0 us)
template <int UNR, class Pre, class Out>
__device__ __forceinline__ void mma_apply(const double* __restrict__ F, const MmaShape sh, int R, const double* xs,
                                          int XS, int vn, double* red, Pre pre, Out out) {
  const int mt = sh.mt, nt = (vn + 7) >> 3, mn = mt * nt, ks = sh.ks;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, gr = lane >> 2, gc = lane & 3;
  // unit u = (s * nt + n) * mt + m: the up sweep (many short units) decodes it once and
  // advances it by MW per round; the down sweep (few long units, registers for the loads in
  // flight) decodes it per unit
  constexpr bool INC = UNR == 2;
  int s = warp / mn, n = (warp - s * mn) / mt, m = warp - s * mn - n * mt;
  for (int u = warp; u < mn * ks; u += MW) {
    if (!INC) {
      s = ks == 1 ? 0 : u / mn;
      const int t = u - s * mn;
      n = t / mt;
      m = t - n * mt;
    }
    const int row = m * 8 + gr, node = n * 8 + 2 * gc;
    const int k0 = s * sh.kper, kn = min(sh.kt4 - k0, sh.kper);
    const double* ap = F + ((size_t)m * sh.kt4 + k0) * 32 + lane;
    const double* bp = xs + min(n * 8 + gr, vn - 1) * XS + k0 * 4 + gc;
    typename Pre::Ctx cx{};
    if (ks == 1 && row < R) pre(node, row, cx);
    double d0 = 0.0, d1 = 0.0, e0 = 0.0, e1 = 0.0;
#pragma unroll(UNR)
    for (int k = 0; k < kn; k += 4) {
      const double a0 = __ldg(ap), a1 = __ldg(ap + 32), a2 = __ldg(ap + 64), a3 = __ldg(ap + 96);
      const double b0 = bp[0], b1 = bp[4], b2 = bp[8], b3 = bp[12];
      dmma8(d0, d1, a0, b0);
      dmma8(e0, e1, a1, b1);
      dmma8(d0, d1, a2, b2);
      dmma8(e0, e1, a3, b3);
      ap += 128;
      bp += 16;
    }
    d0 += e0;
    d1 += e1;
    if (ks == 1) {
      if (row < R) {
        if (node < vn) out(node, row, d0, cx, 0);
        if (node + 1 < vn) out(node + 1, row, d1, cx, 1);
      }
    } else {
      double* rp = red + (size_t)u * 64 + gr * 8 + 2 * gc;
      rp[0] = d0;
      rp[1] = d1;
    }
    if (INC) {
      m += MW;
      while (m >= mt) {
        m -= mt;
        if (++n == nt) { n = 0; ++s; }
      }
    }
  }
  if (ks > 1) {
    __syncthreads();
    for (int i = threadIdx.x; i < mn * 64; i += NT) {
      const int t = i >> 6, e = i & 63, n = t / mt, row = (t - n * mt) * 8 + (e >> 3), node = n * 8 + (e & 7);
      if (row >= R || node >= vn) continue;
      double y = red[i];
      for (int s = 1; s < ks; ++s) y += red[(size_t)s * mn * 64 + i];
      typename Pre::Ctx cx{};
      pre.single(node, row, cx);
      out(node, row, y, cx, 0);
    }
  }
}

// (idx over nodes x width W) decoded incrementally: one division per thread per level
struct Walk {
  int j, c, dj, dc, W;
  __device__ __forceinline__ Walk(int W_) : W(W_) {
    j = threadIdx.x / W; c = threadIdx.x - j * W; dj = NT / W; dc = NT - dj * W;
  }
  __device__ __forceinline__ void next() {
    j += dj; c += dc;
    if (c >= W) { c -= W; ++j; }
  }
};

struct MLevel {       // per fused level, the tensor-core path
  const double *UpF, *SF;
  MmaShape up, dn;
  int tab;            // k_sub_up_mma: offset of the level's index table (ints) in shared memory
};

struct MmaArgs {
  MLevel ml[MAXF];
  int tab_ints;       // k_sub_up_mma: index tables (ints)
  int sl_ints;        // k_sub_down_mma: slot maps (ints)
  int hcap, rcap, xcap;
};

struct NoCtx { int z; };
struct PreNone {
  using Ctx = NoCtx;
  __device__ __forceinline__ void operator()(int, int, Ctx&) const {}
  __device__ __forceinline__ void single(int, int, Ctx&) const {}
};

__global__ void __launch_bounds__(NT, 4) k_sub_up_mma(SubArgs a, MmaArgs m) {
  extern __shared__ double sm[];
  double* Hs = sm;                 // children's fluxes of the current level [child][cs]
  double* Hn = Hs + m.hcap;        // this level's fluxes [node][n12]
  double* r3s = Hn + m.hcap;       // [node][mma_xs(n3)]
  double* red = r3s + m.rcap;      // kRedMma
  int* tab = reinterpret_cast<int*>(red + kRedMma);
  const int b = a.b0 + blockIdx.x, tid = threadIdx.x;
  pdl_trigger();
  // index tables (plan constants) before the dependency wait: per level
  // [g3a (n3) | g3b (n3) | gh (n12)], offsets relative to child 0 of a node
  for (int e = 0; e < a.nf; ++e) {
    const FLevel& L = a.lv[e];
    const int cs = e == a.nf - 1 ? (int)a.hs : L.nbc, n3 = L.n3, n12 = L.n12;
    int* t = tab + m.ml[e].tab;
    for (int i = tid; i < 2 * n3 + n12; i += NT) {
      int v;
      if (i < n3) v = L.i3a[i];
      else if (i < 2 * n3) v = cs + L.i3b[i - n3];
      else {
        const int r = i - 2 * n3;
        v = r < L.n1a ? L.i1a[r] : cs + L.i2b[r - L.n1a];
      }
      t[i] = v;
    }
  }
  pdl_wait();
  {  // the subtree's leaf fluxes: one contiguous block
    const int npn = 1 << (a.nf - 1);
    const double* src = a.Hleaf + 2LL * b * npn * a.hs;
    const int n = 2 * npn * (int)a.hs;
    for (int i = tid; i < n; i += NT) Hs[i] = src[i];
  }
  for (int e = a.nf - 1; e >= 0; --e) {
    const FLevel& L = a.lv[e];
    const MLevel& M = m.ml[e];
    const int npn = 1 << e, node0 = b * npn, n3 = L.n3, n12 = L.n12, XS = mma_xs(n3), W = (n3 + 15) & ~15;
    const int cs = e == a.nf - 1 ? (int)a.hs : L.nbc;
    const int* g3 = tab + M.tab;
    const int* gh = g3 + 2 * n3;
    __syncthreads();
    {
      Walk w(W);
      for (int idx = tid; idx < npn * W; idx += NT, w.next()) {
        double v = 0.0;
        if (w.c < n3) {
          const double* hc = Hs + 2 * w.j * cs;
          v = hc[g3[n3 + w.c]] - hc[g3[w.c]];
          if (a.jump) v = v - a.inv_dt * a.jump[L.j3[(long long)(node0 + w.j) * n3 + w.c]];
        }
        r3s[w.j * XS + w.c] = v;
      }
    }
    __syncthreads();
    // [w3; h - base] = [X33^-1; Tstack X33^-1] r3 for the subtree's nodes of this level
    mma_apply<2>(M.UpF, M.up, L.Up.R, r3s, XS, npn, red, PreNone{},
              [&](int j, int row, double y, NoCtx&, int) {
                if (row < n3) {
                  L.W3[(long long)(node0 + j) * n3 + row] = y;
                  return;
                }
                const int r = row - n3;
                const double h = Hs[2 * j * cs + gh[r]] + y;
                Hn[j * n12 + r] = h;
                if (e == 0) a.H_dF[(long long)(node0 + j) * n12 + r] = h;
              });
    if (a.dF + e == 0) break;  // the root's outer flux is never consumed
    double* t = Hs; Hs = Hn; Hn = t;
  }
}

struct DnCtx { double w[2]; int id[2]; };
struct PreDown {
  using Ctx = DnCtx;
  const double* W3; const int* j3; long long base; int n3, has_w3, vn;
  __device__ __forceinline__ void single(int node, int row, Ctx& c) const {
    const long long nd = base + (long long)node * n3 + row;
    c.w[0] = has_w3 ? W3[nd] : 0.0;
    c.id[0] = j3[nd];
  }
  __device__ __forceinline__ void operator()(int node, int row, Ctx& c) const {  // nodes node, node + 1
    const long long nd = base + (long long)node * n3 + row;
    if (node < vn) {
      c.w[0] = has_w3 ? W3[nd] : 0.0;
      c.id[0] = j3[nd];
    }
    if (node + 1 < vn) {
      c.w[1] = has_w3 ? W3[nd + n3] : 0.0;
      c.id[1] = j3[nd + n3];
    }
  }
};

__global__ void __launch_bounds__(NT, 4) k_sub_down_mma(SubArgs a, MmaArgs m) {
  extern __shared__ double sm[];
  double* red = sm;                        // kRedMma
  double* xs = red + kRedMma;              // [node][mma_xs(n12)]
  double* uloc = xs + m.xcap;              // [nslots]
  int* sls = reinterpret_cast<int*>(uloc + ((a.nslots + 1) & ~1));  // slot maps of every level
  const int b = a.b0 + blockIdx.x, tid = threadIdx.x;
  pdl_trigger();
  const int n12r = a.lv[0].n12;
  const int gi = tid < n12r ? a.gidx_root[(long long)b * n12r + tid] : 0;
  for (int i = tid; i < m.sl_ints; i += NT) sls[i] = a.slots[i];
  pdl_wait();
  for (int col = tid; col < n12r; col += NT) uloc[col] = a.u[col == tid ? gi : a.gidx_root[(long long)b * n12r + col]];
  for (int e = 0; e < a.nf; ++e) {
    const FLevel& L = a.lv[e];
    const MLevel& M = m.ml[e];
    const int npn = 1 << e, node0 = b * npn, n3 = L.n3, n12 = L.n12, jb = a.j3_base[e], XS = mma_xs(n12);
    const int W = (n12 + 15) & ~15;
    const int* sl = sls + a.slot_off[e];
    __syncthreads();
    {
      Walk w(W);
      for (int idx = tid; idx < npn * W; idx += NT, w.next())
        xs[w.j * XS + w.c] = w.c < n12 ? uloc[sl[w.j * n12 + w.c]] : 0.0;
    }
    __syncthreads();
    PreDown pd{L.W3, L.j3, (long long)node0 * n3, n3, a.has_w3, npn};
    mma_apply<4>(M.SF, M.dn, n3, xs, XS, npn, red, pd, [&](int j, int row, double y, DnCtx& c, int h) {
      y = y + c.w[h];
      uloc[jb + j * n3 + row] = y;
      a.u[c.id[h]] = y;
    });
  }
}

// fragment-ordered copy of a column-major panel tile (R x C, column stride TS)
__global__ void k_frag(const double* __restrict__ src, int R, int C, int TS, int mt, int kt4, double* dst) {
  const long long n = (long long)mt * kt4 * 32;
  for (long long i = blockIdx.x * 256LL + threadIdx.x; i < n; i += gridDim.x * 256LL) {
    const int lane = (int)(i & 31);
    const long long t = i >> 5;
    const int k = (int)(t % kt4), mm = (int)(t / kt4);
    const int r = mm * 8 + (lane >> 2), c = k * 4 + (lane & 3);
    dst[i] = (r < R && c < C) ? src[(size_t)c * TS + r] : 0.0;
  }
}

MmaShape mma_shape(int R, int C, int vn) {
  MmaShape s;
  s.mt = (R + 7) / 8;
  s.kt4 = (((C + 3) / 4) + 3) & ~3;
  const int mn = s.mt * ((vn + 7) / 8);
  // column splits of whole 4-step groups: fewest (rounds of units) x (latency + k-steps)
  constexpr int kLat = 24, kRed = 24;
  const int g = s.kt4 / 4;
  long long best = -1;
  s.ks = 1; s.kper = s.kt4;
  for (int ks = 1; ks <= 8 && ks <= g; ++ks) {
    if (ks > 1 && mn * ks > kRedUnits) break;
    const int kper = ((g + ks - 1) / ks) * 4;
    const int used = (s.kt4 + kper - 1) / kper;
    if (used != ks) continue;
    const long long cost = (long long)((mn * ks + MW - 1) / MW) * (kLat + kper) + (ks > 1 ? kRed : 0);
    if (best < 0 || cost < best) { best = cost; s.ks = ks; s.kper = kper; }
  }
  return s;
}

bool sub_mma_enabled() {
  static const bool off = [] {
    const char* e = getenv("HPSB_NO_SUB_MMA");
    return e && e[0] == '1';
  }();
  return !off;
}

void fill_args(const Ops& ops, const Workspace& ws, int k, SubArgs& a) {
  const Plan& P = *ops.plan;
  static const int fold = [] {
    const char* e = getenv("HPSB_NO_SUB_FOLD");
    return e && e[0] == '1' ? 0 : 1;
  }();
  a.fold = fold;
  a.nf = P.depth - P.dF;
  a.dF = P.dF;
  a.k = k;
  int hcap = 0, rcap = 0;
  for (int e = 0; e < a.nf; ++e) {
    const int d = P.dF + e;
    const Level& lv = P.lv[d];
    const LevelOps& lo = ops.lo[d];
    FLevel& L = a.lv[e];
    L.Up = lo.Up; L.S = lo.S;
    L.i1a = lv.i1a; L.i3a = lv.i3a; L.i2b = lv.i2b; L.i3b = lv.i3b; L.j3 = lv.j3; L.gidx = lv.gidx_bnd;
    L.n3 = lv.n3; L.n12 = lv.n12; L.n1a = lv.n1a; L.nbc = lv.nbc;
    L.W3 = ws.W3[d];
    L.W3_k = (long long)lv.c * lv.n3;
    const int npn = 1 << e;
    hcap = std::max(hcap, npn * lv.n12);  // children's fluxes of level e are level e+1's
    rcap = std::max(rcap, npn * ((lv.n3 + 1) & ~1));
  }
  a.hcap = (hcap + 1) & ~1;  // even: the r3 block after the two flux blocks starts 16-byte aligned
  a.rcap = rcap;
  if (P.sub_local) {
    a.slots = P.sub_slots;
    for (int e = 0; e <= a.nf; ++e) a.slot_off[e] = P.sub_slot_off[e];
    for (int e = 0; e < a.nf; ++e) a.j3_base[e] = P.sub_j3_base[e];
    a.nslots = P.sub_nslots;
    a.gidx_root = P.lv[P.dF].gidx_bnd;
  }
  if (P.dF > 0 && P.dF < P.depth) {
    a.H_dF = ws.H[P.dF];
    a.H_k = (long long)P.lv[P.dF].c * P.lv[P.dF].n12;
  }
}

// every fused level holds one (shared) operator tile: row pairs never straddle nodes
bool shared_sub(const SubArgs& a) {
  static const bool off = [] {
    const char* e = getenv("HPSB_NO_SUB_SH");
    return e && e[0] == '1';
  }();
  if (off) return false;
  for (int e = 0; e < a.nf; ++e)
    if (a.lv[e].Up.c != 1 || a.lv[e].S.c != 1) return false;
  return true;
}

// the tensor-core path: shared operators with fragment-ordered copies, one rhs, subtree-local slots
bool fill_mma(const Ops& ops, const SubArgs& a, MmaArgs& m) {
  const Plan& P = *ops.plan;
  if (!sub_mma_enabled() || a.k != 1 || !ops.shared_levels) return false;
  int tab = 0, hcap = 0, rcap = 0, xcap = 0;
  for (int e = 0; e < a.nf; ++e) {
    const LevelOps& lo = ops.lo[P.dF + e];
    if (!lo.UpF || !lo.SF) return false;
    const FLevel& L = a.lv[e];
    const int npn = 1 << e;
    MLevel& M = m.ml[e];
    M.UpF = lo.UpF; M.SF = lo.SF;
    M.up = mma_shape(L.Up.R, L.n3, npn);
    M.dn = mma_shape(L.n3, L.n12, npn);
    M.tab = tab;
    tab += 2 * L.n3 + L.n12;
    const int cs = e == a.nf - 1 ? (int)a.hs : L.nbc;
    hcap = std::max(hcap, std::max(2 * npn * cs, npn * L.n12));
    rcap = std::max(rcap, npn * mma_xs(L.n3));
    xcap = std::max(xcap, npn * mma_xs(L.n12));
  }
  m.tab_ints = tab;
  m.hcap = (hcap + 1) & ~1;
  m.rcap = (rcap + 1) & ~1;
  m.xcap = (xcap + 1) & ~1;
  m.sl_ints = P.sub_local ? (int)P.sub_slot_off[a.nf] : 0;
  return true;
}

template <class K, class... X>
int launch_sub(K kern, int nsub, int KM, int k, size_t smem, const SubArgs& a, cudaStream_t st, const X&... x) {
  if (smem > 227 * 1024) {
    set_error("subtree kernel needs %zu bytes of shared memory", smem);
    return -1;
  }
  static bool attr = false;  // per instantiation
  (void)attr;
  HPSB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  if (nsub <= 0) return 0;
  dim3 grid((unsigned)nsub, (unsigned)cdiv(k, KM));
  HPSB_CUDA(launch_pdl(kern, grid, dim3(NT), smem, st, a, x...));
  HPSB_LAUNCH_CHECK();
  return 0;
}

}  // namespace

// Smallest dF such that every fused level keeps one CTA's operator rows per
// level within kMaxRows and level dF still offers enough subtrees to spread
// over the SMs (or, for small trees, a reasonable share of the leaves).
int fuse_level(const Plan& P) {
  if (P.depth == 0) return 0;
  const long long cmin = std::min<long long>(2LL * kNumSMs, std::max<long long>(1, P.lv[P.depth - 1].c / 8));
  int best = P.depth;
  for (int d = P.depth - 1; d >= 0; --d) {
    if (P.depth - d > MAXF || P.lv[d].c < cmin) break;
    bool ok = true;
    for (int e = d; e < P.depth && ok; ++e) {
      const long long npn = 1LL << (e - d);
      ok = npn * P.lv[e].n12 <= kMaxRows && 2 * npn * P.lv[e].nbc <= 2 * kMaxRows;
    }
    if (!ok) break;
    best = d;
  }
  return best;
}

// fragment-ordered copies of the fused levels' shared operators for the
// tensor-core subtree kernels (not part of an operator dump: rebuilt on load)
int sub_mma_prepare(Ops& O, cudaStream_t st) {
  const Plan& P = *O.plan;
  if (!O.shared_levels || P.dF >= P.depth) return 0;
  for (int d = P.dF; d < P.depth; ++d) {
    LevelOps& lo = O.lo[d];
    if (!lo.Up.base || !lo.S.base || lo.Up.c != 1 || lo.S.c != 1) return 0;
    const int npn = 1 << (d - P.dF);
    const MmaShape u = mma_shape(lo.Up.R, lo.Up.C, npn), s = mma_shape(lo.S.R, lo.S.C, npn);
    const size_t nu = (size_t)u.mt * u.kt4 * 32, ns = (size_t)s.mt * s.kt4 * 32;
    double* p = nullptr;
    if (cudaMalloc(&p, (nu + ns) * 8) != cudaSuccess) { cudaGetLastError(); return 0; }  // SIMT kernels instead
    O.aux.push_back(p);
    k_frag<<<(unsigned)std::min<size_t>((nu + 255) / 256, 1184), 256, 0, st>>>(lo.Up.base, lo.Up.R, lo.Up.C, lo.Up.TS,
                                                                                u.mt, u.kt4, p);
    k_frag<<<(unsigned)std::min<size_t>((ns + 255) / 256, 1184), 256, 0, st>>>(lo.S.base, lo.S.R, lo.S.C, lo.S.TS,
                                                                                s.mt, s.kt4, p + nu);
    HPSB_LAUNCH_CHECK();
    lo.UpF = p;
    lo.SF = p + nu;
  }
  return 0;
}

int mb_subtree_up(const Ops& ops, const Workspace& ws, int k, const double* Hleaf, long long sh, long long hs,
                  int b0, int b1, cudaStream_t st);
int mb_subtree_down(const Ops& ops, const Workspace& ws, int k, bool has_w3, double* u, long long ld_u, int b0,
                    int b1, cudaStream_t st);

int subtree_up(const Ops& ops, const Workspace& ws, int k, const double* Hleaf, long long sh, long long hs,
               const double* jump, long long ld_jump, double inv_dt, int b0, int b1, cudaStream_t st) {
  const Plan& P = *ops.plan;
  if (P.dF >= P.depth) return 0;
  if (ops.shared_levels && k >= kSharedGemmRhs && !jump) {  // many rhs: member-blocked kernels
    const int rc = mb_subtree_up(ops, ws, k, Hleaf, sh, hs, b0, b1, st);
    if (rc != 1) return rc;
  }
  SubArgs a{};
  fill_args(ops, ws, k, a);
  a.b0 = b0;
  a.Hleaf = Hleaf; a.sh = sh; a.hs = hs;
  a.jump = jump; a.jump_k = ld_jump; a.inv_dt = inv_dt;
  const int KM = k == 1 ? 1 : 4;
  const bool shm = KM == 1 && shared_sub(a);
  if (shm) {
    MmaArgs m{};
    if (fill_mma(ops, a, m)) {
      size_t sm2 = (size_t)(2 * m.hcap + m.rcap + kRedMma) * 8 + (size_t)m.tab_ints * 4;
      return launch_sub(k_sub_up_mma, b1 - b0, 1, k, sm2, a, st, m);
    }
  }
  const size_t smem = (size_t)(KM * (2 * a.hcap + a.rcap) + red_doubles(KM, shm)) * 8;
  if (shm) return launch_sub(k_sub_up<1, true>, b1 - b0, 1, k, smem, a, st);
  if (KM == 1) return launch_sub(k_sub_up<1>, b1 - b0, 1, k, smem, a, st);
  return launch_sub(k_sub_up<4>, b1 - b0, 4, k, smem, a, st);
}

int subtree_down(const Ops& ops, const Workspace& ws, int k, bool has_w3, double* u, long long ld_u, int b0,
                 int b1, cudaStream_t st) {
  const Plan& P = *ops.plan;
  if (P.dF >= P.depth) return 0;
  if (ops.shared_levels && k >= kSharedGemmRhs) {
    const int rc = mb_subtree_down(ops, ws, k, has_w3, u, ld_u, b0, b1, st);
    if (rc != 1) return rc;
  }
  SubArgs a{};
  fill_args(ops, ws, k, a);
  a.b0 = b0;
  a.u = u; a.u_k = ld_u; a.has_w3 = has_w3 ? 1 : 0;
  const int KM = k == 1 ? 1 : 4;
  int xcap = 0;
  for (int e = 0; e < a.nf; ++e) xcap = std::max(xcap, (1 << e) * ((a.lv[e].n12 + 1) & ~1));
  const bool shm = KM == 1 && shared_sub(a);
  if (P.sub_local && shm) {
    MmaArgs m{};
    if (fill_mma(ops, a, m)) {
      const size_t sm2 = (size_t)(kRedMma + m.xcap + ((a.nslots + 1) & ~1)) * 8 + (size_t)m.sl_ints * 4;
      if (sm2 <= 200 * 1024) return launch_sub(k_sub_down_mma, b1 - b0, 1, k, sm2, a, st, m);
    }
  }
  if (P.sub_local) {
    const size_t smem = (size_t)(KM * xcap + red_doubles(KM, shm) + ((KM * a.nslots + 1) & ~1)) * 8;
    if (smem <= 200 * 1024) {
      if (shm) return launch_sub(k_sub_down_local<1, true>, b1 - b0, 1, k, smem, a, st);
      if (KM == 1) return launch_sub(k_sub_down_local<1>, b1 - b0, 1, k, smem, a, st);
      return launch_sub(k_sub_down_local<4>, b1 - b0, 4, k, smem, a, st);
    }
  }
  const size_t smem = (size_t)(KM * xcap + red_doubles(KM, shm)) * 8;
  if (shm) return launch_sub(k_sub_down<1, true>, b1 - b0, 1, k, smem, a, st);
  if (KM == 1) return launch_sub(k_sub_down<1>, b1 - b0, 1, k, smem, a, st);
  return launch_sub(k_sub_down<4>, b1 - b0, 4, k, smem, a, st);
}

}  // namespace hpsb
