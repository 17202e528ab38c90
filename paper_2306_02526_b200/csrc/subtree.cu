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

template <class K>
int launch_sub(K kern, int nsub, int KM, int k, size_t smem, const SubArgs& a, cudaStream_t st) {
  if (smem > 227 * 1024) {
    set_error("subtree kernel needs %zu bytes of shared memory", smem);
    return -1;
  }
  static bool attr = false;  // per instantiation
  (void)attr;
  HPSB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  if (nsub <= 0) return 0;
  dim3 grid((unsigned)nsub, (unsigned)cdiv(k, KM));
  HPSB_CUDA(launch_pdl(kern, grid, dim3(NT), smem, st, a));
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
