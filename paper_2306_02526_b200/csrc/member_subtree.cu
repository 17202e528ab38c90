// Member-blocked fused subtree kernels: the deep levels of a many-rhs solve
// on shared (constant-coefficient) operators, e.g. the C5 ensemble.
//
// The level-by-level GEMM over (node, rhs) rows (dedup.cu) writes every deep
// level's fluxes and w3 to HBM and reads the children's back: at k = 64 and
// the deepest level of C2's tree that is ~0.9 GB per level for ~1.4 GFLOP.
// Here one CTA owns one level-dF subtree for a block of KM members and walks
// all fused levels in one launch (solver.py:243-268), the fluxes of the
// subtree (up) and its interface values (down) held in shared memory:
//   up   level e (deepest first): r3 = hb[i3b] - ha[i3a] for the subtree's
//        2^e nodes x KM members, [w3; h - base] = [X33^-1; Tstack X33^-1] r3,
//        w3 to the workspace, h to shared memory (level dF: to the workspace);
//   down level e (root first): the boundary values gathered from the
//        subtree-local slots, u3 = S u_bnd + w3, back into the slots and u.
// Every level apply is one small GEMM Y (R x Q) = Op (R x C) X (C x Q) over
// Q = 2^e KM (node, member) columns: register tiles of TR rows x 8 columns
// (8 columns share each operator load, TR rows each x load), split over the
// columns C in G thread groups when the tiles are few; the group partials
// meet in shared memory in group order (bitwise reproducible).  The operator
// is the level's one row-major copy (L1 / L2 resident: every CTA reads it).
#include <stdlib.h>

#include "hps_plan.cuh"

namespace hpsb {

namespace {

constexpr int MB_NT = 256;
constexpr int MB_TQ = 8;      // (node, member) columns per register tile
constexpr int MB_MAXF = 10;

struct MbLevel {
  const double* op;  // up: (n3 + n12) x ld (root level: n3 x ld); down: n3 x ld
  int ld;
  int R, C;          // operator rows / columns
  int TR, G;         // register-tile rows, column groups
  const int *i1a, *i3a, *i2b, *i3b, *j3;
  int n3, n12, n1a, nbc;
  double* W3; long long W3_k;
};

struct MbArgs {
  int nf, dF, k;
  MbLevel up[MB_MAXF], dn[MB_MAXF];
  const double* Hleaf; long long sh, hs;  // leaf fluxes: member stride, per-leaf stride
  double* H_dF; long long H_k;            // level-dF fluxes (dF > 0)
  double* u; long long u_k; int has_w3;
  const int* slots; long long slot_off[MB_MAXF + 1]; int j3_base[MB_MAXF]; int nslots;
  const int* gidx_root;
  int b0;
  int hcap, xcap_up, xcap_dn;             // shared-memory carve (doubles per member)
};

// X layout: column c of the (node, member) matrix holds Q / 8 tiles of 8
// values; the four 16-byte pairs of a tile are stored pair-major so that the
// threads of a warp (consecutive tiles) read consecutive 16-byte words
// (conflict-free), and rows of the layout are padded by 2 doubles (gathers
// that write along c spread over the banks).
__device__ __forceinline__ int mb_xstride(int Q) { return Q + 2; }
__device__ __forceinline__ int mb_xpos(int c, int q, int Q) {
  const int tq = Q / MB_TQ;
  return c * mb_xstride(Q) + (((q & 7) >> 1) * tq + (q >> 3)) * 2 + (q & 1);
}

// Y = Op X over the R x Q outputs (X: C x Q in the mb_xpos layout, Q a multiple of MB_TQ),
// out(r, q, y) for r < R, q < Q; red: G x tiles x TR x MB_TQ doubles
template <int TR, class Out>
__device__ __forceinline__ void mb_apply_tr(const MbLevel& L, const double* __restrict__ X, int Q, double* red,
                                            Out out) {
  const int tq = Q / MB_TQ, ntile = tq * ((L.R + TR - 1) / TR), G = L.G;
  const int KC = (L.C + G - 1) / G;
  for (int t = threadIdx.x; t < ntile * G; t += MB_NT) {
    const int tile = t % ntile, g = t / ntile;
    const int q0 = (tile % tq) * MB_TQ, r0 = (tile / tq) * TR;
    const int c0 = g * KC, c1 = min(L.C, c0 + KC);
    double acc[TR][MB_TQ];
#pragma unroll
    for (int i = 0; i < TR; ++i)
#pragma unroll
      for (int j = 0; j < MB_TQ; ++j) acc[i][j] = 0.0;
    const double* op[TR];
#pragma unroll
    for (int i = 0; i < TR; ++i) op[i] = L.op + (size_t)min(r0 + i, L.R - 1) * L.ld;
    const int tile_q = tile % tq, xs2 = mb_xstride(Q) / 2;
    const double2* xp = reinterpret_cast<const double2*>(X) + tile_q;
#pragma unroll 2
    for (int c = c0; c < c1; ++c) {
      double o[TR];
#pragma unroll
      for (int i = 0; i < TR; ++i) o[i] = __ldg(op[i] + c);
      double x[MB_TQ];
#pragma unroll
      for (int j = 0; j < MB_TQ / 2; ++j) {
        const double2 v = xp[(size_t)c * xs2 + j * tq];
        x[2 * j] = v.x;
        x[2 * j + 1] = v.y;
      }
#pragma unroll
      for (int i = 0; i < TR; ++i)
#pragma unroll
        for (int j = 0; j < MB_TQ; ++j) acc[i][j] = fma(o[i], x[j], acc[i][j]);
    }
    if (G == 1) {
#pragma unroll
      for (int i = 0; i < TR; ++i)
        if (r0 + i < L.R)
#pragma unroll
          for (int j = 0; j < MB_TQ; ++j) out(r0 + i, q0 + j, acc[i][j]);
    } else {
      double* rp = red + ((size_t)g * ntile + tile) * TR * MB_TQ;
#pragma unroll
      for (int i = 0; i < TR; ++i)
#pragma unroll
        for (int j = 0; j < MB_TQ; ++j) rp[i * MB_TQ + j] = acc[i][j];
    }
  }
  if (G > 1) {
    __syncthreads();
    for (int o = threadIdx.x; o < ntile * TR * MB_TQ; o += MB_NT) {
      const int tile = o / (TR * MB_TQ), w = o % (TR * MB_TQ), i = w / MB_TQ, j = w % MB_TQ;
      const int q0 = (tile % tq) * MB_TQ, r0 = (tile / tq) * TR;
      if (r0 + i >= L.R) continue;
      double y = 0.0;
      for (int g = 0; g < G; ++g) y += red[((size_t)g * ntile + tile) * TR * MB_TQ + w];
      out(r0 + i, q0 + j, y);
    }
  }
}

template <class Out>
__device__ __forceinline__ void mb_apply(const MbLevel& L, const double* X, int Q, double* red, Out out) {
  if (L.TR == 4) mb_apply_tr<4>(L, X, Q, red, out);
  else if (L.TR == 2) mb_apply_tr<2>(L, X, Q, red, out);
  else mb_apply_tr<1>(L, X, Q, red, out);
}

template <int KM>
__global__ void __launch_bounds__(MB_NT, 2) k_mb_up(MbArgs a) {
  extern __shared__ double sm[];
  double* Hs = sm;                   // children's fluxes [child][KM][nbc]
  double* Hn = Hs + KM * a.hcap;     // this level's fluxes [node][KM][n12]
  double* X = Hn + KM * a.hcap;      // r3 [col][node * KM + member]
  double* red = X + KM * a.xcap_up;  // split partials
  const int b = a.b0 + blockIdx.x, kg0 = blockIdx.y * KM;
  pdl_trigger();
  pdl_wait();
  for (int e = a.nf - 1; e >= 0; --e) {
    const MbLevel& L = a.up[e];
    const int npn = 1 << e, node0 = b * npn, n3 = L.n3, n12 = L.n12, nbc = L.nbc, Q0 = npn * KM;
    const int Q = (Q0 + MB_TQ - 1) & ~(MB_TQ - 1);  // padded (node, member) columns
    const bool leafc = e == a.nf - 1;
    auto child = [&](int j, int m, int which) -> const double* {  // which: 0 = alpha, 1 = beta
      if (leafc) return a.Hleaf + (long long)min(kg0 + m, a.k - 1) * a.sh + (2LL * (node0 + j) + which) * a.hs;
      return Hs + ((2 * j + which) * KM + m) * nbc;
    };
    for (int idx = threadIdx.x; idx < n3 * Q; idx += MB_NT) {  // c fastest: coalesced leaf-flux reads
      const int c = idx % n3, q = idx / n3, j = q / KM, m = q % KM;
      X[mb_xpos(c, q, Q)] = q < Q0 ? child(j, m, 1)[L.i3b[c]] - child(j, m, 0)[L.i3a[c]] : 0.0;
    }
    __syncthreads();
    mb_apply(L, X, Q, red, [&](int r, int q, double y) {
      if (q >= Q0) return;
      const int j = q / KM, m = q % KM, kg = kg0 + m;
      if (r < n3) {
        if (kg < a.k) L.W3[kg * L.W3_k + (long long)(node0 + j) * n3 + r] = y;
        return;
      }
      const int rr = r - n3;
      const double base = rr < L.n1a ? child(j, m, 0)[L.i1a[rr]] : child(j, m, 1)[L.i2b[rr - L.n1a]];
      const double h = base + y;
      Hn[(j * KM + m) * n12 + rr] = h;
      if (e == 0 && kg < a.k) a.H_dF[kg * a.H_k + (long long)(node0 + j) * n12 + rr] = h;
    });
    __syncthreads();
    if (a.dF + e == 0) break;  // the root's outer flux is never consumed
    double* t = Hs; Hs = Hn; Hn = t;
  }
}

template <int KM>
__global__ void __launch_bounds__(MB_NT, 2) k_mb_down(MbArgs a) {
  extern __shared__ double sm[];
  double* uloc = sm;                          // [KM][nslots]
  double* X = uloc + ((KM * a.nslots + 1) & ~1);  // [col][node * KM + member]
  double* red = X + KM * a.xcap_dn;
  const int b = a.b0 + blockIdx.x, kg0 = blockIdx.y * KM, ns = a.nslots;
  pdl_trigger();
  pdl_wait();
  {
    const int n12 = a.dn[0].n12;
    for (int idx = threadIdx.x; idx < KM * n12; idx += MB_NT) {
      const int m = idx / n12, col = idx % n12, kg = min(kg0 + m, a.k - 1);
      uloc[m * ns + col] = a.u[kg * a.u_k + a.gidx_root[(long long)b * n12 + col]];
    }
  }
  for (int e = 0; e < a.nf; ++e) {
    const MbLevel& L = a.dn[e];
    const int npn = 1 << e, node0 = b * npn, n3 = L.n3, n12 = L.n12, jb = a.j3_base[e], Q0 = npn * KM;
    const int Q = (Q0 + MB_TQ - 1) & ~(MB_TQ - 1);
    const int* sl = a.slots + a.slot_off[e];
    __syncthreads();
    for (int idx = threadIdx.x; idx < n12 * Q; idx += MB_NT) {
      const int c = idx % n12, q = idx / n12, j = q / KM, m = q % KM;
      X[mb_xpos(c, q, Q)] = q < Q0 ? uloc[m * ns + sl[j * n12 + c]] : 0.0;
    }
    __syncthreads();
    mb_apply(L, X, Q, red, [&](int r, int q, double y) {
      if (q >= Q0) return;
      const int j = q / KM, m = q % KM, kg = kg0 + m;
      const long long nd = (long long)(node0 + j) * n3 + r;
      if (a.has_w3) y = y + L.W3[min(kg, a.k - 1) * L.W3_k + nd];
      uloc[m * ns + jb + j * n3 + r] = y;
      if (kg < a.k) a.u[kg * a.u_k + L.j3[nd]] = y;
    });
  }
}

// register-tile rows and column groups for an R x Q output over C columns:
// enough (tile, group) units for the CTA, at least 8 columns per group
void mb_shape(MbLevel& L, int Q) {
  const int tq = Q / MB_TQ;
  L.TR = 4;
  if (tq * ((L.R + 3) / 4) < MB_NT / 2) L.TR = 2;
  if (tq * ((L.R + 1) / 2) < MB_NT / 2) L.TR = 1;
  const int tiles = tq * ((L.R + L.TR - 1) / L.TR);
  L.G = 1;
  while (tiles * L.G * 2 <= MB_NT && L.C / (L.G * 2) >= 8) L.G *= 2;
}

size_t mb_red_doubles(const MbLevel& L, int Q) {
  if (L.G == 1) return 0;
  return (size_t)L.G * (Q / MB_TQ) * ((L.R + L.TR - 1) / L.TR) * L.TR * MB_TQ;
}

constexpr int MB_KM = 4;

bool mb_fill(const Ops& ops, const Workspace& ws, int k, MbArgs& a, size_t& red) {
  const Plan& P = *ops.plan;
  a.nf = P.depth - P.dF;
  if (a.nf <= 0 || a.nf > MB_MAXF || !ops.shared_levels) return false;
  a.dF = P.dF;
  a.k = k;
  int hcap = 0, xu = 0, xd = 0;
  red = 0;
  for (int e = 0; e < a.nf; ++e) {
    const int d = P.dF + e, npn = 1 << e, Q = (npn * MB_KM + MB_TQ - 1) & ~(MB_TQ - 1);
    const Level& lv = P.lv[d];
    const LevelOps& lo = ops.lo[d];
    if (!lo.Ush || !lo.Ssh) return false;
    for (MbLevel* L : {&a.up[e], &a.dn[e]}) {
      L->i1a = lv.i1a; L->i3a = lv.i3a; L->i2b = lv.i2b; L->i3b = lv.i3b; L->j3 = lv.j3;
      L->n3 = lv.n3; L->n12 = lv.n12; L->n1a = lv.n1a; L->nbc = lv.nbc;
      L->W3 = ws.W3[d];
      L->W3_k = (long long)lv.c * lv.n3;
    }
    a.up[e].op = lo.Ush; a.up[e].ld = lv.ld3; a.up[e].R = lv.n3 + (d > 0 ? lv.n12 : 0); a.up[e].C = lv.n3;
    a.dn[e].op = lo.Ssh; a.dn[e].ld = lv.ld12; a.dn[e].R = lv.n3; a.dn[e].C = lv.n12;
    mb_shape(a.up[e], Q);
    mb_shape(a.dn[e], Q);
    red = std::max({red, mb_red_doubles(a.up[e], Q), mb_red_doubles(a.dn[e], Q)});
    hcap = std::max(hcap, npn * lv.n12);
    xu = std::max(xu, lv.n3 * (Q + 2));   // mb_xstride
    xd = std::max(xd, lv.n12 * (Q + 2));
  }
  a.hcap = (hcap + 1) & ~1;
  a.xcap_up = (xu + MB_KM * 2 - 1) / MB_KM;  // doubles per member (the carve multiplies by KM)
  a.xcap_dn = (xd + MB_KM * 2 - 1) / MB_KM;
  a.xcap_up = (a.xcap_up + 1) & ~1;
  a.xcap_dn = (a.xcap_dn + 1) & ~1;
  if (P.sub_local) {
    a.slots = P.sub_slots;
    for (int e = 0; e <= a.nf; ++e) a.slot_off[e] = P.sub_slot_off[e];
    for (int e = 0; e < a.nf; ++e) a.j3_base[e] = P.sub_j3_base[e];
    a.nslots = P.sub_nslots;
    a.gidx_root = P.lv[P.dF].gidx_bnd;
  }
  if (P.dF > 0) {
    a.H_dF = ws.H[P.dF];
    a.H_k = (long long)P.lv[P.dF].c * P.lv[P.dF].n12;
  }
  return true;
}

template <class K>
int mb_launch(K kern, int nsub, int k, size_t smem, const MbArgs& a, cudaStream_t st) {
  HPSB_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  if (nsub <= 0) return 0;
  dim3 grid((unsigned)nsub, (unsigned)cdiv(k, MB_KM));
  HPSB_CUDA(launch_pdl(kern, grid, dim3(MB_NT), smem, st, a));
  HPSB_LAUNCH_CHECK();
  return 0;
}

}  // namespace

// Off by default: measured slower than the level GEMMs on C5 (k_mb_up 2.16 ms +
// k_mb_down 1.79 ms against ~3.6 ms of deep-level GEMMs, solve 9.8 vs 9.4 ms):
// at 2 CTAs / SM the level-synchronous CTAs sit in barriers and L2 latency
// (ncu: 12-25 % warps active).  HPSB_MB_SUB=1 enables them.
bool mb_enabled() {
  static const bool on = [] {
    const char* e = getenv("HPSB_MB_SUB");
    return e && e[0] == '1';
  }();
  return on;
}

// returns 1 when not applicable (the caller runs the level GEMMs instead)
int mb_subtree_up(const Ops& ops, const Workspace& ws, int k, const double* Hleaf, long long sh, long long hs,
                  int b0, int b1, cudaStream_t st) {
  MbArgs a{};
  size_t red = 0;
  if (!mb_enabled() || !mb_fill(ops, ws, k, a, red)) return 1;
  a.b0 = b0;
  a.Hleaf = Hleaf; a.sh = sh; a.hs = hs;
  const size_t smem = ((size_t)MB_KM * (2 * a.hcap + a.xcap_up) + red) * 8;
  if (smem > 227 * 1024) return 1;
  return mb_launch(k_mb_up<MB_KM>, b1 - b0, k, smem, a, st);
}

int mb_subtree_down(const Ops& ops, const Workspace& ws, int k, bool has_w3, double* u, long long ld_u, int b0,
                    int b1, cudaStream_t st) {
  const Plan& P = *ops.plan;
  MbArgs a{};
  size_t red = 0;
  if (!mb_enabled() || !P.sub_local || !mb_fill(ops, ws, k, a, red)) return 1;
  a.b0 = b0;
  a.u = u; a.u_k = ld_u; a.has_w3 = has_w3 ? 1 : 0;
  const size_t smem = ((size_t)((MB_KM * a.nslots + 1) & ~1) + (size_t)MB_KM * a.xcap_dn + red) * 8;
  if (smem > 227 * 1024) return 1;
  return mb_launch(k_mb_down<MB_KM>, b1 - b0, k, smem, a, st);
}

// whether the fused member-blocked kernels take a k-rhs solve's deep levels
bool mb_applies(const Ops& ops, int k) {
  const Plan& P = *ops.plan;
  MbArgs a{};
  size_t red = 0;
  Workspace ws;
  ws.W3.assign(P.depth, nullptr);
  ws.H.assign(P.depth, nullptr);
  if (!mb_enabled() || !P.sub_local || !mb_fill(ops, ws, k, a, red)) return false;
  const size_t up = ((size_t)MB_KM * (2 * a.hcap + a.xcap_up) + red) * 8;
  const size_t dn = ((size_t)((MB_KM * a.nslots + 1) & ~1) + (size_t)MB_KM * a.xcap_dn + red) * 8;
  return up <= 227 * 1024 && dn <= 227 * 1024;
}

}  // namespace hpsb
