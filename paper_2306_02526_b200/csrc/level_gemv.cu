// Level-batched streaming GEMV for the HPS solve (sm_100a, FP64, HBM-bound).
//
// One launch applies one operator family of one tree level to every node:
//   UP  : r3 = hb[i3b] - ha[i3a] [- jump/dt]                    (solver.py:246-250)
//         w3 = X33^-1 r3, h = [ha[i1a]; hb[i2b]] + (Tstack X33^-1) r3
//         (solver.py:251-254) -- one stacked operator, one pass
//   DOWN: u[j3] = S u[gidx_bnd] (+ w3)                          (solver.py:261-268)
//   LEAF: y    = M x (+ add)   per leaf (variable-coefficient leaves,
//                               solver.py:225-227 and 269-272)
//
// Operators live in the "panel" layout (hps_plan.cuh): the level's row space
// (c nodes x R rows) is cut into 512-row tiles stored column-major.  CTA =
// one tile x one column chunk: it stages the chunk of every touched node's
// input vector in shared memory (mode-specific gather fused in), then each
// of its 256 threads owns two adjacent rows and walks the columns issuing U
// independent 16-byte streaming loads (ld.global.cs) before consuming them,
// so every CTA keeps U*4 KB of one contiguous HBM region in flight.
// Outputs are plain sequential sums.  When a level has too few tiles to fill
// the machine (top levels: 1-64 huge nodes) the columns are split across
// CTAs; partial sums go to the workspace and the last CTA of a tile (counted
// with a semaphore, reset for the next launch) adds them in chunk order, so
// results stay bitwise reproducible.
#include "hps_plan.cuh"
#include "stream.cuh"

namespace hpsb {

// Tile height: 512 rows (256 threads, two rows each) unless that leaves too
// few tiles to spread over the SMs, then down to 64 rows (one warp).  The
// total thread count of a launch is (rows/2) x (column splits), whatever the
// tile height; the height only sets how evenly the tiles land on the SMs.
Panel make_panel(int c, int R, int C, int parts) {
  Panel p;
  p.parts = std::max(1, parts);
  p.c = c / p.parts; p.R = R; p.C = C;
  const long long rows = (long long)p.c * R;
  p.TR = kPanelRows;
  while (p.TR > 64 && cdiv(rows, p.TR) * p.parts < 2LL * kNumSMs) p.TR /= 2;
  p.TS = p.TR;
  p.ntiles = (int)cdiv(rows, p.TR);
  return p;
}

Panel make_panel_nodes(int c, int R, int C, int npn) {
  Panel p;
  p.c = c; p.R = R; p.C = C;
  p.TR = npn * R;
  p.TS = (p.TR + 1) & ~1;
  p.ntiles = (int)cdiv(c, npn);
  return p;
}

namespace {

constexpr int NT = 256;
// threads per launch: ~1K threads per SM, each with up to 2 batches of U=8
// 16-byte loads in flight, cover HBM latency under full load
constexpr int kTargetThreads = kNumSMs * 1024;
constexpr size_t kMaxStage = 64 * 1024;
constexpr int kMaxSplitDefault = 32;  // bounds the serial partial-sum tail of the last CTA
int max_split() {
  static const int v = [] {
    const char* e = getenv("HPSB_MAXSPLIT");
    return e ? std::max(1, atoi(e)) : kMaxSplitDefault;
  }();
  return v;
}

}  // namespace

PanelSplit panel_split(const Panel& pn, int k, int vnodes) {
  PanelSplit s;
  s.KM = k == 1 ? 1 : k <= 4 ? 4 : k <= 8 ? 8 : 16;
  s.kgroups = (int)cdiv(k, s.KM);
  s.nodes = (int)std::min<long long>(pn.c, (pn.TR - 1) / pn.R + 2);
  long long base = (long long)pn.ntiles * vnodes * s.kgroups;
  int ns = (int)std::max<long long>(1, cdiv(kTargetThreads, base * (pn.TR / 2)));
  ns = std::min(ns, std::max(1, pn.C / 16));
  ns = std::min(ns, max_split());
  int CK = (int)cdiv(pn.C, ns);
  auto xs = [](int ck) { return ck | 1; };
  long long cap = (long long)(kMaxStage / 8) / ((long long)s.nodes * s.KM);
  if (xs(CK) > cap) CK = (int)std::max<long long>(1, (cap - 1) & ~1LL);
  s.CK = CK;
  s.nsplit = (int)cdiv(pn.C, CK);
  s.XS = xs(CK);
  s.smem = (size_t)s.nodes * s.KM * s.XS * 8;
  if (s.nsplit > 1) {
    s.part_doubles = (size_t)s.kgroups * s.KM * s.nsplit * pn.ntiles * pn.TR * vnodes;
    s.counters = pn.ntiles * vnodes * s.kgroups;
  }
  return s;
}

namespace {

template <int MODE>
__device__ __forceinline__ double xval(const GemvArgs& a, int node, int kg, int col) {
  if (MODE == GEMV_UP) {
    const double* Ha = a.Hc + kg * a.Hc_k + (long long)(2 * node) * a.Hc_s;
    const double* Hb = Ha + a.Hc_s;
    double v = Hb[a.i3b[col]] - Ha[a.i3a[col]];
    if (a.jump) v = v - a.inv_dt * a.jump[kg * a.jump_k + a.j3[(long long)node * a.n3 + col]];
    return v;
  } else if (MODE == GEMV_DOWN) {
    return a.u[kg * a.u_k + a.gidx[(long long)node * a.n12 + col]];
  } else {
    return a.xin[kg * a.xin_k + (long long)node * a.xin_s + col];
  }
}

template <int MODE>
__device__ __forceinline__ void epilogue(const GemvArgs& a, int node, int r, int kg, double y) {
  if (MODE == GEMV_UP) {
    if (r < a.n3) {
      a.W3[kg * a.W3_k + (long long)node * a.n3 + r] = y;
    } else {
      r -= a.n3;
      const double* Ha = a.Hc + kg * a.Hc_k + (long long)(2 * node) * a.Hc_s;
      const double* Hb = Ha + a.Hc_s;
      double base = (r < a.n1a) ? Ha[a.i1a[r]] : Hb[a.i2b[r - a.n1a]];
      a.Hout[kg * a.Hout_k + (long long)node * a.n12 + r] = base + y;
    }
  } else if (MODE == GEMV_DOWN) {
    double v = y;
    if (a.W3) v = v + a.W3[kg * a.W3_k + (long long)node * a.n3 + r];
    const long long nr = (long long)node * a.n3 + r;
    if (a.yout) a.yout[kg * a.yout_k + nr] = v;   // staging output (row-sharded top levels)
    else a.u[kg * a.u_k + a.j3[nr]] = v;
  } else {
    double v = y;
    if (a.yadd) v = v + a.yadd[kg * a.yadd_k + (long long)node * a.yadd_s + r];
    a.yout[kg * a.yout_k + (long long)node * a.yout_s + r] = v;
  }
}

template <int MODE, int KM, int U>
__global__ void __launch_bounds__(NT) k_panel(GemvArgs a, Panel pn, PanelSplit sp) {
  extern __shared__ double xs[];
  __shared__ unsigned s_last;
  const int tid = threadIdx.x;
  const int vt = blockIdx.x / sp.nsplit, split = blockIdx.x % sp.nsplit;
  // shared operator: virtual tile vt = (node, tile of the one-node panel)
  const int vnode = a.shared ? vt / pn.ntiles : 0;
  const int tile = a.shared ? vt % pn.ntiles : vt;
  const int kg0 = blockIdx.y * KM;
  const int R = pn.R, TR = pn.TR;
  const long long P = (long long)pn.c * R;
  const long long p0 = (long long)tile * TR + a.prow0;
  const int n0 = (int)(p0 / R);
  const int nn = (int)((std::min(P, p0 + TR) - 1) / R) - n0 + 1;
  const int c0 = split * sp.CK, cw = min(sp.CK, pn.C - c0);
  const int XS = sp.XS;
  pdl_trigger();

  const long long pa = p0 + 2 * tid;
  const int cs = TR / 2;
  const double2* M = reinterpret_cast<const double2*>(pn.base + (size_t)tile * pn.C * TR + (size_t)c0 * TR) + tid;
  // the first batch of the operator stream does not depend on x: issue it
  // before the gather so the two latencies overlap
  double2 A[U];
  if (cw >= U) load_batch<U>(A, M, cs, 0);

  pdl_wait();  // vectors below are produced by the previous kernel of the chain

  // stage x chunks of the touched nodes: xs[(node*KM + kk)*XS + col]
  for (int e = tid; e < nn * KM * cw; e += blockDim.x) {
    const int col = e % cw, t2 = e / cw, kk = t2 % KM, nl = t2 / KM, kg = kg0 + kk;
    xs[(nl * KM + kk) * XS + col] = kg < a.k ? xval<MODE>(a, a.shared ? vnode : n0 + nl, kg, c0 + col) : 0.0;
  }
  __syncthreads();

  const int na = (int)(std::min(pa, P - 1) / R) - n0;
  const int nb = (int)(std::min(pa + 1, P - 1) / R) - n0;
  double acc0[KM], acc1[KM];
#pragma unroll
  for (int kk = 0; kk < KM; ++kk) { acc0[kk] = 0.0; acc1[kk] = 0.0; }
  stream_cols<KM, U>(A, M, cs, 0, cw, xs, na * KM * XS, nb * KM * XS, XS, acc0, acc1);

  if (sp.nsplit > 1) {
    const long long Pp = (long long)pn.ntiles * TR * (a.shared ? a.shared : 1);
    const long long pv = pa - a.prow0 + (long long)vnode * pn.ntiles * TR;  // row in the (virtual) row space of the view
    const size_t cidx = ((size_t)vnode * pn.ntiles + tile) * gridDim.y + blockIdx.y;
    double* part = a.part + ((long long)blockIdx.y * KM * sp.nsplit) * Pp;
#pragma unroll
    for (int kk = 0; kk < KM; ++kk) {
      double2 v = make_double2(acc0[kk], acc1[kk]);
      *reinterpret_cast<double2*>(part + ((long long)kk * sp.nsplit + split) * Pp + pv) = v;
    }
    __syncthreads();  // barrier + one thread's acq_rel atomic (hps_common.cuh)
    if (tid == 0) s_last = atom_add_acq_rel(a.cnt + cidx, 1u) == (unsigned)sp.nsplit - 1;
    __syncthreads();
    if (!s_last) return;
#pragma unroll
    for (int kk = 0; kk < KM; ++kk) {
      double s0 = 0.0, s1 = 0.0;
#pragma unroll 8
      for (int s = 0; s < sp.nsplit; ++s) {
        double2 v = __ldcg(reinterpret_cast<const double2*>(part + ((long long)kk * sp.nsplit + s) * Pp + pv));
        s0 += v.x;
        s1 += v.y;
      }
      acc0[kk] = s0;
      acc1[kk] = s1;
    }
    if (tid == 0) a.cnt[cidx] = 0u;
  }
#pragma unroll
  for (int kk = 0; kk < KM; ++kk) {
    const int kg = kg0 + kk;
    if (kg >= a.k) continue;
    const int ra = (int)(pa - (long long)(n0 + na) * R), rb = (int)(pa + 1 - (long long)(n0 + nb) * R);
    if (pa < P) epilogue<MODE>(a, a.shared ? vnode : n0 + na, ra, kg, acc0[kk]);
    if (pa + 1 < P) epilogue<MODE>(a, a.shared ? vnode : n0 + nb, rb, kg, acc1[kk]);
  }
}

// Shared-layout levels with many nodes (the mid levels of the tree): the
// level's single operator (one-node panel, TR-row tiles) is applied to NB
// nodes per CTA.  The CTA stages the NB nodes' whole input vectors in shared
// memory (one gather pass), its 256 threads are G = 256/(TR/2) column groups
// of TR/2 threads (two rows each) streaming K/G columns of the tile from L2,
// the groups' partial sums meet in shared memory (in group order: bitwise
// reproducible) and the TR x NB outputs are spread over all threads for the
// epilogue.  No split-K through global memory, no semaphores: the latency
// chain is gather -> short stream -> reduce -> scatter.
constexpr int kVnThreads = 256;

template <int MODE, int NB, int U>
__global__ void __launch_bounds__(kVnThreads) k_vn(GemvArgs a, Panel pn, int XS) {
  extern __shared__ double sm[];
  double* xs = sm;                    // [NB][XS] input slots
  double* red = sm + NB * XS;         // [G][NB][TR] partial sums
  const int TR = pn.TR, C = pn.C, P2 = TR / 2, G = kVnThreads / P2;
  const int tile = blockIdx.x, tid = threadIdx.x, g = tid / P2, q = tid % P2;
  const int slot0 = blockIdx.y * NB, nslots = a.shared * a.k;
  const int CKg = (C + G - 1) / G, c0 = min(C, g * CKg), c1 = min(C, c0 + CKg);
  const double2* M = reinterpret_cast<const double2*>(pn.base + (size_t)tile * C * TR) + q;
  pdl_trigger();
  double2 A[U];
  if (c1 - c0 >= U) load_batch<U>(A, M, P2, c0);  // operator: independent of the previous kernel
  pdl_wait();
  for (int e = tid; e < NB * C; e += kVnThreads) {
    const int j = e / C, col = e % C, s = slot0 + j;
    xs[j * XS + col] = s < nslots ? xval<MODE>(a, s / a.k, s % a.k, col) : 0.0;
  }
  __syncthreads();
  double acc0[NB], acc1[NB];
#pragma unroll
  for (int j = 0; j < NB; ++j) { acc0[j] = 0.0; acc1[j] = 0.0; }
  stream_cols<NB, U>(A, M, P2, c0, c1, xs, 0, 0, XS, acc0, acc1);
#pragma unroll
  for (int j = 0; j < NB; ++j) {
    red[(g * NB + j) * TR + 2 * q] = acc0[j];
    red[(g * NB + j) * TR + 2 * q + 1] = acc1[j];
  }
  __syncthreads();
  for (int e = tid; e < NB * TR; e += kVnThreads) {
    const int j = e / TR, r = e % TR, row = tile * TR + r, s = slot0 + j;
    if (row >= pn.R || s >= nslots) continue;
    double y = 0.0;
    for (int gg = 0; gg < G; ++gg) y += red[(gg * NB + j) * TR + r];
    epilogue<MODE>(a, s / a.k, row, s % a.k, y);
  }
}

constexpr int kVnNB = 4;
constexpr int kVnMinNodes = 32;      // fewer nodes: the operator stream dominates (panel kernel)
constexpr size_t kVnMaxSmem = 96 * 1024;
constexpr int kVnMaxCols = 64;

size_t vn_smem(const Panel& pn, int& XS) {
  XS = pn.C | 1;
  return ((size_t)kVnNB * XS + (size_t)kVnNB * 2 * kVnThreads) * 8;
}

template <int MODE>
int launch_vn(const GemvArgs& a, const Panel& pn, cudaStream_t st) {
  int XS;
  const size_t smem = vn_smem(pn, XS);
  static bool attr_set = false;
  if (!attr_set) {
    HPSB_CUDA(cudaFuncSetAttribute(k_vn<MODE, kVnNB, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)kVnMaxSmem));
    attr_set = true;
  }
  dim3 grid((unsigned)pn.ntiles, (unsigned)cdiv((long long)a.shared * a.k, kVnNB));
  HPSB_CUDA(launch_pdl(k_vn<MODE, kVnNB, 4>, grid, dim3(kVnThreads), smem, st, a, pn, XS));
  HPSB_LAUNCH_CHECK();
  return 0;
}

bool vn_enabled() {
  static const bool on = [] {
    const char* e = getenv("HPSB_NO_VN");
    return !(e && e[0] == '1');
  }();
  return on;
}

template <int MODE, int KM, int U>
int launch(const GemvArgs& a, const Panel& pn, const PanelSplit& sp, cudaStream_t st) {
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(k_panel<MODE, KM, U>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kMaxStage);
    attr_set = true;
  }
  dim3 grid((unsigned)((long long)pn.ntiles * sp.nsplit * (a.shared ? a.shared : 1)), (unsigned)sp.kgroups);
  HPSB_CUDA(launch_pdl(k_panel<MODE, KM, U>, grid, dim3(pn.TR / 2), sp.smem, st, a, pn, sp));
  HPSB_LAUNCH_CHECK();
  return 0;
}

template <int MODE>
int dispatch(const GemvArgs& a, const Panel& pn, const PanelSplit& sp, cudaStream_t st) {
  switch (sp.KM) {
    case 1: return launch<MODE, 1, 8>(a, pn, sp, st);
    case 4: return launch<MODE, 4, 4>(a, pn, sp, st);
    case 8: return launch<MODE, 8, 4>(a, pn, sp, st);
    default: return launch<MODE, 16, 2>(a, pn, sp, st);
  }
}

__global__ void k_pack(const double* __restrict__ src1, long long s1, int ld1, int R1,
                       const double* __restrict__ src2, long long s2, int ld2, Panel pn) {
  const long long total = (long long)pn.ntiles * pn.C * pn.TS;
  const long long P = (long long)pn.c * pn.R;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < total;
       e += (long long)gridDim.x * blockDim.x) {
    const long long tile = e / ((long long)pn.C * pn.TS);
    const long long rem = e % ((long long)pn.C * pn.TS);
    const int col = (int)(rem / pn.TS), r = (int)(rem % pn.TS);
    const long long p = tile * pn.TR + r;
    double v = 0.0;
    if (r < pn.TR && p < P) {
      const long long node = p / pn.R;
      const int rr = (int)(p % pn.R);
      v = rr < R1 ? src1[node * s1 + (long long)rr * ld1 + col] : src2[node * s2 + (long long)(rr - R1) * ld2 + col];
    }
    pn.base[e] = v;
  }
}

__global__ void k_unpack(Panel pn, int node, int row0, int nrows, double* __restrict__ dst) {
  const long long n = (long long)nrows * pn.C;
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n;
       e += (long long)gridDim.x * blockDim.x) {
    const int row = (int)(e / pn.C) + row0, col = (int)(e % pn.C);
    const long long p = (long long)node * pn.R + row;
    dst[e] = pn.base[(p / pn.TR) * pn.C * pn.TS + (long long)col * pn.TS + p % pn.TR];
  }
}

}  // namespace

int gemv_level(const GemvArgs& a, const Panel& pn, cudaStream_t st) {
  if (pn.c <= 0 || pn.R <= 0 || a.k <= 0) return 0;
  if (pn.TS != pn.TR) {
    set_error("gemv: node-aligned panel passed to the level kernel");
    return -1;
  }
  // (the column chain of one thread, C/G, must stay short: long-K levels
  // -- the down sweep's S -- keep the split-K panel kernel)
  if (a.prow0 == 0 && a.shared >= kVnMinNodes && pn.c == 1 && pn.TR <= 2 * kVnThreads && vn_enabled() &&
      cdiv(pn.C, kVnThreads / (pn.TR / 2)) <= kVnMaxCols) {
    int XS;
    if (vn_smem(pn, XS) <= kVnMaxSmem) {
      switch (a.mode) {
        case GEMV_UP: return launch_vn<GEMV_UP>(a, pn, st);
        case GEMV_DOWN: return launch_vn<GEMV_DOWN>(a, pn, st);
        default: return launch_vn<GEMV_LEAF>(a, pn, st);
      }
    }
  }
  const PanelSplit sp = panel_split(pn, a.k, a.shared ? a.shared : 1);
  if (sp.nsplit > 1 && (!a.part || !a.cnt)) {
    set_error("gemv: split-K needs workspace");
    return -1;
  }
  switch (a.mode) {
    case GEMV_UP: return dispatch<GEMV_UP>(a, pn, sp, st);
    case GEMV_DOWN: return dispatch<GEMV_DOWN>(a, pn, sp, st);
    default: return dispatch<GEMV_LEAF>(a, pn, sp, st);
  }
}

// the node-indexed inputs / outputs of a launch shifted to start at node n0
GemvArgs shift_nodes(GemvArgs a, long long n0) {
  if (n0 == 0) return a;
  if (a.mode == GEMV_UP) {
    a.Hc += 2 * n0 * a.Hc_s;
    a.W3 += n0 * a.n3;
    if (a.Hout) a.Hout += n0 * a.n12;
    if (a.j3) a.j3 += n0 * a.n3;
  } else if (a.mode == GEMV_DOWN) {
    a.gidx += n0 * a.n12;
    a.j3 += n0 * a.n3;
    if (a.W3) a.W3 += n0 * a.n3;
  } else {
    a.xin += n0 * a.xin_s;
    a.yout += n0 * a.yout_s;
    if (a.yadd) a.yadd += n0 * a.yadd_s;
  }
  return a;
}

int gemv_nodes(const GemvArgs& a, const Panel& pn, int n0, int n1, cudaStream_t st) {
  if (n1 <= n0) return 0;
  if (a.shared) {
    GemvArgs b = shift_nodes(a, n0);
    b.shared = n1 - n0;
    return gemv_level(b, pn, st);
  }
  const int cp = pn.c;
  if (n0 % cp || n1 % cp || n1 / cp > pn.parts) {
    set_error("gemv: node range [%d, %d) is not aligned to the panel's parts (%d nodes each)", n0, n1, cp);
    return -1;
  }
  for (int g = n0 / cp; g < n1 / cp; ++g)
    if (int rc = gemv_level(shift_nodes(a, (long long)g * cp), pn.part(g), st)) return rc;
  return 0;
}

int pack_panel2(const double* src1, long long s1, int ld1, int R1, const double* src2, long long s2, int ld2,
                const Panel& pn, cudaStream_t st) {
  if (pn.parts > 1) {
    for (int g = 0; g < pn.parts; ++g) {
      const long long o = (long long)g * pn.c;
      if (int rc = pack_panel2(src1 + o * s1, s1, ld1, R1, src2 + o * s2, s2, ld2, pn.part(g), st)) return rc;
    }
    return 0;
  }
  long long total = (long long)pn.ntiles * pn.C * pn.TS;
  if (total <= 0) return 0;
  unsigned blocks = (unsigned)std::min<long long>(cdiv(total, 256), (long long)kNumSMs * 32);
  k_pack<<<blocks, 256, 0, st>>>(src1, s1, ld1, R1, src2, s2, ld2, pn);
  HPSB_LAUNCH_CHECK();
  return 0;
}

int pack_panel(const double* src, long long s_node, int ld, const Panel& pn, cudaStream_t st) {
  return pack_panel2(src, s_node, ld, pn.R, src, s_node, ld, pn, st);
}

int unpack_panel(const Panel& pn, int node, int row0, int nrows, double* dst, cudaStream_t st) {
  if (pn.parts > 1) return unpack_panel(pn.part(node / pn.c), node % pn.c, row0, nrows, dst, st);
  long long n = (long long)nrows * pn.C;
  if (n <= 0) return 0;
  unsigned blocks = (unsigned)std::min<long long>(cdiv(n, 256), (long long)kNumSMs * 8);
  k_unpack<<<blocks, 256, 0, st>>>(pn, node, row0, nrows, dst);
  HPSB_LAUNCH_CHECK();
  return 0;
}

}  // namespace hpsb
