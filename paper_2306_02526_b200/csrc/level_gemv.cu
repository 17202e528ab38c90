// Level-batched streaming GEMV for the HPS solve (sm_100a, FP64, HBM-bound).
//
// One launch applies one operator family of one tree level to every node:
//   UPX : w3   = X33^-1 (hb[i3b] - ha[i3a] [- jump/dt])        (solver.py:246-251)
//   UPT : h    = [ha[i1a]; hb[i2b]] + Tstack w3                 (solver.py:252-254)
//   DOWN: u[j3] = S u[gidx_bnd] (+ w3)                          (solver.py:261-268)
//   LEAF: y    = M x (+ add)   per leaf (variable-coefficient leaves,
//                               solver.py:225-227 and 269-272)
// Operators are stored node-contiguous, row-major, rows padded to an even
// length, so each node's matrix is one contiguous HBM stream read once per
// solve with 16-byte streaming loads (ld.global.cs).  The gathered input
// vector of each node is staged in shared memory (column chunks), groups of
// G lanes own rows and reduce with xor-shuffles, and the mode-specific
// gather / scatter is fused into the prologue / epilogue.
#include "hps_plan.cuh"

namespace hpsb {

namespace {

constexpr int NT = 256;
constexpr int MAXS = 4;  // rows per lane-group per block

template <int MODE>
__device__ __forceinline__ double xval(const GemvArgs& a, int node, int kg, int col) {
  if (MODE == GEMV_UPX) {
    const double* Ha = a.Hc + kg * a.Hc_k + (long long)(2 * node) * a.nbc;
    const double* Hb = Ha + a.nbc;
    double v = Hb[a.i3b[col]] - Ha[a.i3a[col]];
    if (a.jump) v = v - a.inv_dt * a.jump[kg * a.jump_k + a.j3[(long long)node * a.n3 + col]];
    return v;
  } else if (MODE == GEMV_UPT) {
    return a.W3[kg * a.W3_k + (long long)node * a.n3 + col];
  } else if (MODE == GEMV_DOWN) {
    return a.u[kg * a.u_k + a.gidx[(long long)node * a.n12 + col]];
  } else {
    return a.xin[kg * a.xin_k + (long long)node * a.xin_s + col];
  }
}

template <int MODE>
__device__ __forceinline__ void epilogue(const GemvArgs& a, int node, int r, int kg, double y) {
  if (MODE == GEMV_UPX) {
    a.W3[kg * a.W3_k + (long long)node * a.n3 + r] = y;
  } else if (MODE == GEMV_UPT) {
    const double* Ha = a.Hc + kg * a.Hc_k + (long long)(2 * node) * a.nbc;
    const double* Hb = Ha + a.nbc;
    double base = (r < a.n1a) ? Ha[a.i1a[r]] : Hb[a.i2b[r - a.n1a]];
    a.Hout[kg * a.Hout_k + (long long)node * a.n12 + r] = base + y;
  } else if (MODE == GEMV_DOWN) {
    double v = y;
    if (a.W3) v = v + a.W3[kg * a.W3_k + (long long)node * a.n3 + r];
    a.u[kg * a.u_k + a.j3[(long long)node * a.n3 + r]] = v;
  } else {
    double v = y;
    if (a.yadd) v = v + a.yadd[kg * a.yadd_k + (long long)node * a.yadd_s + r];
    a.yout[kg * a.yout_k + (long long)node * a.yout_s + r] = v;
  }
}

template <int MODE, int G, int KM>
__global__ void __launch_bounds__(NT) k_gemv(GemvArgs a, int npb, int rpb, int CH) {
  extern __shared__ double xs[];
  const int tid = threadIdx.x;
  const int gl = tid & (G - 1);
  const int grp = tid / G;
  constexpr int NGRP = NT / G;
  const int k0 = blockIdx.y * KM;

  int node0, rbeg, rend;
  if (npb > 1 || rpb >= a.R) {
    node0 = blockIdx.x * npb; rbeg = 0; rend = a.R;
  } else {
    int splits = (a.R + rpb - 1) / rpb;
    node0 = blockIdx.x / splits;
    rbeg = (blockIdx.x % splits) * rpb;
    rend = min(a.R, rbeg + rpb);
  }
  const int nn = min(npb, a.c - node0);
  const int rpn = rend - rbeg;
  const int nrows = nn * rpn;

  // per-slot row pointers and shared-memory x offsets (x chunk laid out [node][k][col])
  const double* mp[MAXS];
  int xnode[MAXS];
  bool live[MAXS];
#pragma unroll
  for (int i = 0; i < MAXS; ++i) {
    int s = grp + i * NGRP;
    live[i] = s < nrows;
    int nl = live[i] ? s / rpn : 0;
    int r = live[i] ? rbeg + s % rpn : 0;
    xnode[i] = nl;
    mp[i] = a.M + (long long)(node0 + nl) * a.sM + (long long)r * a.ldm;
  }

  double acc[MAXS][KM];
#pragma unroll
  for (int i = 0; i < MAXS; ++i)
#pragma unroll
    for (int kk = 0; kk < KM; ++kk) acc[i][kk] = 0.0;

  for (int c0 = 0; c0 < a.C; c0 += CH) {
    const int cw = min(CH, a.C - c0);
    const int cwp = (cw + 1) & ~1;
    if (c0 > 0) __syncthreads();
    for (int e = tid; e < nn * KM * cwp; e += NT) {
      int j = e % cwp;
      int t2 = e / cwp;
      int kk = t2 % KM, nl = t2 / KM;
      int kg = k0 + kk, col = c0 + j;
      double v = 0.0;
      if (kg < a.k && col < a.C) v = xval<MODE>(a, node0 + nl, kg, col);
      xs[(nl * KM + kk) * cwp + j] = v;
    }
    __syncthreads();
    const int n2 = cwp >> 1;
#pragma unroll 2
    for (int j2 = gl; j2 < n2; j2 += G) {
      double2 m[MAXS];
#pragma unroll
      for (int i = 0; i < MAXS; ++i)
        if (live[i]) m[i] = __ldcs(reinterpret_cast<const double2*>(mp[i] + c0) + j2);
#pragma unroll
      for (int i = 0; i < MAXS; ++i) {
        if (!live[i]) continue;
#pragma unroll
        for (int kk = 0; kk < KM; ++kk) {
          const double2 x = *reinterpret_cast<const double2*>(xs + (xnode[i] * KM + kk) * cwp + 2 * j2);
          acc[i][kk] = fma(m[i].x, x.x, acc[i][kk]);
          acc[i][kk] = fma(m[i].y, x.y, acc[i][kk]);
        }
      }
    }
  }

#pragma unroll
  for (int i = 0; i < MAXS; ++i) {
#pragma unroll
    for (int kk = 0; kk < KM; ++kk) {
      double v = acc[i][kk];
#pragma unroll
      for (int off = G / 2; off > 0; off >>= 1) v += __shfl_xor_sync(0xffffffffu, v, off, G);
      acc[i][kk] = v;
    }
  }
  if (gl == 0) {
#pragma unroll
    for (int i = 0; i < MAXS; ++i) {
      if (!live[i]) continue;
      int s = grp + i * NGRP;
      int nl = s / rpn, r = rbeg + s % rpn;
#pragma unroll
      for (int kk = 0; kk < KM; ++kk) {
        int kg = k0 + kk;
        if (kg < a.k) epilogue<MODE>(a, node0 + nl, r, kg, acc[i][kk]);
      }
    }
  }
}

template <int MODE, int G, int KM>
int launch(const GemvArgs& a, int npb, int rpb, int CH, unsigned blocks, cudaStream_t st) {
  int cwp = (CH + 1) & ~1;
  size_t smem = (size_t)npb * KM * cwp * sizeof(double);
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(k_gemv<MODE, G, KM>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024);
    attr_set = true;
  }
  dim3 grid(blocks, (unsigned)((a.k + KM - 1) / KM));
  k_gemv<MODE, G, KM><<<grid, NT, smem, st>>>(a, npb, rpb, CH);
  HPSB_LAUNCH_CHECK();
  return 0;
}

template <int MODE>
int dispatch(const GemvArgs& a, int G, int KM, int npb, int rpb, int CH, unsigned blocks,
             cudaStream_t st) {
#define HPSB_G(GG)                                                                   \
  if (G == GG) {                                                                     \
    if (KM == 1) return launch<MODE, GG, 1>(a, npb, rpb, CH, blocks, st);            \
    return launch<MODE, GG, 4>(a, npb, rpb, CH, blocks, st);                         \
  }
  HPSB_G(8) HPSB_G(16) HPSB_G(32)
#undef HPSB_G
  set_error("gemv: bad group size %d", G);
  return -1;
}

}  // namespace

int gemv_level(const GemvArgs& a, cudaStream_t st) {
  if (a.c <= 0 || a.R <= 0 || a.k <= 0) return 0;
  // lane-group size: enough lanes to cover a row with 16-byte loads
  int half = (a.C + 1) / 2;
  int G = 32;
  if (half <= 8) G = 8; else if (half <= 16) G = 16;
  const int ngrp = NT / G;
  const int KM = a.k == 1 ? 1 : 4;
  const int max_rows = ngrp * MAXS;
  const int target_blocks = 4 * kNumSMs;
  int npb = 1, rpb = a.R;
  if (a.R <= max_rows) {
    npb = max_rows / a.R;
    int cap = a.c / target_blocks;
    if (cap < 1) cap = 1;
    if (npb > cap) npb = cap;
    if (npb < 1) npb = 1;
  } else {
    rpb = max_rows;
    while (rpb > ngrp && (long long)a.c * ((a.R + rpb - 1) / rpb) < target_blocks) rpb /= 2;
  }
  // column chunk so the staged x (npb nodes x KM rhs) fits in ~48 KB
  long long cap_cols = (48 * 1024 / 8) / ((long long)npb * KM);
  int CH = (int)(cap_cols & ~1LL);
  if (CH >= a.C) CH = (a.C + 1) & ~1;
  if (CH < 2) { set_error("gemv: chunk too small"); return -1; }
  unsigned blocks;
  if (npb > 1 || rpb >= a.R) blocks = (unsigned)((a.c + npb - 1) / npb);
  else blocks = (unsigned)((long long)a.c * ((a.R + rpb - 1) / rpb));
  switch (a.mode) {
    case GEMV_UPX: return dispatch<GEMV_UPX>(a, G, KM, npb, rpb, CH, blocks, st);
    case GEMV_UPT: return dispatch<GEMV_UPT>(a, G, KM, npb, rpb, CH, blocks, st);
    case GEMV_DOWN: return dispatch<GEMV_DOWN>(a, G, KM, npb, rpb, CH, blocks, st);
    default: return dispatch<GEMV_LEAF>(a, G, KM, npb, rpb, CH, blocks, st);
  }
}

}  // namespace hpsb
