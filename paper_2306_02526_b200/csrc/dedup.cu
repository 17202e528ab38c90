// Shared-layout level applies (constant coefficients).
//
// With constant coefficients every node of a level has bitwise the same
// operators (the reference still stores one copy per node, solver.py:137-151),
// so a level apply is a real GEMM: the level's operator times the matrix
// whose columns are the nodes' input vectors.  Posed node-major,
//     Y (nodes x R) = X (nodes x K) * Op^T,   Op = [X33^-1; Tstack X33^-1] (up)
//                                                   or S (down),
// it is the "NT" product of mma_gemm.cu with the node vectors gathered
// straight into the A tiles (r3 = hb[i3b] - ha[i3a] [- jump/dt] for the up
// pass, u[gidx_bnd] for the down pass) and a scattering epilogue (w3 / the
// node's flux / u[j3]).  The FP64 tensor pipe (DMMA m8n8k4) does the math;
// the operator tiles come from L2.  Levels with fewer than kSharedGemmNodes
// nodes (the top of the tree: few nodes, operators up to hundreds of MB) use
// the streaming panel kernel on a one-node panel, one virtual tile per
// (node, tile): the operator is read from HBM once and re-read from L2.
#include <stdlib.h>

#include "hps_plan.cuh"

namespace hpsb {

namespace {

constexpr int BK = 16;
constexpr int SROW = BK + 4;
constexpr int BM = 64;  // nodes per CTA tile (2 warps of 32 rows)

enum GsMode { GS_UP = 0, GS_DOWN = 1 };

struct GsArgs {
  int M, N, K;                 // nodes x rhs (row m: node m % nodes, rhs m / nodes), operator rows, columns
  int nodes;
  int nsplit, KC;              // split-K: CTA column range [split * KC, +KC) (KC a multiple of BK)
  double* part; unsigned* cnt; // split-K partials (nsplit x M x N) and per-tile semaphores
  const double* B; int ldb;    // operator, N x K row-major
  const double* X;             // non-null: the gathered inputs, M x K row-major (k_gs_gather)
  GemvArgs g;                  // gathers / scatters (same fields as the streaming kernels)
};

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

template <int MODE>
__device__ __forceinline__ double gs_x(const GemvArgs& a, int node, int kg, int col) {
  if (MODE == GS_UP) {
    const double* Ha = a.Hc + kg * a.Hc_k + (long long)(2 * node) * a.Hc_s;
    const double* Hb = Ha + a.Hc_s;
    double v = Hb[a.i3b[col]] - Ha[a.i3a[col]];
    if (a.jump) v = v - a.inv_dt * a.jump[kg * a.jump_k + a.j3[(long long)node * a.n3 + col]];
    return v;
  } else {
    return a.u[kg * a.u_k + a.gidx[(long long)node * a.n12 + col]];
  }
}

// The epilogue in two halves, so that it issues every load of a row group
// (pass-through flux entries / w3, target indices) before its first store --
// the stores may alias the loaded arrays as far as the compiler knows, so a
// fused load-store per output serialises the loads
template <int MODE>
__device__ __forceinline__ void gs_pre(const GemvArgs& a, int node, int r, int kg, double& base, int& t) {
  if (MODE == GS_UP) {
    base = 0.0;
    t = 0;
    if (r >= a.n3) {
      r -= a.n3;
      const double* Ha = a.Hc + kg * a.Hc_k + (long long)(2 * node) * a.Hc_s;
      base = (r < a.n1a) ? Ha[a.i1a[r]] : Ha[a.Hc_s + a.i2b[r - a.n1a]];
    }
  } else {
    base = a.W3 ? a.W3[kg * a.W3_k + (long long)node * a.n3 + r] : 0.0;
    t = a.j3[(long long)node * a.n3 + r];
  }
}

template <int MODE>
__device__ __forceinline__ void gs_put(const GemvArgs& a, int node, int r, int kg, double v, int t) {
  if (MODE == GS_UP) {
    if (r < a.n3) a.W3[kg * a.W3_k + (long long)node * a.n3 + r] = v;
    else a.Hout[kg * a.Hout_k + (long long)node * a.n12 + r - a.n3] = v;
  } else {
    a.u[kg * a.u_k + t] = v;
  }
}

// epilogue of one 8-row group of a warp tile: loads first, then the stores
template <int MODE>
__device__ __forceinline__ void gs_epilogue_row(const GsArgs& a, int m, int rbase, const double (&acc)[4][2]) {
  if (m >= a.M) return;
  const int node = m % a.nodes, kg = m / a.nodes;
  double base[4][2];
  int t[4][2];
#pragma unroll
  for (int j = 0; j < 4; ++j)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int r = rbase + j * 8 + h;
      base[j][h] = 0.0;
      t[j][h] = 0;
      if (r < a.N) gs_pre<MODE>(a.g, node, r, kg, base[j][h], t[j][h]);
    }
#pragma unroll
  for (int j = 0; j < 4; ++j)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int r = rbase + j * 8 + h;
      if (r < a.N) gs_put<MODE>(a.g, node, r, kg, acc[j][h] + base[j][h], t[j][h]);
    }
}

// The (node, rhs) x K input matrix of a level GEMM gathered once: every
// N-tile of the GEMM reads it (the top levels have few (node, rhs) rows but
// thousands of operator rows, i.e. tens of N-tiles that would each repeat the
// index-chasing gathers).
template <int MODE>
__global__ void k_gs_gather(GsArgs a) {
  const long long n = (long long)a.M * a.K;
  pdl_trigger();
  pdl_wait();
  for (long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x; e < n; e += (long long)gridDim.x * blockDim.x) {
    const int m = (int)(e / a.K), col = (int)(e % a.K);
    const_cast<double*>(a.X)[e] = gs_x<MODE>(a.g, m % a.nodes, m / a.nodes, col);
  }
}

// Every (node, rhs) pair is one row of the GEMM: the multi-rhs (ensemble)
// level apply is one tensor-core GEMM over nodes x rhs.
template <int MODE, int WN>
__global__ void __launch_bounds__(64 * WN) k_gs(GsArgs a, int tilesN) {
  constexpr int BN = 32 * WN, NT = 64 * WN;
  constexpr int AE = BM * BK / NT, BE = BN * BK / NT;  // staged elements per thread
  extern __shared__ double sm[];
  __shared__ unsigned s_last;
  double* As = sm;                  // [2][BM][SROW]
  double* Bs = sm + 2 * BM * SROW;  // [2][BN][SROW]
  const int tile = blockIdx.x / a.nsplit, split = blockIdx.x % a.nsplit;
  const int tm = tile / tilesN, tn = tile % tilesN;
  const int m0 = tm * BM, n0 = tn * BN;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp / WN, wn = warp % WN;
  const int kb = split * a.KC / BK;                                   // first k-step of this CTA
  const int nk = (min(a.K, (split + 1) * a.KC) - split * a.KC + BK - 1) / BK;
  pdl_trigger();

  double ra[AE], rb[BE];
  auto load_b = [&](int kt) {  // the operator does not depend on the previous kernel
#pragma unroll
    for (int i = 0; i < BE; ++i) {
      const int e = tid + NT * i, r = e / BK, c = e % BK;
      const int gn = n0 + r, gk = (kb + kt) * BK + c;
      rb[i] = (gn < a.N && gk < a.K) ? a.B[(long long)gn * a.ldb + gk] : 0.0;
    }
  };
  auto load_a = [&](int kt) {
#pragma unroll
    for (int i = 0; i < AE; ++i) {
      const int e = tid + NT * i, r = e / BK, c = e % BK;
      const int gm = m0 + r, gk = (kb + kt) * BK + c;
      ra[i] = (gm < a.M && gk < a.K) ? (a.X ? a.X[(long long)gm * a.K + gk] : gs_x<MODE>(a.g, gm % a.nodes, gm / a.nodes, gk))
                                     : 0.0;
    }
  };
  auto store = [&](int buf) {
#pragma unroll
    for (int i = 0; i < AE; ++i) {
      const int e = tid + NT * i;
      As[(buf * BM + e / BK) * SROW + e % BK] = ra[i];
    }
#pragma unroll
    for (int i = 0; i < BE; ++i) {
      const int e = tid + NT * i;
      Bs[(buf * BN + e / BK) * SROW + e % BK] = rb[i];
    }
  };

  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) { acc[i][j][0] = 0.0; acc[i][j][1] = 0.0; }

  load_b(0);
  pdl_wait();
  load_a(0);
  store(0);
  __syncthreads();
  for (int kt = 0; kt < nk; ++kt) {
    const int buf = kt & 1;
    if (kt + 1 < nk) { load_b(kt + 1); load_a(kt + 1); }
    const double* Ab = As + (buf * BM + wm * 32 + (lane >> 2)) * SROW + (lane & 3);
    const double* Bb = Bs + (buf * BN + wn * 32 + (lane >> 2)) * SROW + (lane & 3);
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double af[4], bf[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) af[i] = Ab[i * 8 * SROW + kk];
#pragma unroll
      for (int j = 0; j < 4; ++j) bf[j] = Bb[j * 8 * SROW + kk];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
    if (kt + 1 < nk) store(buf ^ 1);
    __syncthreads();
  }

  if (a.nsplit > 1) {  // partial tile to the workspace; the last CTA of the tile sums in split order
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int m = m0 + wm * 32 + i * 8 + (lane >> 2);
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int r = n0 + wn * 32 + j * 8 + 2 * (lane & 3) + h;
          if (m < a.M && r < a.N) a.part[((size_t)split * a.M + m) * a.N + r] = acc[i][j][h];
        }
    }
    __syncthreads();  // barrier + one thread's acq_rel atomic (hps_common.cuh)
    if (tid == 0) s_last = atom_add_acq_rel(a.cnt + tile, 1u) == (unsigned)a.nsplit - 1;
    __syncthreads();
    if (!s_last) return;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int m = m0 + wm * 32 + i * 8 + (lane >> 2);
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int r = n0 + wn * 32 + j * 8 + 2 * (lane & 3) + h;
          double y = 0.0;
          if (m < a.M && r < a.N) {
            const double* pp = a.part + (size_t)m * a.N + r;
            const size_t ps = (size_t)a.M * a.N;
            for (int s0 = 0; s0 < a.nsplit; s0 += 4) {  // four loads in flight, summed in split order
              double v[4];
#pragma unroll
              for (int u = 0; u < 4; ++u) v[u] = s0 + u < a.nsplit ? __ldcg(pp + (size_t)(s0 + u) * ps) : 0.0;
#pragma unroll
              for (int u = 0; u < 4; ++u)
                if (s0 + u < a.nsplit) y += v[u];
            }
          }
          acc[i][j][h] = y;
        }
    }
    if (tid == 0) a.cnt[tile] = 0u;
  }

#pragma unroll
  for (int i = 0; i < 4; ++i)
    gs_epilogue_row<MODE>(a, m0 + wm * 32 + i * 8 + (lane >> 2), n0 + wn * 32 + 2 * (lane & 3), acc[i]);
}

// The same GEMM with its operands streamed by a GS_STAGES-deep cp.async
// pipeline (16-byte copies, zero-filled past K) instead of one register-staged
// k-tile: the top levels of a many-rhs solve (X gathered up front, thousands
// of operator rows and columns, few (node, rhs) row tiles) are long k-loops
// whose global latency the two-stage register path leaves exposed.
constexpr int GS_STAGES = 3;

__device__ __forceinline__ void cp16_zfill(double* dst, const double* src, bool ok) {
  const unsigned d = (unsigned)__cvta_generic_to_shared(dst);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(d), "l"(src), "r"(ok ? 16 : 0) : "memory");
}

template <int MODE, int WN>
__global__ void __launch_bounds__(64 * WN) k_gsp(GsArgs a, int tilesN) {
  constexpr int BN = 32 * WN, NT = 64 * WN;
  constexpr int ACH = BM * BK / 2 / NT, BCH = BN * BK / 2 / NT;  // 16-byte chunks per thread and stage
  extern __shared__ double sm[];
  __shared__ unsigned s_last;
  double* As = sm;                           // [GS_STAGES][BM][SROW]
  double* Bs = sm + GS_STAGES * BM * SROW;   // [GS_STAGES][BN][SROW]
  const int tile = blockIdx.x / a.nsplit, split = blockIdx.x % a.nsplit;
  const int tm = tile / tilesN, tn = tile % tilesN;
  const int m0 = tm * BM, n0 = tn * BN;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp / WN, wn = warp % WN;
  const int kb = split * a.KC / BK;
  const int kend = min(a.K, (split + 1) * a.KC);
  const int nk = (kend - split * a.KC + BK - 1) / BK;
  pdl_trigger();
  auto load_b = [&](int kt, int buf) {  // the operator does not depend on the previous kernel
#pragma unroll
    for (int i = 0; i < BCH; ++i) {
      const int e = tid + NT * i, r = e / (BK / 2), c = 2 * (e % (BK / 2));
      const int gn = n0 + r, gk = (kb + kt) * BK + c;
      const bool ok = gn < a.N && gk < kend;
      cp16_zfill(Bs + (buf * BN + r) * SROW + c, ok ? a.B + (long long)gn * a.ldb + gk : a.B, ok);
    }
  };
  auto load_a = [&](int kt, int buf) {
#pragma unroll
    for (int i = 0; i < ACH; ++i) {
      const int e = tid + NT * i, r = e / (BK / 2), c = 2 * (e % (BK / 2));
      const int gm = m0 + r, gk = (kb + kt) * BK + c;
      const bool ok = gm < a.M && gk < kend;
      cp16_zfill(As + (buf * BM + r) * SROW + c, ok ? a.X + (long long)gm * a.K + gk : a.X, ok);
    }
  };
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) { acc[i][j][0] = 0.0; acc[i][j][1] = 0.0; }
  // prologue: the operator's first stages before the dependency wait, the inputs after
#pragma unroll
  for (int s = 0; s < GS_STAGES - 1; ++s)
    if (s < nk) load_b(s, s);
  pdl_wait();
#pragma unroll
  for (int s = 0; s < GS_STAGES - 1; ++s) {
    if (s < nk) load_a(s, s);
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  for (int kt = 0; kt < nk; ++kt) {
    const int buf = kt % GS_STAGES;
    asm volatile("cp.async.wait_group %0;" ::"n"(GS_STAGES - 2) : "memory");
    __syncthreads();  // stage kt landed for every thread; stage kt - 1 is consumed by all
    if (kt + GS_STAGES - 1 < nk) {
      load_b(kt + GS_STAGES - 1, (kt + GS_STAGES - 1) % GS_STAGES);
      load_a(kt + GS_STAGES - 1, (kt + GS_STAGES - 1) % GS_STAGES);
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    const double* Ab = As + (buf * BM + wm * 32 + (lane >> 2)) * SROW + (lane & 3);
    const double* Bb = Bs + (buf * BN + wn * 32 + (lane >> 2)) * SROW + (lane & 3);
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double af[4], bf[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) af[i] = Ab[i * 8 * SROW + kk];
#pragma unroll
      for (int j = 0; j < 4; ++j) bf[j] = Bb[j * 8 * SROW + kk];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");

  if (a.nsplit > 1) {  // partial tile to the workspace; the last CTA of the tile sums in split order
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int m = m0 + wm * 32 + i * 8 + (lane >> 2);
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int r = n0 + wn * 32 + j * 8 + 2 * (lane & 3) + h;
          if (m < a.M && r < a.N) a.part[((size_t)split * a.M + m) * a.N + r] = acc[i][j][h];
        }
    }
    __syncthreads();
    if (tid == 0) s_last = atom_add_acq_rel(a.cnt + tile, 1u) == (unsigned)a.nsplit - 1;
    __syncthreads();
    if (!s_last) return;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int m = m0 + wm * 32 + i * 8 + (lane >> 2);
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int r = n0 + wn * 32 + j * 8 + 2 * (lane & 3) + h;
          double y = 0.0;
          if (m < a.M && r < a.N) {
            const double* pp = a.part + (size_t)m * a.N + r;
            const size_t ps = (size_t)a.M * a.N;
            for (int s0 = 0; s0 < a.nsplit; s0 += 4) {
              double v[4];
#pragma unroll
              for (int u = 0; u < 4; ++u) v[u] = s0 + u < a.nsplit ? __ldcg(pp + (size_t)(s0 + u) * ps) : 0.0;
#pragma unroll
              for (int u = 0; u < 4; ++u)
                if (s0 + u < a.nsplit) y += v[u];
            }
          }
          acc[i][j][h] = y;
        }
    }
    if (tid == 0) a.cnt[tile] = 0u;
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
    gs_epilogue_row<MODE>(a, m0 + wm * 32 + i * 8 + (lane >> 2), n0 + wn * 32 + 2 * (lane & 3), acc[i]);
}

template <int MODE, int WN>
int launch_gsp(GsArgs a, const GsSplit& sp, cudaStream_t st) {
  constexpr int BN = 32 * WN;
  const size_t smem = (size_t)GS_STAGES * (BM + BN) * SROW * 8;
  static bool attr = false;
  if (!attr) {
    HPSB_CUDA(cudaFuncSetAttribute(k_gsp<MODE, WN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr = true;
  }
  a.nsplit = sp.nsplit;
  a.KC = sp.KC;
  const int tilesN = (int)cdiv(a.N, BN);
  dim3 grid((unsigned)(sp.tiles * sp.nsplit));
  HPSB_CUDA(launch_pdl(k_gsp<MODE, WN>, grid, dim3(64 * WN), smem, st, a, tilesN));
  HPSB_LAUNCH_CHECK();
  return 0;
}

static bool gs_pipe_enabled() {
  static const bool on = [] {
    const char* e = getenv("HPSB_NO_GS_PIPE");
    return !(e && e[0] == '1');
  }();
  return on;
}

template <int MODE, int WN>
int launch_gs(GsArgs a, const GsSplit& sp, cudaStream_t st) {
  constexpr int BN = 32 * WN;
  const size_t smem = (size_t)2 * (BM + BN) * SROW * 8;
  static bool attr = false;
  if (!attr) {
    HPSB_CUDA(cudaFuncSetAttribute(k_gs<MODE, WN>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr = true;
  }
  a.nsplit = sp.nsplit;
  a.KC = sp.KC;
  const int tilesN = (int)cdiv(a.N, BN);
  dim3 grid((unsigned)(sp.tiles * sp.nsplit));
  HPSB_CUDA(launch_pdl(k_gs<MODE, WN>, grid, dim3(64 * WN), smem, st, a, tilesN));
  HPSB_LAUNCH_CHECK();
  return 0;
}

static bool gs_gather_enabled() {
  static const bool on = [] {
    const char* e = getenv("HPSB_NO_GS_GATHER");
    return !(e && e[0] == '1');
  }();
  return on;
}

template <int MODE>
int gs(const GsArgs& a, const Workspace& ws, cudaStream_t st) {
  const GsSplit sp = gs_split(a.M, a.N, a.K);
  if (sp.nsplit > 1 && (!ws.part || !ws.cnt)) {
    set_error("gs: split-K needs workspace");
    return -1;
  }
  GsArgs b = a;
  b.part = ws.part;
  b.cnt = ws.cnt;
  b.X = nullptr;
  if (sp.gather_doubles && ws.xg && gs_gather_enabled()) {
    b.X = ws.xg;
    const long long n = (long long)a.M * a.K;
    HPSB_CUDA(launch_pdl(k_gs_gather<MODE>, dim3((unsigned)std::min<long long>(cdiv(n, 256), 148LL * 16)), dim3(256), 0,
                         st, b));
    HPSB_LAUNCH_CHECK();
  }
  // pipelined path: gathered inputs and 16-byte aligned rows of X and of the operator
  // (long k-loops only: with a few k-steps the 2-CTA/SM register path wins)
  if (b.X && gs_pipe_enabled() && sp.KC >= 8 * BK && a.K % 2 == 0 && a.ldb % 2 == 0 && ((uintptr_t)a.B & 15) == 0 &&
      ((uintptr_t)b.X & 15) == 0) {
    if (sp.WN == 1) return launch_gsp<MODE, 1>(b, sp, st);
    if (sp.WN == 2) return launch_gsp<MODE, 2>(b, sp, st);
    return launch_gsp<MODE, 4>(b, sp, st);
  }
  if (sp.WN == 1) return launch_gs<MODE, 1>(b, sp, st);
  if (sp.WN == 2) return launch_gs<MODE, 2>(b, sp, st);
  return launch_gs<MODE, 4>(b, sp, st);
}

}  // namespace

// tile width (operator rows per CTA: enough tiles to fill the SMs, little
// padding waste) and split-K (short column chains when the tiles are few)
GsSplit gs_split(long long M, int N, int K) {
  GsSplit s;
  const long long tilesM = cdiv(M, BM);
  if (N <= 32 || tilesM * cdiv(N, 64) < 2 * kNumSMs) s.WN = 1;
  else if (N <= 64 || tilesM * cdiv(N, 128) < 2 * kNumSMs) s.WN = 2;
  else s.WN = 4;
  s.tiles = (int)(tilesM * cdiv(N, 32 * s.WN));
  const int ksteps = (int)cdiv(K, BK);
  int ns = (int)std::min<long long>(cdiv(2LL * kNumSMs, s.tiles), 16);
  ns = std::max(1, std::min(ns, ksteps / 4));          // >= 4 k-steps per CTA
  s.KC = (int)cdiv(ksteps, ns) * BK;
  s.nsplit = (int)cdiv(K, s.KC);
  if (s.nsplit > 1) {
    s.part_doubles = (size_t)s.nsplit * M * N;
    s.counters = s.tiles;
  }
  // many N-tiles re-read the inputs, or a long k-loop (the pipelined GEMM streams gathered inputs)
  if (cdiv(N, 32 * s.WN) >= 4 || K >= 256) s.gather_doubles = (size_t)M * K;
  return s;
}

// the level apply as a DMMA GEMM over (node, rhs) rows: many nodes, or a
// multi-rhs solve (the streaming kernel otherwise); levels whose one-node
// panel is node-aligned (fused subtree levels) always take the GEMM
bool shared_gemm(const Plan& P, int d, int nodes, int k) {
  if (d >= P.dF) return true;
  static const long long min_rows = [] {  // A/B: HPSB_GS_MIN_ROWS
    const char* e = getenv("HPSB_GS_MIN_ROWS");
    return e ? atoll(e) : 64LL;
  }();
  return (long long)nodes * k >= kSharedGemmNodes || (k >= kSharedGemmRhs && (long long)nodes * k >= min_rows);
}

int shared_level_up(const Ops& ops, const Workspace& ws, int d, int k, const double* Hc, long long Hc_k,
                    long long Hc_s, const double* jump, long long ld_jump, double inv_dt, int n0, int n1,
                    cudaStream_t st) {
  const Plan& P = *ops.plan;
  const Level& lv = P.lv[d];
  const LevelOps& lo = ops.lo[d];
  GemvArgs g{};
  g.k = k; g.part = ws.part; g.cnt = ws.cnt;
  g.Hc = Hc; g.nbc = lv.nbc; g.Hc_k = Hc_k; g.Hc_s = Hc_s;
  g.W3 = ws.W3[d]; g.n3 = lv.n3; g.W3_k = (long long)lv.c * lv.n3;
  g.i1a = lv.i1a; g.i3a = lv.i3a; g.i2b = lv.i2b; g.i3b = lv.i3b; g.n1a = lv.n1a; g.n12 = lv.n12;
  g.jump = jump; g.jump_k = ld_jump; g.inv_dt = inv_dt; g.j3 = lv.j3;
  g.Hout = d > 0 ? ws.H[d] : nullptr; g.Hout_k = (long long)lv.c * lv.n12;
  g.mode = GEMV_UP;
  if (!shared_gemm(P, d, n1 - n0, k)) {
    g.shared = 1;
    return gemv_nodes(g, lo.Up, n0, n1, st);
  }
  GsArgs a{};
  a.nodes = n1 - n0;
  a.M = a.nodes * k;
  a.N = lv.n3 + (d > 0 ? lv.n12 : 0); a.K = lv.n3;
  g = shift_nodes(g, n0);
  a.B = lo.Ush; a.ldb = lv.ld3; a.g = g;
  const int rc = deep_level(g, true, a.nodes, k, a.N, a.K, lo.Ush, lv.ld3, st);  // many rhs, deep levels
  if (rc != 1) return rc;
  return gs<GS_UP>(a, ws, st);
}

int shared_level_down(const Ops& ops, const Workspace& ws, int d, int k, bool has_w3, double* u, long long ld_u,
                      int n0, int n1, cudaStream_t st) {
  const Plan& P = *ops.plan;
  const Level& lv = P.lv[d];
  const LevelOps& lo = ops.lo[d];
  GemvArgs g{};
  g.k = k; g.part = ws.part; g.cnt = ws.cnt;
  g.u = u; g.u_k = ld_u; g.gidx = lv.gidx_bnd; g.j3 = lv.j3; g.n3 = lv.n3; g.n12 = lv.n12;
  g.W3 = has_w3 ? ws.W3[d] : nullptr; g.W3_k = (long long)lv.c * lv.n3;
  g.mode = GEMV_DOWN;
  if (!shared_gemm(P, d, n1 - n0, k)) {
    g.shared = 1;
    return gemv_nodes(g, lo.S, n0, n1, st);
  }
  GsArgs a{};
  a.nodes = n1 - n0;
  a.M = a.nodes * k;
  a.N = lv.n3; a.K = lv.n12;
  g = shift_nodes(g, n0);
  a.B = lo.Ssh; a.ldb = lv.ld12; a.g = g;
  const int rc = deep_level(g, false, a.nodes, k, a.N, a.K, lo.Ssh, lv.ld12, st);
  if (rc != 1) return rc;
  return gs<GS_DOWN>(a, ws, st);
}

}  // namespace hpsb
