// Many-rhs level applies of the deep levels on shared operators (the C5
// ensemble: 64 members sharing one operator set, solver.py:205-213 with a
// stacked k), up (solver.py:243-256) and down (solver.py:258-268).
//
// A deep level has thousands of nodes and small operators (R x K with K =
// n3 or n12 in the tens to hundreds), so its apply is a memory-bound GEMM over
// (node, member) rows whose cost is moving the inputs and outputs, not the
// flops: the generic level GEMM (dedup.cu k_gs) gathers every input element
// through its index map in the A-tile load and every pass-through flux entry
// in the epilogue -- two dependent scattered loads per element at two CTAs per
// SM, ~0.7-1.8 TB/s.  Here one CTA takes BMN consecutive nodes of one member:
//
// * up: the nodes' 2 BMN children's flux rows are ONE contiguous block of the
//   child level's flux array, staged into shared memory by 16-byte cp.async;
//   r3 = hb[i3b] - ha[i3a] and the pass-through entries hb / ha[i1a, i2b] are
//   then shared-memory permutations;
// * down: the nodes' boundary indices (one contiguous block of gidx_bnd) are
//   staged first, then the boundary values are fetched pairwise by cp.async
//   into shared memory (16 bytes where the pair is adjacent and aligned --
//   the runs along leaf edges --, else 2 x 8; all in flight, no registers);
// * the product Y (BMN x R) = X (BMN x K) Op^T runs on the FP64 tensor pipe
//   (DMMA m8n8k4), the operator fragments from L1 / L2 (every CTA reads the
//   same operator) one k-step ahead: wide operators (the up pass, R = n3 +
//   n12) as 32-column chunks per warp over all m-tiles (each operator
//   fragment serves BMN / 8 tiles), short ones (the down pass, R = n3, K =
//   n12 long) split-K over the warps with all BMN / 8 x R / 8 tiles per warp
//   (independent accumulator chains), the warps' partials summed in warp
//   order through shared memory;
// * outputs: w3 and flux rows are contiguous per node (16-byte stores of the
//   accumulator pairs), u3 goes to u[j3] (+ w3).
// Summation order per output is fixed (k-steps in order): bitwise
// reproducible.
#include <stdlib.h>

#include "hps_plan.cuh"

namespace hpsb {

namespace {

constexpr int DW = 4;           // warps per CTA
constexpr int DT = 32 * DW;

enum DeepMode { DEEP_UP = 0, DEEP_DOWN = 1 };

struct DeepArgs {
  int nodes, k;                 // nodes of the level range (node-relative indices), rhs
  int R, K;                     // operator rows / columns
  const double* op; int ldo;    // row-major operator (R x ldo)
  GemvArgs g;                   // gathers / targets (node indices relative to the range)
  int xs;                       // staged row stride of X (doubles)
};

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ unsigned smem_addr(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

// one accumulator pair of Y: node n (CTA-relative), operator rows r, r + 1
template <int MODE>
__device__ __forceinline__ void deep_out(const DeepArgs& a, const double* blk, int nb0, int nv, int kg, int n, int r,
                                         double y0, double y1) {
  const GemvArgs& g = a.g;
  if (n >= nv || r >= a.R) return;  // r even; R, n3 even: both rows valid or both padding
  const long long node = nb0 + n;
  if (MODE == DEEP_UP) {
    if (r < g.n3) {
      *reinterpret_cast<double2*>(g.W3 + kg * g.W3_k + node * g.n3 + r) = make_double2(y0, y1);
    } else {
      const int q = r - g.n3;
      const double* ha = blk + (long long)(2 * n) * g.Hc_s;
      const double b0 = q < g.n1a ? ha[g.i1a[q]] : ha[g.Hc_s + g.i2b[q - g.n1a]];
      const double b1 = q + 1 < g.n1a ? ha[g.i1a[q + 1]] : ha[g.Hc_s + g.i2b[q + 1 - g.n1a]];
      *reinterpret_cast<double2*>(g.Hout + kg * g.Hout_k + node * g.n12 + q) = make_double2(b0 + y0, b1 + y1);
    }
  } else {
    if (g.W3) {
      const double2 w = *reinterpret_cast<const double2*>(g.W3 + kg * g.W3_k + node * g.n3 + r);
      y0 += w.x;
      y1 += w.y;
    }
    double* u = g.u + kg * g.u_k;
    const int p0 = g.j3[node * g.n3 + r], p1 = g.j3[node * g.n3 + r + 1];
    if (p1 == p0 + 1 && (p0 & 1) == 0 && (reinterpret_cast<uintptr_t>(u) & 15) == 0) {
      *reinterpret_cast<double2*>(u + p0) = make_double2(y0, y1);
    } else {
      u[p0] = y0;
      u[p1] = y1;
    }
  }
}

template <int MODE, int BMN, int NT8>  // NT8 = 0: wide operators; else the n-tiles of a short one
__global__ void __launch_bounds__(DT) k_deep(DeepArgs a) {
  constexpr int MT = BMN / 8;   // m-tiles of 8 nodes
  extern __shared__ __align__(16) double dsm[];
  const GemvArgs& g = a.g;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, gr = lane >> 2, gc = lane & 3;
  const int nb0 = blockIdx.x * BMN, kg = blockIdx.y;
  const int nv = min(BMN, a.nodes - nb0);
  double* X = dsm;                                   // [BMN][xs]
  double* blk = dsm + BMN * a.xs;                    // up: [2 BMN][Hc_s] children's flux rows
  int* idx = reinterpret_cast<int*>(blk);            // down: [BMN][n12] boundary ids
  pdl_trigger();
  pdl_wait();
  if (MODE == DEEP_UP) {
    // the children of nodes [nb0, nb0 + nv) are rows [2 nb0, 2 (nb0 + nv)) of the child level
    const double* src = g.Hc + kg * g.Hc_k + (long long)(2 * nb0) * g.Hc_s;
    const int nd = 2 * nv * (int)g.Hc_s;  // doubles (even)
    for (int e = 2 * tid; e < nd; e += 2 * DT)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr(blk + e)), "l"(src + e) : "memory");
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
    __syncthreads();
    for (int e = tid; e < BMN * a.K; e += DT) {
      const int n = e / a.K, c = e - n * a.K;
      double v = 0.0;
      if (n < nv) {
        const double* ha = blk + (long long)(2 * n) * g.Hc_s;
        v = ha[g.Hc_s + g.i3b[c]] - ha[g.i3a[c]];
        if (g.jump) v = v - g.inv_dt * g.jump[kg * g.jump_k + g.j3[(long long)(nb0 + n) * g.n3 + c]];
      }
      X[n * a.xs + c] = v;
    }
  } else {
    const int* isrc = g.gidx + (long long)nb0 * g.n12;
    if ((g.n12 & 3) == 0 && (reinterpret_cast<uintptr_t>(isrc) & 15) == 0) {  // one contiguous block
      for (int e = 4 * tid; e < nv * g.n12; e += 4 * DT)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr(idx + e)), "l"(isrc + e) : "memory");
      asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
    } else {
      for (int e = tid; e < nv * g.n12; e += DT) idx[e] = isrc[e];
    }
    __syncthreads();
    const double* u = g.u + kg * g.u_k;
    // boundary values in pairs: one 16-byte copy where the two DOFs are
    // adjacent and 16-byte aligned (the runs along a leaf edge), else two 8-byte
    const int hk = a.K / 2;
    const bool u16 = ((reinterpret_cast<uintptr_t>(u)) & 15) == 0;
    for (int e = tid; e < BMN * hk; e += DT) {
      const int n = e / hk, c = 2 * (e - n * hk);
      double* dst = X + n * a.xs + c;
      if (n < nv) {
        const int i0 = idx[n * g.n12 + c], i1 = idx[n * g.n12 + c + 1];
        if (u16 && i1 == i0 + 1 && (i0 & 1) == 0) {
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_addr(dst)), "l"(u + i0) : "memory");
        } else {
          asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_addr(dst)), "l"(u + i0) : "memory");
          asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(smem_addr(dst + 1)), "l"(u + i1) : "memory");
        }
      } else {
        dst[0] = 0.0;
        dst[1] = 0.0;
      }
    }
    asm volatile("cp.async.commit_group;\ncp.async.wait_group 0;" ::: "memory");
  }
  __syncthreads();
  if (NT8 == 0) {
    // wide operators (R > 64): warp w takes operator rows [32 (w + DW it), +32) for all MT
    // m-tiles (4 x MT tiles per fragment pair: each operator fragment serves MT tiles)
    const int ksteps = (a.K + 3) / 4;
    for (int r0 = warp * 32; r0 < a.R; r0 += 32 * DW) {
      double acc[MT][4][2];
#pragma unroll
      for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) { acc[i][j][0] = 0.0; acc[i][j][1] = 0.0; }
      const double* orow[4];
      bool rok[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int r = r0 + j * 8 + gr;
        rok[j] = r < a.R;
        orow[j] = a.op + (long long)(rok[j] ? r : 0) * a.ldo;
      }
      double bn[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) bn[j] = (rok[j] && gc < a.K) ? __ldg(orow[j] + gc) : 0.0;
      for (int ks = 0; ks < ksteps; ++ks) {
        const int k = ks * 4 + gc;
        double bf[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) bf[j] = bn[j];
        if (ks + 1 < ksteps) {
#pragma unroll
          for (int j = 0; j < 4; ++j) bn[j] = (rok[j] && k + 4 < a.K) ? __ldg(orow[j] + k + 4) : 0.0;
        }
        double af[MT];
#pragma unroll
        for (int i = 0; i < MT; ++i) af[i] = k < a.K ? X[(i * 8 + gr) * a.xs + k] : 0.0;
#pragma unroll
        for (int i = 0; i < MT; ++i)
#pragma unroll
          for (int j = 0; j < 4; ++j) dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
      }
#pragma unroll
      for (int i = 0; i < MT; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) deep_out<MODE>(a, blk, nb0, nv, kg, i * 8 + gr, r0 + j * 8 + 2 * gc, acc[i][j][0],
                                                   acc[i][j][1]);
    }
    return;
  }
  // short operators (the down pass, R = n3 <= 8 NT8): split-K over the warps
  // -- warp w takes k-steps [w K4 / DW, (w + 1) K4 / DW) for all MT x NT8
  // tiles (MT NT8 independent accumulator chains, each operator fragment
  // serving MT tiles); the warps' partial tiles meet in shared memory (the
  // staged inputs' space) and are summed in warp order
  constexpr int NTA = NT8 > 0 ? NT8 : 1;  // (NT8 = 0 returned above)
  const int ksteps = (a.K + 3) / 4;
  const int ks0 = warp * ksteps / DW, ks1 = (warp + 1) * ksteps / DW;
  double acc[MT][NTA][2];
#pragma unroll
  for (int i = 0; i < MT; ++i)
#pragma unroll
    for (int j = 0; j < NT8; ++j) { acc[i][j][0] = 0.0; acc[i][j][1] = 0.0; }
  const double* orow[NTA];
  bool rok[NTA];
#pragma unroll
  for (int j = 0; j < NT8; ++j) {
    const int r = j * 8 + gr;
    rok[j] = r < a.R;
    orow[j] = a.op + (long long)(rok[j] ? r : 0) * a.ldo;
  }
  double bn[NTA];
  {
    const int k = ks0 * 4 + gc;
#pragma unroll
    for (int j = 0; j < NT8; ++j) bn[j] = (ks0 < ks1 && rok[j] && k < a.K) ? __ldg(orow[j] + k) : 0.0;
  }
  for (int ks = ks0; ks < ks1; ++ks) {
    const int k = ks * 4 + gc;
    double bf[NTA];
#pragma unroll
    for (int j = 0; j < NT8; ++j) bf[j] = bn[j];
    if (ks + 1 < ks1) {  // next k-step's operator fragments in flight
#pragma unroll
      for (int j = 0; j < NT8; ++j) bn[j] = (rok[j] && k + 4 < a.K) ? __ldg(orow[j] + k + 4) : 0.0;
    }
    double af[MT];
#pragma unroll
    for (int i = 0; i < MT; ++i) af[i] = k < a.K ? X[(i * 8 + gr) * a.xs + k] : 0.0;
#pragma unroll
    for (int i = 0; i < MT; ++i)
#pragma unroll
      for (int j = 0; j < NT8; ++j) dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
  }
  __syncthreads();  // every warp is done with X: it takes the partial tiles [DW][BMN][R]
  double* red = X;
#pragma unroll
  for (int i = 0; i < MT; ++i)
#pragma unroll
    for (int j = 0; j < NT8; ++j) {
      const int r = j * 8 + 2 * gc;
      if (r < a.R)
        *reinterpret_cast<double2*>(red + ((long long)warp * BMN + i * 8 + gr) * a.R + r) =
            make_double2(acc[i][j][0], acc[i][j][1]);
    }
  __syncthreads();
  const int hr = a.R / 2;
  for (int o = tid; o < BMN * hr; o += DT) {
    const int n = o / hr, r = 2 * (o - n * hr);
    double y0 = 0.0, y1 = 0.0;
#pragma unroll
    for (int w = 0; w < DW; ++w) {
      const double2 v = *reinterpret_cast<const double2*>(red + ((long long)w * BMN + n) * a.R + r);
      y0 += v.x;
      y1 += v.y;
    }
    deep_out<MODE>(a, blk, nb0, nv, kg, n, r, y0, y1);
  }
}

template <int MODE, int BMN, int NT8>
int launch_deep1(const DeepArgs& a, size_t smem, cudaStream_t st) {
  HPSB_CUDA(cudaFuncSetAttribute(k_deep<MODE, BMN, NT8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  dim3 grid((unsigned)cdiv(a.nodes, BMN), (unsigned)a.k);
  HPSB_CUDA(launch_pdl(k_deep<MODE, BMN, NT8>, grid, dim3(DT), smem, st, a));
  HPSB_LAUNCH_CHECK();
  return 0;
}

template <int MODE, int BMN>
int launch_deep(const DeepArgs& a, size_t smem, cudaStream_t st) {
  // wide operators (the up pass: R = n3 + n12) as column chunks over the warps; short ones (the
  // down pass: R = n3) split-K over the warps with all tiles per warp
  if (a.R > 64) return launch_deep1<MODE, BMN, 0>(a, smem, st);
  if (a.R <= 16) return launch_deep1<MODE, BMN, 2>(a, smem, st);
  if (a.R <= 32) return launch_deep1<MODE, BMN, 4>(a, smem, st);
  return launch_deep1<MODE, BMN, 8>(a, smem, st);
}

}  // namespace

bool deep_enabled() {
  static const bool on = [] {
    const char* e = getenv("HPSB_NO_DEEP");
    return !(e && e[0] == '1');
  }();
  return on;
}

// The deep-level kernel applies to many-rhs levels with many nodes, even
// row / column counts and 16-byte aligned flux rows; returns 1 otherwise.
int deep_level(const GemvArgs& g, bool up, int nodes, int k, int R, int K, const double* op, int ldo,
               cudaStream_t st) {
  // (levels with fewer nodes have larger operators: the tiled GEMM of dedup.cu wins there)
  if (!deep_enabled() || k < kSharedGemmRhs || nodes < 512 || (R & 1) || (K & 1) || (g.n3 & 1)) return 1;
  DeepArgs a{};
  a.nodes = nodes; a.k = k; a.R = R; a.K = K; a.op = op; a.ldo = ldo; a.g = g;
  a.xs = K + 2 - (K & 1);  // even (16-byte rows), offset from multiples of 32 doubles
  if (a.xs % 32 == 0) a.xs += 2;
  if (R <= 64) a.xs = std::max(a.xs, DW * R);  // the split-K partials reuse the staged inputs' space
  if (up) {
    if ((g.Hc_s & 1) || (g.Hc_k & 1) || (reinterpret_cast<uintptr_t>(g.Hc) & 15) || !g.Hout) return 1;
    for (int bmn : {32, 16}) {
      const size_t smem = ((size_t)bmn * a.xs + 2 * (size_t)bmn * g.Hc_s) * 8;
      if (smem <= 72 * 1024 || bmn == 16) {
        if (smem > 200 * 1024) return 1;
        return bmn == 32 ? launch_deep<DEEP_UP, 32>(a, smem, st) : launch_deep<DEEP_UP, 16>(a, smem, st);
      }
    }
  } else {
    for (int bmn : {32, 16}) {
      const size_t smem = (size_t)bmn * a.xs * 8 + (((size_t)bmn * g.n12 * 4 + 15) & ~(size_t)15);
      if (smem <= 72 * 1024 || bmn == 16) {
        if (smem > 200 * 1024) return 1;
        return bmn == 32 ? launch_deep<DEEP_DOWN, 32>(a, smem, st) : launch_deep<DEEP_DOWN, 16>(a, smem, st);
      }
    }
  }
  return 1;
}

}  // namespace hpsb
