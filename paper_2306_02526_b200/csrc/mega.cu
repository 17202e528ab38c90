// Persistent dataflow kernel for the wide levels of a shared-layout solve.
//
// The wide levels (0..dF-1) of the up and down sweeps (solver.py:243-268)
// are ~2*dF dependent level applies; as one launch each, every level pays a
// kernel drain + fill and the slowest CTA of the level (the split-K
// reducers).  Here one persistent launch runs all of them as a task list:
//
//   task = (segment = (pass, level), node group of NB nodes, 64-row block,
//           column split)
//
// in topological order (deepest level first for the up pass, root first for
// the down pass).  A task waits only for what it reads -- the up pass for the
// two children of each of its nodes, the down pass for the parents and for its
// own nodes' up results -- through per-node completion counters (one count per
// finished row block).  CTAs take tasks in increasing order from a ticket
// counter and every task depends only on lower-numbered ones, so the lowest
// unfinished task is always held by a running CTA and can run, whichever of
// the CTAs are resident (another stream's kernel may hold SMs).  The one
// exception is opt-in (HPSB_MEGA_DEDICATED=1, an exclusive GPU): the root
// pair's head tasks bound to the last CTAs of the grid.
//
// Within a task the CTA is 8 column groups x 32 threads; a thread owns two
// adjacent rows of the block and walks its group's columns of the split
// (16-byte loads of the column-major one-node panel), the groups' sums meet in
// shared memory in group order, and a split > 1 goes through workspace
// partials summed in split order by the last CTA (semaphore) -- outputs are
// bitwise reproducible.  Data produced inside the launch are read with
// ld.global.cg (L2; L1 is not coherent).  The last CTA to exit resets every
// counter for the next solve.
#include <stdio.h>

#include "hps_plan.cuh"
#include "stream.cuh"

namespace hpsb {

namespace {

constexpr int MT = 256;        // threads per CTA
constexpr int MRB = 64;        // rows per row block
constexpr int MGRP = 8;        // column groups (MT / (MRB / 2))
constexpr int MNB = 4;         // nodes per group
constexpr int MKC = 256;       // max operator columns per task (32 per thread)
constexpr int MAXSEG = 24;
constexpr int MXS = MKC + 2;   // even: 16-byte x loads (every lane of a group reads the same x: broadcasts)
constexpr int MTS = 6;         // trace stamps per task
constexpr int MU = 4;          // 16-byte operator loads per batch (two batches in flight)

struct MSeg {
  int up;                      // 1 = up pass, 0 = down pass
  int n0, nn;                  // node range [n0, n0 + nn)
  int R, K;                    // operator rows / columns
  int dmul;                    // completion counters bumped per node (1; 2 = one per child: level pairs)
  const double* op; int TR;    // one-node panel (tiles of TR rows, column-major)
  int RB, NG, S, KC;           // row blocks, node groups, splits, columns per split
  int task0, ntasks;
  // gathers / epilogue (global node numbering; k = 1)
  const double* Hc; long long Hc_s; const int *i1a, *i3a, *i2b, *i3b; int n1a, n3, n12;
  const double* jump; double inv_dt; const int* j3; const int* gidx;
  double* W3; double* Hout; double* u;
  // dataflow
  unsigned* done;              // [nodes of the level] row blocks finished
  const unsigned* wchild; int wchild_t;   // up: children's counters (level d+1), target
  const unsigned* wpar; int wpar_t;       // down: parents' counters (level d-1; wpar_sh = 2: level d-2, see the pairs)
  const unsigned* wup; int wup_t;         // down: own nodes' up counters
  int Rc, Rp, Ru;              // pn: rows per node of the waited-on segments (targets vary per node)
  double* part; unsigned* sem; // split partials [S][NG*NB][R], semaphores [NG*RB]
  // root pair: the root's down product S u_bnd needs only the Dirichlet data,
  // so its tasks run at the head of the list;
  // the root's up tasks (w3 = X33^-1 r3) and down tasks share one semaphore per
  // row block and the last arriver writes u3 = S u_bnd + w3 = sum of both
  // partial sets (down splits first, then up splits)
  int pair;
  const double *pdn, *pup; int Sdn, Sup;
  // the root's up segment with the Dirichlet product S u_bnd precomputed for
  // this solve (hps_root_dirichlet): the emitting task also writes u3 = w3 + pre
  const double* rootpre;
};

struct MProg {
  int nseg, ntasks;
  int head, dedicated;          // opt-in (mega_dedicated): the first `head` tasks (the root's down
                                // product) run on the last `dedicated` CTAs; every other task is
                                // taken by ticket.  Default 0 / 0: every task by ticket
  unsigned* ticket;             // next task after the head (reset at exit)
  unsigned long long* trace;    // debug (HPSB_MEGA_TRACE): per task start / inputs ready / staged /
                                // streamed / emitted / end, ns (MTS stamps)
  unsigned* reset; int nreset;  // counters to zero at exit (incl. the exit counter at the end)
  MSeg s[MAXSEG];
};

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void wait_count(const unsigned* p, unsigned target) {
  long long spins = 0;
  while (ld_acquire(p) < target) {
    __nanosleep(32);
    if (++spins > (1LL << 24)) __trap();  // a lost dependency must fail, not hang the GPU
  }
}

// sum of n split partials p[s * stride] in split order, eight loads in flight
__device__ __forceinline__ double sum_splits(const double* p, size_t stride, int n, double y) {
  for (int s0 = 0; s0 < n; s0 += 8) {
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = s0 + u < n ? __ldcg(p + (size_t)(s0 + u) * stride) : 0.0;
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (s0 + u < n) y += v[u];
  }
  return y;
}

// pn: number of 64-row blocks of a row space of R rows per node that touch node n
__device__ __forceinline__ unsigned blocks_of(int n, int R) {
  return (unsigned)(((n + 1) * R - 1) / MRB - (n * R) / MRB + 1);
}

__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// PN: per-node operators -- a task's 64 rows tile the level's row space
// (node * R + r) and may span up to MNB nodes; NG = 1
template <bool PN>
__global__ void __launch_bounds__(MT) k_mega(MProg p, unsigned* exit_count) {
  __shared__ __align__(16) double xs[MNB][MXS];              // the task's inputs
  __shared__ double red[MGRP][MNB][MRB];       // column-group partial sums
  __shared__ int sidx[MNB][MKC];               // gather indices (down: per node; up: i3a / i3b rows 0 / 1)
  __shared__ unsigned s_last;
  const int tid = threadIdx.x, grp = tid >> 5, q = tid & 31;
  pdl_wait();
  const int G = gridDim.x, KR = p.dedicated;
  const bool ded = KR > 0 && (int)blockIdx.x >= G - KR;
  // the dedicated CTAs first take the head tasks round-robin, then every CTA
  // takes the remaining tasks in list order from a ticket counter (each task
  // depends only on lower-numbered ones, all taken by resident CTAs)
  __shared__ int s_ticket;
  int t = ded ? (int)blockIdx.x - (G - KR) : p.ntasks;
  for (;;) {
    if (!(ded && t < p.head)) {
      __syncthreads();
      if (tid == 0) s_ticket = p.head + (int)atomicAdd(p.ticket, 1u);
      __syncthreads();
      t = s_ticket;
      if (t >= p.ntasks) break;
    }
    int si = 0;
    while (t >= p.s[si].task0 + p.s[si].ntasks) ++si;
    const MSeg& g = p.s[si];
    int local = t - g.task0;
    const int split = local % g.S;
    local /= g.S;
    const int rb = local % g.RB, ng = local / g.RB;
    // rows of the task: shared -> rows of the one-node operator for MNB nodes;
    // pn -> 64 rows of the level's row space, nodes [node0, node0 + nv)
    const int nrows = PN ? g.nn * g.R : g.R;
    int node0, nv;
    if (PN) {
      const int r0 = rb * MRB, r1 = min(r0 + MRB, nrows) - 1;
      node0 = g.n0 + r0 / g.R;
      nv = r1 / g.R - r0 / g.R + 1;
    } else {
      node0 = g.n0 + ng * MNB;
      nv = min(MNB, g.n0 + g.nn - node0);
    }
    if (p.trace && tid == 0) p.trace[MTS * t] = gtime();
    // ---- nothing below depends on the inputs: the operator's first batch,
    // the gather indices and this thread's epilogue index are in flight while
    // the task waits for its inputs
    const int c0 = split * g.KC, cw = min(g.KC, g.K - c0);
    // column groups of an even width (16-byte x loads in the shared-operator stream)
    const int cg = ((cw + MGRP - 1) / MGRP + 1) & ~1, a0 = min(cw, grp * cg), a1 = min(cw, a0 + cg);
    const int row = rb * MRB + 2 * q;  // rows row, row + 1 (R and TR are even: both valid or both padding)
    const bool rows_ok = row < nrows;
    const int cs = g.TR / 2;           // column stride in double2
    const int rowc = min(row, nrows - 2);
    const int jn = PN ? g.n0 + rowc / g.R - node0 : 0;  // pn: the node of both rows (R even)
    const double2* M =
        reinterpret_cast<const double2*>(g.op + (size_t)(rowc / g.TR) * g.K * g.TR + rowc % g.TR) + (size_t)c0 * cs;
    double2 A[MU];
    if (rows_ok && a1 - a0 >= MU) load_batch<MU>(A, M, cs, a0);
    if (g.up) {
      for (int i = tid; i < 2 * cw; i += MT) sidx[i / cw][i % cw] = (i < cw ? g.i3a : g.i3b)[c0 + i % cw];
    } else {
      for (int i = tid; i < nv * cw; i += MT) sidx[i / cw][i % cw] = g.gidx[(long long)(node0 + i / cw) * g.n12 + c0 + i % cw];
    }
    // one output per thread (shared: MT = MNB * MRB); pn: the block's 64 rows
    int oj, orow;
    bool ovalid;
    if (PN) {
      const int gr = min(rb * MRB + tid, nrows - 1);
      oj = g.n0 + gr / g.R - node0;
      orow = gr % g.R;
      ovalid = tid < MRB && rb * MRB + tid < nrows;
    } else {
      oj = tid / MRB;
      orow = rb * MRB + tid % MRB;
      ovalid = oj < nv && orow < g.R;
    }
    int oidx = 0;  // epilogue index: up -> child flux position (flux rows), down -> global DOF
    if (ovalid) {
      if (g.up) {
        const int r = orow - g.n3;
        if (r >= 0) oidx = r < g.n1a ? g.i1a[r] : g.i2b[r - g.n1a];
      } else {
        oidx = g.j3[(long long)(node0 + oj) * g.n3 + orow];
      }
    }
    // ---- dependencies
    if (g.up) {
      if (g.wchild && tid < 2 * nv) {
        const int ch = 2 * node0 + tid;
        wait_count(g.wchild + ch, PN ? blocks_of(ch, g.Rc) : g.wchild_t);
      }
    } else {
      if (g.wpar && tid < nv) {
        const int pa = (node0 + tid) / 2;
        wait_count(g.wpar + pa, PN ? blocks_of(pa, g.Rp) : g.wpar_t);
      }
      if (g.wup && tid >= 32 && tid < 32 + nv) {
        const int nd = node0 + tid - 32;
        wait_count(g.wup + nd, PN ? blocks_of(nd, g.Ru) : g.wup_t);
      }
    }
    __syncthreads();
    if (p.trace && tid == 0) p.trace[MTS * t + 1] = gtime();
    // the epilogue's additive term (child flux / w3) is ready now: load it
    // while the inputs are gathered and the columns streamed
    double oadd = 0.0;
    if (ovalid && !g.pair) {
      const int node = node0 + oj;
      if (g.up) {
        const int rr = orow - g.n3;
        if (rr >= 0) {
          const double* Ha = g.Hc + (long long)(2 * node) * g.Hc_s;
          oadd = rr < g.n1a ? __ldcg(Ha + oidx) : __ldcg(Ha + g.Hc_s + oidx);
        }
      } else if (g.W3) {
        oadd = __ldcg(g.W3 + (long long)node * g.n3 + orow);
      }
    }
    // ---- stage the group's inputs for this split's columns
    {  // every thread's loads issued before any is consumed
      constexpr int GE = MNB * MKC / MT;
      double va[GE], vb[GE];
#pragma unroll
      for (int u = 0; u < GE; ++u) {
        const int e = tid + u * MT, j = e / cw, col = e - j * cw;
        va[u] = 0.0; vb[u] = 0.0;
        if (e < MNB * cw && j < nv) {
          if (g.up) {
            const double* Ha = g.Hc + (long long)(2 * (node0 + j)) * g.Hc_s;
            vb[u] = __ldcg(Ha + g.Hc_s + sidx[1][col]);
            va[u] = __ldcg(Ha + sidx[0][col]);
          } else {
            vb[u] = __ldcg(g.u + sidx[j][col]);
          }
        }
      }
#pragma unroll
      for (int u = 0; u < GE; ++u) {
        const int e = tid + u * MT, j = e / cw, col = e - j * cw;
        if (e < MNB * cw) {
          double v = vb[u] - va[u];
          if (g.up && g.jump && j < nv) v = v - g.inv_dt * g.jump[g.j3[(long long)(node0 + j) * g.n3 + c0 + col]];
          xs[j][col] = v;
        }
      }
    }
    __syncthreads();
    if (p.trace && tid == 0) p.trace[MTS * t + 2] = gtime();
    // ---- stream: group grp walks columns [a0, a1) of the split for rows 2q, 2q+1 of the block
    if (PN) {
      double acc0[1] = {0.0}, acc1[1] = {0.0};
      if (rows_ok) stream_cols<1, MU>(A, M, cs, a0, a1, &xs[0][0], jn * MXS, jn * MXS, MXS, acc0, acc1);
      red[grp][0][2 * q] = acc0[0];
      red[grp][0][2 * q + 1] = acc1[0];
    } else {
      double acc0[MNB], acc1[MNB];
#pragma unroll
      for (int j = 0; j < MNB; ++j) { acc0[j] = 0.0; acc1[j] = 0.0; }
      if (rows_ok) stream_pairs_nb<MNB, MU>(A, M + (size_t)a0 * cs, cs, a1 - a0, &xs[0][a0], MXS, acc0, acc1);
#pragma unroll
      for (int j = 0; j < MNB; ++j) {
        red[grp][j][2 * q] = acc0[j];
        red[grp][j][2 * q + 1] = acc1[j];
      }
    }
    __syncthreads();
    if (p.trace && tid == 0) p.trace[MTS * t + 3] = gtime();
    // ---- group sums (in group order), then split partials or the epilogue
    const int r = tid % MRB, rj = PN ? 0 : oj;
    double y = 0.0;
#pragma unroll
    for (int gg = 0; gg < MGRP; ++gg) y += red[gg][rj][r];
    bool emit_now = true;
    if (g.S > 1 || g.pair) {
      const size_t slot = PN ? (size_t)rb * MRB + r : (size_t)(ng * MNB + oj) * g.R + orow;
      const size_t pstride = PN ? (size_t)g.RB * MRB : (size_t)g.NG * MNB * g.R;
      if (ovalid) g.part[(size_t)split * pstride + slot] = y;
      // barrier + one thread's acq_rel atomic publishes the CTA's partials; the
      // last arriver's barrier after it orders the CTA's partial reads after them
      __syncthreads();
      const unsigned total = g.pair ? (unsigned)(g.Sdn + g.Sup) : (unsigned)g.S;
      if (tid == 0) s_last = atom_add_acq_rel(g.sem + ng * g.RB + rb, 1u) == total - 1;
      __syncthreads();
      emit_now = s_last;
      if (emit_now) {
        y = 0.0;
        if (ovalid) {
          if (g.pair) {
            y = sum_splits(g.pdn + slot, pstride, g.Sdn, y);
            y = sum_splits(g.pup + slot, pstride, g.Sup, y);
          } else {
            y = sum_splits(g.part + slot, pstride, g.S, y);
          }
        }
      }
    }
    if (emit_now && g.pair) {
      if (ovalid) g.u[g.j3[(long long)(node0 + oj) * g.n3 + orow]] = y;
    } else if (emit_now) {
      if (ovalid) {
        const int node = node0 + oj;
        if (g.up) {
          if (orow < g.n3) {
            g.W3[(long long)node * g.n3 + orow] = y;
            if (g.rootpre) g.u[g.j3[orow]] = y + g.rootpre[orow];
          } else {
            g.Hout[(long long)node * g.n12 + orow - g.n3] = oadd + y;
          }
        } else {
          g.u[oidx] = y + oadd;
        }
      }
    }
    if (emit_now) {
      __syncthreads();
      if (tid < nv) {
        unsigned* dn = g.done + (node0 + tid) * g.dmul;
        red_add_release(dn, 1u);
        if (g.dmul == 2) red_add_release(dn + 1, 1u);
      }
      if (p.trace && tid == 0) p.trace[MTS * t + 4] = gtime();
    }
    __syncthreads();  // xs / red / sidx are reused by the next task
    if (p.trace && tid == 0) p.trace[MTS * t + 5] = gtime();
    if (ded && t < p.head) t += KR;
  }
  // the last CTA out resets the counters for the next solve
  __syncthreads();
  if (tid == 0) s_last = atom_add_acq_rel(exit_count, 1u) == gridDim.x - 1;
  __syncthreads();
  if (s_last) {
    for (int i = tid; i < p.nreset; i += MT) p.reset[i] = 0u;
    __syncthreads();
    if (tid == 0) *exit_count = 0u;
  }
}

}  // namespace

// ---- the root's Dirichlet product for several solves at once
// Y[s][r] = sum_c S_root[r][c] fb_s[bpos[c]], s < ns <= RDN: the root's down
// operator (the largest of the solve) streamed once per step instead of once
// per stage solve.  Task = (64-row block, 256-column split): 8 column groups x
// 32 lanes x two rows, ns accumulators per row; split partials summed in split
// order by k_root_sum (bitwise reproducible).
constexpr int RDN = 8;
constexpr int RDK = 512;

__global__ void __launch_bounds__(MT) k_root_dir(const double* __restrict__ S, int R, int C, int TR,
                                                 const int* __restrict__ bpos, const double* __restrict__ fb,
                                                 long long ld_f, int ns, double* __restrict__ part) {
  static_assert(MGRP * MRB <= RDK, "the group sums reuse the x buffer");
  __shared__ __align__(16) double buf[RDN * RDK];
  double (*xs)[RDK] = reinterpret_cast<double (*)[RDK]>(buf);           // inputs, then ...
  double (*red)[RDN][MRB] = reinterpret_cast<double (*)[RDN][MRB]>(buf);  // ... the group sums
  const int rb = blockIdx.x, split = blockIdx.y, tid = threadIdx.x, grp = tid >> 5, q = tid & 31;
  const int c0 = split * RDK, cw = min(RDK, C - c0);
  for (int i = tid; i < ns * cw; i += MT) {
    const int s = i / cw, c = i - s * cw;
    xs[s][c] = fb[s * ld_f + bpos[c0 + c]];
  }
  __syncthreads();
  const int cg = ((cw + MGRP - 1) / MGRP + 1) & ~1, a0 = min(cw, grp * cg), a1 = min(cw, a0 + cg);
  const int row = rb * MRB + 2 * q, rowc = min(row, R - 2);
  const double2* M = reinterpret_cast<const double2*>(S + (size_t)(rowc / TR) * C * TR + rowc % TR) +
                     (size_t)(c0 + a0) * (TR / 2);
  double acc0[RDN], acc1[RDN];
#pragma unroll
  for (int j = 0; j < RDN; ++j) { acc0[j] = 0.0; acc1[j] = 0.0; }
  if (row < R) {
    int c = a0;
    for (; c + 4 <= a1; c += 4) {  // four column loads in flight
      double2 m[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) { m[u] = __ldcs(M); M += TR / 2; }
#pragma unroll
      for (int u = 0; u < 4; ++u)
#pragma unroll
        for (int j = 0; j < RDN; ++j) {
          if (j < ns) {
            acc0[j] = fma(m[u].x, xs[j][c + u], acc0[j]);
            acc1[j] = fma(m[u].y, xs[j][c + u], acc1[j]);
          }
        }
    }
    for (; c < a1; ++c) {
      const double2 m = __ldcs(M);
      M += TR / 2;
#pragma unroll
      for (int j = 0; j < RDN; ++j) {
        if (j < ns) {
          acc0[j] = fma(m.x, xs[j][c], acc0[j]);
          acc1[j] = fma(m.y, xs[j][c], acc1[j]);
        }
      }
    }
  }
  __syncthreads();  // every x read is done: the buffer takes the group sums
#pragma unroll
  for (int j = 0; j < RDN; ++j) {
    red[grp][j][2 * q] = acc0[j];
    red[grp][j][2 * q + 1] = acc1[j];
  }
  __syncthreads();
  for (int i = tid; i < ns * MRB; i += MT) {
    const int j = i / MRB, r = i - j * MRB;
    double y = 0.0;
#pragma unroll
    for (int gg = 0; gg < MGRP; ++gg) y += red[gg][j][r];
    if (rb * MRB + r < R) part[((size_t)split * ns + j) * R + rb * MRB + r] = y;
  }
}

__global__ void k_root_sum(const double* __restrict__ part, int nsplit, int ns, int R, double* __restrict__ out,
                           long long ld_out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= ns * R) return;
  const int j = i / R, r = i - j * R;
  double y = 0.0;
  for (int s0 = 0; s0 < nsplit; s0 += 8) {  // eight loads in flight, summed in split order
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) v[u] = s0 + u < nsplit ? part[((size_t)(s0 + u) * ns + j) * R + r] : 0.0;
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (s0 + u < nsplit) y += v[u];
  }
  out[j * ld_out + r] = y;
}

size_t root_dirichlet_scratch(const Plan& P, int ns) {
  if (P.depth == 0) return 0;
  return (size_t)((P.lv[0].n12 + RDK - 1) / RDK) * ns * P.lv[0].n3 * 8;
}

int root_dirichlet(const Ops& ops, int ns, const double* fb, long long ld_f, double* out, long long ld_out,
                   double* scratch, cudaStream_t st) {
  const Plan& P = *ops.plan;
  if (P.depth == 0 || !P.root_bpos || ns <= 0 || ns > RDN) {
    set_error("root_dirichlet: not available (depth %d, %d rows)", P.depth, ns);
    return -1;
  }
  const Panel& pn = ops.lo[0].S;
  if (!pn.base || pn.TS != pn.TR || (pn.TR & 1) || pn.R != P.lv[0].n3 || pn.C != P.lv[0].n12) {
    set_error("root_dirichlet: unexpected root operator layout");
    return -1;
  }
  const int R = pn.R, C = pn.C, nsplit = (C + RDK - 1) / RDK;
  HPSB_CUDA(launch_plain(k_root_dir, dim3((unsigned)cdiv(R, MRB), (unsigned)nsplit), dim3(MT), 0, st, pn.base, R,
                         C, pn.TR, (const int*)P.root_bpos, fb, ld_f, ns, scratch));
  HPSB_LAUNCH_CHECK();
  HPSB_CUDA(launch_plain(k_root_sum, dim3((unsigned)cdiv((long long)ns * R, 256)), dim3(256), 0, st,
                         (const double*)scratch, nsplit, ns, R, out, ld_out));
  HPSB_LAUNCH_CHECK();
  return 0;
}

static bool pair_enabled() {
  static const bool on = [] {
    const char* e = getenv("HPSB_NO_ROOT_PAIR");
    return !(e && e[0] == '1');
  }();
  return on;
}

// The root pair's head tasks on dedicated CTAs stream the root's down product
// beside the up sweep (12 us per plain C2 solve faster), but a level-1 down
// task then spins on work bound to specific CTAs, which needs every CTA of the
// grid resident at once: only on an exclusive GPU, by opt-in.  By default the
// head tasks are simply the first tickets (deadlock-free on a shared GPU).
static bool mega_dedicated() {
  static const bool on = [] {
    const char* e = getenv("HPSB_MEGA_DEDICATED");
    return e && e[0] == '1';
  }();
  return on;
}

bool mega_enabled() {
  static const bool on = [] {
    const char* e = getenv("HPSB_NO_MEGA");
    return !(e && e[0] == '1');
  }();
  return on;
}

// Levels [0, mega_depth) may run in the persistent launch.  Shared operators:
// all.  Per-node operators: the persistent kernel streams ~8% below the
// per-level panel kernel but saves a level's drain / fill (~5 us), which pays
// only while a level's operators are small; levels from the first one whose
// up or down operators exceed HPSB_PN_MEGA_MB (default 256 MB) down to the
// leaves run as per-level launches.
int mega_depth(const Ops& ops) {
  const Plan& P = *ops.plan;
  if (ops.shared_levels) return P.depth;
  const char* e = getenv("HPSB_PN_MEGA_MB");  // read per call: tests lower it to exercise k_panel
  const double cap = (e ? atof(e) : 256.0) * 1048576.0;
  int d = 0;
  for (; d < P.depth; ++d) {
    const Level& lv = P.lv[d];
    const double up = (double)lv.c * (lv.n3 + (d ? lv.n12 : 0)) * lv.n3 * 8.0;
    const double dn = (double)lv.c * lv.n3 * lv.n12 * 8.0;
    if (std::max(up, dn) > cap) break;
  }
  return d;
}

// ---- level pairs of the down sweep ------------------------------------------
// The down sweep is a chain of dependent level phases (~9 us each whatever
// their size).  For a pair (d, d + 1) the children's interface values follow
// from the parent's boundary values directly: with u_bnd(c) = [u_bnd(p)[A];
// u3(p)[B]] and u3(p) = S_p u_bnd(p) + w3(p),
//   u3(c) = (S_c[:, A] E_A + S_c[:, B] S_p) u_bnd(p) + S_c[:, B] w3(p) + w3(c),
// so level d + 1 runs in the same phase as level d: one down segment over the
// level-d nodes with the stacked operator C1 = [C1_alpha; C1_beta], and (off the
// critical path, during the up sweep) one segment for the adjusted load
// w3c(c) = w3(c) + S_c[:, B] w3(p).  Both are ordinary down segments of
// k_mega: only their tables differ.
static int pair_min_level() {
  static const int v = [] {
    if (const char* e = getenv("HPSB_NO_MEGA_PAIRS")) if (e[0] == '1') return 1 << 20;
    const char* e = getenv("HPSB_MEGA_PAIR_MIN");
    return e ? std::max(1, atoi(e)) : 2;
  }();
  return v;
}

__global__ void k_pair_gather(const double* __restrict__ Sc, int n3c, int n12c, const int* __restrict__ i3a,
                              const int* __restrict__ i3b, int n3p, double* __restrict__ PU) {
  const long long n = 2LL * n3c * n3p;
  for (long long i = blockIdx.x * 256LL + threadIdx.x; i < n; i += gridDim.x * 256LL) {
    const int t = (int)(i % n3p), r = (int)(i / n3p);
    PU[i] = r < n3c ? Sc[(long long)r * n12c + i3a[t]] : Sc[(long long)(r - n3c) * n12c + i3b[t]];
  }
}

__global__ void k_pair_scatter(const double* __restrict__ Sc, int n3c, int n12c, const int* __restrict__ i1a,
                               const int* __restrict__ i2b, int n1a, int n12p, double* __restrict__ C1) {
  const long long n = 2LL * n3c * n12p;
  for (long long i = blockIdx.x * 256LL + threadIdx.x; i < n; i += gridDim.x * 256LL) {
    const int col = (int)(i % n12p), r = (int)(i / n12p);
    if (r < n3c) {
      if (col < n1a) C1[i] += Sc[(long long)r * n12c + i1a[col]];
    } else if (col >= n1a) {
      C1[i] += Sc[(long long)(r - n3c) * n12c + i2b[col - n1a]];
    }
  }
}

int mega_pairs_prepare(Ops& O, cudaStream_t st) {
  const Plan& P = *O.plan;
  O.pairs.clear();
  if (!O.shared_levels || P.nparts != 1) return 0;
  Workspace w0;
  carve_workspace(P, 1, reinterpret_cast<void*>((uintptr_t)4096), w0);
  for (int d = pair_min_level(); d + 1 < P.dF && d + 1 < P.depth; ++d) {
    const Level &lp = P.lv[d], &lc = P.lv[d + 1];
    const LevelOps &op = O.lo[d], &oc = O.lo[d + 1];
    if (!op.S.base || !oc.S.base || op.S.c != 1 || oc.S.c != 1) continue;
    const int n3p = lp.n3, n12p = lp.n12, n3c = lc.n3, n12c = lc.n12, n1a = lp.n1a;
    if (lp.nbc != n12c || lc.c != 2 * lp.c) continue;
    {  // the children's boundary order against the parent's (node 0 / its two children)
      std::vector<int> gp(n12p), jp(n3p), ga(n12c), gb(n12c);
      HPSB_CUDA(cudaMemcpyAsync(gp.data(), lp.gidx_bnd, n12p * 4, cudaMemcpyDeviceToHost, st));
      HPSB_CUDA(cudaMemcpyAsync(jp.data(), lp.j3, n3p * 4, cudaMemcpyDeviceToHost, st));
      HPSB_CUDA(cudaMemcpyAsync(ga.data(), lc.gidx_bnd, n12c * 4, cudaMemcpyDeviceToHost, st));
      HPSB_CUDA(cudaMemcpyAsync(gb.data(), lc.gidx_bnd + n12c, n12c * 4, cudaMemcpyDeviceToHost, st));
      HPSB_CUDA(cudaStreamSynchronize(st));
      bool ok = (int)lp.h_i1a.size() == n1a && (int)lp.h_i3a.size() == n3p && (int)lp.h_i3b.size() == n3p &&
                (int)lp.h_i2b.size() == n12p - n1a;
      for (int r = 0; ok && r < n1a; ++r) ok = ga[lp.h_i1a[r]] == gp[r];
      for (int r = 0; ok && r < n12p - n1a; ++r) ok = gb[lp.h_i2b[r]] == gp[n1a + r];
      for (int t = 0; ok && t < n3p; ++t) ok = ga[lp.h_i3a[t]] == jp[t] && gb[lp.h_i3b[t]] == jp[t];
      if (!ok) continue;
    }
    MegaPair mp;
    mp.d = d;
    mp.C1 = make_panel(1, 2 * n3c, n12p);
    mp.PU = make_panel(1, 2 * n3c, n3p);
    const size_t nS = (size_t)n3c * n12c + (size_t)n3p * n12p, nPU = (size_t)2 * n3c * n3p,
                 nC = (size_t)2 * n3c * n12p;
    double *tmp = nullptr, *pan = nullptr;
    int* tab = nullptr;
    if (cudaMalloc(&tmp, (nS + nPU + nC) * 8) != cudaSuccess) { cudaGetLastError(); break; }
    if (cudaMalloc(&pan, (mp.C1.total() + mp.PU.total()) * 8) != cudaSuccess ||
        cudaMalloc(&tab, ((size_t)lp.c * n3p + (size_t)lp.c * 2 * n3c) * 4) != cudaSuccess) {
      cudaGetLastError();
      cudaFree(tmp);
      if (pan) cudaFree(pan);
      break;
    }
    O.aux.push_back(pan);
    O.aux.push_back(tab);
    mp.C1.base = pan;
    mp.PU.base = pan + mp.C1.total();
    double *Sc = tmp, *Sp = tmp + (size_t)n3c * n12c, *PU = tmp + nS, *C1 = PU + nPU;
    int rc = unpack_panel(oc.S, 0, 0, n3c, Sc, st);
    if (!rc) rc = unpack_panel(op.S, 0, 0, n3p, Sp, st);
    if (rc) { cudaFree(tmp); return rc; }
    k_pair_gather<<<(unsigned)std::min<size_t>((nPU + 255) / 256, 2368), 256, 0, st>>>(Sc, n3c, n12c, lp.i3a, lp.i3b,
                                                                                       n3p, PU);
    GemmArgs g{};
    g.M = 2 * n3c; g.N = n12p; g.K = n3p; g.alpha = 1.0; g.beta = 0.0;
    g.A = PU; g.lda = n3p; g.B = Sp; g.ldb = n12p; g.C = C1; g.ldc = n12p; g.batch = 1;
    rc = gemm(g, st);
    if (rc) { cudaFree(tmp); return rc; }
    k_pair_scatter<<<(unsigned)std::min<size_t>((nC + 255) / 256, 2368), 256, 0, st>>>(Sc, n3c, n12c, lp.i1a, lp.i2b,
                                                                                       n1a, n12p, C1);
    HPSB_CUDA(cudaMemsetAsync(pan, 0, (mp.C1.total() + mp.PU.total()) * 8, st));
    rc = pack_panel(C1, 0, n12p, mp.C1, st);
    if (!rc) rc = pack_panel(PU, 0, n3p, mp.PU, st);
    if (rc) { cudaFree(tmp); return rc; }
    // tables of the adjusted-load segment (inputs and outputs relative to W3[d])
    mp.off = w0.W3c[d + 1] - w0.W3[d];
    std::vector<int> h((size_t)lp.c * n3p + (size_t)lp.c * 2 * n3c);
    for (size_t i = 0; i < (size_t)lp.c * n3p; ++i) h[i] = (int)i;
    for (size_t i = 0; i < (size_t)lp.c * 2 * n3c; ++i) h[(size_t)lp.c * n3p + i] = (int)(mp.off + (long long)i);
    HPSB_CUDA(cudaMemcpyAsync(tab, h.data(), h.size() * 4, cudaMemcpyHostToDevice, st));
    HPSB_CUDA(cudaStreamSynchronize(st));
    cudaFree(tmp);
    mp.iota = tab;
    mp.out = tab + (size_t)lp.c * n3p;
    O.pairs.push_back(mp);
  }
  return 0;
}

static const MegaPair* pair_at(const Ops& ops, int d) {
  for (const MegaPair& mp : ops.pairs)
    if (mp.d == d) return &mp;
  return nullptr;
}

// rows / columns -> row blocks, node groups, splits of a shared-operator segment
static void seg_dims(int R, int K, int nn, int& RB, int& NG, int& S, int& KC) {
  RB = (R + MRB - 1) / MRB;
  NG = (nn + MNB - 1) / MNB;
  S = std::max(1, (K + MKC - 1) / MKC);
  KC = (K + S - 1) / S;
  S = (K + KC - 1) / KC;
}

// Counter / partial space of the workspace's mega region for one plan: every
// wide level's nodes twice (up, down), semaphores and split partials of every
// possible segment.  Sized generously from the plan alone.
static void mega_dims(const Level& lv, bool root, bool up, int nn, int& RB, int& NG, int& S, int& KC, int& R,
                      int& K, bool pn = false) {
  R = up ? lv.n3 + (root ? 0 : lv.n12) : lv.n3;
  K = up ? lv.n3 : lv.n12;
  RB = pn ? (int)(((long long)nn * R + MRB - 1) / MRB) : (R + MRB - 1) / MRB;
  NG = pn ? 1 : (nn + MNB - 1) / MNB;
  S = std::max(1, (K + MKC - 1) / MKC);
  KC = (K + S - 1) / S;
  S = (K + KC - 1) / KC;
}

void mega_scratch(const Plan& P, size_t& counters, size_t& part_doubles) {
  counters = 2;  // exit counter, task ticket
  part_doubles = 0;
  for (int d = 0; d < P.depth; ++d) {
    const Level& lv = P.lv[d];
    counters += 2 * (size_t)lv.c;
    for (int up = 0; up < 2; ++up) {
      int RB, NG, S, KC, R, K;
      mega_dims(lv, d == 0, up, lv.c, RB, NG, S, KC, R, K);
      size_t sems = (size_t)RB * NG, parts = (size_t)S * NG * MNB * R;
      mega_dims(lv, d == 0, up, lv.c, RB, NG, S, KC, R, K, true);  // per-node row blocks
      sems = std::max(sems, (size_t)RB);
      parts = std::max(parts, (size_t)S * RB * MRB);
      counters += sems;
      if (S > 1 || d == 0) part_doubles += parts;  // the root pair always uses partials
    }
    if (d >= 1 && d + 1 < P.depth) {  // a level pair (d, d + 1): two more segments over the level-d nodes
      const int R2 = 2 * P.lv[d + 1].n3;
      counters += (size_t)lv.c;       // completion counters of the adjusted-load segment
      for (int K : {lv.n12, lv.n3}) {
        int RB, NG, S, KC;
        seg_dims(R2, K, lv.c, RB, NG, S, KC);
        counters += (size_t)RB * NG;
        if (S > 1) part_doubles += (size_t)S * NG * MNB * R2;
      }
    }
  }
}

// resident CTAs of the dataflow kernel on this device
static int mega_max_ctas(bool pnm) {
  static int max_ctas_pn[2] = {0, 0};
  int& max_ctas = max_ctas_pn[pnm];
  if (!max_ctas) {
    int per_sm = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pnm ? k_mega<true> : k_mega<false>, MT, 0) !=
        cudaSuccess) {
      cudaGetLastError();
      per_sm = 1;
    }
    int dev = 0, sms = kNumSMs;
    if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    max_ctas = std::max(1, per_sm) * sms;
  }
  return max_ctas;
}

// Runs the up levels [u0, u1) (deepest first) and the down levels [d0, d1)
// (root first) of nodes range(level) as one launch.  Returns 1 when the
// levels are not eligible (caller falls back to per-level launches).
int mega_levels(const Ops& ops, const Workspace& ws, int u0, int u1, int d0, int d1, int part0, int part1,
                const double* Hleaf, long long hs, const double* jump, double inv_dt, bool has_w3, double* u,
                cudaStream_t st, const double* root_pre) {
  const Plan& P = *ops.plan;
  if (!mega_enabled() || !ws.mega_cnt) return 1;
  // root_pre: the root's down product is precomputed, so the root's up tasks
  // write its interface and level 1's down tasks wait on them (no root pair)
  const bool rpre = root_pre && u0 == 0 && u1 > 0 && d0 == 0 && d1 > 0 && has_w3 && !jump;
  const bool pnm = !ops.shared_levels;  // per-node operators
  MProg p{};
  // counter carve: [exit][per level: up nodes, down nodes][sems...]
  unsigned* cnt = ws.mega_cnt;
  unsigned* exit_count = cnt;
  std::vector<unsigned*> dup(P.depth), ddn(P.depth);
  unsigned* c = cnt + 1;
  for (int d = 0; d < P.depth; ++d) { dup[d] = c; c += P.lv[d].c; ddn[d] = c; c += P.lv[d].c; }
  double* part = ws.mega_part;
  int task = 0;
  // level pairs of the down sweep (whole shared-layout solves with a body load)
  const bool pairs_on = !pnm && !ops.pairs.empty() && P.nparts == 1 && u0 == 0 && d0 == 0 && u1 == d1 && has_w3;
  // pairs are taken greedily from the top while both segments of the phase fit one round of
  // the resident CTAs: a phase that needs a second round of tasks gains nothing (measured)
  std::vector<const MegaPair*> sel(P.depth + 2, nullptr);
  if (pairs_on) {
    static const double frac = [] { const char* e = getenv("HPSB_MEGA_PAIR_FRAC"); return e ? atof(e) : 1.0; }();
    for (int d = 1; d + 1 < d1;) {
      const MegaPair* mp = pair_at(ops, d);
      if (mp && ws.W3c[d + 1] && ws.W3c[d + 1] - ws.W3[d] == mp->off) {
        int RB, NG, S, KC, R, K, RB2, NG2, S2, KC2;
        mega_dims(P.lv[d], d == 0, false, P.lv[d].c, RB, NG, S, KC, R, K);
        seg_dims(2 * P.lv[d + 1].n3, P.lv[d].n12, P.lv[d].c, RB2, NG2, S2, KC2);
        if ((double)RB * NG * S + (double)RB2 * NG2 * S2 <= frac * mega_max_ctas(false)) {
          sel[d] = mp;
          d += 2;
          continue;
        }
      }
      ++d;
    }
  }
  auto pair_parent = [&](int d) -> const MegaPair* { return d >= 1 && d + 1 < d1 ? sel[d] : nullptr; };
  std::vector<unsigned*> dpu(P.depth, nullptr);  // completion counters of the adjusted-load segments
  std::vector<int> rb_pu(P.depth, 0), rb_c1(P.depth, 0);
  // a segment over the level-d nodes with its own operator and tables (the pairs)
  auto add_custom = [&](int d, const Panel& pn, int K, const int* gidx, const int* j3, const double* W3add,
                        double* uvec, unsigned* done, int dmul) -> MSeg* {
    if (p.nseg >= MAXSEG) return nullptr;
    const Level& lv = P.lv[d];
    MSeg& g = p.s[p.nseg];
    g.up = 0; g.dmul = dmul;
    g.n0 = 0; g.nn = lv.c;
    g.R = pn.R; g.K = K;
    seg_dims(g.R, g.K, g.nn, g.RB, g.NG, g.S, g.KC);
    if (pn.C != K || g.KC > MKC || pn.TS != pn.TR || (pn.TR & 1)) return nullptr;
    g.op = pn.base; g.TR = pn.TR;
    g.task0 = task; g.ntasks = g.RB * g.NG * g.S;
    task += g.ntasks;
    g.n3 = pn.R; g.n12 = K;
    g.gidx = gidx; g.j3 = j3;
    g.W3 = const_cast<double*>(W3add);
    g.u = uvec;
    g.done = done;
    g.sem = c; c += (size_t)g.RB * g.NG;
    if (g.S > 1) { g.part = part; part += (size_t)g.S * g.NG * MNB * g.R; }
    ++p.nseg;
    return &g;
  };
  auto add = [&](int d, bool up) -> bool {
    if (p.nseg >= MAXSEG) return false;
    const Level& lv = P.lv[d];
    const LevelOps& lo = ops.lo[d];
    const Panel& pn = up ? lo.Up : lo.S;
    if (!pn.base || pn.c != (pnm ? lv.c : 1) || pn.parts != 1 || pn.TS != pn.TR || (pn.TR & 1) ||
        (pnm && pn.TR % MRB))
      return false;
    MSeg& g = p.s[p.nseg];
    int n0 = 0, n1 = lv.c;  // levels >= lstar: the parts' nodes
    if (d >= P.lstar) { n0 = part0 * (lv.c / P.nparts); n1 = part1 * (lv.c / P.nparts); }
    if (pnm && n0 != 0) return false;  // per-node panels of a part range: per-level launches
    g.up = up;
    g.dmul = 1;
    g.n0 = n0; g.nn = n1 - n0;
    mega_dims(lv, d == 0, up, g.nn, g.RB, g.NG, g.S, g.KC, g.R, g.K, pnm);
    if (g.R != pn.R || g.K != pn.C || g.KC > MKC) return false;
    // pn: both rows of a thread in one node (R even), a row block spans <= MNB nodes
    if (pnm && ((g.R & 1) || (MRB - 2) / g.R + 2 > MNB)) return false;
    g.op = pn.base; g.TR = pn.TR;
    g.task0 = task; g.ntasks = g.RB * g.NG * g.S;
    task += g.ntasks;
    const bool leafc = d == P.depth - 1;
    g.Hc = leafc ? Hleaf : ws.H[d + 1];
    g.Hc_s = leafc ? hs : lv.nbc;
    g.i1a = lv.i1a; g.i3a = lv.i3a; g.i2b = lv.i2b; g.i3b = lv.i3b; g.n1a = lv.n1a; g.n3 = lv.n3; g.n12 = lv.n12;
    g.jump = jump; g.inv_dt = inv_dt; g.j3 = lv.j3; g.gidx = lv.gidx_bnd;
    g.W3 = (up || has_w3) ? ws.W3[d] : nullptr;
    g.Hout = d > 0 ? ws.H[d] : nullptr;
    g.u = u;
    g.done = up ? dup[d] : ddn[d];
    g.sem = c; c += (size_t)g.RB * g.NG;
    const size_t seg_part = pnm ? (size_t)g.S * g.RB * MRB : (size_t)g.S * g.NG * MNB * g.R;
    if (g.S > 1) { g.part = part; part += seg_part; }
    // dependencies inside this launch
    if (up) {
      const bool child_here = d + 1 < u1;
      g.wchild = child_here ? dup[d + 1] : nullptr;
      int RBc = 0, NGc, Sc, KCc, Rc, Kc;
      if (child_here) mega_dims(P.lv[d + 1], false, true, 1, RBc, NGc, Sc, KCc, Rc, Kc);
      g.wchild_t = RBc;
      g.Rc = child_here ? Rc : 0;
    } else {
      const bool par_here = d - 1 >= d0 && d > 0;
      const bool from_up = rpre && d == 1;  // the root's interface comes from its up tasks
      g.wpar = par_here ? (from_up ? dup[0] : ddn[d - 1]) : nullptr;
      int RBp = 0, x1, x2, x3, x4 = 0, x5;
      if (par_here) mega_dims(P.lv[d - 1], d - 1 == 0, from_up, 1, RBp, x1, x2, x3, x4, x5);
      // the parent level is a pair's child: its counters (one per child) are bumped by
      // the grandparents' own tasks and by the pair's tasks
      if (par_here && d >= 2 && pair_parent(d - 2)) {
        mega_dims(P.lv[d - 2], d - 2 == 0, false, 1, RBp, x1, x2, x3, x4, x5);
        RBp += rb_c1[d - 2];
      }
      g.wpar_t = RBp;
      g.Rp = par_here ? x4 : 0;
      const bool up_here = d >= u0 && d < u1;
      g.wup = up_here && has_w3 ? dup[d] : nullptr;
      int RBu = 0;
      if (up_here) mega_dims(lv, d == 0, true, 1, RBu, x1, x2, x3, x4, x5);
      g.wup_t = RBu;
      g.Ru = up_here ? x4 : 0;
    }
    ++p.nseg;
    return true;
  };
  // the root pair: the root's down product first (no inputs from this launch)
  const bool pair = !rpre && u0 == 0 && u1 > 0 && d0 == 0 && d1 > 0 && has_w3 && !jump && pair_enabled();
  int iroot_dn = -1;
  if (pair) {
    iroot_dn = p.nseg;
    if (!add(0, false)) return 1;
  }
  for (int d = u1 - 1; d >= u0; --d) {
    if (!add(d, true)) return 1;
    // adjusted loads w3c = w3(c) + S_c[:, B] w3(p) of the pair (d + 1, d + 2): both levels' up
    // tasks are lower-numbered; runs beside the rest of the up sweep
    if (const MegaPair* mp = pair_parent(d + 1)) {
      const int dp = d + 1;
      dpu[dp] = c; c += P.lv[dp].c;
      MSeg* g = add_custom(dp, mp->PU, P.lv[dp].n3, mp->iota, mp->out, ws.W3[dp + 1], ws.W3[dp], dpu[dp], 1);
      if (!g) return 1;
      g->wup = dup[dp];
      int x1, x2, x3, x4, x5;
      mega_dims(P.lv[dp], dp == 0, true, 1, g->wup_t, x1, x2, x3, x4, x5);
      rb_pu[dp] = g->RB;
      rb_c1[dp] = (2 * P.lv[dp + 1].n3 + MRB - 1) / MRB;
    }
  }
  if (rpre)
    for (int i = 0; i < p.nseg; ++i)
      if (p.s[i].up && p.s[i].Hout == nullptr) p.s[i].rootpre = root_pre;  // the root's up segment
  for (int d = (pair || rpre) ? 1 : d0; d < d1; ++d) {
    if (!add(d, false)) return 1;
    if (const MegaPair* mp = pair_parent(d)) {
      // level d + 1 in the same phase: one segment over the level-d nodes with the stacked
      // operator; both segments count on the children's counters
      MSeg& par = p.s[p.nseg - 1];
      par.dmul = 2;
      par.done = ddn[d + 1];
      MSeg* g = add_custom(d, mp->C1, P.lv[d].n12, P.lv[d].gidx_bnd, P.lv[d + 1].j3, ws.W3c[d + 1], u, ddn[d + 1], 2);
      if (!g) return 1;
      g->wpar = par.wpar; g->wpar_t = par.wpar_t;
      g->wup = dpu[d]; g->wup_t = rb_pu[d];
      ++d;  // level d + 1 is done by the pair
    }
  }
  if (pair) {
    MSeg& dn = p.s[iroot_dn];
    MSeg* upp = nullptr;
    for (int i = 0; i < p.nseg; ++i)
      if (p.s[i].up && p.s[i].Hout == nullptr) upp = &p.s[i];  // the root's up segment (no flux rows)
    if (!upp || upp->RB != dn.RB || upp->NG != dn.NG || upp->R != dn.R) return 1;
    for (MSeg* g : {&dn, upp}) {
      g->pair = 1;
      g->Sdn = dn.S; g->Sup = upp->S;
      g->wup = nullptr;
      g->done = dn.done;             // level 1's down tasks wait on the root's u3
      g->sem = dn.sem;               // one semaphore per row block for both
      if (!g->part) {
        g->part = part;
        part += pnm ? (size_t)g->S * g->RB * MRB : (size_t)g->S * g->NG * MNB * g->R;
      }
    }
    dn.pdn = upp->pdn = dn.part;
    dn.pup = upp->pup = upp->part;
  }
  if (p.nseg == 0) return 0;
  p.ntasks = task;
  p.ticket = c++;
  p.reset = cnt + 1;
  p.nreset = (int)(c - (cnt + 1));
  const int max_ctas = mega_max_ctas(pnm);
  int grid = std::min(max_ctas, p.ntasks);
  if (pair && mega_dedicated()) {  // a quarter of the CTAs stream the root's down product while the up sweep climbs
    grid = max_ctas;
    p.head = p.s[iroot_dn].ntasks;
    p.dedicated = std::max(1, grid / 4);
  }
  const char* tr = getenv("HPSB_MEGA_TRACE");  // debug: per-task timeline appended to this file
  unsigned long long* dtrace = nullptr;
  if (tr) {
    HPSB_CUDA(cudaMalloc(&dtrace, (size_t)MTS * p.ntasks * 8));
    HPSB_CUDA(cudaMemsetAsync(dtrace, 0, (size_t)MTS * p.ntasks * 8, st));
    p.trace = dtrace;
  }
  if (pnm)
    HPSB_CUDA(launch_pdl(k_mega<true>, dim3(grid), dim3(MT), 0, st, p, exit_count));
  else
    HPSB_CUDA(launch_pdl(k_mega<false>, dim3(grid), dim3(MT), 0, st, p, exit_count));
  HPSB_LAUNCH_CHECK();
  if (tr) {
    std::vector<unsigned long long> h((size_t)MTS * p.ntasks);
    HPSB_CUDA(cudaStreamSynchronize(st));
    HPSB_CUDA(cudaMemcpy(h.data(), dtrace, h.size() * 8, cudaMemcpyDeviceToHost));
    cudaFree(dtrace);
    if (FILE* f = fopen(tr, "a")) {
      fprintf(f, "launch grid=%d tasks=%d segs=%d\n", grid, p.ntasks, p.nseg);
      for (int i = 0; i < p.nseg; ++i) {
        const MSeg& g = p.s[i];
        fprintf(f, "seg %d up=%d nodes=%d R=%d K=%d RB=%d NG=%d S=%d tasks=%d:%d\n", i, g.up, g.nn, g.R, g.K, g.RB,
                g.NG, g.S, g.task0, g.ntasks);
      }
      for (int t = 0; t < p.ntasks; ++t) {
        fprintf(f, "%d", t);
        for (int i = 0; i < MTS; ++i) fprintf(f, " %llu", h[(size_t)MTS * t + i]);
        fprintf(f, "\n");
      }
      fclose(f);
    }
  }
  return 0;
}

}  // namespace hpsb
