// The per-stage HPS solve (solver.py:201-276) as a sequence of level-batched
// launches on one stream: boundary scatter, leaf upward pass, level upward
// merges (deepest first), level downward sweep (root first), leaf downward
// reconstruction.  No host synchronisation; capturable in a CUDA graph.
#include <stdlib.h>

#include "hps_plan.cuh"

namespace hpsb {

namespace {

__global__ void k_bnd_scatter(int k, int nbd, const int* __restrict__ ids, const double* __restrict__ fb,
                              long long ld_f, double* __restrict__ u, long long ld_u) {
  pdl_trigger();
  pdl_wait();
  long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  if (e >= (long long)k * nbd) return;
  int kk = (int)(e / nbd), i = (int)(e % nbd);
  u[kk * ld_u + ids[i]] = fb[kk * ld_f + i];
}

// ub rows of nl leaves (rhs stride `per`); lbg and ub point at the first leaf
__global__ void k_leaf_gather(int k, int nl, int nb, long long per, const int* __restrict__ lbg,
                              const double* __restrict__ u, long long ld_u, double* __restrict__ ub) {
  pdl_trigger();
  pdl_wait();
  long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long cnt = (long long)nl * nb;
  if (e >= (long long)k * cnt) return;
  int kk = (int)(e / cnt);
  long long r = e % cnt;
  ub[kk * per + r] = u[kk * ld_u + lbg[r]];
}

}  // namespace

// every panel a solve may launch (with its rhs multiplier), for sizing the
// split-K scratch: per-node wide levels, and the shared layout's one-node
// panels whose launches carry (nodes x rhs) right-hand sides
static void solve_panels(const Plan& P, std::vector<std::pair<Panel, int>>& out) {
  out.clear();
  out.push_back({make_panel(P.L, P.ni, P.ni, P.nparts), 1});
  out.push_back({make_panel(P.L, P.ni, P.nb, P.nparts), 1});
  for (const Level& lv : P.lv)
    if (lv.c < kSharedGemmNodes)
      for (int v = lv.c; v >= 1 && v >= lv.c / P.nparts; v /= 2) {  // node ranges of part ranges
        out.push_back({make_panel(1, lv.n3 + lv.n12, lv.n3), v});
        out.push_back({make_panel(1, lv.n3, lv.n12), v});
      }
  for (int d = 0; d < P.dF; ++d) {  // wide levels only; fused levels use no split-K
    const Level& lv = P.lv[d];
    const int parts = d >= P.lstar ? P.nparts : 1;
    out.push_back({make_panel(lv.c, lv.n3 + (d > 0 ? lv.n12 : 0), lv.n3, parts), 1});
    out.push_back({make_panel(lv.c, lv.n3, lv.n12, parts), 1});
  }
}

static void scratch_sizes(const Plan& P, int k, size_t& part, size_t& cnt, size_t* xg = nullptr) {
  std::vector<std::pair<Panel, int>> pns;
  solve_panels(P, pns);
  part = 0; cnt = 0;
  for (const auto& pk : pns) {
    PanelSplit sp = panel_split(pk.first, k, pk.second);
    part = std::max(part, sp.part_doubles);
    cnt = std::max(cnt, (size_t)sp.counters);
  }
  // shared-layout GEMM level applies (dedup.cu) over every part range
  for (int d = 0; d < P.depth; ++d) {
    const Level& lv = P.lv[d];
    for (int np = 1; np <= (d >= P.lstar ? P.nparts : 1); np *= 2) {
      const long long M = (long long)(lv.c / np) * k;
      for (const GsSplit& sp : {gs_split(M, lv.n3 + (d > 0 ? lv.n12 : 0), lv.n3), gs_split(M, lv.n3, lv.n12)}) {
        part = std::max(part, sp.part_doubles);
        cnt = std::max(cnt, (size_t)sp.counters);
        if (xg) *xg = std::max(*xg, sp.gather_doubles);
      }
    }
  }
}

size_t workspace_bytes(const Plan& P, int k) {
  size_t n = 0;
  auto add = [&](long long cnt) { n += ((size_t)cnt * k * 8 + 255) & ~(size_t)255; };
  add((long long)P.L * (P.ni + P.nb));
  add((long long)P.L * P.nb);
  add((long long)P.L * P.nb);
  for (int d = 0; d < P.depth; ++d) {
    if (d >= 1) add((long long)P.lv[d].c * P.lv[d].n12);
    add((long long)P.lv[d].c * P.lv[d].n3);
  }
  if (k == 1)
    for (int d = 1; d < std::min(P.depth, P.dF); ++d) add((long long)P.lv[d].c * P.lv[d].n3);
  size_t part, cnt, xg = 0;
  scratch_sizes(P, k, part, cnt, &xg);
  n += (part * 8 + 255) & ~(size_t)255;
  n += (cnt * 4 + 255) & ~(size_t)255;
  size_t mc, mp;
  mega_scratch(P, mc, mp);
  n += (mc * 4 + 255) & ~(size_t)255;
  n += (mp * 8 + 255) & ~(size_t)255;
  n += (xg * 8 + 255) & ~(size_t)255;
  return n + 256;
}

void carve_workspace(const Plan& P, int k, void* base, Workspace& ws) {
  char* p = (char*)(((uintptr_t)base + 255) & ~(uintptr_t)255);
  auto take = [&](long long cnt) {
    double* r = (double*)p;
    p += ((size_t)cnt * k * 8 + 255) & ~(size_t)255;
    return r;
  };
  ws.W = take((long long)P.L * (P.ni + P.nb));
  ws.Hleaf = take((long long)P.L * P.nb);
  ws.Ub = take((long long)P.L * P.nb);
  ws.H.assign(P.depth, nullptr);
  ws.W3.assign(P.depth, nullptr);
  for (int d = 0; d < P.depth; ++d) {
    if (d >= 1) ws.H[d] = take((long long)P.lv[d].c * P.lv[d].n12);
    ws.W3[d] = take((long long)P.lv[d].c * P.lv[d].n3);
  }
  ws.W3c.assign(P.depth, nullptr);
  if (k == 1)
    for (int d = 1; d < std::min(P.depth, P.dF); ++d) ws.W3c[d] = take((long long)P.lv[d].c * P.lv[d].n3);
  size_t part, cnt, xg = 0;
  scratch_sizes(P, k, part, cnt, &xg);
  ws.part = (double*)p;
  p += (part * 8 + 255) & ~(size_t)255;
  ws.cnt = (unsigned*)p;  // zeroed by the caller when the workspace is created
  p += (cnt * 4 + 255) & ~(size_t)255;
  size_t mc, mp;
  mega_scratch(P, mc, mp);
  ws.mega_cnt = (unsigned*)p;  // zeroed likewise
  p += (mc * 4 + 255) & ~(size_t)255;
  ws.mega_part = (double*)p;
  p += (mp * 8 + 255) & ~(size_t)255;
  ws.xg = xg ? (double*)p : nullptr;
}

// one level's upward merge over nodes [n0, n1) (solver.py:243-256)
static int level_up(const Ops& ops, const Workspace& ws, int d, int n0, int n1, int k, const double* Hleaf,
                    long long sh, long long hs, const double* jump, long long ld_jump, double inv_dt,
                    cudaStream_t st) {
  const Plan& P = *ops.plan;
  const Level& lv = P.lv[d];
  const bool leafc = d == P.depth - 1;
  const double* Hc = leafc ? Hleaf : ws.H[d + 1];
  const long long Hc_k = leafc ? sh : (long long)P.lv[d + 1].c * P.lv[d + 1].n12;
  const long long Hc_s = leafc ? hs : lv.nbc;
  if (ops.shared_levels)
    return shared_level_up(ops, ws, d, k, Hc, Hc_k, Hc_s, jump, ld_jump, inv_dt, n0, n1, st);
  GemvArgs a{};
  a.k = k; a.part = ws.part; a.cnt = ws.cnt;
  a.Hc = Hc; a.nbc = lv.nbc; a.Hc_k = Hc_k; a.Hc_s = Hc_s;
  a.W3 = ws.W3[d]; a.n3 = lv.n3; a.W3_k = (long long)lv.c * lv.n3;
  a.i1a = lv.i1a; a.i3a = lv.i3a; a.i2b = lv.i2b; a.i3b = lv.i3b; a.n1a = lv.n1a;
  a.n12 = lv.n12;
  a.jump = jump; a.jump_k = ld_jump; a.inv_dt = inv_dt; a.j3 = lv.j3;
  a.mode = GEMV_UP;  // the root's panel has no flux rows (its outer flux is never consumed)
  a.Hout = d > 0 ? ws.H[d] : nullptr; a.Hout_k = (long long)lv.c * lv.n12;
  return gemv_nodes(a, ops.lo[d].Up, n0, n1, st);
}

// one level's downward sweep over nodes [n0, n1) (solver.py:258-268)
static int level_down(const Ops& ops, const Workspace& ws, int d, int n0, int n1, int k, bool has_w3, double* u,
                      long long ld_u, cudaStream_t st) {
  const Plan& P = *ops.plan;
  const Level& lv = P.lv[d];
  if (ops.shared_levels) return shared_level_down(ops, ws, d, k, has_w3, u, ld_u, n0, n1, st);
  GemvArgs a{};
  a.mode = GEMV_DOWN; a.k = k; a.part = ws.part; a.cnt = ws.cnt;
  a.u = u; a.u_k = ld_u; a.gidx = lv.gidx_bnd; a.j3 = lv.j3;
  a.n3 = lv.n3; a.n12 = lv.n12;
  a.W3 = has_w3 ? ws.W3[d] : nullptr; a.W3_k = (long long)lv.c * lv.n3;
  return gemv_nodes(a, ops.lo[d].S, n0, n1, st);
}

// byte offsets of level d's w3 and flux blocks in a k-rhs workspace (-1: none)
void level_offsets(const Plan& P, int k, int d, long long& w3, long long& h) {
  Workspace ws;
  carve_workspace(P, k, nullptr, ws);
  w3 = (long long)(uintptr_t)ws.W3[d];
  h = d >= 1 ? (long long)(uintptr_t)ws.H[d] : -1;
}

// One top level (d < lstar) of a subtree-sharded solve, row-sharded over
// nranks GPUs: this rank applies its contiguous share of the level's operator
// tiles (up: [X33^-1; Tstack X33^-1], down: S) for every node of the level.
// Up: w3 / flux rows into the workspace's level-d blocks, zeroed first, so a
// sum over the ranks completes them; down: u3 rows into `stage` (k x c x n3,
// zeroed first), summed over the ranks and scattered to u[j3] by the caller.
int top_level(const Ops& ops, int d, bool down, int rank, int nranks, int k, double* u, long long ld_u,
              double* stage, void* wsp, size_t ws_bytes, cudaStream_t st) {
  const Plan& P = *ops.plan;
  if (d < 0 || d >= P.lstar || rank < 0 || rank >= nranks || k <= 0) {
    set_error("top_level: level %d (lstar %d), rank %d of %d", d, P.lstar, rank, nranks);
    return -1;
  }
  if (ws_bytes < workspace_bytes(P, k)) {
    set_error("top_level: workspace too small");
    return -1;
  }
  Workspace ws;
  carve_workspace(P, k, wsp, ws);
  const Level& lv = P.lv[d];
  const LevelOps& lo = ops.lo[d];
  const Panel& full = down ? lo.S : lo.Up;
  if (!full.base || full.parts != 1 || full.TS != full.TR || (ops.shared_levels && full.c != 1)) {
    set_error("top_level: level %d has no streaming panel", d);
    return -1;
  }
  const int T = full.ntiles, t0 = (int)((long long)T * rank / nranks), t1 = (int)((long long)T * (rank + 1) / nranks);
  Panel view = full;
  view.base = full.base + (size_t)t0 * full.C * full.TS;
  view.ntiles = t1 - t0;
  GemvArgs a{};
  a.k = k; a.part = ws.part; a.cnt = ws.cnt;
  a.prow0 = (long long)t0 * full.TR;
  a.shared = ops.shared_levels ? lv.c : 0;
  a.n3 = lv.n3; a.n12 = lv.n12;
  a.W3 = ws.W3[d]; a.W3_k = (long long)lv.c * lv.n3;
  if (!down) {
    HPSB_CUDA(cudaMemsetAsync(ws.W3[d], 0, (size_t)k * lv.c * lv.n3 * 8, st));
    if (d > 0) HPSB_CUDA(cudaMemsetAsync(ws.H[d], 0, (size_t)k * lv.c * lv.n12 * 8, st));
    a.mode = GEMV_UP;
    a.Hc = ws.H[d + 1]; a.nbc = lv.nbc;
    a.Hc_k = (long long)P.lv[d + 1].c * P.lv[d + 1].n12; a.Hc_s = lv.nbc;
    a.i1a = lv.i1a; a.i3a = lv.i3a; a.i2b = lv.i2b; a.i3b = lv.i3b; a.n1a = lv.n1a;
    a.j3 = lv.j3;
    a.Hout = d > 0 ? ws.H[d] : nullptr; a.Hout_k = (long long)lv.c * lv.n12;
  } else {
    if (!stage) { set_error("top_level: down pass needs a staging vector"); return -1; }
    HPSB_CUDA(cudaMemsetAsync(stage, 0, (size_t)k * lv.c * lv.n3 * 8, st));
    a.mode = GEMV_DOWN;
    a.u = u; a.u_k = ld_u; a.gidx = lv.gidx_bnd; a.j3 = lv.j3;
    a.yout = stage; a.yout_k = (long long)lv.c * lv.n3;  // u3 to the staging vector
  }
  if (view.ntiles <= 0) return 0;
  return gemv_level(a, view, st);
}

size_t exchange_offset(const Plan& P, int k) {
  Workspace ws;
  carve_workspace(P, k, nullptr, ws);
  return (size_t)(uintptr_t)ws.H[P.lstar];
}

// Phases of one solve over the parts [part0, part1) (SOLVE_ALL over every
// part = the whole solve of solver.py:201-276).
int solve(const Ops& ops, int phases, int part0, int part1, int k, const double* fb, long long ld_f,
          const double* g, long long ld_g, const double* jump, long long ld_jump, double inv_dt, double* u,
          long long ld_u, void* wsp, size_t ws_bytes, cudaStream_t st, double* lu, long long ld_lu,
          double* guard, const double* root_pre, const StageTerms* terms) {
  const Plan& P = *ops.plan;
  if (k <= 0) return 0;
  if (ws_bytes < workspace_bytes(P, k)) {
    set_error("solve: workspace too small (%zu < %zu)", ws_bytes, workspace_bytes(P, k));
    return -1;
  }
  const int NP = P.nparts, ls = P.lstar;
  if (part0 < 0 || part1 > NP || part0 >= part1) {
    set_error("solve: part range [%d, %d) outside [0, %d)", part0, part1, NP);
    return -1;
  }
  Workspace ws;
  carve_workspace(P, k, wsp, ws);
  const long long Lni = (long long)P.L * P.ni, Lnb = (long long)P.L * P.nb;
  const int T = 256;
  const int lpp = P.L / NP, leaf0 = part0 * lpp, nleaf = (part1 - part0) * lpp;
  auto range = [&](int d, int& n0, int& n1) {  // the parts' nodes on level d >= lstar
    const int per = P.lv[d].c / NP;
    n0 = part0 * per;
    n1 = part1 * per;
  };

  const bool up = (g != nullptr) || (jump != nullptr);
  const int nw = P.ni + P.nb;
  bool mb_applies(const Ops& ops, int k);

// fused subtree kernels for the deep levels, except for many-rhs solves on
  // shared operators: there every level is one tensor-core GEMM over
  // (node, rhs) rows (dedup.cu)
  static const int sub_rhs_max = [] {  // A/B: HPSB_SUB_RHS_MAX=n fuses the deep levels up to n rhs
    const char* e = getenv("HPSB_SUB_RHS_MAX");
    return e ? atoi(e) : kSharedGemmRhs - 1;
  }();
  // ... unless the member-blocked subtree kernels take them (member_subtree.cu)
  const bool many = ops.shared_levels && k > sub_rhs_max;
  const bool fused = P.dF < P.depth && (!many || (!jump && k >= kSharedGemmRhs && mb_applies(ops, k)));
  const int dW = fused ? P.dF : P.depth;  // levels [lstar, dW) run level by level
  // leaf outputs: W (row stride ldw, rhs stride sw) and H (child stride hs, rhs stride sh)
  long long ldw = P.ni, sw = Lni, hs = P.nb, sh = Lnb;
  const double* Hleaf = ws.Hleaf;
  // tensor-product leaves: h only on the way up, u_int = A_ii^-1 (r - A_ib u_b) on the way down
  const bool fd_down = ops.shared_leaf && ops.fd && leaf_fd_down_enabled();
  const bool stacked = g && ops.shared_leaf && !fd_down;  // [w | h] rows of one GEMM / the tensor-product solve
  if (stacked) {
    ldw = nw; sw = (long long)P.L * nw; hs = nw; sh = sw;
    Hleaf = ws.W + P.ni;
  }

  bool bnd_done = false;  // Dirichlet data already written by the leaf kernel
  if (phases & SOLVE_UP) {
    // (2) leaf particular solutions and their fluxes (solver.py:219-230)
    if (terms && fd_down) {
      // the stage combination formed by the leaf kernel (no combination pass), written out for the
      // downward sweep; the Dirichlet data too
      const bool bnd = (phases & SOLVE_TOP) && P.nbd > 0;
      if (int rc = leaf_fd_up_terms(ops, k, nleaf, terms->nterm, terms->tv, terms->tld, terms->tdc,
                                    terms->rout + (long long)leaf0 * P.ni, terms->ld_rout,
                                    ws.Hleaf + (long long)leaf0 * P.nb, Lnb, st, bnd ? P.nbd : 0, P.boundary_ids,
                                    fb, ld_f, u, ld_u))
        return rc;
      bnd_done = bnd;
    } else if (g && fd_down) {
      // a whole solve: the leaf kernel also writes the Dirichlet data (no separate scatter launch)
      const bool bnd = (phases & SOLVE_TOP) && P.nbd > 0;
      if (int rc = leaf_fd_up_h(ops, k, nleaf, g, ld_g, ws.Hleaf + (long long)leaf0 * P.nb, Lnb, st,
                                bnd ? P.nbd : 0, P.boundary_ids, fb, ld_f, u, ld_u))
        return rc;
      bnd_done = bnd;
    } else if (g && ops.shared_leaf && ops.fd) {
      // tensor-product leaf solve: same [W | H] rows, 5x fewer flops
      if (int rc = leaf_fd(ops, k, nleaf, g, ld_g, ws.W + (long long)leaf0 * nw, sw, st)) return rc;
    } else if (g && ops.shared_leaf) {
      // [W | H] (L x (ni+nb)) = G_int (L x ni) * [Ainv; D_bi Ainv]^T, one GEMM per rhs
      GemmArgs a{};
      a.M = nleaf; a.N = nw; a.K = P.ni; a.alpha = 1.0; a.beta = 0.0;
      a.A = g; a.lda = P.ni; a.sA = ld_g; a.tA = 0;
      a.B = ops.Ainv; a.ldb = P.ldi; a.sB = 0; a.tB = 1;
      a.C = ws.W + (long long)leaf0 * nw; a.ldc = nw; a.sC = sw; a.batch = k;
      if (int rc = gemm_nt(a, st)) return rc;
    } else if (g) {
      GemvArgs a{};
      a.mode = GEMV_LEAF; a.k = k; a.part = ws.part; a.cnt = ws.cnt;
      // xin is addressed by global leaf index: g's (virtual) leaf-0 origin
      a.xin = (const double*)((uintptr_t)g - (uintptr_t)leaf0 * P.ni * sizeof(double));
      a.xin_k = ld_g; a.xin_s = P.ni;
      a.yout = ws.W; a.yout_k = Lni; a.yout_s = P.ni;
      if (int rc = gemv_nodes(a, ops.pAinv, leaf0, leaf0 + nleaf, st)) return rc;
      // H (nleaf x nb) = W (nleaf x ni) * D_bi^T per rhs
      GemmArgs h{};
      h.M = nleaf; h.N = P.nb; h.K = P.ni; h.alpha = 1.0; h.beta = 0.0;
      h.A = ws.W + (long long)leaf0 * P.ni; h.lda = P.ni; h.sA = Lni; h.tA = 0;
      h.B = ops.D_bi; h.ldb = P.ni; h.sB = 0; h.tB = 1;
      h.C = ws.Hleaf + (long long)leaf0 * P.nb; h.ldc = P.nb; h.sC = Lnb; h.batch = k;
      if (int rc = gemm_nt(h, st)) return rc;
    } else if (jump) {
      for (int kk = 0; kk < k; ++kk)
        HPSB_CUDA(cudaMemsetAsync(ws.Hleaf + kk * Lnb + (long long)leaf0 * P.nb, 0, (size_t)nleaf * P.nb * 8, st));
    }
    // (3) upward merges of the fused subtree levels in one launch (solver.py:243-256)
    if (up && fused) {
      int b0, b1;
      range(P.dF, b0, b1);
      if (int rc = subtree_up(ops, ws, k, Hleaf, sh, hs, jump, ld_jump, inv_dt, b0, b1, st)) return rc;
    }
  }
  if (phases & SOLVE_TOP) {
    // (1) Dirichlet data into u (solver.py:259-260); the up sweep never reads u
    long long n = bnd_done ? 0 : (long long)k * P.nbd;
    if (n > 0) {
      HPSB_CUDA(launch_pdl(k_bnd_scatter, dim3((unsigned)cdiv(n, T)), dim3(T), 0, st, k, P.nbd, P.boundary_ids,
                           fb, ld_f, u, ld_u));
      HPSB_LAUNCH_CHECK();
    }
  }
  // (3, 4) the wide levels: up [uA, uB) deepest first, then down [dA, dB) root
  // first (solver.py:243-268) -- the parts' nodes on levels >= lstar, every
  // node above.  Shared operators, one rhs: one persistent dataflow launch
  // (mega.cu); otherwise one launch per level and pass.
  const int uA = (phases & SOLVE_TOP) ? 0 : ls, uB = up ? ((phases & SOLVE_UP) ? dW : ls) : uA;
  const int dA = (phases & SOLVE_TOP) ? 0 : ls, dB = (phases & SOLVE_DOWN) ? dW : ls;
  // levels >= dm (large per-node operators) always run per level
  const int dm = k == 1 && mega_enabled() ? mega_depth(ops) : 0;
  auto ups = [&](int d1, int d0) -> int {  // per-level up merges d1 - 1 .. d0
    for (int d = d1 - 1; d >= d0; --d) {
      int n0 = 0, n1 = P.lv[d].c;
      if (d >= ls) range(d, n0, n1);
      if (int rc = level_up(ops, ws, d, n0, n1, k, Hleaf, sh, hs, jump, ld_jump, inv_dt, st)) return rc;
    }
    return 0;
  };
  auto downs = [&](int d0, int d1) -> int {
    for (int d = d0; d < d1; ++d) {
      int n0 = 0, n1 = P.lv[d].c;
      if (d >= ls) range(d, n0, n1);
      if (int rc = level_down(ops, ws, d, n0, n1, k, up, u, ld_u, st)) return rc;
    }
    return 0;
  };
  if (int rc = ups(uB, std::max(uA, dm))) return rc;
  const int mu1 = std::min(uB, dm), md1 = std::min(dB, dm);
  int rc_mega = 1;
  if (mu1 > uA || md1 > dA)
    rc_mega = mega_levels(ops, ws, uA, std::max(uA, mu1), dA, std::max(dA, md1), part0, part1, Hleaf, hs, jump,
                          inv_dt, up, u, st, root_pre);
  if (rc_mega < 0) return rc_mega;
  if (rc_mega == 1) {
    if (int rc = ups(std::max(uA, mu1), uA)) return rc;
    if (int rc = downs(dA, std::max(dA, md1))) return rc;
  }
  if (int rc = downs(std::max(dA, dm), dB)) return rc;

  if (terms && fd_down) { g = terms->rout; ld_g = terms->ld_rout; }  // the formed body load
  if (phases & SOLVE_DOWN) {
    if (fused) {
      int b0, b1;
      range(P.dF, b0, b1);
      if (int rc = subtree_down(ops, ws, k, up, u, ld_u, b0, b1, st)) return rc;
    }
    // (5) leaf interiors: u_int = S_leaf u_bnd + w (solver.py:269-276)
    if (fd_down)
      return leaf_fd_down(ops, k, nleaf, g, ld_g, P.leaf_bnd_gidx + (long long)leaf0 * P.nb, u, ld_u,
                          u + (long long)leaf0 * P.ni, ld_u, lu, ld_lu, guard, st);
    if (lu) {
      set_error("solve: the fused stage history needs the tensor-product leaf solve");
      return -1;
    }
    long long n = (long long)k * nleaf * P.nb;
    HPSB_CUDA(launch_pdl(k_leaf_gather, dim3((unsigned)cdiv(n, T)), dim3(T), 0, st, k, nleaf, P.nb, Lnb,
                         (const int*)(P.leaf_bnd_gidx + (long long)leaf0 * P.nb), (const double*)u, ld_u,
                         ws.Ub + (long long)leaf0 * P.nb));
    HPSB_LAUNCH_CHECK();
    if (ops.shared_leaf) {
      GemmArgs a{};
      a.M = nleaf; a.N = P.ni; a.K = P.nb; a.alpha = 1.0;
      a.A = ws.Ub + (long long)leaf0 * P.nb; a.lda = P.nb; a.sA = Lnb; a.tA = 0;
      a.B = ops.S_leaf; a.ldb = P.ldb; a.sB = 0; a.tB = 1;
      a.beta = g ? 1.0 : 0.0; a.D = g ? ws.W + (long long)leaf0 * ldw : nullptr; a.ldd = ldw; a.sD = sw;
      a.C = u + (long long)leaf0 * P.ni; a.ldc = P.ni; a.sC = ld_u; a.batch = k;
      if (int rc = gemm_nt(a, st)) return rc;
    } else {
      GemvArgs a{};
      a.mode = GEMV_LEAF; a.k = k; a.part = ws.part; a.cnt = ws.cnt;
      a.xin = ws.Ub; a.xin_k = Lnb; a.xin_s = P.nb;
      a.yout = u; a.yout_k = ld_u; a.yout_s = P.ni;
      a.yadd = g ? ws.W : nullptr; a.yadd_k = Lni; a.yadd_s = P.ni;
      if (int rc = gemv_nodes(a, ops.pSleaf, leaf0, leaf0 + nleaf, st)) return rc;
    }
  }
  return 0;
}

}  // namespace hpsb
