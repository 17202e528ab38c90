// The per-stage HPS solve (solver.py:201-276) as a sequence of level-batched
// launches on one stream: boundary scatter, leaf upward pass, level upward
// merges (deepest first), level downward sweep (root first), leaf downward
// reconstruction.  No host synchronisation; capturable in a CUDA graph.
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

__global__ void k_leaf_gather(int k, int L, int nb, const int* __restrict__ lbg, const double* __restrict__ u,
                              long long ld_u, double* __restrict__ ub) {
  pdl_trigger();
  pdl_wait();
  long long e = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  long long per = (long long)L * nb;
  if (e >= (long long)k * per) return;
  int kk = (int)(e / per);
  long long r = e % per;
  ub[kk * per + r] = u[kk * ld_u + lbg[r]];
}

}  // namespace

// every panel a solve may launch (with its rhs multiplier), for sizing the
// split-K scratch: per-node wide levels, and the shared layout's one-node
// panels whose launches carry (nodes x rhs) right-hand sides
static void solve_panels(const Plan& P, std::vector<std::pair<Panel, int>>& out) {
  out.clear();
  out.push_back({make_panel(P.L, P.ni, P.ni), 1});
  out.push_back({make_panel(P.L, P.ni, P.nb), 1});
  for (const Level& lv : P.lv)
    if (lv.c < kSharedGemmNodes) {
      out.push_back({make_panel(1, lv.n3 + lv.n12, lv.n3), lv.c});
      out.push_back({make_panel(1, lv.n3, lv.n12), lv.c});
    }
  for (int d = 0; d < P.dF; ++d) {  // wide levels only; fused levels use no split-K
    const Level& lv = P.lv[d];
    out.push_back({make_panel(lv.c, lv.n3 + (d > 0 ? lv.n12 : 0), lv.n3), 1});
    out.push_back({make_panel(lv.c, lv.n3, lv.n12), 1});
  }
}

static void scratch_sizes(const Plan& P, int k, size_t& part, size_t& cnt) {
  std::vector<std::pair<Panel, int>> pns;
  solve_panels(P, pns);
  part = 0; cnt = 0;
  for (const auto& pk : pns) {
    PanelSplit sp = panel_split(pk.first, k, pk.second);
    part = std::max(part, sp.part_doubles);
    cnt = std::max(cnt, (size_t)sp.counters);
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
  size_t part, cnt;
  scratch_sizes(P, k, part, cnt);
  n += (part * 8 + 255) & ~(size_t)255;
  n += (cnt * 4 + 255) & ~(size_t)255;
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
  size_t part, cnt;
  scratch_sizes(P, k, part, cnt);
  ws.part = (double*)p;
  p += (part * 8 + 255) & ~(size_t)255;
  ws.cnt = (unsigned*)p;  // zeroed by the caller when the workspace is created
}

int solve(const Ops& ops, int k, const double* fb, long long ld_f, const double* g, long long ld_g,
          const double* jump, long long ld_jump, double inv_dt, double* u, long long ld_u,
          void* wsp, size_t ws_bytes, cudaStream_t st) {
  const Plan& P = *ops.plan;
  if (k <= 0) return 0;
  if (ws_bytes < workspace_bytes(P, k)) {
    set_error("solve: workspace too small (%zu < %zu)", ws_bytes, workspace_bytes(P, k));
    return -1;
  }
  Workspace ws;
  carve_workspace(P, k, wsp, ws);
  const long long Lni = (long long)P.L * P.ni, Lnb = (long long)P.L * P.nb;
  const int T = 256;

  // (1) Dirichlet data into u (solver.py:259-260)
  {
    long long n = (long long)k * P.nbd;
    if (n > 0) {
      HPSB_CUDA(launch_pdl(k_bnd_scatter, dim3((unsigned)cdiv(n, T)), dim3(T), 0, st, k, P.nbd, P.boundary_ids,
                           fb, ld_f, u, ld_u));
      HPSB_LAUNCH_CHECK();
    }
  }

  const bool up = (g != nullptr) || (jump != nullptr);
  const int nw = P.ni + P.nb;
  // leaf outputs: W (row stride ldw, rhs stride sw) and H (child stride hs, rhs stride sh)
  long long ldw = P.ni, sw = Lni, hs = P.nb, sh = Lnb;
  const double* Hleaf = ws.Hleaf;
  // (2) leaf particular solutions and their fluxes (solver.py:219-230)
  if (g) {
    if (ops.shared_leaf && ops.fd) {
      // tensor-product leaf solve: same [W | H] rows, 5x fewer flops
      if (int rc = leaf_fd(ops, k, g, ld_g, ws.W, (long long)P.L * nw, st)) return rc;
      ldw = nw; sw = (long long)P.L * nw; hs = nw; sh = sw;
      Hleaf = ws.W + P.ni;
    } else if (ops.shared_leaf) {
      // [W | H] (L x (ni+nb)) = G_int (L x ni) * [Ainv; D_bi Ainv]^T, one GEMM per rhs
      GemmArgs a{};
      a.M = P.L; a.N = nw; a.K = P.ni; a.alpha = 1.0; a.beta = 0.0;
      a.A = g; a.lda = P.ni; a.sA = ld_g; a.tA = 0;
      a.B = ops.Ainv; a.ldb = P.ldi; a.sB = 0; a.tB = 1;
      a.C = ws.W; a.ldc = nw; a.sC = (long long)P.L * nw; a.batch = k;
      if (int rc = gemm_nt(a, st)) return rc;
      ldw = nw; sw = (long long)P.L * nw; hs = nw; sh = sw;
      Hleaf = ws.W + P.ni;
    } else {
      GemvArgs a{};
      a.mode = GEMV_LEAF; a.k = k; a.part = ws.part; a.cnt = ws.cnt;
      a.xin = g; a.xin_k = ld_g; a.xin_s = P.ni;
      a.yout = ws.W; a.yout_k = Lni; a.yout_s = P.ni;
      if (int rc = gemv_level(a, ops.pAinv, st)) return rc;
      // H (k*L x nb) = W (k*L x ni) * D_bi^T
      GemmArgs h{};
      h.M = k * P.L; h.N = P.nb; h.K = P.ni; h.alpha = 1.0; h.beta = 0.0;
      h.A = ws.W; h.lda = P.ni; h.sA = 0; h.tA = 0;
      h.B = ops.D_bi; h.ldb = P.ni; h.sB = 0; h.tB = 1;
      h.C = ws.Hleaf; h.ldc = P.nb; h.sC = 0; h.batch = 1;
      if (int rc = gemm_nt(h, st)) return rc;
    }
  } else if (jump) {
    HPSB_CUDA(cudaMemsetAsync(ws.Hleaf, 0, (size_t)k * Lnb * 8, st));
  }

  // (3) upward merges, deepest level first (solver.py:243-256): the fused
  // subtree levels in one launch, then one launch per family on wide levels
  if (up) {
    if (int rc = subtree_up(ops, ws, k, Hleaf, sh, hs, jump, ld_jump, inv_dt, st)) return rc;
    for (int d = P.dF - 1; d >= 0; --d) {
      const Level& lv = P.lv[d];
      const LevelOps& lo = ops.lo[d];
      const bool leafc = d == P.depth - 1;
      const double* Hc = leafc ? Hleaf : ws.H[d + 1];
      const long long Hc_k = leafc ? sh : (long long)P.lv[d + 1].c * P.lv[d + 1].n12;
      const long long Hc_s = leafc ? hs : lv.nbc;
      if (ops.shared_levels) {
        if (int rc = shared_level_up(ops, ws, d, k, Hc, Hc_k, Hc_s, jump, ld_jump, inv_dt, st)) return rc;
        continue;
      }
      GemvArgs a{};
      a.k = k; a.part = ws.part; a.cnt = ws.cnt;
      a.Hc = Hc; a.nbc = lv.nbc; a.Hc_k = Hc_k; a.Hc_s = Hc_s;
      a.W3 = ws.W3[d]; a.n3 = lv.n3; a.W3_k = (long long)lv.c * lv.n3;
      a.i1a = lv.i1a; a.i3a = lv.i3a; a.i2b = lv.i2b; a.i3b = lv.i3b; a.n1a = lv.n1a;
      a.n12 = lv.n12;
      a.jump = jump; a.jump_k = ld_jump; a.inv_dt = inv_dt; a.j3 = lv.j3;
      a.mode = GEMV_UP;  // the root's panel has no flux rows (its outer flux is never consumed)
      a.Hout = d > 0 ? ws.H[d] : nullptr; a.Hout_k = (long long)lv.c * lv.n12;
      if (int rc = gemv_level(a, lo.Up, st)) return rc;
    }
  }

  // (4) downward sweep, root first (solver.py:258-268)
  for (int d = 0; d < P.dF; ++d) {
    const Level& lv = P.lv[d];
    const LevelOps& lo = ops.lo[d];
    if (ops.shared_levels) {
      if (int rc = shared_level_down(ops, ws, d, k, up, u, ld_u, st)) return rc;
      continue;
    }
    GemvArgs a{};
    a.mode = GEMV_DOWN; a.k = k; a.part = ws.part; a.cnt = ws.cnt;
    a.u = u; a.u_k = ld_u; a.gidx = lv.gidx_bnd; a.j3 = lv.j3;
    a.n3 = lv.n3; a.n12 = lv.n12;
    a.W3 = up ? ws.W3[d] : nullptr; a.W3_k = (long long)lv.c * lv.n3;
    if (int rc = gemv_level(a, lo.S, st)) return rc;
  }
  if (int rc = subtree_down(ops, ws, k, up, u, ld_u, st)) return rc;

  // (5) leaf interiors: u_int = S_leaf u_bnd + w (solver.py:269-276)
  {
    long long n = (long long)k * Lnb;
    HPSB_CUDA(launch_pdl(k_leaf_gather, dim3((unsigned)cdiv(n, T)), dim3(T), 0, st, k, P.L, P.nb,
                         (const int*)P.leaf_bnd_gidx, (const double*)u, ld_u, ws.Ub));
    HPSB_LAUNCH_CHECK();
    if (ops.shared_leaf) {
      GemmArgs a{};
      a.M = P.L; a.N = P.ni; a.K = P.nb; a.alpha = 1.0;
      a.A = ws.Ub; a.lda = P.nb; a.sA = Lnb; a.tA = 0;
      a.B = ops.S_leaf; a.ldb = P.ldb; a.sB = 0; a.tB = 1;
      a.beta = g ? 1.0 : 0.0; a.D = g ? ws.W : nullptr; a.ldd = ldw; a.sD = sw;
      a.C = u; a.ldc = P.ni; a.sC = ld_u; a.batch = k;
      if (int rc = gemm_nt(a, st)) return rc;
    } else {
      GemvArgs a{};
      a.mode = GEMV_LEAF; a.k = k; a.part = ws.part; a.cnt = ws.cnt;
      a.xin = ws.Ub; a.xin_k = Lnb; a.xin_s = P.nb;
      a.yout = u; a.yout_k = ld_u; a.yout_s = P.ni;
      a.yadd = g ? ws.W : nullptr; a.yadd_k = Lni; a.yadd_s = P.ni;
      if (int rc = gemv_level(a, ops.pSleaf, st)) return rc;
    }
  }
  return 0;
}

}  // namespace hpsb
