// C ABI (include/hpstep_b200.h): plan / operator-set lifecycle and solve.
#include <math.h>
#include <stdlib.h>
#include <stdarg.h>
#include <string.h>

#include <algorithm>
#include <map>
#include <mutex>
#include <unordered_map>
#include <vector>

#include "../../include/hpstep_b200.h"
#include "hps_plan.cuh"

namespace hpsb {

std::atomic<long long> g_launches{0};
std::atomic<int> g_ktimer_on{0};

// ---- per-kernel event timing (hps_ktimer_*)
struct KRec { cudaEvent_t a, b; const void* fn; };
static std::mutex g_kt_mu;
static std::vector<KRec> g_kt_recs;
static std::vector<cudaEvent_t> g_kt_pool;

static cudaEvent_t kt_event() {
  if (!g_kt_pool.empty()) { cudaEvent_t e = g_kt_pool.back(); g_kt_pool.pop_back(); return e; }
  cudaEvent_t e = nullptr;
  cudaEventCreate(&e);
  return e;
}

cudaEvent_t ktimer_begin(cudaStream_t st) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(st, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) return nullptr;
  std::lock_guard<std::mutex> lk(g_kt_mu);
  cudaEvent_t a = kt_event();
  if (a) cudaEventRecord(a, st);
  return a;
}

void ktimer_end(cudaEvent_t a, const void* fn, cudaStream_t st) {
  std::lock_guard<std::mutex> lk(g_kt_mu);
  cudaEvent_t b = kt_event();
  if (!b) return;
  cudaEventRecord(b, st);
  g_kt_recs.push_back({a, b, fn});
}
static thread_local char g_err[1024] = {0};
static thread_local long long g_err_node = -1;

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}
void set_error_node(long long node) { g_err_node = node; }

bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("HPSB_NO_PDL");
    return !(e && e[0] == '1');
  }();
  return on;
}

int gj_invert(int n, int batch, double* A, double* X, int ldx, long long sX, double* stats, cudaStream_t st);
int leaf_assemble(int Lc, int ni, int nb, const double* cv, int has_c1, int has_c2, int has_c,
                  const double* D2x, const double* D2y, const double* D1x, const double* D1y, double sigma,
                  double dtg, double* Aii, double* Aib, cudaStream_t st);
int merge_gather(int c, int n3, int n1a, int n2b, int nbc, const double* Tc, long long sTc, const int* i1a,
                 const int* i3a, const int* i2b, const int* i3b, double* X33, double* R, double* Tst, int ld3,
                 double* Tnew, cudaStream_t st);

static const double kPivotRtol = 1e-13;  // linalg.py:17

// Subtree-local slot numbering for the fused levels (see Plan::sub_slots),
// built from subtree b; false if some id is not covered.
static bool subtree_slots(const Plan& P, const int* const* gb, const int* const* j3, const int* lbg, int b,
                          std::vector<int>& slots, std::vector<long long>& off, std::vector<int>& jbase,
                          int& nslots) {
  const int nf = P.depth - P.dF;
  std::unordered_map<int, int> m;
  int ns = 0;
  const Level& R = P.lv[P.dF];
  for (int col = 0; col < R.n12; ++col) m[gb[P.dF][(size_t)b * R.n12 + col]] = ns++;
  jbase.assign(nf, 0);
  for (int e = 0; e < nf; ++e) {
    const int d = P.dF + e, npn = 1 << e;
    const Level& L = P.lv[d];
    jbase[e] = ns;
    for (int j = 0; j < npn; ++j)
      for (int r = 0; r < L.n3; ++r) m[j3[d][((size_t)b * npn + j) * L.n3 + r]] = ns++;
  }
  nslots = ns;
  slots.clear();
  off.assign(nf + 1, 0);
  auto slot = [&](int id, int& out) {
    auto it = m.find(id);
    if (it == m.end()) return false;
    out = it->second;
    return true;
  };
  for (int e = 0; e < nf; ++e) {
    const int d = P.dF + e, npn = 1 << e;
    const Level& L = P.lv[d];
    off[e] = (long long)slots.size();
    for (int j = 0; j < npn; ++j)
      for (int col = 0; col < L.n12; ++col) {
        int sl;
        if (!slot(gb[d][((size_t)b * npn + j) * L.n12 + col], sl)) return false;
        slots.push_back(sl);
      }
  }
  off[nf] = (long long)slots.size();
  const int nl = 1 << nf;
  for (int j = 0; j < nl; ++j)
    for (int col = 0; col < P.nb; ++col) {
      int sl;
      if (!slot(lbg[((size_t)b * nl + j) * P.nb + col], sl)) return false;
      slots.push_back(sl);
    }
  return true;
}

template <class T>
static int upload(const T* host, size_t count, T** dev) {
  *dev = nullptr;
  if (count == 0) return 0;
  HPSB_CUDA(cudaMalloc((void**)dev, count * sizeof(T)));
  HPSB_CUDA(cudaMemcpy(*dev, host, count * sizeof(T), cudaMemcpyHostToDevice));
  return 0;
}

static int even(int n) { return (n + 1) & ~1; }

// Returns the first failing batch entry (or -1) under the reference policy.
static int check_pivots(const double* dstats, int batch, int n, std::vector<double>& hs, cudaStream_t st) {
  hs.resize(2 * (size_t)batch);
  if (cudaStreamSynchronize(st) != cudaSuccess) return -2;
  if (cudaMemcpy(hs.data(), dstats, hs.size() * 8, cudaMemcpyDeviceToHost) != cudaSuccess) return -2;
  for (int b = 0; b < batch; ++b) {
    double pmin = hs[2 * b], pmax = hs[2 * b + 1];
    if (n > 0 && (!(pmax > 0.0) || !(pmin > kPivotRtol * pmax))) return b;
  }
  return -1;
}

static int singular(int n, double pmin, double pmax, const char* kind, long long node) {
  set_error("matrix of size %d is singular to tolerance %g (min/max pivot = %.3e/%.3e) [%s node %lld]", n,
            kPivotRtol, pmin, pmax, kind, node);
  set_error_node(node);
  return HPS_ERR_SINGULAR;
}

// Accuracy of the explicit inverses the solve applies.  Gauss-Jordan gives
// X ~ A^-1 with a relative residual of ~kappa*eps; the solves chain these
// products through every level of the tree and the time stepper applies the
// same operators thousands of times, so a residual that is systematic (the
// same every step) accumulates linearly.  One Newton step
// X <- X + X (I - A X) squares the residual; the products that use X in the
// build (S = X R) get one step of residual correction S <- S + X (R - A S).
// HPSB_NO_REFINE=1 skips both (A/B).
static bool refine_enabled() {
  static const bool on = [] {
    const char* e = getenv("HPSB_NO_REFINE");
    return !(e && e[0] == '1');
  }();
  return on;
}

// X (n x n per batch entry, ld ldx, stride sX) <- X + X (I - A X); A n x n dense (stride sA), batch entries.
// tmp: 2 * batch * n * n doubles; ident: n * n identity.
static int newton_inverse(int n, int batch, const double* A, long long sA, double* X, int ldx, long long sX,
                          double* tmp, const double* ident, cudaStream_t st) {
  double* E = tmp;
  double* Xn = tmp + (size_t)batch * n * n;
  GemmArgs r{};  // E = I - A X
  r.M = n; r.N = n; r.K = n; r.alpha = -1.0; r.beta = 1.0;
  r.A = A; r.lda = n; r.sA = sA; r.B = X; r.ldb = ldx; r.sB = sX;
  r.D = ident; r.ldd = n; r.sD = 0; r.C = E; r.ldc = n; r.sC = (long long)n * n; r.batch = batch;
  if (int rc = gemm(r, st)) return rc;
  GemmArgs u{};  // Xn = X + X E
  u.M = n; u.N = n; u.K = n; u.alpha = 1.0; u.beta = 1.0;
  u.A = X; u.lda = ldx; u.sA = sX; u.B = E; u.ldb = n; u.sB = (long long)n * n;
  u.D = X; u.ldd = ldx; u.sD = sX; u.C = Xn; u.ldc = n; u.sC = (long long)n * n; u.batch = batch;
  if (int rc = gemm(u, st)) return rc;
  HPSB_CUDA(cudaMemcpy2DAsync(X, (size_t)ldx * 8, Xn, (size_t)n * 8, (size_t)n * 8, (size_t)batch * n,
                              cudaMemcpyDeviceToDevice, st));
  (void)sX;
  return 0;
}

// S (M x N, ld lds, stride sS) = alpha X R refined once: S <- S + alpha X (R - A S / alpha) where X ~ A^-1.
// Implemented for the two uses: S = X R (alpha 1) and S = -X R (alpha -1).  tmp: batch * M * N doubles.
static int refine_solve(int M, int N, int batch, double alpha, const double* A, long long sA, const double* X,
                        int ldx, long long sX, const double* R, int ldr, long long sR, double* S, int lds,
                        long long sS, double* tmp, cudaStream_t st) {
  // residual of X^-1 S = alpha R:  Res = alpha R - A S
  GemmArgs r{};
  r.M = M; r.N = N; r.K = M; r.alpha = -1.0; r.beta = alpha;
  r.A = A; r.lda = M; r.sA = sA; r.B = S; r.ldb = lds; r.sB = sS;
  r.D = R; r.ldd = ldr; r.sD = sR; r.C = tmp; r.ldc = N; r.sC = (long long)M * N; r.batch = batch;
  if (int rc = gemm(r, st)) return rc;
  GemmArgs u{};  // S = S + X Res
  u.M = M; u.N = N; u.K = M; u.alpha = 1.0; u.beta = 1.0;
  u.A = X; u.lda = ldx; u.sA = sX; u.B = tmp; u.ldb = N; u.sB = (long long)M * N;
  u.D = S; u.ldd = lds; u.sD = sS; u.C = S; u.ldc = lds; u.sC = sS; u.batch = batch;
  return gemm(u, st);
}

}  // namespace hpsb

using namespace hpsb;


extern "C" {

int hps_version(void) { return 1; }

void hps_ktimer_enable(int on) { g_ktimer_on.store(on ? 1 : 0); }

int hps_ktimer_collect(char* names, int names_len, double* ms, long long* counts, int max) {
  if (cudaDeviceSynchronize() != cudaSuccess) { set_error("hps_ktimer_collect: device error"); return HPS_ERR_CUDA; }
  std::map<std::string, std::pair<double, long long>> agg;
  {
    std::lock_guard<std::mutex> lk(g_kt_mu);
    for (const KRec& r : g_kt_recs) {
      float t = 0.f;
      cudaEventElapsedTime(&t, r.a, r.b);
      const char* nm = nullptr;
      if (cudaFuncGetName(&nm, r.fn) != cudaSuccess || !nm) nm = "?";
      auto& v = agg[nm];
      v.first += t;
      v.second += 1;
      g_kt_pool.push_back(r.a);
      g_kt_pool.push_back(r.b);
    }
    g_kt_recs.clear();
  }
  // names: '\n'-separated, in the same order as ms / counts
  int n = 0;
  std::string all;
  for (auto& kv : agg) {
    if (n >= max) break;
    if (ms) ms[n] = kv.second.first;
    if (counts) counts[n] = kv.second.second;
    all += kv.first;
    all += '\n';
    ++n;
  }
  if (names && names_len > 0) {
    const size_t m = std::min((size_t)names_len - 1, all.size());
    memcpy(names, all.data(), m);
    names[m] = 0;
  }
  return n;
}

int hps_merge_node(int nbc, const double* Tc, int n1a, int n2b, int n3, const int* i1a, const int* i3a,
                   const int* i2b, const int* i3b, long long node_index, double* Xinv, double* S,
                   double* Tstack, double* T, void* stream) {
  if (nbc <= 0 || n3 <= 0 || n1a < 0 || n2b < 0 || !Tc || !i3a || !i3b || !Xinv || !S || !Tstack || !T) {
    set_error("hps_merge_node: bad arguments");
    return HPS_ERR_ARG;
  }
  cudaStream_t st = (cudaStream_t)stream;
  const int n12 = n1a + n2b;
  double *X33 = nullptr, *R = nullptr, *stats = nullptr;
  auto done = [&](int rc) {
    cudaFree(X33); cudaFree(R); cudaFree(stats);
    return rc;
  };
  if (cudaMalloc(&X33, (size_t)n3 * n3 * 8) != cudaSuccess || cudaMalloc(&R, (size_t)n3 * n12 * 8 + 8) != cudaSuccess ||
      cudaMalloc(&stats, 16) != cudaSuccess) {
    set_error("hps_merge_node: out of device memory");
    return done(HPS_ERR_CUDA);
  }
  // X33, [-T_a31 | T_b32], Tstack and the block diagonal of T (build.cu k_merge_gather, one node)
  if (int rc = merge_gather(1, n3, n1a, n2b, nbc, Tc, (long long)nbc * nbc, i1a, i3a, i2b, i3b, X33, R, Tstack,
                            n3, T, st))
    return done(rc);
  if (int rc = gj_invert(n3, 1, X33, Xinv, n3, (long long)n3 * n3, stats, st)) return done(rc);
  std::vector<double> hs;
  const int bad = check_pivots(stats, 1, n3, hs, st);
  if (bad == -2) { set_error("cuda error during merge"); return done(HPS_ERR_CUDA); }
  if (bad >= 0) return done(singular(n3, hs[0], hs[1], "merge", node_index));
  GemmArgs a{};  // S = Xinv [-T_a31 | T_b32]
  a.M = n3; a.N = n12; a.K = n3; a.alpha = 1.0; a.beta = 0.0;
  a.A = Xinv; a.lda = n3; a.B = R; a.ldb = n12; a.C = S; a.ldc = n12; a.batch = 1;
  if (int rc = gemm(a, st)) return done(rc);
  GemmArgs t{};  // T = blkdiag + Tstack S
  t.M = n12; t.N = n12; t.K = n3; t.alpha = 1.0; t.beta = 1.0;
  t.A = Tstack; t.lda = n3; t.B = S; t.ldb = n12; t.D = T; t.ldd = n12; t.C = T; t.ldc = n12; t.batch = 1;
  if (int rc = gemm(t, st)) return done(rc);
  if (cudaStreamSynchronize(st) != cudaSuccess) { set_error("cuda error during merge"); return done(HPS_ERR_CUDA); }
  return done(0);
}
long long hps_launch_count(void) { return g_launches.load(); }

int hps_ops_level_pairs(const hps_ops* ops) { return ops ? (int)ops->O.pairs.size() : 0; }
const char* hps_last_error(void) { return g_err; }
long long hps_last_error_node(void) { return g_err_node; }

int hps_plan_create(const hps_plan_desc* d, hps_plan** out) {
  *out = nullptr;
  g_err_node = -1;
  if (!d || d->n1 <= 0 || d->n2 <= 0 || d->p < 4 || d->depth < 0) {
    set_error("hps_plan_create: invalid descriptor");
    return HPS_ERR_ARG;
  }
  hps_plan* h = new hps_plan();
  Plan& P = h->P;
  P.n1 = d->n1; P.n2 = d->n2; P.p = d->p; P.q = d->p - 2;
  P.ni = d->ni; P.nb = d->nb; P.L = d->L; P.depth = d->depth; P.nbd = d->nbd; P.N = d->N;
  P.ldi = even(P.ni); P.ldb = even(P.nb);
  P.lv.resize(P.depth);
  int rc = 0;
  auto up = [&](const int* src, size_t n, int** dst) {
    if (rc) return;
    rc = upload(src, n, dst);
    if (!rc && *dst) h->allocs.push_back(*dst);
  };
  for (int l = 0; l < P.depth && !rc; ++l) {
    Level& lv = P.lv[l];
    lv.c = d->lvl_shape[5 * l]; lv.n3 = d->lvl_shape[5 * l + 1]; lv.n1a = d->lvl_shape[5 * l + 2];
    lv.n2b = d->lvl_shape[5 * l + 3]; lv.nbc = d->lvl_shape[5 * l + 4];
    lv.n12 = lv.n1a + lv.n2b; lv.ld3 = even(lv.n3); lv.ld12 = even(lv.n12);
    lv.h_i1a.assign(d->lvl_i1a[l], d->lvl_i1a[l] + lv.n1a);
    lv.h_i3a.assign(d->lvl_i3a[l], d->lvl_i3a[l] + lv.n3);
    lv.h_i2b.assign(d->lvl_i2b[l], d->lvl_i2b[l] + lv.n2b);
    lv.h_i3b.assign(d->lvl_i3b[l], d->lvl_i3b[l] + lv.n3);
    up(d->lvl_i1a[l], lv.n1a, &lv.i1a);
    up(d->lvl_i3a[l], lv.n3, &lv.i3a);
    up(d->lvl_i2b[l], lv.n2b, &lv.i2b);
    up(d->lvl_i3b[l], lv.n3, &lv.i3b);
    up(d->lvl_gidx_bnd[l], (size_t)lv.c * lv.n12, &lv.gidx_bnd);
    up(d->lvl_j3[l], (size_t)lv.c * lv.n3, &lv.j3);
    lv.node_index.assign(d->lvl_node_index[l], d->lvl_node_index[l] + lv.c);
  }
  // subtree partition: nparts = 2^lstar parts below a parent level lstar; the
  // fused subtree levels must lie inside one part
  P.nparts = d->nparts > 1 ? d->nparts : 1;
  while ((1 << P.lstar) < P.nparts) ++P.lstar;
  if ((1 << P.lstar) != P.nparts || (P.nparts > 1 && P.lstar >= P.depth)) {
    set_error("hps_plan_create: nparts = %d must be a power of two below 2^depth (depth %d)", d->nparts, P.depth);
    hps_plan_destroy(h);
    return HPS_ERR_ARG;
  }
  P.dF = std::max(fuse_level(P), P.lstar);
  if (const char* e = getenv("HPSB_FUSE_LEVEL"))  // A/B: first fused level (depth = none)
    P.dF = std::min(P.depth, std::max(P.lstar, atoi(e)));
  if (!rc && P.dF < P.depth) {
    std::vector<int> s0, s1;
    std::vector<long long> o0, o1;
    std::vector<int> j0, j1;
    int n0 = 0, n1 = 0;
    const int last = P.lv[P.dF].c - 1;
    bool ok = subtree_slots(P, d->lvl_gidx_bnd, d->lvl_j3, d->leaf_bnd_gidx, 0, s0, o0, j0, n0) &&
              subtree_slots(P, d->lvl_gidx_bnd, d->lvl_j3, d->leaf_bnd_gidx, last, s1, o1, j1, n1) &&
              s0 == s1 && n0 == n1;
    if (ok) {
      P.sub_local = true;
      P.sub_nslots = n0;
      P.sub_slot_off = o0;
      P.sub_j3_base = j0;
      up(s0.data(), s0.size(), &P.sub_slots);
    }
  }
  up(d->leaf_bnd_gidx, (size_t)P.L * P.nb, &P.leaf_bnd_gidx);
  up(d->boundary_ids, (size_t)P.nbd, &P.boundary_ids);
  if (P.depth > 0 && P.nbd > 0) {  // the root's boundary is the domain boundary: its position in fb order
    std::unordered_map<int, int> pos;
    for (int i = 0; i < P.nbd; ++i) pos[d->boundary_ids[i]] = i;
    const int n12 = P.lv[0].n12;
    std::vector<int> bp(n12, -1);
    bool all = true;
    for (int c = 0; c < n12 && all; ++c) {
      auto it = pos.find(d->lvl_gidx_bnd[0][c]);
      if (it == pos.end()) all = false;
      else bp[c] = it->second;
    }
    if (all) up(bp.data(), (size_t)n12, &P.root_bpos);
  }
  {  // boundary position of every edge DOF (the final stage combination writes the Dirichlet data itself)
    const long long e0 = (long long)P.L * P.ni, ne = P.N - e0;
    std::vector<int> eb((size_t)std::max(0LL, ne), -1);
    bool ok = true;
    for (int i = 0; i < P.nbd && ok; ++i) {
      const long long g = d->boundary_ids[i] - e0;
      if (g < 0 || g >= ne) ok = false;
      else eb[(size_t)g] = i;
    }
    if (ok && ne > 0) up(eb.data(), (size_t)ne, &P.edge_bpos);
  }
  P.leaf_node_index.assign(d->leaf_node_index, d->leaf_node_index + P.L);
  if (rc) { hps_plan_destroy(h); return rc; }
  *out = h;
  return HPS_OK;
}

void hps_plan_destroy(hps_plan* h) {
  if (!h) return;
  for (void* p : h->allocs) cudaFree(p);
  delete h;
}

static double* ops_alloc(Ops& O, size_t doubles, bool zero) {
  double* p = nullptr;
  if (doubles == 0) doubles = 1;
  if (cudaMalloc(&p, doubles * 8) != cudaSuccess) return nullptr;
  if (zero) cudaMemset(p, 0, doubles * 8);
  O.allocs.push_back(p);
  O.alloc_bytes.push_back(doubles * 8);
  O.bytes += doubles * 8;
  return p;
}

void hps_ops_destroy(hps_ops* h) {
  if (!h) return;
  for (void* p : h->O.allocs) cudaFree(p);
  for (void* p : h->O.aux) cudaFree(p);
  delete h;
}

size_t hps_ops_device_bytes(const hps_ops* h) { return h ? h->O.bytes : 0; }

int hps_ops_build(const hps_plan* hp, const hps_build_desc* d, void* stream, hps_ops** out) {
  *out = nullptr;
  g_err_node = -1;
  if (!hp || !d) { set_error("hps_ops_build: null argument"); return HPS_ERR_ARG; }
  cudaStream_t st = (cudaStream_t)stream;
  const Plan& P = hp->P;
  hps_ops* h = new hps_ops();
  Ops& O = h->O;
  O.plan = const_cast<Plan*>(&P);
  O.sigma = d->sigma; O.dtg = d->dt_gamma;
  O.shared_leaf = d->shared_leaf ? 1 : 0;
  if (d->layout == HPS_LAYOUT_SHARED && !O.shared_leaf) {
    set_error("hps_ops_build: the shared layout needs constant coefficients");
    delete h;
    return HPS_ERR_ARG;
  }
  O.shared_levels = d->layout == HPS_LAYOUT_SHARED ? 1 : 0;
  O.Lc = O.shared_leaf ? 1 : P.L;
  O.lo.resize(P.depth);
  const int ni = P.ni, nb = P.nb, m = ni + nb, Lc = O.Lc;
  std::vector<void*> tmp;
  auto fail = [&](int rc) {
    for (void* p : tmp) cudaFree(p);
    hps_ops_destroy(h);
    return rc;
  };
  auto talloc = [&](size_t doubles) -> double* {
    double* p = nullptr;
    if (doubles == 0) doubles = 1;
    if (cudaMalloc(&p, doubles * 8) != cudaSuccess) return nullptr;
    tmp.push_back(p);
    return p;
  };
  auto tfree = [&](double* p) {
    if (!p) return;
    auto it = std::find(tmp.begin(), tmp.end(), (void*)p);
    if (it != tmp.end()) { cudaFree(p); tmp.erase(it); }
  };
  // an n x n identity (Newton refinement of the explicit inverses)
  auto ident = [&](int n) -> double* {
    std::vector<double> h((size_t)n * n, 0.0);
    for (int i = 0; i < n; ++i) h[(size_t)i * n + i] = 1.0;
    double* p = talloc((size_t)n * n);
    if (p && cudaMemcpy(p, h.data(), h.size() * 8, cudaMemcpyHostToDevice) != cudaSuccess) return nullptr;
    return p;
  };
  const bool refine = refine_enabled();
  // stencil rows, coefficients
  double *dD2x, *dD2y, *dD1x, *dD1y, *dcoef;
  std::vector<double> Dbi((size_t)nb * ni), Dbb((size_t)nb * nb);
  for (int r = 0; r < nb; ++r) {
    for (int c = 0; c < ni; ++c) Dbi[(size_t)r * ni + c] = d->D_bnd[(size_t)r * m + c];
    for (int c = 0; c < nb; ++c) Dbb[(size_t)r * nb + c] = d->D_bnd[(size_t)r * m + ni + c];
  }
  double* dDbb;
  if (int rc = upload(d->D2x, (size_t)ni * m, &dD2x)) return fail(rc);
  tmp.push_back(dD2x);
  if (int rc = upload(d->D2y, (size_t)ni * m, &dD2y)) return fail(rc);
  tmp.push_back(dD2y);
  if (int rc = upload(d->D1x, (size_t)ni * m, &dD1x)) return fail(rc);
  tmp.push_back(dD1x);
  if (int rc = upload(d->D1y, (size_t)ni * m, &dD1y)) return fail(rc);
  tmp.push_back(dD1y);
  if (int rc = upload(d->coef, (size_t)Lc * 5 * ni, &dcoef)) return fail(rc);
  tmp.push_back(dcoef);
  if (int rc = upload(Dbb.data(), Dbb.size(), &dDbb)) return fail(rc);
  tmp.push_back(dDbb);
  O.D_bi = ops_alloc(O, (size_t)nb * ni, false);
  if (!O.D_bi) { set_error("out of device memory"); return fail(HPS_ERR_CUDA); }
  if (cudaMemcpy(O.D_bi, Dbi.data(), Dbi.size() * 8, cudaMemcpyHostToDevice) != cudaSuccess) {
    set_error("copy failed");
    return fail(HPS_ERR_CUDA);
  }

  // ---- leaves (solver.py:53-64, 112-125)
  double* Aii = talloc((size_t)Lc * ni * ni);
  double* Aib = talloc((size_t)Lc * ni * nb);
  double* stats = talloc(2 * (size_t)std::max(Lc, 1));
  // shared leaf: row-major operands of the leaf GEMMs; per-leaf: build row-major, then pack
  // shared leaf: rows ni..ni+nb-1 hold D_bi Ainv, so the solve's leaf pass is one GEMM for [w | h]
  double* Ainv = O.shared_leaf ? ops_alloc(O, (size_t)(ni + nb) * P.ldi, true) : talloc((size_t)Lc * ni * P.ldi);
  double* Sl = O.shared_leaf ? ops_alloc(O, (size_t)Lc * ni * P.ldb, true) : talloc((size_t)Lc * ni * P.ldb);
  double* Tleaf = d->keep_dtn ? ops_alloc(O, (size_t)Lc * nb * nb, false) : talloc((size_t)Lc * nb * nb);
  if (!Aii || !Aib || !stats || !Ainv || !Sl || !Tleaf) {
    set_error("out of device memory (leaf build)");
    return fail(HPS_ERR_CUDA);
  }
  if (!O.shared_leaf) {
    cudaMemsetAsync(Ainv, 0, (size_t)Lc * ni * P.ldi * 8, st);
    cudaMemsetAsync(Sl, 0, (size_t)Lc * ni * P.ldb * 8, st);
  }
  if (d->keep_dtn) O.T_leaf = Tleaf;
  if (int rc = leaf_assemble(Lc, ni, nb, dcoef, d->has_c1, d->has_c2, d->has_c, dD2x, dD2y, dD1x, dD1y,
                             d->sigma, d->dt_gamma, Aii, Aib, st))
    return fail(rc);
  double* Aii0 = refine ? talloc((size_t)Lc * ni * ni) : nullptr;  // A_ii (Gauss-Jordan overwrites it)
  if (refine) {
    if (!Aii0) { set_error("out of device memory (leaf build)"); return fail(HPS_ERR_CUDA); }
    HPSB_CUDA(cudaMemcpyAsync(Aii0, Aii, (size_t)Lc * ni * ni * 8, cudaMemcpyDeviceToDevice, st));
  }
  if (int rc = gj_invert(ni, Lc, Aii, Ainv, P.ldi, (long long)ni * P.ldi, stats, st)) return fail(rc);
  {
    std::vector<double> hs;
    int bad = check_pivots(stats, Lc, ni, hs, st);
    if (bad == -2) { set_error("cuda error during leaf build"); return fail(HPS_ERR_CUDA); }
    if (bad >= 0) return fail(singular(ni, hs[2 * bad], hs[2 * bad + 1], "leaf", P.leaf_node_index[bad]));
  }
  if (refine) {
    double* I = ident(ni);
    double* tmp = talloc(2 * (size_t)Lc * ni * std::max(ni, nb));
    if (!I || !tmp) { set_error("out of device memory (leaf refinement)"); return fail(HPS_ERR_CUDA); }
    if (int rc = newton_inverse(ni, Lc, Aii0, (long long)ni * ni, Ainv, P.ldi, (long long)ni * P.ldi, tmp, I, st))
      return fail(rc);
    tfree(tmp); tfree(I);
  }
  {
    GemmArgs a{};  // S = -Ainv A_ib
    a.M = ni; a.N = nb; a.K = ni; a.alpha = -1.0; a.beta = 0.0;
    a.A = Ainv; a.lda = P.ldi; a.sA = (long long)ni * P.ldi; a.tA = 0;
    a.B = Aib; a.ldb = nb; a.sB = (long long)ni * nb; a.tB = 0;
    a.C = Sl; a.ldc = P.ldb; a.sC = (long long)ni * P.ldb; a.batch = Lc;
    if (int rc = gemm(a, st)) return fail(rc);
    if (refine) {
      double* tmp = talloc((size_t)Lc * ni * nb);
      if (!tmp) { set_error("out of device memory (leaf refinement)"); return fail(HPS_ERR_CUDA); }
      if (int rc = refine_solve(ni, nb, Lc, -1.0, Aii0, (long long)ni * ni, Ainv, P.ldi, (long long)ni * P.ldi, Aib,
                                nb, (long long)ni * nb, Sl, P.ldb, (long long)ni * P.ldb, tmp, st))
        return fail(rc);
      tfree(tmp);
    }
    GemmArgs t{};  // T = D_bi S + D_bb
    t.M = nb; t.N = nb; t.K = ni; t.alpha = 1.0; t.beta = 1.0;
    t.A = O.D_bi; t.lda = ni; t.sA = 0; t.tA = 0;
    t.B = Sl; t.ldb = P.ldb; t.sB = (long long)ni * P.ldb; t.tB = 0;
    t.D = dDbb; t.ldd = nb; t.sD = 0;
    t.C = Tleaf; t.ldc = nb; t.sC = (long long)nb * nb; t.batch = Lc;
    if (int rc = gemm(t, st)) return fail(rc);
  }
  if (O.shared_leaf) {
    GemmArgs e{};  // E = D_bi Ainv (nb x ni) below Ainv
    e.M = nb; e.N = ni; e.K = ni; e.alpha = 1.0; e.beta = 0.0;
    e.A = O.D_bi; e.lda = ni; e.sA = 0; e.tA = 0;
    e.B = Ainv; e.ldb = P.ldi; e.sB = 0; e.tB = 0;
    e.C = Ainv + (size_t)ni * P.ldi; e.ldc = P.ldi; e.sC = 0; e.batch = 1;
    if (int rc = gemm(e, st)) return fail(rc);
    O.Ainv = Ainv;
    O.S_leaf = Sl;
  } else {
    O.pAinv = make_panel(P.L, ni, ni, P.nparts);
    O.pSleaf = make_panel(P.L, ni, nb, P.nparts);
    O.pAinv.base = ops_alloc(O, O.pAinv.total(), false);
    O.pSleaf.base = ops_alloc(O, O.pSleaf.total(), false);
    if (!O.pAinv.base || !O.pSleaf.base) { set_error("out of device memory (leaf panels)"); return fail(HPS_ERR_CUDA); }
    if (int rc = pack_panel(Ainv, (long long)ni * P.ldi, P.ldi, O.pAinv, st)) return fail(rc);
    if (int rc = pack_panel(Sl, (long long)ni * P.ldb, P.ldb, O.pSleaf, st)) return fail(rc);
    tfree(Ainv);
    tfree(Sl);
  }
  tfree(Aii); tfree(Aib); tfree(stats); tfree(Aii0);

  // ---- merges, deepest level first (solver.py:127-155)
  double* Tchild = Tleaf;
  long long sTchild = O.shared_leaf ? 0 : (long long)nb * nb;
  for (int l = P.depth - 1; l >= 0; --l) {
    const Level& lv = P.lv[l];
    LevelOps& lo = O.lo[l];
    const int ce = O.shared_leaf ? 1 : lv.c;
    const int n3 = lv.n3, n12 = lv.n12;
    double* Xinv = talloc((size_t)ce * n3 * lv.ld3);
    double* Tst = talloc((size_t)ce * n12 * lv.ld3);
    double* S = talloc((size_t)ce * n3 * lv.ld12);
    // every level's DtN map feeds its parent; the root's is kept (solver.py:155)
    const bool keepT = d->keep_dtn || l == 0;
    double* Tnew = keepT ? ops_alloc(O, (size_t)ce * n12 * n12, false) : talloc((size_t)ce * n12 * n12);
    double* X33 = talloc((size_t)ce * n3 * n3);
    double* R = talloc((size_t)ce * n3 * n12);
    double* lst = talloc(2 * (size_t)ce);
    const int nup = n3 + (l > 0 ? n12 : 0);
    if (O.shared_levels && l >= P.dF) {  // fused levels: ONE one-node tile read by every subtree CTA
      lo.Up = make_panel_nodes(1, nup, n3, 1);
      lo.S = make_panel_nodes(1, n3, n12, 1);
    } else if (O.shared_levels) {  // wide levels: one-node panels (or GEMM operands only)
      if (lv.c < kSharedGemmNodes) {
        lo.Up = make_panel(1, nup, n3);
        lo.S = make_panel(1, n3, n12);
      }
    } else if (l >= P.dF) {  // fused subtree levels: node-aligned tiles
      const int npn = 1 << (l - P.dF);
      lo.Up = make_panel_nodes(lv.c, nup, n3, npn);
      lo.S = make_panel_nodes(lv.c, n3, n12, npn);
    } else {  // wide levels: below lstar every part gets its own tiles
      const int parts = l >= P.lstar ? P.nparts : 1;
      lo.Up = make_panel(lv.c, nup, n3, parts);
      lo.S = make_panel(lv.c, n3, n12, parts);
    }
    if (lo.Up.c) lo.Up.base = ops_alloc(O, lo.Up.total(), false);
    if (lo.S.c) lo.S.base = ops_alloc(O, lo.S.total(), false);
    if (O.shared_levels) {
      lo.Ush = ops_alloc(O, (size_t)nup * lv.ld3, true);
      lo.Ssh = ops_alloc(O, (size_t)n3 * lv.ld12, true);
    }
    double* TX = l > 0 ? talloc((size_t)ce * n12 * lv.ld3) : nullptr;
    const bool ok_ops = O.shared_levels ? (lo.Ush && lo.Ssh && (!lo.Up.c || (lo.Up.base && lo.S.base)))
                                        : (lo.Up.base && lo.S.base);
    if (!Xinv || !Tst || !S || !Tnew || !X33 || !R || !lst || !ok_ops || (l > 0 && !TX)) {
      set_error("out of device memory (merge level %d)", l);
      return fail(HPS_ERR_CUDA);
    }
    cudaMemsetAsync(Xinv, 0, (size_t)ce * n3 * lv.ld3 * 8, st);
    cudaMemsetAsync(Tst, 0, (size_t)ce * n12 * lv.ld3 * 8, st);
    cudaMemsetAsync(S, 0, (size_t)ce * n3 * lv.ld12 * 8, st);
    if (int rc = merge_gather(ce, n3, lv.n1a, lv.n2b, lv.nbc, Tchild, sTchild, lv.i1a, lv.i3a, lv.i2b, lv.i3b,
                              X33, R, Tst, lv.ld3, Tnew, st))
      return fail(rc);
    double* X330 = refine ? talloc((size_t)ce * n3 * n3) : nullptr;  // X33 (Gauss-Jordan overwrites it)
    if (refine) {
      if (!X330) { set_error("out of device memory (merge level %d)", l); return fail(HPS_ERR_CUDA); }
      HPSB_CUDA(cudaMemcpyAsync(X330, X33, (size_t)ce * n3 * n3 * 8, cudaMemcpyDeviceToDevice, st));
    }
    if (int rc = gj_invert(n3, ce, X33, Xinv, lv.ld3, (long long)n3 * lv.ld3, lst, st)) return fail(rc);
    {
      std::vector<double> hs;
      int bad = check_pivots(lst, ce, n3, hs, st);
      if (bad == -2) { set_error("cuda error during merge build"); return fail(HPS_ERR_CUDA); }
      if (bad >= 0) return fail(singular(n3, hs[2 * bad], hs[2 * bad + 1], "merge", lv.node_index[bad]));
    }
    if (refine) {
      double* I = ident(n3);
      double* tmp = talloc(2 * (size_t)ce * n3 * n3);
      if (!I || !tmp) { set_error("out of device memory (merge level %d)", l); return fail(HPS_ERR_CUDA); }
      if (int rc = newton_inverse(n3, ce, X330, (long long)n3 * n3, Xinv, lv.ld3, (long long)n3 * lv.ld3, tmp, I, st))
        return fail(rc);
      tfree(tmp); tfree(I);
    }
    GemmArgs a{};  // S = Xinv [-Ta31 | Tb32]
    a.M = n3; a.N = n12; a.K = n3; a.alpha = 1.0; a.beta = 0.0;
    a.A = Xinv; a.lda = lv.ld3; a.sA = (long long)n3 * lv.ld3; a.tA = 0;
    a.B = R; a.ldb = n12; a.sB = (long long)n3 * n12; a.tB = 0;
    a.C = S; a.ldc = lv.ld12; a.sC = (long long)n3 * lv.ld12; a.batch = ce;
    if (int rc = gemm(a, st)) return fail(rc);
    if (refine) {
      double* tmp = talloc((size_t)ce * n3 * n12);
      if (!tmp) { set_error("out of device memory (merge level %d)", l); return fail(HPS_ERR_CUDA); }
      if (int rc = refine_solve(n3, n12, ce, 1.0, X330, (long long)n3 * n3, Xinv, lv.ld3, (long long)n3 * lv.ld3, R,
                                n12, (long long)n3 * n12, S, lv.ld12, (long long)n3 * lv.ld12, tmp, st))
        return fail(rc);
      tfree(tmp);
      tfree(X330);
    }
    {
      GemmArgs t{};  // T = blkdiag + Tstack S
      t.M = n12; t.N = n12; t.K = n3; t.alpha = 1.0; t.beta = 1.0;
      t.A = Tst; t.lda = lv.ld3; t.sA = (long long)n12 * lv.ld3; t.tA = 0;
      t.B = S; t.ldb = lv.ld12; t.sB = (long long)n3 * lv.ld12; t.tB = 0;
      t.D = Tnew; t.ldd = n12; t.sD = (long long)n12 * n12;
      t.C = Tnew; t.ldc = n12; t.sC = (long long)n12 * n12; t.batch = ce;
      if (int rc = gemm(t, st)) return fail(rc);
    }
    // pack into the streaming layout; constant coefficients: every node of a
    // level is identical (solver.py stores one copy per node, so do we)
    const long long bx = ce < lv.c ? 0 : 1;
    if (l > 0) {
      GemmArgs x{};  // TX = Tstack X33^-1: the flux rows of the stacked up-pass operator
      x.M = n12; x.N = n3; x.K = n3; x.alpha = 1.0; x.beta = 0.0;
      x.A = Tst; x.lda = lv.ld3; x.sA = (long long)n12 * lv.ld3; x.tA = 0;
      x.B = Xinv; x.ldb = lv.ld3; x.sB = (long long)n3 * lv.ld3; x.tB = 0;
      x.C = TX; x.ldc = lv.ld3; x.sC = (long long)n12 * lv.ld3; x.batch = ce;
      if (int rc = gemm(x, st)) return fail(rc);
    }
    if (lo.Up.base) {
      if (int rc = pack_panel2(Xinv, bx * n3 * lv.ld3, lv.ld3, n3, l > 0 ? TX : Xinv, bx * n12 * lv.ld3, lv.ld3,
                               lo.Up, st))
        return fail(rc);
      if (int rc = pack_panel(S, bx * n3 * lv.ld12, lv.ld12, lo.S, st)) return fail(rc);
    }
    if (O.shared_levels) {
      HPSB_CUDA(cudaMemcpyAsync(lo.Ush, Xinv, (size_t)n3 * lv.ld3 * 8, cudaMemcpyDeviceToDevice, st));
      if (l > 0)
        HPSB_CUDA(cudaMemcpyAsync(lo.Ush + (size_t)n3 * lv.ld3, TX, (size_t)n12 * lv.ld3 * 8,
                                  cudaMemcpyDeviceToDevice, st));
      HPSB_CUDA(cudaMemcpyAsync(lo.Ssh, S, (size_t)n3 * lv.ld12 * 8, cudaMemcpyDeviceToDevice, st));
    }
    if (l == 0) {  // the reference keeps every merge's Tstack; the solve never reads the root's
      O.root_Tst = ops_alloc(O, (size_t)n12 * lv.ld3, false);
      if (!O.root_Tst) { set_error("out of device memory (root Tstack)"); return fail(HPS_ERR_CUDA); }
      HPSB_CUDA(cudaMemcpyAsync(O.root_Tst, Tst, (size_t)n12 * lv.ld3 * 8, cudaMemcpyDeviceToDevice, st));
    }
    tfree(Xinv); tfree(Tst); tfree(S); tfree(TX);
    if (!d->keep_dtn) tfree(Tchild);
    tfree(X33); tfree(R); tfree(lst);
    if (keepT) lo.T = Tnew;
    Tchild = Tnew;
    sTchild = O.shared_leaf ? 0 : (long long)n12 * n12;
  }
  if (P.depth > 0) O.root_T = O.lo[0].T;
  if (int rc = sub_mma_prepare(O, st)) return fail(rc);
  if (int rc = mega_pairs_prepare(O, st)) return fail(rc);
  if (cudaStreamSynchronize(st) != cudaSuccess) {
    set_error("cuda error at end of build: %s", cudaGetErrorString(cudaGetLastError()));
    return fail(HPS_ERR_CUDA);
  }
  for (void* p : tmp) cudaFree(p);
  *out = h;
  return HPS_OK;
}

static int copy_panel_block(const Panel& pn, int node, double* host, int row0 = 0, int nrows = -1) {
  double* tmp = nullptr;
  if (nrows < 0) nrows = pn.R;
  HPSB_CUDA(cudaDeviceSynchronize());
  HPSB_CUDA(cudaMalloc(&tmp, (size_t)nrows * pn.C * 8 + 8));
  int rc = unpack_panel(pn, node, row0, nrows, tmp, 0);
  if (!rc && cudaMemcpy(host, tmp, (size_t)nrows * pn.C * 8, cudaMemcpyDeviceToHost) != cudaSuccess) {
    set_error("copy failed");
    rc = HPS_ERR_CUDA;
  }
  cudaFree(tmp);
  return rc;
}

int hps_ops_get_leaf(const hps_ops* h, int which, int leaf, double* host) {
  if (!h) return HPS_ERR_ARG;
  const Ops& O = h->O;
  const Plan& P = *O.plan;
  int l = O.shared_leaf ? 0 : leaf;
  if (leaf < 0 || leaf >= P.L) { set_error("leaf out of range"); return HPS_ERR_ARG; }
  if (!O.shared_leaf && which <= 1) return copy_panel_block(which == 0 ? O.pAinv : O.pSleaf, leaf, host);
  const double* src; int rows, cols, ld;
  if (which == 0) { src = O.Ainv + (size_t)l * P.ni * P.ldi; rows = P.ni; cols = P.ni; ld = P.ldi; }
  else if (which == 1) { src = O.S_leaf + (size_t)l * P.ni * P.ldb; rows = P.ni; cols = P.nb; ld = P.ldb; }
  else if (which == 2 && O.T_leaf) { src = O.T_leaf + (size_t)l * P.nb * P.nb; rows = P.nb; cols = P.nb; ld = P.nb; }
  else { set_error("leaf block %d not available", which); return HPS_ERR_ARG; }
  HPSB_CUDA(cudaDeviceSynchronize());
  HPSB_CUDA(cudaMemcpy2D(host, cols * 8, src, ld * 8, cols * 8, rows, cudaMemcpyDeviceToHost));
  return HPS_OK;
}

int hps_ops_get_merge(const hps_ops* h, int level, int node, int which, double* host) {
  if (!h) return HPS_ERR_ARG;
  const Ops& O = h->O;
  const Plan& P = *O.plan;
  if (level < 0 || level >= P.depth) { set_error("level out of range"); return HPS_ERR_ARG; }
  const Level& lv = P.lv[level];
  const LevelOps& lo = O.lo[level];
  if (node < 0 || node >= lv.c) { set_error("node out of range"); return HPS_ERR_ARG; }
  if (O.shared_levels && (which == 0 || which == 2 || which == 4)) {  // one operator for every node
    const double* src = which == 0 ? lo.Ush : which == 4 ? lo.Ush + (size_t)lv.n3 * lv.ld3 : lo.Ssh;
    const int rows = which == 4 ? lv.n12 : lv.n3, cols = which == 2 ? lv.n12 : lv.n3;
    const int ld = which == 2 ? lv.ld12 : lv.ld3;
    if (which == 4 && level == 0) { set_error("the root has no flux rows"); return HPS_ERR_ARG; }
    HPSB_CUDA(cudaDeviceSynchronize());
    HPSB_CUDA(cudaMemcpy2D(host, cols * 8, src, ld * 8, cols * 8, rows, cudaMemcpyDeviceToHost));
    return HPS_OK;
  }
  if (which == 0) return copy_panel_block(lo.Up, node, host, 0, lv.n3);
  if (which == 1) {
    if (level > 0) { set_error("Tstack of level %d is stored as Tstack X33^-1 (which=4)", level); return HPS_ERR_ARG; }
    HPSB_CUDA(cudaDeviceSynchronize());
    HPSB_CUDA(cudaMemcpy2D(host, lv.n3 * 8, O.root_Tst, lv.ld3 * 8, lv.n3 * 8, lv.n12, cudaMemcpyDeviceToHost));
    return HPS_OK;
  }
  if (which == 4) {
    if (level == 0) { set_error("the root has no flux rows"); return HPS_ERR_ARG; }
    return copy_panel_block(lo.Up, node, host, lv.n3, lv.n12);
  }
  if (which == 2) return copy_panel_block(lo.S, node, host);
  if (which == 3 && lo.T) {
    int nn = O.shared_leaf ? 0 : node;
    HPSB_CUDA(cudaDeviceSynchronize());
    HPSB_CUDA(cudaMemcpy(host, lo.T + (size_t)nn * lv.n12 * lv.n12, (size_t)lv.n12 * lv.n12 * 8,
                         cudaMemcpyDeviceToHost));
    return HPS_OK;
  }
  set_error("merge block %d not available", which);
  return HPS_ERR_ARG;
}

size_t hps_solve_workspace_bytes(const hps_plan* h, int k) { return h ? workspace_bytes(h->P, k) : 0; }

int hps_solve(const hps_ops* h, int k, const double* fb, long long ld_f, const double* g, long long ld_g,
              const double* jump, long long ld_jump, double inv_dt, double* u, long long ld_u, void* ws,
              size_t ws_bytes, void* stream) {
  if (!h || !fb || !u || !ws) { set_error("hps_solve: null argument"); return HPS_ERR_ARG; }
  return solve(h->O, SOLVE_ALL, 0, h->O.plan->nparts, k, fb, ld_f, g, ld_g, jump, ld_jump, inv_dt, u, ld_u, ws,
               ws_bytes, (cudaStream_t)stream);
}

int hps_solve_stage(const hps_ops* h, int k, const double* fb, long long ld_f, const double* g, long long ld_g,
                    double* u, long long ld_u, double* lu_int, long long ld_lu, double* guard,
                    const double* root_pre, void* ws, size_t ws_bytes, void* stream) {
  if (!h || !fb || !u || !ws) { set_error("hps_solve_stage: null argument"); return HPS_ERR_ARG; }
  const Ops& O = h->O;
  if (!(O.shared_leaf && O.fd && leaf_fd_down_enabled())) {
    set_error("hps_solve_stage: needs the tensor-product leaf solve (constant coefficients)");
    return HPS_ERR_ARG;
  }
  if (root_pre && k != 1) { set_error("hps_solve_stage: root_pre needs k = 1"); return HPS_ERR_ARG; }
  return solve(O, SOLVE_ALL, 0, O.plan->nparts, k, fb, ld_f, g, ld_g, nullptr, 0, 0.0, u, ld_u, ws, ws_bytes,
               (cudaStream_t)stream, lu_int, ld_lu, guard, root_pre);
}

int hps_solve_stage_terms(const hps_ops* h, const double* fb, int nterms, const double* dcoefs,
                          const double* const* vecs, double* r_out, double* u, double* lu_int, double* guard,
                          const double* root_pre, void* ws, size_t ws_bytes, void* stream) {
  if (!h || !fb || !u || !ws || !r_out || !dcoefs || !vecs) {
    set_error("hps_solve_stage_terms: null argument");
    return HPS_ERR_ARG;
  }
  const Ops& O = h->O;
  if (!(O.shared_leaf && O.fd && leaf_fd_down_enabled())) {
    set_error("hps_solve_stage_terms: needs the tensor-product leaf solve (constant coefficients)");
    return HPS_ERR_ARG;
  }
  if (nterms < 1 || nterms > 12) { set_error("hps_solve_stage_terms: %d terms (1..12)", nterms); return HPS_ERR_ARG; }
  StageTerms T;
  T.nterm = nterms; T.tdc = dcoefs; T.rout = r_out;
  for (int t = 0; t < nterms; ++t) T.tv[t] = vecs[t];
  const long long N = h->O.plan->N;
  T.ld_rout = N;
  return solve(O, SOLVE_ALL, 0, O.plan->nparts, 1, fb, 0, r_out, 0, nullptr, 0, 0.0, u, N, ws, ws_bytes,
               (cudaStream_t)stream, lu_int, N, guard, root_pre, &T);
}

int hps_solve_stage_terms_k(const hps_ops* h, int k, const double* fb, long long ld_f, int nterms,
                            const double* dcoefs, const double* const* vecs, const long long* vec_ld, double* r_out,
                            long long ld_r, double* u, long long ld_u, double* lu_int, long long ld_lu, double* guard,
                            void* ws, size_t ws_bytes, void* stream) {
  if (!h || !fb || !u || !ws || !r_out || !dcoefs || !vecs || !vec_ld || k <= 0) {
    set_error("hps_solve_stage_terms_k: null argument or k <= 0");
    return HPS_ERR_ARG;
  }
  const Ops& O = h->O;
  if (!(O.shared_leaf && O.fd && leaf_fd_down_enabled())) {
    set_error("hps_solve_stage_terms_k: needs the tensor-product leaf solve (constant coefficients)");
    return HPS_ERR_ARG;
  }
  if (nterms < 1 || nterms > 12) { set_error("hps_solve_stage_terms_k: %d terms (1..12)", nterms); return HPS_ERR_ARG; }
  StageTerms T;
  T.nterm = nterms; T.tdc = dcoefs; T.rout = r_out; T.ld_rout = ld_r;
  for (int t = 0; t < nterms; ++t) { T.tv[t] = vecs[t]; T.tld[t] = vec_ld[t]; }
  return solve(O, SOLVE_ALL, 0, O.plan->nparts, k, fb, ld_f, r_out, ld_r, nullptr, 0, 0.0, u, ld_u, ws, ws_bytes,
               (cudaStream_t)stream, lu_int, ld_lu, guard, nullptr, &T);
}

size_t hps_root_dirichlet_scratch(const hps_ops* h, int ns) { return h ? root_dirichlet_scratch(*h->O.plan, ns) : 0; }

int hps_root_dirichlet(const hps_ops* h, int ns, const double* fb, long long ld_f, double* out, long long ld_out,
                       void* scratch, size_t scratch_bytes, void* stream) {
  if (!h || !fb || !out || !scratch) { set_error("hps_root_dirichlet: null argument"); return HPS_ERR_ARG; }
  if (scratch_bytes < root_dirichlet_scratch(*h->O.plan, ns)) {
    set_error("hps_root_dirichlet: scratch too small");
    return HPS_ERR_ARG;
  }
  if (root_dirichlet(h->O, ns, fb, ld_f, out, ld_out, (double*)scratch, (cudaStream_t)stream)) return HPS_ERR_ARG;
  return HPS_OK;
}

int hps_leaf_lu(const hps_ops* h, int leaf0, int nleaf, int k, const double* u, long long ld_u, double* lu_int,
                long long ld_lu, double* guard, void* stream) {
  if (!h || !u || !lu_int) { set_error("hps_leaf_lu: null argument"); return HPS_ERR_ARG; }
  const Ops& O = h->O;
  const Plan& P = *O.plan;
  if (!(O.shared_leaf && O.fd)) {
    set_error("hps_leaf_lu: needs the tensor-product leaf solve (constant coefficients)");
    return HPS_ERR_ARG;
  }
  if (leaf0 < 0 || nleaf < 0 || leaf0 + nleaf > P.L || k <= 0) {
    set_error("hps_leaf_lu: leaf range [%d, %d) of %d, k = %d", leaf0, leaf0 + nleaf, P.L, k);
    return HPS_ERR_ARG;
  }
  if (leaf_fd_lu(O, k, nleaf, P.leaf_bnd_gidx + (long long)leaf0 * P.nb, u, ld_u, u + (long long)leaf0 * P.ni,
                 lu_int, ld_lu, guard, (cudaStream_t)stream))
    return HPS_ERR_CUDA;
  return HPS_OK;
}

int hps_plan_partition(const hps_plan* h, int k, int* nparts, int* lstar, int* n12, long long* flux_offset) {
  if (!h) { set_error("hps_plan_partition: null plan"); return HPS_ERR_ARG; }
  const Plan& P = h->P;
  if (nparts) *nparts = P.nparts;
  if (lstar) *lstar = P.lstar;
  if (n12) *n12 = P.nparts > 1 ? P.lv[P.lstar].n12 : 0;
  if (flux_offset) *flux_offset = P.nparts > 1 && k > 0 ? (long long)exchange_offset(P, k) : -1;
  return HPS_OK;
}

int hps_plan_fused_level(const hps_plan* h) { return h ? h->P.dF : -1; }

int hps_workspace_level(const hps_plan* h, int k, int level, long long* w3_off, long long* h_off) {
  if (!h || k <= 0 || level < 0 || level >= h->P.depth) {
    set_error("hps_workspace_level: bad arguments");
    return HPS_ERR_ARG;
  }
  long long w = -1, f = -1;
  level_offsets(h->P, k, level, w, f);
  if (w3_off) *w3_off = w;
  if (h_off) *h_off = f;
  return HPS_OK;
}

int hps_top_level(const hps_ops* h, int level, int down, int rank, int nranks, int k, double* u, long long ld_u,
                  double* stage, void* ws, size_t ws_bytes, void* stream) {
  if (!h || !u || !ws) { set_error("hps_top_level: null argument"); return HPS_ERR_ARG; }
  return top_level(h->O, level, down != 0, rank, nranks, k, u, ld_u, stage, ws, ws_bytes, (cudaStream_t)stream);
}

int hps_solve_phase(const hps_ops* h, int phases, int part0, int part1, int k, const double* fb, long long ld_f,
                    const double* g, long long ld_g, const double* jump, long long ld_jump, double inv_dt,
                    double* u, long long ld_u, void* ws, size_t ws_bytes, void* stream) {
  if (!h || !u || !ws || ((phases & SOLVE_TOP) && !fb)) { set_error("hps_solve_phase: null argument"); return HPS_ERR_ARG; }
  if (phases <= 0 || phases > SOLVE_ALL) { set_error("hps_solve_phase: bad phase mask %d", phases); return HPS_ERR_ARG; }
  return solve(h->O, phases, part0, part1, k, fb, ld_f, g, ld_g, jump, ld_jump, inv_dt, u, ld_u, ws, ws_bytes,
               (cudaStream_t)stream);
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Operator-set persistence (solver.py:294-337): the device buffers and the
// structure that points into them, as one flat host byte stream.  Pointers are
// stored as indices of the owning allocation.
// ---------------------------------------------------------------------------
namespace {

constexpr unsigned long long kDumpMagic = 0x32425350484244ULL;  // "DBHPSB2"

struct Writer {
  std::vector<unsigned char>* out;
  template <class T>
  void put(const T& v) {
    const unsigned char* p = reinterpret_cast<const unsigned char*>(&v);
    out->insert(out->end(), p, p + sizeof(T));
  }
};

struct Reader {
  const unsigned char* p;
  size_t left;
  bool ok = true;
  template <class T>
  T get() {
    T v{};
    if (left < sizeof(T)) { ok = false; return v; }
    memcpy(&v, p, sizeof(T));
    p += sizeof(T);
    left -= sizeof(T);
    return v;
  }
};

long long alloc_index(const Ops& O, const void* ptr) {
  if (!ptr) return -1;
  for (size_t i = 0; i < O.allocs.size(); ++i)
    if (O.allocs[i] == ptr) return (long long)i;
  return -2;
}

void put_panel(Writer& w, const Ops& O, const Panel& pn) {
  w.put(pn.c); w.put(pn.R); w.put(pn.C); w.put(pn.TR); w.put(pn.TS); w.put(pn.ntiles); w.put(pn.parts);
  w.put(alloc_index(O, pn.base));
}

void get_panel(Reader& r, Panel& pn, long long& idx) {
  pn.c = r.get<int>(); pn.R = r.get<int>(); pn.C = r.get<int>(); pn.TR = r.get<int>(); pn.TS = r.get<int>();
  pn.ntiles = r.get<int>(); pn.parts = r.get<int>();
  idx = r.get<long long>();
}

// the structure (everything but the raw buffers)
bool write_structure(const Ops& O, Writer& w) {
  const Plan& P = *O.plan;
  w.put(kDumpMagic);
  w.put(O.sigma); w.put(O.dtg); w.put(O.shared_leaf); w.put(O.shared_levels); w.put(O.Lc);
  w.put(P.depth); w.put(P.L); w.put(P.ni); w.put(P.nb); w.put(P.N); w.put(P.nparts);
  std::vector<long long> ptrs = {alloc_index(O, O.Ainv), alloc_index(O, O.S_leaf), alloc_index(O, O.T_leaf),
                                 alloc_index(O, O.D_bi), alloc_index(O, O.root_T), alloc_index(O, O.root_Tst),
                                 alloc_index(O, O.fd)};
  for (long long i : ptrs) { if (i == -2) return false; w.put(i); }
  put_panel(w, O, O.pAinv);
  put_panel(w, O, O.pSleaf);
  for (const LevelOps& lo : O.lo) {
    put_panel(w, O, lo.Up);
    put_panel(w, O, lo.S);
    for (const void* q : {(const void*)lo.Ush, (const void*)lo.Ssh, (const void*)lo.T}) {
      long long i = alloc_index(O, q);
      if (i == -2) return false;
      w.put(i);
    }
  }
  w.put((long long)O.allocs.size());
  for (size_t b : O.alloc_bytes) w.put((unsigned long long)b);
  return true;
}

}  // namespace

extern "C" {

long long hps_ops_dump_size(const hps_ops* h) {
  if (!h) return -1;
  std::vector<unsigned char> head;
  Writer w{&head};
  if (!write_structure(h->O, w)) return -1;
  size_t n = head.size();
  for (size_t b : h->O.alloc_bytes) n += b;
  return (long long)n;
}

int hps_ops_dump(const hps_ops* h, void* host, long long size) {
  if (!h || !host) { set_error("hps_ops_dump: null argument"); return HPS_ERR_ARG; }
  std::vector<unsigned char> head;
  Writer w{&head};
  if (!write_structure(h->O, w)) { set_error("hps_ops_dump: unowned operator pointer"); return HPS_ERR_ARG; }
  if (size < hps_ops_dump_size(h)) { set_error("hps_ops_dump: buffer too small"); return HPS_ERR_ARG; }
  unsigned char* dst = (unsigned char*)host;
  memcpy(dst, head.data(), head.size());
  dst += head.size();
  HPSB_CUDA(cudaDeviceSynchronize());
  for (size_t i = 0; i < h->O.allocs.size(); ++i) {
    HPSB_CUDA(cudaMemcpy(dst, h->O.allocs[i], h->O.alloc_bytes[i], cudaMemcpyDeviceToHost));
    dst += h->O.alloc_bytes[i];
  }
  return HPS_OK;
}

int hps_ops_load(const hps_plan* hp, const void* host, long long size, hps_ops** out) {
  *out = nullptr;
  if (!hp || !host) { set_error("hps_ops_load: null argument"); return HPS_ERR_ARG; }
  const Plan& P = hp->P;
  Reader r{(const unsigned char*)host, (size_t)size};
  if (r.get<unsigned long long>() != kDumpMagic) { set_error("hps_ops_load: not an operator dump"); return HPS_ERR_ARG; }
  hps_ops* h = new hps_ops();
  Ops& O = h->O;
  O.plan = const_cast<Plan*>(&P);
  O.sigma = r.get<double>(); O.dtg = r.get<double>(); O.shared_leaf = r.get<int>();
  O.shared_levels = r.get<int>(); O.Lc = r.get<int>();
  const int depth = r.get<int>(), L = r.get<int>(), ni = r.get<int>(), nb = r.get<int>();
  const long long N = r.get<long long>();
  const int nparts = r.get<int>();
  if (!r.ok || depth != P.depth || L != P.L || ni != P.ni || nb != P.nb || N != P.N || nparts != P.nparts) {
    delete h;
    set_error("hps_ops_load: dump was made for a different tree");
    return HPS_ERR_ARG;
  }
  long long ptr[7];
  for (long long& i : ptr) i = r.get<long long>();
  long long iA, iS;
  get_panel(r, O.pAinv, iA);
  get_panel(r, O.pSleaf, iS);
  O.lo.resize(depth);
  std::vector<long long> lidx((size_t)depth * 5);
  for (int d = 0; d < depth; ++d) {
    get_panel(r, O.lo[d].Up, lidx[5 * d]);
    get_panel(r, O.lo[d].S, lidx[5 * d + 1]);
    for (int j = 2; j < 5; ++j) lidx[5 * d + j] = r.get<long long>();
  }
  const long long na = r.get<long long>();
  std::vector<size_t> sizes;
  for (long long i = 0; i < na && r.ok; ++i) sizes.push_back((size_t)r.get<unsigned long long>());
  size_t need = 0;
  for (size_t b : sizes) need += b;
  if (!r.ok || r.left < need) { delete h; set_error("hps_ops_load: truncated dump"); return HPS_ERR_ARG; }
  for (size_t b : sizes) {
    void* p = nullptr;
    if (cudaMalloc(&p, b ? b : 8) != cudaSuccess) {
      hps_ops_destroy(h);
      set_error("hps_ops_load: out of device memory");
      return HPS_ERR_CUDA;
    }
    O.allocs.push_back(p);
    O.alloc_bytes.push_back(b);
    O.bytes += b;
    if (cudaMemcpy(p, r.p, b, cudaMemcpyHostToDevice) != cudaSuccess) {
      hps_ops_destroy(h);
      set_error("hps_ops_load: copy failed");
      return HPS_ERR_CUDA;
    }
    r.p += b;
    r.left -= b;
  }
  auto at = [&](long long i) -> double* { return i >= 0 && i < na ? (double*)O.allocs[(size_t)i] : nullptr; };
  O.Ainv = at(ptr[0]); O.S_leaf = at(ptr[1]); O.T_leaf = at(ptr[2]); O.D_bi = at(ptr[3]);
  O.root_T = at(ptr[4]); O.root_Tst = at(ptr[5]); O.fd = at(ptr[6]);
  O.pAinv.base = at(iA); O.pSleaf.base = at(iS);
  for (int d = 0; d < depth; ++d) {
    LevelOps& lo = O.lo[d];
    lo.Up.base = at(lidx[5 * d]); lo.S.base = at(lidx[5 * d + 1]);
    lo.Ush = at(lidx[5 * d + 2]); lo.Ssh = at(lidx[5 * d + 3]); lo.T = at(lidx[5 * d + 4]);
  }
  if (int rc = sub_mma_prepare(O, 0)) { hps_ops_destroy(h); return rc; }
  if (int rc = mega_pairs_prepare(O, 0)) { hps_ops_destroy(h); return rc; }
  if (cudaDeviceSynchronize() != cudaSuccess) {
    hps_ops_destroy(h);
    set_error("hps_ops_load: %s", cudaGetErrorString(cudaGetLastError()));
    return HPS_ERR_CUDA;
  }
  *out = h;
  return HPS_OK;
}

}  // extern "C"

extern "C" int hps_ops_set_leaf_fd(hps_ops* h, const double* host, int count) {
  if (!h) { set_error("hps_ops_set_leaf_fd: null ops"); return HPS_ERR_ARG; }
  Ops& O = h->O;
  const Plan& P = *O.plan;
  if (!host) { O.fd = nullptr; return HPS_OK; }  // disable (the buffer stays owned)
  const int q = P.q;
  if (!O.shared_leaf || !leaf_fd_supported(q) || count != 5 * q * q + 8 * q + 513) {
    set_error("hps_ops_set_leaf_fd: needs constant coefficients, q in [4, 14] and %d values",
              5 * q * q + 8 * q + 513);
    return HPS_ERR_ARG;
  }
  double* d = ops_alloc(O, (size_t)count, false);
  if (!d) { set_error("out of device memory"); return HPS_ERR_CUDA; }
  HPSB_CUDA(cudaMemcpy(d, host, (size_t)count * 8, cudaMemcpyHostToDevice));
  O.fd = d;
  return HPS_OK;
}
