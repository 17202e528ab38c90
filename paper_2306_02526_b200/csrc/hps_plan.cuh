// Internal plan / operator-set structures (device-resident, level-contiguous).
#pragma once

#include <algorithm>
#include <vector>

#include "hps_common.cuh"

namespace hpsb {

// One parent level of the binary tree (level 0 = root).  All nodes of a
// level share the same shapes and the same child-local index maps
// (i1a, i3a, i2b, i3b); only the global ids (gidx_bnd, j3) differ per node.
struct Level {
  int c = 0;       // nodes on the level
  int n3 = 0;      // |J3| interface size
  int n1a = 0;     // |J1| (alpha's outer boundary)
  int n2b = 0;     // |J2|
  int n12 = 0;     // n1a + n2b = node boundary size
  int nbc = 0;     // child boundary size (= n1a + n3 = n2b + n3)
  int ld3 = 0;     // even-padded row length for n3-column matrices
  int ld12 = 0;    // even-padded row length for n12-column matrices
  int *i1a = nullptr, *i3a = nullptr, *i2b = nullptr, *i3b = nullptr;  // device
  int* gidx_bnd = nullptr;  // device, c x n12 global ids
  int* j3 = nullptr;        // device, c x n3 global ids
  std::vector<long long> node_index;  // host: DFS node index (error reports)
  std::vector<int> h_i1a, h_i3a, h_i2b, h_i3b;
};

struct Plan {
  int n1 = 0, n2 = 0, p = 0, q = 0, ni = 0, nb = 0, L = 0, depth = 0, nbd = 0;
  long long N = 0;
  std::vector<Level> lv;          // depth entries, root first
  int* leaf_bnd_gidx = nullptr;   // device L x nb
  int* boundary_ids = nullptr;    // device nbd
  int* root_bpos = nullptr;       // device lv[0].n12: fb position of each root boundary DOF (null: not all on the boundary)
  int* edge_bpos = nullptr;       // device N - L*ni: fb position of each edge DOF, -1 off the domain boundary
  std::vector<long long> leaf_node_index;  // host
  int dF = 0;                     // levels d >= dF run as fused subtree kernels
  // subtree-local numbering of the DOFs a fused subtree touches (the same for
  // every level-dF subtree): slots [0, n12_dF) = the subtree root's boundary,
  // then every subtree node's interface (j3) level by level.  sub_slots maps
  // each fused level's gidx_bnd (and the leaves' boundaries) to slots.
  bool sub_local = false;
  int sub_nslots = 0;
  int* sub_slots = nullptr;                 // device
  std::vector<long long> sub_slot_off;      // per fused level, then the leaves
  std::vector<int> sub_j3_base;             // first slot of level e's interfaces
  int ldi = 0;                    // even-padded ni
  int ldb = 0;                    // even-padded nb
  // subtree partition: the level-lstar nodes (nparts = 2^lstar)
  // root independent subtrees; levels >= lstar and the leaves can be solved
  // per contiguous part range, levels < lstar ("top") need every part's flux
  int nparts = 1, lstar = 0;
};

// Streaming layout of one operator family of a level ("panel"): the level's
// c matrices (R x C each) are stacked into a row space of c*R rows (node-major),
// cut into tiles of TR consecutive rows, and every tile is stored column-major
// ([C][TR], rows zero-padded).  A CTA streams one tile (or a column chunk of
// it) as one contiguous run; each thread owns two adjacent rows (16-byte
// loads), so no cross-lane reduction is needed and every output is a
// sequential sum (bitwise reproducible).
constexpr int kPanelRows = 512;

struct Panel {
  double* base = nullptr;
  int c = 0, R = 0, C = 0;
  int TR = kPanelRows;  // logical rows per tile
  int TS = kPanelRows;  // stored rows per tile (even; > TR only for node-aligned tiles)
  int ntiles = 0;
  int parts = 1;        // > 1: c is the node count of one part; `parts` such panels back to back
  size_t doubles() const { return (size_t)ntiles * C * TS; }    // one part
  size_t total() const { return doubles() * parts; }
  Panel part(int g) const {
    Panel q = *this;
    q.base = base ? base + (size_t)g * doubles() : nullptr;
    q.parts = 1;
    return q;
  }
};
// wide levels: power-of-two tiles (TS = TR); parts > 1 tiles each of `parts`
// equal node ranges separately (no tile straddles a part boundary)
Panel make_panel(int c, int R, int C, int parts = 1);
// fused (subtree) levels: one tile = the npn nodes of one subtree, so one
// CTA finds all of its operator rows for a level in one contiguous tile
Panel make_panel_nodes(int c, int R, int C, int npn);

// launch-time split of a panel for k right-hand sides (split-K over columns)
struct PanelSplit {
  int KM = 1, kgroups = 1;  // rhs per pass, passes
  int nsplit = 1, CK = 0;   // column chunks
  int nodes = 1;            // max nodes touched by one tile
  int XS = 1;               // staged x row stride (odd)
  size_t smem = 0;
  size_t part_doubles = 0;  // split-K partials
  int counters = 0;         // split-K semaphores
};
PanelSplit panel_split(const Panel& pn, int k, int vnodes = 1);

struct LevelOps {
  // up-pass operator of a node: [X33^-1; Tstack X33^-1], (n3 + n12) x n3
  // (root: X33^-1 only).  Both halves act on the same r3, so w3 and the
  // node's outgoing flux h = [ha; hb] + (Tstack X33^-1) r3 come out of one pass.
  Panel Up;
  Panel S;                 // n3 x n12
  // shared layout (constant coefficients): the level's single operator pair,
  // row-major (GEMM operands, levels with >= kSharedGemmNodes nodes) or as
  // one-node panels (streaming kernel over virtual node tiles, other levels)
  double* Ush = nullptr;   // (n3 + n12) x ld3
  double* Ssh = nullptr;   // n3 x ld12
  double* T = nullptr;     // c x n12 x n12 row-major (only when keep_dtn)
  // fused subtree levels, shared layout: fragment-ordered Up / S for the
  // tensor-core subtree kernels (subtree.cu, sub_mma_prepare), or null
  const double* UpF = nullptr;
  const double* SF = nullptr;
};

// Level pair (d, d + 1) of the dataflow kernel's down sweep (mega.cu): level
// d + 1's interface values straight from level d's boundary values,
//   [u3_a; u3_b] = C1 u_bnd(p) + (PU w3(p) + [w3_a; w3_b]),
// so the two levels are one dependent phase instead of two.
struct MegaPair {
  int d = -1;              // parent level
  Panel C1;                // (2 n3_{d+1}) x n12_d: [S_c[:, A] E + S_c[:, B] S_p] for the alpha, beta child
  Panel PU;                // (2 n3_{d+1}) x n3_d:  [S_c[:, i3a]; S_c[:, i3b]]
  int* iota = nullptr;     // device c_d x n3_d: w3(p) positions relative to W3[d]
  int* out = nullptr;      // device c_d x 2 n3_{d+1}: positions of the adjusted w3 rows relative to W3[d]
  long long off = 0;       // W3c[d + 1] - W3[d] in doubles (workspace carve, k = 1) the tables were built for
};

struct Ops {
  Plan* plan = nullptr;
  double sigma = 0.0, dtg = 0.0;
  int shared_leaf = 1;         // constant coefficients: one leaf operator set
  int shared_levels = 0;       // HPS_LAYOUT_SHARED: one operator per level
  int Lc = 1;                  // number of stored leaf operator sets (1 or L)
  double* Ainv = nullptr;      // shared leaf: [Ainv; D_bi Ainv], (ni+nb) x ldi row-major (GEMM operand)
  double* S_leaf = nullptr;    // shared leaf: ni x ldb row-major
  Panel pAinv, pSleaf;         // per-leaf operators (variable coefficients)
  double* fd = nullptr;        // tensor-product leaf solve data (leaf_fd.cu), or null
  double* T_leaf = nullptr;    // Lc x nb x nb (kept only when keep_dtn)
  double* D_bi = nullptr;      // nb x ni (shared stencil rows)
  std::vector<LevelOps> lo;    // depth entries, root first
  double* root_T = nullptr;    // n12 x n12 of the root (keep_dtn)
  double* root_Tst = nullptr;  // root Tstack, n12 x ld3 row-major (test hooks only)
  size_t bytes = 0;            // device bytes owned
  std::vector<void*> allocs;
  std::vector<size_t> alloc_bytes;
  std::vector<void*> aux;      // derived device data rebuilt after build / load (not dumped)
  std::vector<MegaPair> pairs; // level pairs of the dataflow kernel's down sweep (derived, shared layout)
};
int sub_mma_prepare(Ops& O, cudaStream_t st);
int mega_pairs_prepare(Ops& O, cudaStream_t st);

int pack_panel(const double* src, long long s_node, int ld, const Panel& pn, cudaStream_t st);
// rows [0, R1) of each node from src1, rows [R1, R) from src2
int pack_panel2(const double* src1, long long s1, int ld1, int R1, const double* src2, long long s2, int ld2,
                const Panel& pn, cudaStream_t st);
int unpack_panel(const Panel& pn, int node, int row0, int nrows, double* dst, cudaStream_t st);  // nrows x C

// per-solve workspace carve-up (per-rhs strides in doubles)
struct Workspace {
  double* W = nullptr;      // k x L x (ni+nb): [w | h] rows (shared leaf) or w (ld ni)
  double* Hleaf = nullptr;  // k x L x nb
  double* Ub = nullptr;     // k x L x nb
  std::vector<double*> H;   // per level d (d>=1): k x c x n12
  std::vector<double*> W3;  // per level: k x c x n3
  std::vector<double*> W3c; // k = 1, per level d >= 1: c x n3, w3 adjusted by the parent's (level pairs, mega.cu)
  double* part = nullptr;   // split-K partials
  unsigned* cnt = nullptr;  // split-K semaphores (zero between launches)
  unsigned* mega_cnt = nullptr;  // persistent level kernel: completion counters (zero between launches)
  double* mega_part = nullptr;   // ... and its split partials
  double* xg = nullptr;          // shared-layout GEMMs: the gathered (node, rhs) x K inputs (GsSplit)
};
size_t workspace_bytes(const Plan& P, int k);
void carve_workspace(const Plan& P, int k, void* base, Workspace& ws);

// level GEMV launcher (see level_gemv.cu)
enum GemvMode { GEMV_UP = 0, GEMV_DOWN = 2, GEMV_LEAF = 3 };
constexpr int kSharedGemmNodes = 1024;  // shared layout: levels with at least this many (node, rhs) rows use the GEMM
constexpr int kSharedGemmRhs = 16;      // ... and multi-rhs solves from this many rhs on (fused subtree kernels off)

struct GemvArgs {
  int mode;
  int k;                        // right-hand sides
  // UPX / UPT
  const double* Hc; int nbc; long long Hc_k, Hc_s;  // child fluxes: per-child stride Hc_s
  double* Hout; int n12; long long Hout_k;
  double* W3; int n3; long long W3_k;
  const int *i1a, *i3a, *i2b, *i3b; int n1a;
  const double* jump; long long jump_k; double inv_dt; const int* j3;
  // DOWN
  double* u; long long u_k; const int* gidx;
  // LEAF: y[b] = M[b] x[b] (+ add[b])
  const double* xin; long long xin_k, xin_s;
  double* yout; long long yout_k, yout_s;
  const double* yadd; long long yadd_k, yadd_s;
  // split-K scratch
  double* part; unsigned* cnt;
  // shared layout: the one-node panel is applied to `shared` nodes (virtual
  // tiles = node x tile); 0 = per-node panels
  int shared;
  // row-sharded launches (top levels over several GPUs): the panel passed is a
  // view starting at tile t0 of the level's panel; prow0 = t0 * TR is its
  // first row in the level's row space.  DOWN with yout set: u3 goes to
  // yout[kg * yout_k + node * n3 + r] (a staging vector) instead of u[j3].
  long long prow0;
};
int gemv_level(const GemvArgs& a, const Panel& pn, cudaStream_t st);
// nodes [n0, n1) of a level: per-part panels are launched part by part (the
// range must be part-aligned), one-node (shared) panels over the node range
int gemv_nodes(const GemvArgs& a, const Panel& pn, int n0, int n1, cudaStream_t st);
GemvArgs shift_nodes(GemvArgs a, long long n0);

// fused subtree kernels (subtree.cu) for the narrow levels dF..depth-1
int fuse_level(const Plan& P);
// level-dF subtrees [b0, b1)
int subtree_up(const Ops& ops, const Workspace& ws, int k, const double* Hleaf, long long sh, long long hs,
               const double* jump, long long ld_jump, double inv_dt, int b0, int b1, cudaStream_t st);
int subtree_down(const Ops& ops, const Workspace& ws, int k, bool has_w3, double* u, long long ld_u, int b0,
                 int b1, cudaStream_t st);

// shared-layout level applies (dedup.cu)
// nodes [n0, n1) of level d
int shared_level_up(const Ops& ops, const Workspace& ws, int d, int k, const double* Hc, long long Hc_k,
                    long long Hc_s, const double* jump, long long ld_jump, double inv_dt, int n0, int n1,
                    cudaStream_t st);
int shared_level_down(const Ops& ops, const Workspace& ws, int d, int k, bool has_w3, double* u, long long ld_u,
                      int n0, int n1, cudaStream_t st);
bool shared_gemm(const Plan& P, int d, int nodes, int k);
// many-rhs deep levels (deep.cu): staged contiguous inputs, DMMA product; 1 = not eligible
bool deep_enabled();
int deep_level(const GemvArgs& g, bool up, int nodes, int k, int R, int K, const double* op, int ldo,
               cudaStream_t st);
struct GsSplit {
  int WN = 1, tiles = 0, nsplit = 1, KC = 0;
  size_t part_doubles = 0;
  int counters = 0;
  size_t gather_doubles = 0;  // > 0: the (node, rhs) x K input matrix is gathered once up front
};
GsSplit gs_split(long long M, int N, int K);  // (node, rhs) rows x operator rows x operator columns

// tensor-product leaf solve (leaf_fd.cu): [w | h] rows from the body load
// nleaf leaves: g and WH point at the first one
int leaf_fd(const Ops& ops, int k, int nleaf, const double* g, long long ld_g, double* WH, long long ld_wh,
            cudaStream_t st);
bool leaf_fd_supported(int q);
// tensor-product leaf solve split over the two sweeps: the up sweep writes only
// the fluxes h, the down sweep solves u_int = A_ii^-1 (r - A_ib u_b) directly
bool leaf_fd_down_enabled();
// (nbd > 0: also the Dirichlet data u[bids[i]] = fb[i], see FdArgs)
int leaf_fd_up_h(const Ops& ops, int k, int nleaf, const double* g, long long ld_g, double* H, long long ld_h,
                 cudaStream_t st, int nbd = 0, const int* bids = nullptr, const double* fb = nullptr,
                 long long ld_f = 0, double* u = nullptr, long long ld_u = 0);
int leaf_fd_down(const Ops& ops, int k, int nleaf, const double* g, long long ld_g, const int* lbg, const double* u,
                 long long ld_u, double* uint, long long ld_uint, double* lu, long long ld_lu, double* guard,
                 cudaStream_t st);
// L u at the interiors of nleaf leaves of a given state (the leaf grid's two
// DMMA products of the fused stage, without the solve); lbg / uint / lu at the first leaf
int leaf_fd_lu(const Ops& ops, int k, int nleaf, const int* lbg, const double* u, long long ld_u, const double* uint,
               double* lu, long long ld_lu, double* guard, cudaStream_t st);

// the up sweep's leaf kernel forming the body load sum_t tdc[t] tv[t] (leaf
// interiors; k rhs rows, term t's row stride tld[t], 0 = one row for every rhs)
// itself and writing it to rout (row stride ld_rout) for the downward sweep
int leaf_fd_up_terms(const Ops& ops, int k, int nleaf, int nterm, const double* const* tv, const long long* tld,
                     const double* tdc, double* rout, long long ld_rout, double* H, long long ld_h, cudaStream_t st,
                     int nbd, const int* bids, const double* fb, long long ld_f, double* u, long long ld_u);
struct StageTerms {
  int nterm = 0;
  const double* tv[12] = {};
  long long tld[12] = {};   // rhs row strides (0: one row shared by every rhs)
  const double* tdc = nullptr;
  double* rout = nullptr;
  long long ld_rout = 0;
};

// persistent dataflow kernel for the wide levels (mega.cu): up
// levels [u0, u1) deepest first, then down levels [d0, d1) root first, over
// the parts' nodes on levels >= lstar; returns 1 when not eligible
bool mega_enabled();
int mega_depth(const Ops& ops);  // levels [0, mega_depth) are eligible
void mega_scratch(const Plan& P, size_t& counters, size_t& part_doubles);
// root_pre: the root's Dirichlet product S u_bnd of this solve, precomputed
// (root_dirichlet); the launch then has no root down tasks
int mega_levels(const Ops& ops, const Workspace& ws, int u0, int u1, int d0, int d1, int part0, int part1,
                const double* Hleaf, long long hs, const double* jump, double inv_dt, bool has_w3, double* u,
                cudaStream_t st, const double* root_pre = nullptr);
// S_root u_bnd for ns (<= 8) rows of boundary data (fb order), streaming the
// root's down operator once for all of them (mega.cu); scratch >= root_dirichlet_scratch
size_t root_dirichlet_scratch(const Plan& P, int ns);
int root_dirichlet(const Ops& ops, int ns, const double* fb, long long ld_f, double* out, long long ld_out,
                   double* scratch, cudaStream_t st);

// solve entry (solve.cu).  phases: SOLVE_UP (leaves + levels >= lstar of parts
// [part0, part1)), SOLVE_TOP (Dirichlet data, levels < lstar up and down),
// SOLVE_DOWN (levels >= lstar + leaves of the parts); all three = the whole
// solve.  g is indexed from the first leaf of part0.
enum SolvePhase { SOLVE_UP = 1, SOLVE_TOP = 2, SOLVE_DOWN = 4, SOLVE_ALL = 7 };
int solve(const Ops& ops, int phases, int part0, int part1, int k, const double* fb, long long ld_f,
          const double* g, long long ld_g, const double* jump, long long ld_jump, double inv_dt, double* u,
          long long ld_u, void* ws, size_t ws_bytes, cudaStream_t st, double* lu = nullptr, long long ld_lu = 0,
          double* guard = nullptr, const double* root_pre = nullptr, const StageTerms* terms = nullptr);
// byte offset of level lstar's flux block (k x nparts x n12) in a workspace
size_t exchange_offset(const Plan& P, int k);
void level_offsets(const Plan& P, int k, int d, long long& w3, long long& h);
int top_level(const Ops& ops, int d, bool down, int rank, int nranks, int k, double* u, long long ld_u,
              double* stage, void* wsp, size_t ws_bytes, cudaStream_t st);

}  // namespace hpsb

// opaque handles of the C ABI (include/hpstep_b200.h)
struct hps_plan { hpsb::Plan P; std::vector<void*> allocs; };
struct hps_ops { hpsb::Ops O; };
