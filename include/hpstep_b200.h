/*
 * hpstep_b200.h -- C ABI of the B200 (sm_100a) HPS stage-solve library.
 *
 * Drop-in boundary for the per-ESDIRK-stage HPS solve of arXiv 2306.02526's
 * reference package `hpstep` (/root/reference/pkg/src/hpstep).  The reference
 * is pure Python, so its "plugin boundary" is the Python class API; each entry
 * point below replaces the reference code cited beside it, and the Python
 * package `paper_2306_02526_b200` binds them with ctypes exactly as a
 * maintainer would from `hpstep`.
 *
 * Conventions
 *   - plain C types only; every `const double* / double*` argument named
 *     "device" is a CUDA device pointer owned by the caller (e.g. a torch
 *     tensor); host descriptors are copied during the call.
 *   - `stream` is a cudaStream_t passed as void*; all device work is
 *     stream-ordered and never synchronises the host, except
 *     hps_ops_build (which must read pivots to report singular nodes).
 *   - return value 0 = success; < 0 = failure with a message available from
 *     hps_last_error() (thread-local).  HPS_ERR_SINGULAR additionally sets
 *     hps_last_error_node() to the DFS node index of the first singular
 *     block (reference: SingularMatrixError context "leaf node i" /
 *     "merge node i", linalg.py:36-42, solver.py:60,72).
 *   - operator sets are immutable after build; any number of concurrent
 *     solves may share one (solver.py:84-89) as long as each passes its own
 *     workspace.
 */
#ifndef HPSTEP_B200_H
#define HPSTEP_B200_H

#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

#define HPS_OK 0
#define HPS_ERR_ARG (-1)
#define HPS_ERR_CUDA (-2)
#define HPS_ERR_SINGULAR (-3)

typedef struct hps_plan hps_plan; /* tree shape + per-level index maps (device) */
typedef struct hps_ops hps_ops;   /* device operator set of one shift        */

/* Tree description (host arrays, copied).  Replaces the DomainTree numbering
 * consumed by the solver (tree.py:123-156, 216-280, 374-404).
 * Levels are the parent levels of the binary tree, root first.
 * lvl_shape[5*d + {0..4}] = {c, n3, n1a, n2b, nbc}: node count, |J3|, |J1|,
 * |J2| and the child boundary size.  The per-level child-local maps i1a,
 * i3a, i2b, i3b are shared by every node of a level; gidx_bnd (c x n12) and
 * j3 (c x n3) are the global DOF ids of each node's boundary / interface. */
typedef struct {
  int n1, n2, p;
  int depth;              /* number of parent levels = log2(n1*n2)          */
  long long N;            /* global DOFs                                     */
  int L, ni, nb, nbd;     /* leaves, interior / boundary DOFs per leaf, |boundary| */
  const int* lvl_shape;
  const int* const* lvl_i1a;
  const int* const* lvl_i3a;
  const int* const* lvl_i2b;
  const int* const* lvl_i3b;
  const int* const* lvl_gidx_bnd;
  const int* const* lvl_j3;
  const long long* const* lvl_node_index; /* DFS node index per level node  */
  const int* leaf_bnd_gidx;                /* L x nb                          */
  const long long* leaf_node_index;        /* L                               */
  const int* boundary_ids;                 /* nbd, ascending                  */
  int nparts;             /* subtree partition for multi-GPU solves (SURVEY.md
                             8(e)): 0 or 1 = none, else 2^lstar parts = the
                             subtrees of the lstar-th parent level, lstar < depth */
} hps_plan_desc;

/* Build inputs (host arrays, copied).  Replaces build_leaf / merge / _build
 * (solver.py:53-158) for the shifted operator sigma*I + dt_gamma*A. */
typedef struct {
  double sigma, dt_gamma;
  int shared_leaf;     /* 1: constant coefficients, one leaf operator set   */
  int keep_dtn;        /* keep every level's DtN map T (tests, save/load)    */
  const double* coef;  /* Lc x 5 x ni: c11,c22,c1,c2,c at interior points (Lc = 1 or L) */
  int has_c1, has_c2, has_c;
  const double* D2x;   /* ni x m interior stencil rows (operators.py:180-181) */
  const double* D2y;
  const double* D1x;
  const double* D1y;
  const double* D_bnd; /* nb x m flux rows (operators.py:188-190)            */
  int layout;          /* HPS_LAYOUT_PER_NODE: one operator copy per node,
                          streamed from HBM every solve (what the reference
                          stores, solver.py:137-151); HPS_LAYOUT_SHARED: one
                          copy per level, level applies run as tensor-core
                          GEMMs (constant coefficients only, where every node
                          of a level has bitwise the same operators)          */
} hps_build_desc;

#define HPS_LAYOUT_PER_NODE 0
#define HPS_LAYOUT_SHARED 1

int hps_version(void);
long long hps_launch_count(void); /* kernels launched by this library so far */
const char* hps_last_error(void);
long long hps_last_error_node(void);

int hps_plan_create(const hps_plan_desc* desc, hps_plan** out);
void hps_plan_destroy(hps_plan* plan);

/* HpsOperatorSet.__init__ / build() (solver.py:91-158, 380-390). */
int hps_ops_build(const hps_plan* plan, const hps_build_desc* desc, void* stream, hps_ops** out);
void hps_ops_destroy(hps_ops* ops);
size_t hps_ops_device_bytes(const hps_ops* ops);
/* Diagnostics: number of level pairs prepared for the down sweep of the
 * dataflow kernel (shared layout; 0 = none).  A pair (d, d + 1) computes level
 * d + 1's interface values of solver.py:262-265 straight from level d's
 * boundary values through a composite operator, in level d's phase. */
int hps_ops_level_pairs(const hps_ops* ops);

/* Enable the tensor-product leaf solve for a constant-coefficient operator
 * set (leaf_fd.cu): host = Vx^-1, Vy^-T, Vx, Vy^T, rden (q x q each, row-major;
 * rden[a][b] = 1 / (lx_a + ly_b + sigma + dtg c)), then the interior parts of the
 * flux rows d1x[0], d1x[p-1], d1y[0], d1y[p-1] (q each), then the couplings of
 * the interior points to the boundary, dtg(-c11 d2x + c1 d1x)[1..p-2][0],
 * ...[1..p-2][p-1], dtg(-c22 d2y + c2 d1y)[1..p-2][0], ...[1..p-2][p-1]
 * (q each), then Mx = c11 d2x - c1 d1x and My = c22 d2y - c2 d1y (p x p
 * zero-padded to 16 x 16, row-major) and c -- the interior L u of the stage
 * history is Mx G + G My^T - c G on the leaf grid G; count = 5q^2 + 8q + 513.
 * host = NULL disables it.  Replaces the dense A_ii^-1 apply of
 * solver.py:221-228 with the Kronecker-sum factorisation of A_ii. */
int hps_ops_set_leaf_fd(hps_ops* ops, const double* host, int count);

/* Measurement hooks (bench.py): per-kernel CUDA-event timing of this
 * library's launches on streams that are not being captured.  While enabled,
 * each launch is bracketed by two events (this serialises the programmatic-
 * dependent-launch overlap of neighbouring kernels).  hps_ktimer_collect
 * synchronises the device and returns the number of distinct kernels (<= max):
 * names ('\n'-separated, mangled), total milliseconds and launch counts,
 * then clears the records. */
void hps_ktimer_enable(int on);
int hps_ktimer_collect(char* names, int names_len, double* ms, long long* counts, int max);

/* merge(T_alpha, T_beta, node) (solver.py:67-81) on the device for one node:
 * Tc = [T_alpha; T_beta], two nbc x nbc row-major DtN maps (a smaller child's
 * map zero-padded), i1a/i3a/i2b/i3b the node's child-local index maps (device
 * int arrays).  Forms X33 = T_a33 - T_b33, inverts it by pivoted Gauss-Jordan
 * under the reference's singularity rule (linalg.py:17,36-42: min pivot <=
 * 1e-13 max pivot -> HPS_ERR_SINGULAR naming "merge node <node_index>"), and
 * writes Xinv (n3 x n3), S = X33^-1 [-T_a31 | T_b32] (n3 x n12), Tstack
 * (n12 x n3) and T = blkdiag(T_a11, T_b22) + Tstack S (n12 x n12), all
 * row-major device arrays.  Synchronises the stream (the pivot check). */
int hps_merge_node(int nbc, const double* Tc, int n1a, int n2b, int n3, const int* i1a, const int* i3a,
                   const int* i2b, const int* i3b, long long node_index, double* Xinv, double* S,
                   double* Tstack, double* T, void* stream);

/* Copy one operator block to host memory (test hooks leaf_operators /
 * merge_operators, solver.py:339-348).  which: leaf 0=Ainv (ni x ni),
 * 1=S (ni x nb), 2=T (nb x nb, keep_dtn only); merge 0=Xinv (n3 x n3),
 * 1=Tstack (n12 x n3, root only), 2=S (n3 x n12), 3=T (n12 x n12, keep_dtn
 * or root), 4=Tstack Xinv (n12 x n3, non-root: the flux rows of the stacked
 * up-pass operator; Tstack = (Tstack Xinv) Xinv^-1).
 * `level` is the parent level (root = 0), `node` the position on it. */
int hps_ops_get_leaf(const hps_ops* ops, int which, int leaf, double* host_out);
int hps_ops_get_merge(const hps_ops* ops, int level, int node, int which, double* host_out);

/* Operator-set persistence (HpsOperatorSet.save / .load, solver.py:294-337):
 * hps_ops_dump writes the operator set into a host buffer of
 * hps_ops_dump_size(ops) bytes; hps_ops_load rebuilds it on the device for a
 * plan of the same tree (no build). */
long long hps_ops_dump_size(const hps_ops* ops);
int hps_ops_dump(const hps_ops* ops, void* host, long long size);
int hps_ops_load(const hps_plan* plan, const void* host, long long size, hps_ops** out);

size_t hps_solve_workspace_bytes(const hps_plan* plan, int k);

/* HpsOperatorSet._solve (solver.py:201-276) for k stacked right-hand sides:
 *   fb   device k x nbd Dirichlet values (row stride ld_f; ld_f = 0 broadcasts)
 *   g    device body load, read at leaf interiors [0, L*ni) only, row stride
 *        ld_g; NULL = homogeneous solve (solve_homogeneous)
 *   jump device interface flux jumps (row stride ld_jump) or NULL; with
 *        inv_dt = 1/dt this is solve_penalized (solver.py:188-199, 249-250)
 *   u    device k x N output (row stride ld_u), every DOF written
 *   ws   device workspace of >= hps_solve_workspace_bytes(plan, k) bytes,
 *        256-byte aligned and zero-filled before its first use (its
 *        semaphores and completion counters return to zero after every solve) */
int hps_solve(const hps_ops* ops, int k, const double* fb, long long ld_f, const double* g,
              long long ld_g, const double* jump, long long ld_jump, double inv_dt, double* u,
              long long ld_u, void* ws, size_t ws_bytes, void* stream);

/* Fused ARK stage (timestep.py:259-261 after solver.py:201-276): hps_solve
 * of the stage body load, plus the next stage's history L u at the leaf
 * interiors (lu_int, k x L*ni rows of stride ld_lu, operators.py:276-301 at
 * interior points) and guard = max(guard, max |u|) over the leaves' grids
 * (timestep.py:198-203), computed by the leaf kernel of the downward sweep
 * while the leaf's grid is on chip.  Constant coefficients with the
 * tensor-product leaf solve only (HPS_ERR_ARG otherwise: use hps_solve +
 * hps_leaf_eval).  lu_int may be NULL (the last stage: solve + guard only).
 * root_pre (k = 1, may be NULL): this solve's root Dirichlet product from
 * hps_root_dirichlet. */
int hps_solve_stage(const hps_ops* ops, int k, const double* fb, long long ld_f, const double* g,
                    long long ld_g, double* u, long long ld_u, double* lu_int, long long ld_lu,
                    double* guard, const double* root_pre, void* ws, size_t ws_bytes, void* stream);

/* hps_solve_stage for one rhs (k = 1) with the stage body load given as its
 * combination (timestep.py:255-257): r = sum_t dcoefs[t] vecs[t] over the
 * leaf interiors [0, L*ni) (device coefficients, 1..12 terms, term order as
 * hps_combine), formed by the upward sweep's leaf kernel -- no separate
 * combination pass -- and written to r_out for the downward sweep.  lu_int
 * and guard as hps_solve_stage (row strides N); root_pre as hps_solve_stage. */
int hps_solve_stage_terms(const hps_ops* ops, const double* fb, int nterms, const double* dcoefs,
                          const double* const* vecs, double* r_out, double* u, double* lu_int,
                          double* guard, const double* root_pre, void* ws, size_t ws_bytes,
                          void* stream);

/* hps_solve_stage_terms for k rhs rows (an ensemble stage, timestep.py:255-257
 * over the stacked members): term t has row stride vec_ld[t] (0 = one row
 * shared by every rhs), r_out / u / lu_int rows of stride ld_r / ld_u / ld_lu,
 * fb rows of stride ld_f; no root_pre. */
int hps_solve_stage_terms_k(const hps_ops* ops, int k, const double* fb, long long ld_f, int nterms,
                            const double* dcoefs, const double* const* vecs, const long long* vec_ld,
                            double* r_out, long long ld_r, double* u, long long ld_u, double* lu_int,
                            long long ld_lu, double* guard, void* ws, size_t ws_bytes, void* stream);

/* The root's Dirichlet product S_root u_bnd (solver.py:262-265 at the root,
 * whose boundary is the domain boundary) for ns <= 8 rows of boundary data
 * fb (nbd values each, row stride ld_f) in one pass over the root operator:
 * out[s * ld_out + r], r < n3 of the root.  A step computes it once for all of
 * its stage times and passes row s to hps_solve_stage as root_pre (k = 1), so
 * the per-stage solves skip the root's down product.  scratch holds
 * hps_root_dirichlet_scratch(ops, ns) bytes. */
size_t hps_root_dirichlet_scratch(const hps_ops* ops, int ns);
int hps_root_dirichlet(const hps_ops* ops, int ns, const double* fb, long long ld_f, double* out,
                       long long ld_out, void* scratch, size_t scratch_bytes, void* stream);

/* Stage history of an explicit stage (timestep.py:259-261, the first ARK
 * stage's L u_n): lu_int = L u at the interiors of leaves [leaf0, leaf0 +
 * nleaf) (operators.py:276-301 at interior points; rows start at leaf0's
 * interior) and guard = max(guard, max |u|) over those leaves' grids
 * (guard may be NULL).  The same leaf-grid products as hps_solve_stage,
 * without the solve.  Constant coefficients with the tensor-product leaf
 * solve only (HPS_ERR_ARG otherwise: use hps_leaf_eval_range). */
int hps_leaf_lu(const hps_ops* ops, int leaf0, int nleaf, int k, const double* u, long long ld_u,
                double* lu_int, long long ld_lu, double* guard, void* stream);

/* Subtree-sharded solve (the reference solves the whole tree
 * in one call, solver.py:201-276).  With a plan created with nparts = 2^lstar,
 * part r is the subtree of node r on parent level lstar.  Phases:
 *   HPS_PHASE_UP    leaves + levels >= lstar of parts [part0, part1): leaf
 *                   solves and upward merges; leaves the parts' level-lstar
 *                   fluxes in the workspace's exchange block;
 *   HPS_PHASE_TOP   Dirichlet data, then the levels < lstar up and down (needs
 *                   every part's flux in the exchange block: all-gather it
 *                   between the phases when the parts live on other GPUs);
 *   HPS_PHASE_DOWN  levels >= lstar + leaf reconstruction of the parts.
 * g is indexed from the first leaf of part0 (row stride ld_g) and only read
 * by the UP phase; pass the same g / jump to every phase (its nullness selects
 * the data flow).  u rows are global (N DOFs); a phase writes only the DOFs it
 * owns: TOP the boundary and the interfaces of levels < lstar, DOWN the
 * interfaces and leaf interiors inside its parts.  HPS_PHASE_ALL over all
 * parts is hps_solve. */
#define HPS_PHASE_UP 1
#define HPS_PHASE_TOP 2
#define HPS_PHASE_DOWN 4
#define HPS_PHASE_ALL 7
int hps_solve_phase(const hps_ops* ops, int phases, int part0, int part1, int k, const double* fb,
                    long long ld_f, const double* g, long long ld_g, const double* jump,
                    long long ld_jump, double inv_dt, double* u, long long ld_u, void* ws,
                    size_t ws_bytes, void* stream);

/* Partition of a plan: nparts, lstar, the level-lstar flux length n12 and the
 * byte offset in a k-rhs workspace of the exchange block (k x nparts x n12
 * doubles, part r's fluxes at [r*n12, (r+1)*n12) of each rhs row; -1 when
 * nparts = 1). */
int hps_plan_partition(const hps_plan* plan, int k, int* nparts, int* lstar, int* n12,
                       long long* flux_offset);

/* The first parent level the fused subtree kernels run (levels >= it);
 * levels above run in the wide-level dataflow kernel / per-level launches.
 * Measurement only (bench.py's per-kernel algorithmic bytes). */
int hps_plan_fused_level(const hps_plan* plan);

/* Row-sharded top levels of a subtree-sharded solve (the
 * levels < lstar, which every rank would otherwise run whole).  Between the
 * UP phase (+ the level-lstar flux all-gather) and the DOWN phase, each rank
 * runs, for level = lstar-1 .. 0, hps_top_level(level, down = 0): its share
 * rank/nranks of the level's up operator tiles for every node, writing w3 and
 * flux rows into the workspace's level blocks (zeroed first, so a sum over
 * the ranks completes them -- hps_workspace_level gives their byte offsets),
 * then for level = 0 .. lstar-1 hps_top_level(level, down = 1): its share of
 * the S tiles, u3 = S u_bnd + w3 rows into `stage` (k x c x n3, zeroed
 * first), to be summed over the ranks and scattered to u[j3] of the level.
 * u must hold the Dirichlet data (hps_put_boundary) and every interface value
 * of the levels above.  Replaces HPS_PHASE_TOP (solver.py:243-268 for the top
 * levels) with 1/nranks of its operator traffic per rank. */
int hps_workspace_level(const hps_plan* plan, int k, int level, long long* w3_off, long long* h_off);
int hps_top_level(const hps_ops* ops, int level, int down, int rank, int nranks, int k, double* u, long long ld_u,
                  double* stage, void* ws, size_t ws_bytes, void* stream);

/* ------------------------------------------------------------------------
 * Stage right-hand-side assembly (timestep.py:237-266 and the leaf-local
 * evaluations of operators.py:276-346).
 * ------------------------------------------------------------------------ */
typedef struct hps_disc hps_disc; /* device leaf stencil + coefficient samples */

/* EllipticDiscretization (operators.py:219-236) as seen by the evaluations:
 * 1D CGL derivative matrices of the leaf grid (p x p, descending nodes) and
 * the edge-local ones on the p-2 interior nodes (operators.py:192-213),
 * coefficient samples at the m = ni + nb leaf-local points, the reference's
 * leaf_bnd_sign (tree.py:382-403) as int8. */
typedef struct {
  const double *d1x, *d2x, *d1y, *d2y; /* p x p  */
  const double *ex1, *ex2, *ey1, *ey2; /* (p-2) x (p-2) */
  int Lc;                              /* 1 (constant) or L sample sets        */
  const double* coef;                  /* Lc x 5 x m: c11, c22, c1, c2, c       */
  int has_c1, has_c2, has_c;
  const signed char* leaf_bnd_sign;    /* L x nb, 0 on the domain boundary     */
} hps_disc_desc;

int hps_disc_create(const hps_plan* plan, const hps_disc_desc* desc, hps_disc** out);
void hps_disc_destroy(hps_disc* disc);

/* One pass over the leaves of k stacked grid vectors u (row stride ld_u).
 * Each non-NULL output (row stride ld_o) receives:
 *   lu_int  L u at leaf-interior DOFs [0, L*ni) only (stage history)
 *   lu      apply_lop (operators.py:276-301), interface-averaged, every DOF
 *   ux, uy  gradient (operators.py:303-317), interface-averaged
 *   jump    flux_jump (operators.py:319-336), zero off the interfaces
 * guard (device double, may be NULL) is raised to max |u| over every DOF
 * (NaN sticks), the divergence guard of timestep.py:198-203. */
int hps_leaf_eval(const hps_disc* disc, int k, const double* u, long long ld_u, double* lu_int,
                  double* lu, double* ux, double* uy, double* jump, long long ld_o, double* guard,
                  void* stream);

/* hps_leaf_eval over leaves [leaf0, leaf0 + nleaf) (a subtree part): lu_int
 * rows are indexed from leaf0's first interior DOF, the other outputs are
 * global N-DOF rows.  Edge DOFs receive only these leaves' contributions
 * (the interface mean adds 1/2 of each abutting leaf), so an edge shared with
 * leaves outside the range holds a partial sum the caller completes (e.g. an
 * all-reduce over the GPUs of a sharded run). */
int hps_leaf_eval_range(const hps_disc* disc, int leaf0, int nleaf, int k, const double* u,
                        long long ld_u, double* lu_int, double* lu, double* ux, double* uy,
                        double* jump, long long ld_o, double* guard, void* stream);

/* out[r][0:n) = sum_t coefs[t] * vecs[t][r*lds[t] + (0:n)] for r < k
 * (lds[t] = 0 broadcasts one vector over the rows); at most 24 terms.
 * The ARK stage combinations of timestep.py:255-257 and 263-264. */
int hps_combine(int k, long long n, int nterms, const double* coefs, const double* const* vecs,
                const long long* lds, double* out, long long ld_out, double* guard, void* stream);

/* As hps_combine with the coefficients read from device memory at run time
 * (dcoefs[t]), so a captured CUDA graph replays with per-step coefficients. */
int hps_combine_dev(int k, long long n, int nterms, const double* dcoefs, const double* const* vecs,
                    const long long* lds, double* out, long long ld_out, double* guard, void* stream);

/* As hps_combine_dev with per-row coefficients: row r of out takes
 * dcoefs[r * ld_c + t] (the boundary data f(t_i) of every stage time of a
 * step, timestep.py:245,265, in one launch). */
int hps_combine_dev_rows(int k, long long n, int nterms, const double* dcoefs, long long ld_c,
                         const double* const* vecs, const long long* lds, double* out, long long ld_out,
                         double* guard, void* stream);

/* guard = max(guard, max |x|) over k rows of n values. */
int hps_maxabs(int k, long long n, const double* x, long long ld, double* guard, void* stream);

/* The step's final combination with the Dirichlet data and the guard in one
 * pass (timestep.py:263-266): out[k][e] = sum_t c_t vecs[t][k][e] over all N
 * DOFs, then fb at the domain-boundary DOFs, guard = max(guard, max |out|).
 * Coefficients from the host (coefs) or device memory (dcoefs, graph replay). */
int hps_combine_bnd(const hps_plan* plan, int k, int nterms, const double* coefs, const double* dcoefs,
                    const double* const* vecs, const long long* lds, const double* fb, long long ld_f,
                    double* out, long long ld_out, double* guard, void* stream);

/* u[r][boundary_ids] = fb[r] (timestep.py:265). */
int hps_put_boundary(const hps_plan* plan, int k, const double* fb, long long ld_f, double* u,
                     long long ld_u, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* HPSTEP_B200_H */
