"""Drop-in ``HpsOperatorSet`` / ``build`` backed by the sm_100a library.

Mirrors the reference API (solver.py:84-390 of hpstep): same constructor,
``solve_with_body_load`` / ``solve_homogeneous`` / ``solve_penalized``, the
``sigma`` / ``dt_gamma`` / ``shift`` properties, the squeeze rule, the
boundary-shape ``ValueError``, ``InvalidStepError`` for dt <= 0 and
``SingularMatrixError`` naming the node.  The build and every solve run on
the GPU (no CPU fallback): numpy inputs are copied to the device and the
result copied back; torch CUDA tensors stay on the device.
"""

import contextlib
import ctypes
import hashlib
import json
import os
import threading

import numpy as np

from . import _lib
from .device import cuda_device, current_stream_handle, ndim, torch
from .errors import HpstepError, InvalidStepError
from .operators import EllipticDiscretization

FORMAT_VERSION = 1

# Solve workspaces (level fluxes, w3, split partials, dataflow counters) are
# per plan and per stream, so solves on different streams never share one
# (solver.py:84-89: solves are re-entrant and concurrent-safe).  A captured
# CUDA graph owns its own workspace instead: it replays on whatever stream
# the caller uses, so its key is the capturing owner's token
# (graph_workspace), set for the warm pass that precedes the capture (which
# allocates it outside the capture) and for the capture itself.
_tls = threading.local()


@contextlib.contextmanager
def graph_workspace(token):
    prev = getattr(_tls, "graph", None)
    _tls.graph = ("graph", token)
    try:
        yield
    finally:
        _tls.graph = prev


def _workspace_key(k):
    tok = getattr(_tls, "graph", None)
    if tok is not None:
        return (k, tok)
    if torch.cuda.is_current_stream_capturing():
        return (k, ("graph", None))
    return (k, torch.cuda.current_stream().cuda_stream)


class DevicePlan:
    """Device copy of the tree numbering (one per tree, partition and device).

    ``nparts`` > 1 cuts the tree into the 2^lstar subtrees of parent level
    lstar so a solve can run part by part (multi-GPU)."""

    def __init__(self, tree, nparts=1):
        lib = _lib.load()
        cuda_device()  # raises without a GPU
        self.tree = tree
        lms = tree.level_maps
        keep = []

        def arr(a, dt=np.int32):
            a = np.ascontiguousarray(a, dtype=dt)
            keep.append(a)
            return a

        shape = arr([v for lm in lms for v in (lm.count, lm.n3, lm.n1a, lm.n2b, lm.nbc)] or [0])
        IP = _lib.c_int_p * max(1, len(lms))
        LP = _lib.c_ll_p * max(1, len(lms))

        def ptrs(key, dt=np.int32, T=IP, conv=_lib.int_ptr):
            return T(*[conv(arr(getattr(lm, key), dt)) for lm in lms])

        d = _lib.PlanDesc()
        d.n1, d.n2, d.p, d.depth = tree.n1, tree.n2, tree.p, tree.depth
        d.N, d.L, d.ni, d.nb = tree.N, tree.L, tree.ni, tree.nb
        d.nbd = tree.boundary_ids.size
        d.lvl_shape = _lib.int_ptr(shape)
        d.lvl_i1a, d.lvl_i3a = ptrs("i1a"), ptrs("i3a")
        d.lvl_i2b, d.lvl_i3b = ptrs("i2b"), ptrs("i3b")
        d.lvl_gidx_bnd, d.lvl_j3 = ptrs("gidx_bnd"), ptrs("j3")
        d.lvl_node_index = ptrs("node_index", np.int64, LP, _lib.ll_ptr)
        d.leaf_bnd_gidx = _lib.int_ptr(arr(tree.leaf_bnd_gidx))
        d.leaf_node_index = _lib.ll_ptr(arr(tree.leaves, np.int64))
        d.boundary_ids = _lib.int_ptr(arr(tree.boundary_ids))
        d.nparts = int(nparts)
        h = ctypes.c_void_p()
        _lib.check(lib.hps_plan_create(ctypes.byref(d), ctypes.byref(h)), "hps_plan_create")
        self.handle = h
        self._lib = lib
        self._ws = {}
        npt, ls, n12 = ctypes.c_int(), ctypes.c_int(), ctypes.c_int()
        _lib.check(lib.hps_plan_partition(h, 1, ctypes.byref(npt), ctypes.byref(ls), ctypes.byref(n12), None),
                   "hps_plan_partition")
        self.nparts, self.lstar, self.flux_n12 = npt.value, ls.value, n12.value
        dev = cuda_device()
        self.boundary_ids = torch.as_tensor(tree.boundary_ids, device=dev)

    def workspace(self, k):
        """The solve workspace of ``k`` right-hand sides for the current
        stream (or the graph being captured / warmed, see graph_workspace)."""
        key = _workspace_key(k)
        ws = self._ws.get(key)
        if ws is None:
            nbytes = self._lib.hps_solve_workspace_bytes(self.handle, k)
            ws = torch.zeros(nbytes, dtype=torch.uint8, device=cuda_device())  # split-K semaphores start at 0
            self._ws[key] = ws
        return ws

    def level_blocks(self, k, level):
        """(k, c * n3) view of level ``level``'s w3 block and (k, c * n12) view
        of its flux block (None for the root) in the current workspace."""
        w3, h = ctypes.c_longlong(), ctypes.c_longlong()
        _lib.check(self._lib.hps_workspace_level(self.handle, k, int(level), ctypes.byref(w3), ctypes.byref(h)),
                   "hps_workspace_level")
        lm = self.tree.level_maps[level]
        ws = self.workspace(k)

        def view(off, n):
            return ws[off:off + 8 * k * n].view(torch.float64).view(k, n)
        return view(w3.value, lm.count * lm.n3), (None if h.value < 0 else view(h.value, lm.count * lm.n12))

    def flux_block(self, k):
        """(k, nparts, n12) view of the workspace's level-lstar flux block
        (what the UP phase leaves for the TOP phase; all-gathered between
        GPUs in a sharded solve)."""
        off = ctypes.c_longlong()
        _lib.check(self._lib.hps_plan_partition(self.handle, k, None, None, None, ctypes.byref(off)),
                   "hps_plan_partition")
        if off.value < 0:
            raise HpstepError("plan has no subtree partition")
        ws = self.workspace(k)
        n = k * self.nparts * self.flux_n12
        return ws[off.value:off.value + 8 * n].view(torch.float64).view(k, self.nparts, self.flux_n12)

    def __del__(self):
        try:
            if self.handle:
                self._lib.hps_plan_destroy(self.handle)
        except Exception:
            pass


def device_plan(tree, nparts=1):
    cache = getattr(tree, "_device_plans", None)
    if cache is None:
        cache = tree._device_plans = {}
    p = cache.get(int(nparts))
    if p is None:
        p = cache[int(nparts)] = DevicePlan(tree, nparts)
    return p


class _InverseFactor:
    """Stand-in for ``DenseFactorization`` over a downloaded explicit inverse."""

    def __init__(self, inv):
        self.inv = inv
        self.n = inv.shape[0]

    def solve(self, B):
        return self.inv @ np.asarray(B, dtype=float)


class LeafOperators:
    def __init__(self, S, T, Aii_factor, D_edge):
        self.S, self.T, self.Aii_factor, self.D_edge = S, T, Aii_factor, D_edge


class MergeOperators:
    def __init__(self, S, X33_factor, Tstack, T=None):
        self.S, self.X33_factor, self.Tstack, self.T = S, X33_factor, Tstack, T


def build_leaf(disc, leaf_id, sigma=0.0, dt_gamma=1.0):
    """One leaf's operators S = -A_ii^-1 A_ib, T = D_bi S + D_bb (reference
    solver.py:53-64), from a device build of the operator set (the leaf build
    is batched over every leaf); SingularMatrixError names "leaf node {i}"."""
    ops = build(disc.tree, disc.coeffs, sigma=sigma, dt_gamma=dt_gamma, disc=disc, keep_dtn=True)
    return ops.leaf_operators(leaf_id)


def merge(T_alpha, T_beta, node):
    """Merge two children's DtN maps across their interface (reference
    solver.py:67-81) on the device (``hps_merge_node``): the same X33 / S /
    Tstack / T and the same singularity rule, raising SingularMatrixError
    naming "merge node {node.index}"."""
    lib = _lib.load()
    dev = cuda_device()
    Ta = np.asarray(T_alpha, dtype=float)
    Tb = np.asarray(T_beta, dtype=float)
    nbc = max(Ta.shape[0], Tb.shape[0])
    Tc = np.zeros((2, nbc, nbc))
    Tc[0, :Ta.shape[0], :Ta.shape[1]] = Ta
    Tc[1, :Tb.shape[0], :Tb.shape[1]] = Tb
    maps = [torch.as_tensor(np.ascontiguousarray(getattr(node, k), dtype=np.int32), device=dev)
            for k in ("i1a", "i3a", "i2b", "i3b")]
    n1a, n3, n2b = maps[0].numel(), maps[1].numel(), maps[2].numel()
    n12 = n1a + n2b
    dTc = torch.as_tensor(Tc, device=dev)
    Xinv = torch.empty((n3, n3), dtype=torch.float64, device=dev)
    S = torch.empty((n3, n12), dtype=torch.float64, device=dev)
    Tst = torch.empty((n12, n3), dtype=torch.float64, device=dev)
    T = torch.empty((n12, n12), dtype=torch.float64, device=dev)
    rc = lib.hps_merge_node(nbc, dTc.data_ptr(), n1a, n2b, n3, *[m.data_ptr() for m in maps],
                            int(node.index), Xinv.data_ptr(), S.data_ptr(), Tst.data_ptr(), T.data_ptr(),
                            current_stream_handle())
    _lib.check(rc, "hps_merge_node")
    return MergeOperators(S=S.cpu().numpy(), X33_factor=_InverseFactor(Xinv.cpu().numpy()),
                          Tstack=Tst.cpu().numpy(), T=T.cpu().numpy())


class HpsOperatorSet:
    """Per-node HPS operators of ``sigma*I + dt_gamma*A``, resident on the GPU.

    Read-only after construction; concurrent solves on different streams are
    safe (each stream gets its own workspace, ``DevicePlan.workspace``).
    """

    def __init__(self, disc, sigma, dt_gamma, keep_dtn=False, threads=None, layout=None, nparts=1):
        self.disc = disc
        self.tree = disc.tree
        self.sigma = float(sigma)
        self.dt_gamma = float(dt_gamma)
        self.keep_dtn = bool(keep_dtn)
        self.layout = resolve_layout(layout, disc.coeffs)
        st = disc.stencil
        self.D_bi = st.D_bnd[:, :st.ni]
        self.plan = device_plan(self.tree, nparts)
        self._build()

    @property
    def shift(self):
        return self.dt_gamma

    def _build(self):
        disc, st = self.disc, self.disc.stencil
        lib = self.plan._lib
        ni = st.ni
        samp = disc.coefficient_samples()[:, :, :ni]          # interior points only
        cf = disc.coeffs
        keep = [np.ascontiguousarray(samp, dtype=float)]
        rows = [np.ascontiguousarray(M[:ni], dtype=float) for M in (st.D2x, st.D2y, st.D1x, st.D1y)]
        dbnd = np.ascontiguousarray(st.D_bnd, dtype=float)
        keep += rows + [dbnd]
        d = _lib.BuildDesc()
        d.sigma, d.dt_gamma = self.sigma, self.dt_gamma
        d.shared_leaf = 1 if cf.is_constant else 0
        d.keep_dtn = 1 if self.keep_dtn else 0
        d.coef = _lib.dbl_ptr(keep[0])
        d.has_c1 = int(cf.c1 is not None)
        d.has_c2 = int(cf.c2 is not None)
        d.has_c = int(cf.c is not None)
        d.D2x, d.D2y, d.D1x, d.D1y = (_lib.dbl_ptr(r) for r in rows)
        d.D_bnd = _lib.dbl_ptr(dbnd)
        d.layout = _lib.LAYOUT_SHARED if self.layout == "shared" else _lib.LAYOUT_PER_NODE
        h = ctypes.c_void_p()
        rc = lib.hps_ops_build(self.plan.handle, ctypes.byref(d), current_stream_handle(),
                               ctypes.byref(h))
        _lib.check(rc, "hps_ops_build")
        self.handle = h
        self._lib = lib
        self.parent_order = [int(i) for lm in self.tree.level_maps for i in lm.node_index]
        self.leaf_solve = "dense"  # "tensor": Kronecker-sum leaf solve (csrc/leaf_fd.cu)
        fd = tensor_leaf_factors(disc, self.sigma, self.dt_gamma)
        if fd is not None and os.environ.get("HPSB_NO_FD") != "1":
            fd = np.ascontiguousarray(fd, dtype=float)
            _lib.check(lib.hps_ops_set_leaf_fd(h, _lib.dbl_ptr(fd), fd.size), "hps_ops_set_leaf_fd")
            self.leaf_solve = "tensor"

    def __del__(self):
        try:
            if getattr(self, "handle", None):
                self._lib.hps_ops_destroy(self.handle)
                self.handle = None
        except Exception:
            pass

    @property
    def device_bytes(self):
        return int(self._lib.hps_ops_device_bytes(self.handle))

    # -- solves ------------------------------------------------------------------
    def solve_homogeneous(self, f):
        return self._solve(f, None, None, None)

    def solve_with_body_load(self, f, g):
        return self._solve(f, g, None, None)

    def solve_penalized(self, f, g, flux_jump, dt):
        if dt <= 0:
            raise InvalidStepError(f"time step must be positive, got {dt}")
        return self._solve(f, g, flux_jump, 1.0 / dt)

    def _boundary_values(self, f, dev):
        """(kf, nbd) device tensor from scalar / (nbd,) / (N,) / stacked data
        (reference solver.py:162-174)."""
        tree = self.tree
        nbd = tree.boundary_ids.size
        if torch.is_tensor(f):
            F = f.to(device=dev, dtype=torch.float64)
        else:
            F = np.asarray(f, dtype=float)
            if F.ndim == 0:
                return torch.full((1, nbd), float(F), dtype=torch.float64, device=dev)
            if F.shape[-1] == tree.N:
                F = np.atleast_2d(F)[:, tree.boundary_ids]
            elif F.shape[-1] != nbd:
                raise ValueError(f"boundary data must have trailing size {nbd} or {tree.N}, "
                                 f"got {F.shape}")
            return torch.as_tensor(np.ascontiguousarray(np.atleast_2d(F)), device=dev)
        if F.ndim == 0:
            return F.reshape(1, 1).expand(1, nbd).contiguous()
        if F.shape[-1] == tree.N:
            return torch.atleast_2d(F)[:, self.plan.boundary_ids].contiguous()
        if F.shape[-1] == nbd:
            return torch.atleast_2d(F).contiguous()
        raise ValueError(f"boundary data must have trailing size {nbd} or {tree.N}, "
                         f"got {tuple(F.shape)}")

    def _solve(self, f, g, flux_jump, inv_dt, out=None):
        tree = self.tree
        dev = cuda_device()
        as_numpy = not any(torch.is_tensor(x) for x in (f, g, flux_jump))
        fb = self._boundary_values(f, dev)
        k = fb.shape[0]
        squeeze = (ndim(f) <= 1) if g is None else (ndim(g) == 1)
        G = None
        if g is not None:
            G = torch.atleast_2d(torch.as_tensor(g, dtype=torch.float64, device=dev))
            k = max(k, G.shape[0])
        J = None
        if flux_jump is not None:
            J = torch.atleast_2d(torch.as_tensor(flux_jump, dtype=torch.float64, device=dev))
            if G is None:
                k = max(k, J.shape[0])
        ld_f = fb.shape[1] if fb.shape[0] > 1 else 0
        if fb.shape[0] not in (1, k):
            raise ValueError(f"boundary data has {fb.shape[0]} rows for {k} right-hand sides")
        for name, X in (("body load", G), ("flux jump", J)):
            if X is not None and (X.shape[-1] != tree.N or X.shape[0] not in (1, k)):
                raise ValueError(f"{name} must have shape ({k}, {tree.N}), got {tuple(X.shape)}")
        G = None if G is None else G.contiguous()
        J = None if J is None else J.contiguous()
        U = out if out is not None else torch.empty((k, tree.N), dtype=torch.float64, device=dev)
        ws = self.plan.workspace(k)
        ld_g = 0 if G is None or G.shape[0] == 1 else tree.N
        ld_j = 0 if J is None or J.shape[0] == 1 else tree.N
        rc = self._lib.hps_solve(
            self.handle, k, fb.data_ptr(), ld_f,
            None if G is None else G.data_ptr(), ld_g,
            None if J is None else J.data_ptr(), ld_j,
            0.0 if inv_dt is None else float(inv_dt),
            U.data_ptr(), tree.N, ws.data_ptr(), ws.numel(), current_stream_handle())
        _lib.check(rc, "hps_solve")
        res = U[0] if squeeze else U
        if as_numpy:
            return res.cpu().numpy()
        return res

    def solve_device(self, fb, body, out, jump=None, inv_dt=None):
        """Stream-ordered device solve without validation or host copies (the
        stepper's entry).  ``fb`` (1 or k, nbd); ``body`` (k, >= L*ni) read at
        leaf interiors only, or None; ``jump`` (k, N) or None; ``out`` (k, N)."""
        k = out.shape[0]
        ld_f = 0 if fb.shape[0] == 1 else fb.stride(0)
        ld_g = 0 if body is None or body.shape[0] == 1 else body.stride(0)
        ld_j = 0 if jump is None or jump.shape[0] == 1 else jump.stride(0)
        ws = self.plan.workspace(k)
        rc = self._lib.hps_solve(
            self.handle, k, fb.data_ptr(), ld_f, None if body is None else body.data_ptr(), ld_g,
            None if jump is None else jump.data_ptr(), ld_j,
            0.0 if inv_dt is None else float(inv_dt), out.data_ptr(), out.stride(0),
            ws.data_ptr(), ws.numel(), current_stream_handle())
        _lib.check(rc, "hps_solve")
        return out

    @property
    def fuses_stage_history(self):
        """Whether ``solve_stage_device`` can return the stage history L u
        (tensor-product leaf solve, constant coefficients)."""
        return self.leaf_solve == "tensor" and os.environ.get("HPSB_NO_FUSED_LU") != "1" \
            and os.environ.get("HPSB_NO_FD_DOWN") is None and os.environ.get("HPSB_FD_SIMT") is None

    def solve_stage_device(self, fb, body, out, lu, guard, root_pre=None):
        """``solve_device`` plus the interior L u of the solution into ``lu``
        (k, >= L*ni) and max |u| into ``guard`` (hps_solve_stage)."""
        k = out.shape[0]
        ld_f = 0 if fb.shape[0] == 1 else fb.stride(0)
        ld_g = 0 if body is None or body.shape[0] == 1 else body.stride(0)
        ws = self.plan.workspace(k)
        rc = self._lib.hps_solve_stage(
            self.handle, k, fb.data_ptr(), ld_f, None if body is None else body.data_ptr(), ld_g,
            out.data_ptr(), out.stride(0), None if lu is None else lu.data_ptr(), 0 if lu is None else lu.stride(0),
            None if guard is None else guard.data_ptr(), None if root_pre is None else root_pre.data_ptr(),
            ws.data_ptr(), ws.numel(), current_stream_handle())
        _lib.check(rc, "hps_solve_stage")
        return out

    def solve_stage_terms_device(self, fb, dcoef_ptr, vecs, rout, out, lu, guard, root_pre=None):
        """The fused stage solve (one rhs) with its body load given as the
        combination sum_t c_t vecs[t] over the leaf interiors (coefficients in
        device memory at ``dcoef_ptr``), formed by the upward sweep's leaf
        kernel and written to ``rout`` (hps_solve_stage_terms)."""
        ws = self.plan.workspace(1)
        vp = (ctypes.c_void_p * len(vecs))(*[v.data_ptr() for v in vecs])
        rc = self._lib.hps_solve_stage_terms(
            self.handle, fb.data_ptr(), len(vecs), dcoef_ptr, vp, rout.data_ptr(), out.data_ptr(),
            None if lu is None else lu.data_ptr(), None if guard is None else guard.data_ptr(),
            None if root_pre is None else root_pre.data_ptr(), ws.data_ptr(), ws.numel(), current_stream_handle())
        _lib.check(rc, "hps_solve_stage_terms")
        return out

    def solve_stage_terms_k_device(self, fb, dcoef_ptr, vecs, rout, out, lu, guard):
        """solve_stage_terms_device for k rhs rows (hps_solve_stage_terms_k):
        vecs are (rows, N) views with rows 1 (shared by every rhs) or k."""
        k = out.shape[0]
        ws = self.plan.workspace(k)
        vp = (ctypes.c_void_p * len(vecs))(*[v.data_ptr() for v in vecs])
        lds = (ctypes.c_longlong * len(vecs))(*[0 if v.shape[0] == 1 else v.stride(0) for v in vecs])
        rc = self._lib.hps_solve_stage_terms_k(
            self.handle, k, fb.data_ptr(), fb.stride(0) if fb.shape[0] > 1 else 0, len(vecs), dcoef_ptr, vp, lds,
            rout.data_ptr(), rout.stride(0), out.data_ptr(), out.stride(0),
            None if lu is None else lu.data_ptr(), 0 if lu is None else lu.stride(0),
            None if guard is None else guard.data_ptr(), ws.data_ptr(), ws.numel(), current_stream_handle())
        _lib.check(rc, "hps_solve_stage_terms_k")
        return out

    @property
    def root_dirichlet_ok(self):
        """Whether the root's Dirichlet product can be batched over a step's
        stages (hps_root_dirichlet: the root boundary is the domain boundary)."""
        return self.tree.depth > 0 and self.plan.nparts == 1 and \
            os.environ.get("HPSB_NO_ROOT_BATCH") != "1"

    def root_dirichlet_device(self, fb_rows, out):
        """S_root u_bnd for each row of boundary data (fb order) into out
        (ns, n3_root): one pass over the root operator per 8 rows
        (hps_root_dirichlet)."""
        ns = fb_rows.shape[0]
        nbytes = self._lib.hps_root_dirichlet_scratch(self.handle, min(ns, 8))
        scratch = torch.empty(max(1, (nbytes + 7) // 8), dtype=torch.float64, device=out.device)
        for r0 in range(0, ns, 8):  # eight rows per pass (tableaus with more stages: several passes)
            m = min(8, ns - r0)
            rc = self._lib.hps_root_dirichlet(self.handle, m, fb_rows[r0].data_ptr(), fb_rows.stride(0),
                                              out[r0].data_ptr(), out.stride(0), scratch.data_ptr(),
                                              scratch.numel() * 8, current_stream_handle())
            _lib.check(rc, "hps_root_dirichlet")
        return out

    def leaf_lu_device(self, u, lu, guard=None, leaves=None):
        """Interior L u of the (k, N) device state ``u`` into ``lu`` (rows from
        the first leaf's interior) and max |u| into ``guard``, by the leaf-grid
        products of the fused stage (hps_leaf_lu; needs ``fuses_stage_history``).
        ``leaves = (leaf0, nleaf)`` restricts it to a leaf range."""
        k = u.shape[0]
        leaf0, nleaf = (0, self.tree.L) if leaves is None else leaves
        rc = self._lib.hps_leaf_lu(self.handle, leaf0, nleaf, k, u.data_ptr(), u.stride(0), lu.data_ptr(),
                                   lu.stride(0), None if guard is None else guard.data_ptr(),
                                   current_stream_handle())
        _lib.check(rc, "hps_leaf_lu")
        return lu

    def solve_phase(self, phases, part0, part1, fb, body, out, jump=None, inv_dt=None):
        """One or more phases of a subtree-partitioned solve (hps_solve_phase):
        ``_lib.HPS_PHASE_UP`` / ``TOP`` / ``DOWN`` over parts [part0, part1).
        ``body`` rows start at the first leaf of part0 (or None); ``out`` (k, N)
        rows are global."""
        k = out.shape[0]
        ld_f = 0 if fb.shape[0] == 1 else fb.stride(0)
        ld_g = 0 if body is None or body.shape[0] == 1 else body.stride(0)
        ld_j = 0 if jump is None or jump.shape[0] == 1 else jump.stride(0)
        ws = self.plan.workspace(k)
        rc = self._lib.hps_solve_phase(
            self.handle, int(phases), int(part0), int(part1), k, fb.data_ptr(), ld_f,
            None if body is None else body.data_ptr(), ld_g,
            None if jump is None else jump.data_ptr(), ld_j,
            0.0 if inv_dt is None else float(inv_dt), out.data_ptr(), out.stride(0),
            ws.data_ptr(), ws.numel(), current_stream_handle())
        _lib.check(rc, "hps_solve_phase")
        return out

    def top_level(self, level, down, rank, nranks, out, stage=None):
        """This rank's share of one top level (< lstar) of a row-sharded
        subtree-partitioned solve (hps_top_level): up -> w3 / flux rows into
        the workspace's level blocks (``plan.level_blocks``), down -> u3 rows
        into ``stage`` (k, c * n3); the caller sums both over the ranks."""
        k = out.shape[0]
        ws = self.plan.workspace(k)
        rc = self._lib.hps_top_level(self.handle, int(level), 1 if down else 0, int(rank), int(nranks), k,
                                     out.data_ptr(), out.stride(0), None if stage is None else stage.data_ptr(),
                                     ws.data_ptr(), ws.numel(), current_stream_handle())
        _lib.check(rc, "hps_top_level")
        return stage

    # -- operator views (reference solver.py:339-348) ---------------------------------
    def _leaf_block(self, which, leaf):
        st = self.disc.stencil
        shape = {0: (st.ni, st.ni), 1: (st.ni, st.nb), 2: (st.nb, st.nb)}[which]
        out = np.empty(shape)
        _lib.check(self._lib.hps_ops_get_leaf(self.handle, which, leaf, _lib.dbl_ptr(out)),
                   "hps_ops_get_leaf")
        return out

    def _merge_block(self, level, pos, which):
        lm = self.tree.level_maps[level]
        if which == 1 and level > 0:
            # stored as the flux rows Tstack X33^-1 of the stacked up-pass operator
            return self._merge_block(level, pos, 4) @ np.linalg.inv(self._merge_block(level, pos, 0))
        shape = {0: (lm.n3, lm.n3), 1: (lm.n12, lm.n3), 2: (lm.n3, lm.n12), 3: (lm.n12, lm.n12),
                 4: (lm.n12, lm.n3)}[which]
        out = np.empty(shape)
        _lib.check(self._lib.hps_ops_get_merge(self.handle, level, pos, which, _lib.dbl_ptr(out)),
                   "hps_ops_get_merge")
        return out

    def leaf_operators(self, leaf_id):
        T = self._leaf_block(2, leaf_id) if self.keep_dtn else None
        return LeafOperators(S=self._leaf_block(1, leaf_id), T=T,
                             Aii_factor=_InverseFactor(self._leaf_block(0, leaf_id)),
                             D_edge=self.disc.stencil.D_bnd)

    def _locate(self, node_index):
        for d, lm in enumerate(self.tree.level_maps):
            hit = np.nonzero(lm.node_index == node_index)[0]
            if hit.size:
                return d, int(hit[0])
        raise KeyError(node_index)

    def merge_operators(self, node_index):
        d, pos = self._locate(node_index)
        T = self._merge_block(d, pos, 3) if (self.keep_dtn or d == 0) else None
        return MergeOperators(S=self._merge_block(d, pos, 2),
                              X33_factor=_InverseFactor(self._merge_block(d, pos, 0)),
                              Tstack=self._merge_block(d, pos, 1), T=T)

    @property
    def merges(self):
        return {i: _LazyMerge(self, i) for i in self.parent_order}

    @property
    def leaf_factors(self):
        return _LeafFactors(self)

    @property
    def S_leaf(self):
        S0 = self._leaf_block(1, 0)
        if self.disc.coeffs.is_constant:
            return np.broadcast_to(S0, (self.tree.L,) + S0.shape)
        return np.stack([self._leaf_block(1, l) for l in range(self.tree.L)])

    @property
    def root_T(self):
        return self._merge_block(0, 0, 3) if self.tree.depth > 0 else None

    # -- persistence (reference solver.py:280-337) -----------------------------------
    _DUMP_MAGIC = b"HPSB200OPS\n"

    def save(self, path):
        """Binary dump so repeated runs can skip the build (solver.py:294-306):
        the versioned header, then the device operator set."""
        lib = self._lib
        n = int(lib.hps_ops_dump_size(self.handle))
        if n < 0:
            raise HpstepError("hps_ops_dump_size failed: " + _lib.last_error())
        buf = np.empty(n, dtype=np.uint8)
        _lib.check(lib.hps_ops_dump(self.handle, buf.ctypes.data_as(ctypes.c_void_p), n), "hps_ops_dump")
        head = json.dumps({"header": _jsonable(self.header()), "layout": self.layout,
                           "keep_dtn": self.keep_dtn, "nparts": self.plan.nparts}).encode()
        with open(path, "wb") as fh:
            fh.write(self._DUMP_MAGIC)
            fh.write(len(head).to_bytes(8, "little"))
            fh.write(head)
            fh.write(buf.tobytes())

    @classmethod
    def load(cls, path, disc, sigma, dt_gamma):
        """Load a dumped operator set, validating the versioned header
        (solver.py:308-337): a dump made for another tree, coefficient field or
        shift raises HpstepError."""
        obj = cls.__new__(cls)
        obj.disc, obj.tree = disc, disc.tree
        obj.sigma, obj.dt_gamma = float(sigma), float(dt_gamma)
        st = disc.stencil
        obj.D_bi = st.D_bnd[:, :st.ni]
        with open(path, "rb") as fh:
            if fh.read(len(cls._DUMP_MAGIC)) != cls._DUMP_MAGIC:
                raise HpstepError(f"{path} is not an operator dump of this package")
            n = int.from_bytes(fh.read(8), "little")
            meta = json.loads(fh.read(n).decode())
            payload = np.frombuffer(fh.read(), dtype=np.uint8)
        if meta["header"] != _jsonable(obj.header()):
            raise HpstepError("operator dump does not match the requested configuration "
                              f"(dump header {meta['header']})")
        obj.layout, obj.keep_dtn = meta["layout"], bool(meta["keep_dtn"])
        obj.plan = device_plan(obj.tree, meta.get("nparts", 1))
        lib = obj.plan._lib
        h = ctypes.c_void_p()
        _lib.check(lib.hps_ops_load(obj.plan.handle, payload.ctypes.data_as(ctypes.c_void_p), payload.size,
                                    ctypes.byref(h)), "hps_ops_load")
        obj.handle, obj._lib = h, lib
        obj.parent_order = [int(i) for lm in obj.tree.level_maps for i in lm.node_index]
        return obj

    def header(self):
        tree = self.tree
        return {"version": FORMAT_VERSION, "dim": tree.dim, "bounds": tree.bounds, "n1": tree.n1,
                "n2": tree.n2, "p": tree.p, "sigma": self.sigma, "dt_gamma": self.dt_gamma,
                "coeff_hash": coefficient_hash(self.disc)}


class _LazyMerge:
    def __init__(self, ops, idx):
        self._ops, self._idx = ops, idx

    def __getattr__(self, name):
        mo = self._ops.merge_operators(self._idx)
        return getattr(mo, name)


class _LeafFactors:
    def __init__(self, ops):
        self._ops = ops

    def __len__(self):
        return self._ops.tree.L

    def __getitem__(self, i):
        return _InverseFactor(self._ops._leaf_block(0, i))


_EIG_CACHE = {}


def _accurate_eig(A, cond_max):
    """(lam, V, V^-1) of the real q x q matrix A, computed in 34-digit
    arithmetic (mpmath) and rounded to double, or None when A has complex or
    ill-conditioned eigenvectors.  The factors are applied at every stage
    solve of every step, so their error is a fixed perturbation of the leaf
    operator that accumulates coherently over a trajectory: LAPACK's double
    eigenvectors of these non-normal Chebyshev blocks give the tensor-product
    leaf solve a ~1e-14 relative error (a linear drift of ~5e-13 per C2 step
    against the reference), correctly rounded factors ~3e-16."""
    key = A.tobytes()
    if key in _EIG_CACHE:
        return _EIG_CACHE[key]
    lam, V = np.linalg.eig(A)
    scale = max(1.0, float(np.abs(lam).max()))
    res = None
    if np.abs(lam.imag).max() <= 1e-12 * scale and np.abs(V.imag).max() <= 1e-12 and \
            np.linalg.cond(V.real) <= cond_max:
        try:
            import mpmath
        except ImportError:      # no extended-precision eigensolver: the dense leaf path is used
            mpmath = None
        if mpmath is not None:
            ctx = mpmath.mp.clone() if hasattr(mpmath.mp, "clone") else mpmath.mp
            old = ctx.dps
            ctx.dps = 34
            try:
                E, ER = ctx.eig(ctx.matrix(A.tolist()))
                q = A.shape[0]
                order = np.argsort([float(ctx.re(e)) for e in E])
                lam = np.array([float(ctx.re(E[j])) for j in order])
                Vm = ctx.matrix(q, q)
                for a in range(q):
                    for j, b in enumerate(order):
                        Vm[a, j] = ctx.re(ER[a, b])
                Vi = Vm ** -1
                V = np.array(Vm.tolist(), dtype=float)
                res = (lam, V, np.array(Vi.tolist(), dtype=float))
            finally:
                ctx.dps = old
    _EIG_CACHE[key] = res
    return res


def tensor_leaf_factors(disc, sigma, dt_gamma, cond_max=1e6):
    """Kronecker-sum factorisation of the interior leaf block for constant
    coefficients (see csrc/leaf_fd.cu): [Vx^-1, Vy^-T, Vx, Vy^T, 1/den] (q x q)
    and the interior parts of the four flux rows, or None when the block is
    not a Kronecker sum with a real, well-conditioned eigenbasis."""
    cf, st, tree = disc.coeffs, disc.stencil, disc.tree
    q = tree.q
    if not cf.is_constant or not 4 <= q <= 14:
        return None
    v = lambda f: 0.0 if f is None else float(f)
    c11, c22, c1, c2, c0 = v(cf.c11), v(cf.c22), v(cf.c1), v(cf.c2), v(cf.c)
    i = slice(1, tree.p - 1)
    Ax = dt_gamma * (-c11 * st.d2x[i, i] + c1 * st.d1x[i, i])
    Ay = dt_gamma * (-c22 * st.d2y[i, i] + c2 * st.d1y[i, i])
    out = []
    for Amat in (Ax, Ay):
        f = _accurate_eig(Amat, cond_max)
        if f is None:
            return None
        out.append(f)
    (lx, Vx, Vxi), (ly, Vy, Vyi) = out
    den = lx[:, None] + ly[None, :] + (sigma + dt_gamma * c0)
    if np.abs(den).min() <= 1e-13 * np.abs(den).max():
        return None
    den = 1.0 / den                      # the kernel multiplies
    p = tree.p
    edges = [st.d1x[0, i], st.d1x[p - 1, i], st.d1y[0, i], st.d1y[p - 1, i]]
    # interior -> boundary couplings of the shifted operator (A_ib of solver.py:53-64)
    cpl = [dt_gamma * (-c11 * st.d2x[i, 0] + c1 * st.d1x[i, 0]),
           dt_gamma * (-c11 * st.d2x[i, p - 1] + c1 * st.d1x[i, p - 1]),
           dt_gamma * (-c22 * st.d2y[i, 0] + c2 * st.d1y[i, 0]),
           dt_gamma * (-c22 * st.d2y[i, p - 1] + c2 * st.d1y[i, p - 1])]
    # interior L u of the stage history on the leaf grid G: Mx G + G My^T - c G
    Mx = np.zeros((16, 16))
    My = np.zeros((16, 16))
    Mx[:p, :p] = c11 * st.d2x - c1 * st.d1x
    My[:p, :p] = c22 * st.d2y - c2 * st.d1y
    return np.concatenate([Vxi.ravel(), Vyi.T.ravel(), Vx.ravel(), Vy.T.ravel(), den.ravel()]
                          + [e.ravel() for e in edges] + [c.ravel() for c in cpl]
                          + [Mx.ravel(), My.ravel(), [c0]])


def _jsonable(v):
    if isinstance(v, dict):
        return {k: _jsonable(x) for k, x in v.items()}
    if isinstance(v, (list, tuple)):
        return [_jsonable(x) for x in v]
    return v


def coefficient_hash(disc):
    """Hash of coefficient samples identifying the operator (solver.py:351-361)."""
    pts = [disc.leaf_points(0)]
    if disc.tree.leaf_count > 1:
        pts.append(disc.leaf_points(disc.tree.leaf_count - 1))
    h = hashlib.sha256()
    for p in pts:
        s = disc.coeffs.evaluate(p)
        for key in sorted(s):
            h.update(np.ascontiguousarray(s[key]).tobytes())
    return h.hexdigest()


def resolve_layout(layout, coeffs):
    """Operator storage: "per_node" streams one operator copy per node from
    HBM every solve (the reference's storage, solver.py:137-151); "shared"
    keeps one copy per level and runs the level applies as tensor-core GEMMs
    (constant coefficients only).  None / "auto" picks "shared" when the
    coefficients are constant; the environment variable HPSB_LAYOUT
    overrides the automatic choice."""
    if layout in (None, "auto"):
        layout = os.environ.get("HPSB_LAYOUT", "auto")
        if layout == "auto":
            layout = "shared" if coeffs.is_constant else "per_node"
    if layout not in ("per_node", "shared"):
        raise ValueError(f"unknown operator layout {layout!r}")
    if layout == "shared" and not coeffs.is_constant:
        layout = "per_node"      # every node differs: nothing to share
    return layout


def build(tree, coeffs, sigma=0.0, dt_gamma=1.0, disc=None, keep_dtn=False, threads=None, layout=None,
          nparts=1):
    """Build the operator set for ``sigma*I + dt_gamma*A`` on the GPU."""
    if disc is None:
        disc = EllipticDiscretization(tree, coeffs)
    return HpsOperatorSet(disc, sigma=sigma, dt_gamma=dt_gamma, keep_dtn=keep_dtn, threads=threads,
                          layout=layout, nparts=nparts)
