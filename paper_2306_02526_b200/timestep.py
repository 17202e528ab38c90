"""IMEX ARK time stepping with every stage on the GPU (drop-in for
``hpstep.timestep``, reference timestep.py:36-333).

The stage formulation (timestep.py:237-266) is the hot path:

    (I - dt*gamma*L) u_i = u^n + dt*sum_{j<i} a_ij L u_j + dt*sum_{j<i} ahat_ij (q_j + g_j)

Device data flow per stage i (k stacked right-hand sides, N DOFs):

* ``L u_j`` is kept only at the leaf-interior DOFs ``[0, L*ni)`` -- the solve
  reads its body load nowhere else (solver.py:220) -- as ``(k, L*ni)``
  history rows written by one ``hps_leaf_eval`` pass over ``u_j``;
* ``q`` is either a :class:`SeparableField` (spatial parts resident on the
  device, time factors folded into the combination coefficients, nothing
  stored per stage) or any callable, evaluated per stage into a history row;
* ``g(t, u, u_x, u_y)`` receives device tensors (u and the interface-averaged
  gradient from ``hps_leaf_eval``); a callable that cannot run on torch
  tensors is evaluated on the host from downloaded arrays;
* one ``hps_combine`` forms the stage body load over ``[0, L*ni)``, one
  ``hps_solve`` produces ``u_i``, the divergence guard (timestep.py:198-203)
  is a max|u| reduction fused into the next leaf pass and checked on the host
  once per step (or once per ``run`` chunk), raising ``DivergenceError`` with
  the step index the reference would report;
* the update ``u_s + dt*sum_j (bhat_j - ahat_sj)(q_j + g_j)`` is one more
  ``hps_combine`` over all N DOFs followed by the boundary overwrite.

Backward Euler (timestep.py:231-235) and the slope / penalized-slope
formulations (timestep.py:268-328) reuse the same device pieces.
"""

import ctypes
import gc
import os
import sys

import numpy as np

from . import _lib
from .device import cuda_device, current_stream_handle, torch
from . import npgpu
from .errors import DivergenceError, HpstepError, UnsupportedConfigurationError
from .operators import EllipticDiscretization
from .solver import HpsOperatorSet, device_plan, graph_workspace
from .tableaux import ButcherPair, load_tableau

DIVERGENCE_LIMIT = 1e12


# ---------------------------------------------------------------------------
# problem data
# ---------------------------------------------------------------------------

class SeparableField:
    """A field ``F(t, pts) = sum_m s_m(t) * phi_m(pts)``.

    Callable exactly like the reference's field callables (``F(t, pts)``), so
    problems written with it run unchanged on the reference.  The device
    stepper evaluates every ``phi_m`` once at the grid points, keeps it
    resident, and folds ``s_m(t)`` into scalar coefficients: no per-stage
    field evaluation or host traffic.  ``s_m = None`` means constant in time.
    ``phi_m(pts)`` returns ``(n,)`` or ``(ncomp, n)``.
    """

    def __init__(self, terms):
        self.terms = [(phi, s) for phi, s in terms]

    @classmethod
    def product(cls, phi, s=None):
        return cls([(phi, s)])

    def factors(self, t):
        return [1.0 if s is None else float(s(t)) for _, s in self.terms]

    def __call__(self, t, pts):
        out = 0.0
        for (phi, _), f in zip(self.terms, self.factors(t)):
            out = out + f * np.asarray(phi(pts), dtype=float)
        return out


class ParabolicProblem:
    """``u_t = L u + q + g(u)`` with Dirichlet data ``f`` (reference
    timestep.py:36-61); ``coeffs`` holds ``A = -L``."""

    def __init__(self, coeffs, q=None, g=None, f=None, f_t=None, u0=None,
                 time_independent_bc=False, ncomp=1, name="problem"):
        self.coeffs = coeffs
        self.q = q
        self.g = g
        self.f = f
        self.f_t = f_t
        self.u0 = u0
        self.time_independent_bc = time_independent_bc
        self.ncomp = ncomp
        self.name = name

    @property
    def is_linear(self):
        return self.g is None


class StepperState:
    """Time and solution.  The solution stays on the device between steps;
    ``.u`` materialises a host array (cached) for reference-style callers."""

    def __init__(self, t, u):
        self.t = float(t)
        self.u = u

    @property
    def u(self):
        if self._host is None:
            self._host = self._dev.cpu().numpy()
        return self._host.numpy() if torch.is_tensor(self._host) else self._host

    @u.setter
    def u(self, v):
        if torch.is_tensor(v) and v.is_cuda:
            self._dev, self._host = v, None
        elif torch.is_tensor(v):          # host tensor (e.g. pinned): copied on first use
            self._dev, self._host = None, v
        else:
            self._dev, self._host = None, np.asarray(v, dtype=float)

    @property
    def u_device(self):
        if self._dev is None:
            src = self._host if torch.is_tensor(self._host) else torch.from_numpy(self._host)
            self._dev = src.to(cuda_device(), non_blocking=True)
        return self._dev


# ---------------------------------------------------------------------------
# device leaf evaluations (apply_lop / gradient / flux_jump)
# ---------------------------------------------------------------------------

class DeviceDiscretization:
    """Device side of ``EllipticDiscretization`` (operators.py:276-346)."""

    def __init__(self, disc):
        lib = _lib.load()
        self.disc, self.tree = disc, disc.tree
        self.plan = device_plan(self.tree)
        st, cf = disc.stencil, disc.coeffs
        samp = np.ascontiguousarray(disc.coefficient_samples(), dtype=float)
        keep = [np.ascontiguousarray(a, dtype=float)
                for a in (st.d1x, st.d2x, st.d1y, st.d2y, st.ex1, st.ex2, st.ey1, st.ey2)]
        sign = np.ascontiguousarray(self.tree.leaf_bnd_sign, dtype=np.int8)
        d = _lib.DiscDesc()
        d.d1x, d.d2x, d.d1y, d.d2y, d.ex1, d.ex2, d.ey1, d.ey2 = (_lib.dbl_ptr(a) for a in keep)
        d.Lc = samp.shape[0]
        d.coef = _lib.dbl_ptr(samp)
        d.has_c1, d.has_c2, d.has_c = (int(v is not None) for v in (cf.c1, cf.c2, cf.c))
        d.leaf_bnd_sign = sign.ctypes.data_as(ctypes.POINTER(ctypes.c_byte))
        h = ctypes.c_void_p()
        _lib.check(lib.hps_disc_create(self.plan.handle, ctypes.byref(d), ctypes.byref(h)),
                   "hps_disc_create")
        self.handle, self._lib = h, lib
        self.Lni = self.tree.L * self.tree.ni

    def __del__(self):
        try:
            if self.handle:
                self._lib.hps_disc_destroy(self.handle)
        except Exception:
            pass

    def eval(self, U, lu_int=None, lu=None, ux=None, uy=None, jump=None, guard=None, ld_o=None,
             leaves=None):
        """One leaf pass over the (k, N) device tensor U (row stride U.stride(0)).
        ``leaves = (leaf0, nleaf)`` restricts it to a leaf range (lu_int rows
        then start at leaf0's interior; see hps_leaf_eval_range)."""
        outs = [lu_int, lu, ux, uy, jump]
        if ld_o is None:
            ld_o = next((o.stride(0) for o in outs if o is not None), 0)
        ptr = lambda o: None if o is None else o.data_ptr()
        leaf0, nleaf = (0, self.tree.L) if leaves is None else leaves
        rc = self._lib.hps_leaf_eval_range(self.handle, leaf0, nleaf, U.shape[0], U.data_ptr(), U.stride(0),
                                           *[ptr(o) for o in outs], ld_o, ptr(guard),
                                           current_stream_handle())
        _lib.check(rc, "hps_leaf_eval")

    def _prep(self, u):
        as_numpy = not torch.is_tensor(u)
        squeeze = (np.ndim(u) if as_numpy else u.dim()) == 1
        U = torch.atleast_2d(torch.as_tensor(u, dtype=torch.float64, device=cuda_device()))
        return U.contiguous(), as_numpy, squeeze

    @staticmethod
    def _ret(X, as_numpy, squeeze):
        X = X[0] if squeeze else X
        return X.cpu().numpy() if as_numpy else X

    def apply_lop(self, u):
        U, a, s = self._prep(u)
        out = torch.empty_like(U)
        self.eval(U, lu=out)
        return self._ret(out, a, s)

    def apply_lop_interior(self, U, out):
        self.eval(U, lu_int=out)
        return out

    def gradient(self, u):
        U, a, s = self._prep(u)
        ux, uy = torch.empty_like(U), torch.empty_like(U)
        self.eval(U, ux=ux, uy=uy)
        return self._ret(ux, a, s), self._ret(uy, a, s)

    def flux_jump(self, u):
        U, a, s = self._prep(u)
        out = torch.empty_like(U)
        self.eval(U, jump=out)
        return self._ret(out, a, s)


def device_discretization(disc):
    dd = disc._device.get("eval")
    if dd is None:
        dd = DeviceDiscretization(disc)
        disc._device["eval"] = dd
    return dd


class _CoefSink:
    """Coefficient table of one captured step.  While a step is captured into
    a CUDA graph every ``combine`` takes its coefficients from a device table
    (slots in call order) instead of kernel arguments; a *dry* pass of the same
    step code recomputes the table for the next time level without launching
    anything, and the host copies it in before each replay."""

    current = None

    def __init__(self, dev=None, dry=False):
        self.vals, self.dev, self.dry = [], dev, dry

    def take(self, vals):
        off = len(self.vals)
        self.vals.extend(vals)
        if self.dry:
            return None
        if len(self.vals) > self.dev.numel():
            raise HpstepError("coefficient table overflow")
        return self.dev.data_ptr() + 8 * off


def combine(terms, out, n=None, guard=None):
    """out[:, :n] = sum c * v over (coef, tensor) terms (rows broadcast when a
    term has a single row)."""
    lib = _lib.load()
    sink = _CoefSink.current
    if sink is None:
        terms = [(float(c), v) for c, v in terms if c != 0.0]
    else:
        terms = [(float(c), v) for c, v in terms]   # fixed slots: zeros may become nonzero later
    k = out.shape[0]
    n = out.shape[1] if n is None else n
    nt = len(terms)
    dptr = sink.take([c for c, _ in terms]) if sink is not None else None
    if sink is not None and sink.dry:
        return out
    vecs = (ctypes.c_void_p * max(1, nt))(*[v.data_ptr() for _, v in terms])
    lds = (ctypes.c_longlong * max(1, nt))(*[0 if v.shape[0] == 1 else v.stride(0)
                                              for _, v in terms])
    gptr = None if guard is None else guard.data_ptr()
    if sink is None:
        coefs = (ctypes.c_double * max(1, nt))(*[c for c, _ in terms])
        rc = lib.hps_combine(k, n, nt, coefs, vecs, lds, out.data_ptr(), out.stride(0), gptr,
                             current_stream_handle())
    else:
        rc = lib.hps_combine_dev(k, n, nt, dptr, vecs, lds, out.data_ptr(), out.stride(0), gptr,
                                 current_stream_handle())
    _lib.check(rc, "hps_combine")
    return out


def combine_bnd(plan, terms, fb, out, guard):
    """out = sum c * v over all DOFs, the Dirichlet data fb at the boundary
    DOFs and guard = max(guard, max |out|), one pass (hps_combine_bnd)."""
    lib = _lib.load()
    sink = _CoefSink.current
    terms = [(float(c), v) for c, v in terms]
    nt = len(terms)
    dptr = sink.take([c for c, _ in terms]) if sink is not None else None
    if sink is not None and sink.dry:
        return out
    vecs = (ctypes.c_void_p * max(1, nt))(*[v.data_ptr() for _, v in terms])
    lds = (ctypes.c_longlong * max(1, nt))(*[0 if v.shape[0] == 1 else v.stride(0) for _, v in terms])
    coefs = (ctypes.c_double * max(1, nt))(*[c for c, _ in terms]) if sink is None else None
    rc = lib.hps_combine_bnd(plan.handle, out.shape[0], nt, coefs, dptr, vecs, lds, fb.data_ptr(),
                             0 if fb.shape[0] == 1 else fb.stride(0), out.data_ptr(), out.stride(0),
                             None if guard is None else guard.data_ptr(), current_stream_handle())
    _lib.check(rc, "hps_combine_bnd")
    return out


def combine_rows(coefs, vecs, out):
    """out[r] = sum_t coefs[r][t] * vecs[t] (single-row terms) for every row r
    of ``out`` in one launch (hps_combine_dev_rows)."""
    lib = _lib.load()
    k, nt = out.shape[0], len(vecs)
    flat = [float(c) for row in coefs for c in row]
    sink = _CoefSink.current
    if sink is not None:
        dptr = sink.take(flat)
        if sink.dry:
            return out
        dc = None
    else:
        dc = torch.tensor(flat, dtype=torch.float64, device=out.device)
        dptr = dc.data_ptr()
    vp = (ctypes.c_void_p * max(1, nt))(*[v.data_ptr() for v in vecs])
    lds = (ctypes.c_longlong * max(1, nt))(*([0] * nt))
    rc = lib.hps_combine_dev_rows(k, out.shape[1], nt, dptr, nt, vp, lds, out.data_ptr(), out.stride(0), None,
                                  current_stream_handle())
    _lib.check(rc, "hps_combine_dev_rows")
    return out


def scalar_stability_function(pair, z):
    """Amplification factor of the implicit half on u' = lambda u (reference
    timestep.py:331-333)."""
    return pair.stability_function(z)


def evaluate_nonlinear(disc, problem, t, u):
    """Pointwise g with leaf-local spectral derivatives (timestep.py:64-78)."""
    as_numpy = not torch.is_tensor(u)
    squeeze = (np.ndim(u) if as_numpy else u.dim()) == 1
    dd = device_discretization(disc)
    U = torch.atleast_2d(torch.as_tensor(u, dtype=torch.float64, device=cuda_device())).contiguous()
    if problem.g is None:
        out = torch.zeros_like(U)
    else:
        ux, uy = torch.empty_like(U), torch.empty_like(U)
        dd.eval(U, ux=ux, uy=uy)
        out = _call_g(problem.g, t, U, ux, uy)
    out = out[0] if squeeze else out
    return out.cpu().numpy() if as_numpy else out


def gradient_use(g):
    """Which gradient components ``g(t, u, u_x, u_y)`` reads: ``(True, True)``
    unless ``g`` declares otherwise through :func:`declare_nonlinear`."""
    use = getattr(g, "grad_use", None)
    return (True, True) if use is None else (bool(use[0]), bool(use[1]))


def is_pure(g):
    """Whether ``g`` is declared a pure device function (see declare_nonlinear)."""
    return bool(getattr(g, "pure", False))


def declare_nonlinear(g, ux=True, uy=True, pure=False):
    """Declare properties of a nonlinear term ``g(t, u, u_x, u_y)`` that the
    device stepper may exploit (an extension of the reference API, which
    always evaluates both gradient components, timestep.py:192-196, and
    calls g afresh every stage).  Returns ``g``, so it can wrap a lambda.

    * ``ux`` / ``uy`` False: that gradient component is never read; it is
      not computed and ``g`` receives a buffer of unspecified contents.
    * ``pure`` True: ``g`` is a fixed composition of torch operations on its
      device tensor arguments -- independent of ``t``, of host state and of
      data-dependent Python control flow -- so the step's CUDA graph may
      capture it.  Undeclared terms are called eagerly at every stage (the
      captured step is cut around them), with the stage time of that step.

    A declaration is the caller's promise for every (t, u)."""
    try:
        g.grad_use = (bool(ux), bool(uy))
        g.pure = bool(pure)
    except AttributeError as e:
        raise TypeError(f"cannot attach a declaration to {g!r}") from e
    return g


def _is_fresh(r, refs):
    """Whether the tensor ``r`` a call returned owns fresh storage.  ``refs``
    counts the references to ``r`` including the caller's own: a cast copies;
    otherwise ``r`` must not be a view and nobody else may hold it."""
    return r.dtype != torch.float64 or (refs <= 1 and r._base is None)


def _call_g(g, t, U, ux, uy):
    """g on device tensors when it accepts them, else on host copies."""
    if getattr(g, "_hb_torch", True):
        try:
            r = g(t, U, ux, uy)
            if torch.is_tensor(r) and r.is_cuda:
                try:
                    g._hb_torch = True
                except AttributeError:
                    pass
                # a tensor nobody else references that is not a view of other
                # storage is g's own fresh result: it may serve as stage-history
                # storage (no copy); anything else (u, u_x, a persistent out=
                # buffer, a view) is copied by the caller
                refs = sys.getrefcount(r) - 1     # alone in a statement: no stack reference
                fresh = _is_fresh(r, refs)
                out = torch.broadcast_to(r.to(torch.float64), U.shape)
                out._hb_fresh = fresh
                return out
        except Exception:
            pass
        try:
            g._hb_torch = False
        except AttributeError:
            pass
    # numpy code: on device arrays whose ufuncs run with torch (npgpu), once it has matched the host call
    if getattr(g, "_hb_npdev", None) is not False and os.environ.get("HPSB_NO_DEVICE_FIELDS") != "1":
        try:
            r = npgpu.plain(g(t, npgpu.wrap(U), npgpu.wrap(ux), npgpu.wrap(uy)))
        except Exception:
            r = None
        ok = r is not None and r.is_cuda == U.is_cuda
        if ok and getattr(g, "_hb_npdev", None) is None:
            h = np.asarray(g(t, U.cpu().numpy(), ux.cpu().numpy(), uy.cpu().numpy()), dtype=float)
            ok = npgpu.matches_host(torch.broadcast_to(r, U.shape), np.broadcast_to(h, U.shape))
        try:
            g._hb_npdev = ok
        except AttributeError:
            pass
        if ok:
            return torch.broadcast_to(r, U.shape).contiguous()
    r = np.asarray(g(t, U.cpu().numpy(), ux.cpu().numpy(), uy.cpu().numpy()), dtype=float)
    return torch.as_tensor(np.broadcast_to(r, U.shape), device=U.device).contiguous()


# ---------------------------------------------------------------------------
# the stepper
# ---------------------------------------------------------------------------

class _CaptureFailed(Exception):
    pass


class _SegmentedGraph:
    """A captured step cut at its host work: graph segments replayed in order
    with each cut's host function (a nonlinear term, a field evaluation, a
    collective) run eagerly in between, on the replaying stream."""

    def __init__(self):
        self.parts = []          # (CUDAGraph, host function or None)

    def replay(self):
        for g, fn in self.parts:
            g.replay()
            if fn is not None:
                fn()


class _Field:
    """Device evaluation of a field callable at a fixed point set."""

    def __init__(self, fn, pts, k, dev):
        self.fn, self.pts, self.k, self.dev = fn, pts, k, dev
        self.n = pts.shape[0]
        self.sep = None
        if fn is None:
            self.zero = torch.zeros((1, self.n), dtype=torch.float64, device=dev)
        elif isinstance(fn, SeparableField):
            self.sep = [self._stack(phi(pts)) for phi, _ in fn.terms]

    def _stack(self, vals):
        a = np.asarray(vals, dtype=float)
        a = a.reshape(self.k, self.n) if (a.ndim > 1 or self.k == 1) else a.reshape(1, self.n)
        return torch.as_tensor(np.ascontiguousarray(a), device=self.dev)

    _pool = None       # host threads for chunked evaluations (shared)
    _pointwise = None  # per field: whether fn(t, pts) evaluates point by point (checked on first use)
    _device_ok = None  # per field: whether fn runs on device arrays and agrees with the host (first use)
    _pts_dev = None

    def device_eval(self, t):
        """fn(t, pts) with the points as a device array whose numpy ufuncs run
        on the GPU (npgpu.DeviceArray), as a (k or 1, n) tensor; None when fn
        leaves the device (an unmapped numpy call, a numpy result) or its first
        device result differs from the host call beyond rounding."""
        if self._device_ok is False or os.environ.get("HPSB_NO_DEVICE_FIELDS") == "1":
            return None
        if self._pts_dev is None:
            self._pts_dev = torch.as_tensor(np.ascontiguousarray(self.pts, dtype=float), device=self.dev)
        try:
            r = npgpu.plain(self.fn(t, npgpu.wrap(self._pts_dev)))
        except Exception:
            r = None
        if r is None or r.numel() not in (self.n, self.k * self.n):
            self._device_ok = False
            return None
        r = r.reshape(self.k, self.n) if (r.ndim > 1 or self.k == 1) else r.reshape(1, self.n)
        if self._device_ok is None:
            h = np.asarray(self.fn(t, self.pts), dtype=float)
            h = h.reshape(self.k, self.n) if (h.ndim > 1 or self.k == 1) else h.reshape(1, self.n)
            self._device_ok = npgpu.matches_host(r, h)
            if not self._device_ok:
                return None
        return r

    def eval_now(self, t):
        """F(t) of a non-separable F as a device tensor: on the device when F
        runs there, else on the host (chunked when pointwise) and copied."""
        v = self.device_eval(t)
        return v if v is not None else self._stack(self.host_eval(t))

    def host_eval(self, t):
        """fn(t, pts) on the host.  A field callable is a function of the
        points; when it is evaluated point by point (checked once: the chunked
        evaluation equals the whole-array call bitwise) large point sets are
        evaluated in chunks on all host cores (numpy releases the GIL), else
        as one call, as the reference does."""
        fn, pts = self.fn, self.pts
        if self._pointwise is False or self.n < (1 << 16) or os.environ.get("HPSB_NO_FIELD_THREADS") == "1":
            return np.asarray(fn(t, pts), dtype=float)
        if _Field._pool is None:
            from concurrent.futures import ThreadPoolExecutor
            _Field._pool = ThreadPoolExecutor(max_workers=max(1, min(32, os.cpu_count() or 1)))
            # a forked child does not inherit the threads: it starts its own pool
            os.register_at_fork(after_in_child=lambda: setattr(_Field, "_pool", None))
        nw = _Field._pool._max_workers
        cuts = [self.n * i // nw for i in range(nw + 1)]
        parts = list(_Field._pool.map(lambda i: np.asarray(fn(t, pts[cuts[i]:cuts[i + 1]]), dtype=float),
                                      range(nw)))
        if any(p.shape[-1:] != (cuts[i + 1] - cuts[i],) for i, p in enumerate(parts)):
            self._pointwise = False
            return np.asarray(fn(t, pts), dtype=float)
        chunked = np.concatenate(parts, axis=-1)
        if self._pointwise is None:
            full = np.asarray(fn(t, pts), dtype=float)
            self._pointwise = full.shape == chunked.shape and np.array_equal(full, chunked)
            return full
        return chunked

    stepper = None     # the TimeStepper whose step may be captured (host evaluations become cuts)

    def _host_value(self, t):
        """F(t) of a non-separable F: evaluated on the host now, or -- while a
        step is captured -- at this point of every replay, with the replayed
        step's time (the captured step is cut here)."""
        st = self.stepper
        if st is not None and st._dry:
            return st._dummy((1, self.n))
        if st is not None and st._seg is not None:
            return st._cut_field(self, t)
        return self.eval_now(t)

    def terms(self, t, scale=1.0):
        """(coef, tensor) terms of scale*F(t); evaluates non-separable F now."""
        if self.fn is None:
            return []
        if self.sep is not None:
            return [(scale * f, phi) for f, phi in zip(self.fn.factors(t), self.sep)]
        return [(scale, self._host_value(t))]

    def values(self, times):
        """(len(times), n) tensor of F at each time in one launch, for a
        separable F of single-row terms (None otherwise: use value)."""
        if self.fn is None or self.sep is None or any(v.shape[0] != 1 for v in self.sep):
            return None
        out = torch.empty((len(times), self.n), dtype=torch.float64, device=self.dev)
        return combine_rows([self.fn.factors(t) for t in times], self.sep, out)

    def value(self, t, out=None):
        """(k or 1, n) tensor of F(t)."""
        if self.fn is None:
            return self.zero
        if self.sep is not None:
            rows = max(v.shape[0] for v in self.sep)
            out = torch.empty((rows, self.n), dtype=torch.float64, device=self.dev) \
                if out is None else out
            return combine(self.terms(t), out)
        return self._host_value(t)


class TimeStepper:
    """Fixed-step IMEX integrator (reference timestep.py:89-328) whose stages
    run on the GPU.  Same constructor, ``set_dt`` / ``shift`` / ``step`` /
    ``run`` / ``initial_state`` and exceptions."""

    def __init__(self, tree, problem, tableau, dt, formulation="stage", disc=None, threads=None,
                 layout=None):
        if formulation not in ("stage", "slope", "slope-penalized"):
            raise UnsupportedConfigurationError(f"unknown formulation {formulation!r}")
        self.tree = tree
        self.problem = problem
        self.pair = tableau if hasattr(tableau, "Ahat") else load_tableau(tableau)
        self.formulation = formulation
        self.penalized = formulation == "slope-penalized"
        self.disc = disc or EllipticDiscretization(tree, problem.coeffs)
        self.threads = threads
        self.layout = layout
        self._step_count = 0
        if formulation != "stage":
            if not problem.is_linear and not problem.time_independent_bc:
                raise UnsupportedConfigurationError(
                    "slope formulation with a nonlinear term requires time-independent boundary "
                    "data (slope variables have no boundary interpretation otherwise)")
            if (problem.is_linear and not problem.time_independent_bc
                    and problem.f is not None and problem.f_t is None):
                raise UnsupportedConfigurationError(
                    "slope formulation with time-dependent boundary data requires f_t")
        if not problem.is_linear and self.pair.Ahat is None and self.pair.s > 1:
            raise UnsupportedConfigurationError(
                f"tableau {self.pair.name} has no explicit half for g")
        self._bnd_pts = tree.points[tree.boundary_ids]
        self._all_pts = tree.points
        self._dev = cuda_device()
        self._dd = device_discretization(self.disc)
        self._plan = device_plan(tree)
        k = problem.ncomp
        self._k = k
        self._F = _Field(problem.f, self._bnd_pts, k, self._dev)
        self._bc_batch = os.environ.get("HPSB_NO_BC_BATCH") != "1"
        self._Ft = _Field(None if problem.time_independent_bc else problem.f_t, self._bnd_pts, k,
                          self._dev)
        self._Q = _Field(problem.q, self._all_pts, k, self._dev)
        for F in (self._F, self._Ft, self._Q):
            F.stepper = self
        self._bufs = {}
        self._seg = None           # while a step is captured: the graph segments (see _eager)
        self._replay_t = 0.0       # time of the step being replayed (host work at the cuts)
        self._cut_bufs = []
        # the leaf-interior DOF range this process steps (everything on one GPU;
        # a subtree part range in sharding.ShardedTimeStepper)
        self._ir = (0, self._dd.Lni)
        self._nloc = self._dd.Lni
        self._dry = False          # dry pass: record combination coefficients only
        self._graph = None         # captured CUDA graph of one step (see _run_graph)
        self._graph_failed = False
        self.solve_timer = None
        self.dt = None
        self.ops = None
        self.ops_id = None
        self.set_dt(dt)

    # -- operator cache ------------------------------------------------------------------
    @property
    def shift(self):
        return self.dt * self.pair.gamma

    def set_dt(self, dt):
        """Set the step size, rebuilding the cached operator set (timestep.py:142-157)."""
        if dt <= 0:
            raise ValueError(f"dt must be positive, got {dt}")
        if self.dt == dt and self.ops is not None:
            return
        self.dt = float(dt)
        self.ops = HpsOperatorSet(self.disc, sigma=1.0, dt_gamma=self.dt * self.pair.gamma,
                                  threads=self.threads, layout=self.layout,
                                  nparts=getattr(self, "_nparts", 1))
        if self.formulation != "stage" and self.ops_id is None:
            self.ops_id = HpsOperatorSet(self.disc, sigma=1.0, dt_gamma=0.0, threads=self.threads,
                                         layout=self.layout)

    def _check_ops(self):
        if self.ops is None or self.ops.dt_gamma != self.dt * self.pair.gamma \
                or self.ops.sigma != 1.0:
            raise UnsupportedConfigurationError(
                "cached operator set does not match dt*gamma; call set_dt")

    # -- device buffers ------------------------------------------------------------------
    def _buf(self, name, shape):
        b = self._bufs.get(name)
        if b is None or tuple(b.shape) != tuple(shape):
            b = torch.empty(shape, dtype=torch.float64, device=self._dev)
            self._bufs[name] = b
        return b

    def _bc(self, t):
        return self._F.value(t)

    def _bc_t(self, t):
        return self._Ft.value(t)

    def _g(self, t, U, out=None):
        """g(t, U) with the interface-averaged device gradient (timestep.py:192-196).
        The gradient is always evaluated, as the reference does, unless g
        declares that it reads neither component (:func:`declare_nonlinear`).
        While a step is captured, a g not declared pure is cut out of the graph:
        it runs at every replay with that step's stage time, into ``out`` (or a
        buffer of its own)."""
        if self.problem.g is None:
            return None
        ux, uy = self._buf("gx", U.shape), self._buf("gy", U.shape)
        if self._dry:
            return ux if out is None else out
        g = self.problem.g
        if any(gradient_use(g)):  # both components: one pass of the gradient kernel
            self._dd.eval(U, ux=ux, uy=uy)
        if self._seg is not None and not is_pure(g):
            tgt = out if out is not None else self._cut_buf(tuple(U.shape))
            self._eager(lambda tc=t: tgt.copy_(_call_g(g, self._replay_t + tc, U, ux, uy)))
            return tgt
        r = _call_g(g, t, U, ux, uy)
        if out is not None:
            out.copy_(r)
            return out
        return r

    # -- host work inside a captured step: the graph is cut there ------------------------
    def _eager(self, fn):
        """Run ``fn`` now; while a step is being captured, cut the graph here
        and run ``fn`` at this point of every replay instead."""
        if self._seg is None:
            fn()
        else:
            self._seg_end(fn)
            self._seg_begin()

    def _cut_buf(self, shape):
        """A persistent buffer for the result of one cut (allocated from the
        capture's pool; lives as long as the stepper)."""
        b = torch.empty(shape, dtype=torch.float64, device=self._dev)
        self._cut_bufs.append(b)
        return b

    def _cut_field(self, F, t):
        a = np.asarray(F.fn(t, F.pts), dtype=float)      # shape only (host)
        rows = F.k if (a.ndim > 1 or F.k == 1) else 1
        tgt = self._cut_buf((rows, F.n))
        self._eager(lambda tc=t: tgt.copy_(F.eval_now(self._replay_t + tc)))
        return tgt

    def _dummy(self, shape):
        return self._buf("dummy%dx%d" % shape, shape)

    def initial_state(self):
        u0 = np.asarray(self.problem.u0(self._all_pts), dtype=float)
        k, N = self._k, self.tree.N
        u0 = u0.reshape(k, N) if (u0.ndim > 1 or k == 1) else np.broadcast_to(u0, (k, N))
        return StepperState(0.0, u0 if k > 1 else u0[0])

    # -- stepping ------------------------------------------------------------------------
    def step(self, state):
        """Advance one step of size dt, returning a new state (timestep.py:211-224)."""
        if self._graph_eligible():
            try:
                return self._run_graph(state, 1, check_every=1)
            except _CaptureFailed:
                pass
        new, guards = self._advance(state)
        self._raise_if_diverged(self._reduce_guards(guards), self._step_count)
        self._step_count += 1
        return new

    def run(self, state, nsteps, check_every=32):
        """``nsteps`` steps; the divergence guard is read back once per
        ``check_every`` steps (the first failing step is reported exactly)."""
        g = self.problem.g
        if nsteps > 1 and g is not None and is_pure(g) and getattr(g, "_hb_torch", None) is None and \
                self._graph_eligible(probe=True):
            state = self.step(state)           # one eager step probes g on device tensors
            nsteps -= 1
        if nsteps > 0 and self._graph_eligible():
            try:
                return self._run_graph(state, nsteps, check_every)
            except _CaptureFailed:
                pass
        pending = []
        for _ in range(nsteps):
            state, guards = self._advance(state)
            pending.append(guards)
            if len(pending) >= check_every:
                self._drain(pending)
        self._drain(pending)
        return state

    # -- CUDA-graph stepping -------------------------------------------------------------
    def _graph_eligible(self, probe=False):
        """One step is captured once and replayed for the stage formulation and
        BE.  Field callables other than SeparableField and a g not declared
        pure run on the host / eagerly at cuts of the captured step; a g
        declared pure is captured and must run on device tensors (probed by an
        eager step)."""
        if os.environ.get("HPSB_NO_GRAPH") == "1" or self.solve_timer is not None or self._graph_failed:
            return False
        if self.pair.s > 1 and self.formulation != "stage":
            return False
        g = self.problem.g
        return g is None or not is_pure(g) or probe or getattr(g, "_hb_torch", None) is True

    def _step_body(self, t, u, guards, out):
        if self.pair.s == 1:
            return self._step_backward_euler(t, u, guards, out=out)
        return self._step_stage(t, u, guards, out=out)

    def _dry_coefs(self, t, u, guards):
        self._dry, _CoefSink.current = True, _CoefSink(dry=True)
        try:
            self._step_body(t, u, guards, u)
            return _CoefSink.current.vals
        finally:
            self._dry, _CoefSink.current = False, None

    def _capture(self, t, gin):
        s, dev = self.pair.s, self._dev
        guards = torch.zeros(s, dtype=torch.float64, device=dev)
        vals = self._dry_coefs(t, gin, guards)
        coef = torch.zeros(len(vals) + 8, dtype=torch.float64, device=dev)
        coef[:len(vals)] = torch.as_tensor(vals, dtype=torch.float64)
        # warm the captured code path once (kernel attributes, workspaces) on scratch
        # data; the warm pass and the capture use this stepper's graph workspaces
        # (allocated here, outside the capture)
        scratch = gin.clone()
        with graph_workspace(id(self)):
            _CoefSink.current = _CoefSink(dev=coef)
            try:
                self._step_body(t, scratch, guards, scratch)
            finally:
                _CoefSink.current = None
            torch.cuda.synchronize()

            def body():
                # captured at t = 0: the time enters only through the coefficient
                # table (recomputed per replay) and the cuts, which evaluate at
                # replay time t_step + (stage offset), the reference's t + c_i dt
                _CoefSink.current = _CoefSink(dev=coef)
                try:
                    guards.zero_()
                    self._step_body(0.0, gin, guards, gin)
                finally:
                    _CoefSink.current = None

            # a finalizer that frees device memory (an operator set or plan collected
            # by the GC) would invalidate the capture: collect now, none during it
            gc.collect()
            gc.disable()
            try:
                graph = self._capture_graph(body)
            finally:
                gc.enable()
        ring = 4
        self._graph = dict(graph=graph, gin=gin, guards=guards, coef=coef, ncoef=len(vals), key=self._graph_key(gin),
                           pinned=[torch.zeros(len(vals) + 8, dtype=torch.float64).pin_memory() for _ in range(ring)],
                           events=[None] * ring, slot=0)

    def _capture_graph(self, body):
        """``body`` captured as CUDA-graph segments cut at its host work
        (``_eager``: a nonlinear term not declared pure, a field callable, a
        collective); returns an object whose ``replay()`` replays the segments
        in order with the host work in between."""
        seg = _SegmentedGraph()
        stream = torch.cuda.Stream()
        stream.wait_stream(torch.cuda.current_stream())
        self._seg = dict(graph=seg, pool=torch.cuda.graph_pool_handle(), cur=None)
        try:
            with torch.cuda.stream(stream):
                self._seg_begin()
                body()
                self._seg_end(None)
        except Exception:
            cur = self._seg["cur"]
            if cur is not None:
                try:
                    cur.capture_end()
                except Exception:
                    pass
            raise
        finally:
            self._seg = None
            torch.cuda.current_stream().wait_stream(stream)
        return seg

    def _seg_begin(self):
        g = torch.cuda.CUDAGraph()
        g.capture_begin(pool=self._seg["pool"])
        self._seg["cur"] = g

    def _seg_end(self, fn):
        g = self._seg["cur"]
        self._seg["cur"] = None
        g.capture_end()
        self._seg["graph"].parts.append((g, fn))

    def _graph_key(self, u):
        return (tuple(u.shape), self.dt, id(self.ops))

    def _run_graph(self, state, nsteps, check_every):
        self._check_ops()
        src = state.u_device
        squeeze = src.dim() == 1
        src = torch.atleast_2d(src).to(torch.float64)
        G = self._graph
        if G is None or G["key"] != self._graph_key(src):
            self._graph = None
            try:
                self._capture(state.t, src.clone())
            except Exception as e:  # e.g. an op in g that cannot be captured
                self._graph, self._graph_failed = None, True
                torch.cuda.synchronize()
                raise _CaptureFailed(str(e)) from e
            G = self._graph
        gin, guards, coef = G["gin"], G["guards"], G["coef"]
        if src.data_ptr() != gin.data_ptr():
            gin.copy_(src)
        hist = torch.empty((max(1, min(check_every, nsteps)), guards.numel()), dtype=torch.float64,
                           device=self._dev)
        t = state.t
        done = 0
        for step in range(nsteps):
            vals = self._dry_coefs(t, gin, guards)
            if len(vals) != G["ncoef"]:
                raise HpstepError("captured step and coefficient pass disagree")
            slot = G["slot"]
            G["slot"] = (slot + 1) % len(G["pinned"])
            if G["events"][slot] is not None:
                G["events"][slot].synchronize()      # the copy that last read this buffer is done
            buf = G["pinned"][slot]
            buf[:len(vals)] = torch.as_tensor(vals, dtype=torch.float64)
            coef.copy_(buf, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record()
            G["events"][slot] = ev
            self._replay_t = t
            G["graph"].replay()
            hist[(step - done) % hist.shape[0]].copy_(guards)
            t += self.dt
            if step + 1 - done == hist.shape[0] or step + 1 == nsteps:
                host = self._reduce_guards(hist[:step + 1 - done]).cpu().numpy()
                for g in host:
                    self._raise_if_diverged(g, self._step_count, host_vals=True)
                    self._step_count += 1
                done = step + 1
        u = gin.clone()
        return StepperState(t, u[0] if squeeze else u)

    # -- host-resident states: copies overlapped with the neighbouring steps ---------------
    def step_host(self, t, u_in, u_out, check_every=32):
        """One step of the host state ``u_in`` at time ``t`` into the host
        tensor ``u_out`` (both pinned for asynchrony), enqueued without host
        synchronisation: the input copy runs on a copy stream, the step (one
        CUDA-graph replay) on the current stream, the result copy on a second
        copy stream, ordered by events -- so consecutive calls on independent
        states overlap one call's copies with the neighbouring calls' compute.
        Returns the event that completes the result copy.  The divergence guard
        is checked every ``check_every`` calls and by ``sync_host()``."""
        uin = torch.atleast_2d(u_in)
        uout = torch.atleast_2d(u_out)
        if not self._graph_eligible():
            s = self.step(StepperState(t, u_in))
            uout.copy_(torch.atleast_2d(s.u_device))
            ev = torch.cuda.Event()
            ev.record()
            return ev
        # two device buffers, each with its own captured step that runs in place
        # on it: the input is copied straight into the buffer and the result
        # straight out of it (no device-side copies on the compute stream)
        io = getattr(self, "_io", None)
        key = self._graph_key(uin)
        if io is None or io["key"] != key:
            dev = self._dev
            io = self._io = dict(key=key, h2d=torch.cuda.Stream(), d2h=torch.cuda.Stream(),
                                 buf=[torch.zeros(uin.shape, dtype=torch.float64, device=dev) for _ in range(2)],
                                 G=[None, None], free=[None, None], slot=0, pending=[])
            saved = self._graph
            try:
                for b in range(2):
                    self._capture(t, io["buf"][b])
                    io["G"][b] = self._graph
            except Exception:  # e.g. an op in g that cannot be captured: step eagerly from now on
                self._graph_failed, self._io = True, None
                torch.cuda.synchronize()
                return self.step_host(t, u_in, u_out, check_every)
            finally:
                self._graph = saved
        cs = torch.cuda.current_stream()
        slot = io["slot"]
        io["slot"] ^= 1
        G, buf = io["G"][slot], io["buf"][slot]
        with torch.cuda.stream(io["h2d"]):
            if io["free"][slot] is not None:
                io["h2d"].wait_event(io["free"][slot])   # the result copy that last read this buffer
            buf.copy_(uin, non_blocking=True)
            ev_in = torch.cuda.Event()
            ev_in.record(io["h2d"])
        cs.wait_event(ev_in)
        guards, coef = G["guards"], G["coef"]
        vals = self._dry_coefs(t, buf, guards)
        if len(vals) != G["ncoef"]:
            raise HpstepError("captured step and coefficient pass disagree")
        cslot = G["slot"]
        G["slot"] = (cslot + 1) % len(G["pinned"])
        if G["events"][cslot] is not None:
            G["events"][cslot].synchronize()
        pin = G["pinned"][cslot]
        pin[:len(vals)] = torch.as_tensor(vals, dtype=torch.float64)
        coef.copy_(pin, non_blocking=True)
        ev = torch.cuda.Event()
        ev.record()
        G["events"][cslot] = ev
        self._replay_t = t
        G["graph"].replay()
        io["pending"].append(guards.clone())
        done = torch.cuda.Event()
        done.record(cs)
        with torch.cuda.stream(io["d2h"]):
            io["d2h"].wait_event(done)
            uout.copy_(buf, non_blocking=True)
            ev_out = torch.cuda.Event()
            ev_out.record(io["d2h"])
        io["free"][slot] = ev_out
        if len(io["pending"]) >= check_every:
            self.sync_host()
        return ev_out

    def sync_host(self):
        """Wait for every ``step_host`` call and check their divergence guards."""
        io = getattr(self, "_io", None)
        if io is None:
            return
        torch.cuda.current_stream().synchronize()
        io["h2d"].synchronize()
        io["d2h"].synchronize()
        self._drain(io["pending"])

    def _drain(self, pending):
        if not pending:
            return
        host = self._reduce_guards(torch.stack(pending)).cpu().numpy()
        for g in host:
            self._raise_if_diverged(g, self._step_count, host_vals=True)
            self._step_count += 1
        pending.clear()

    def _raise_if_diverged(self, guards, step, host_vals=False):
        """guards = [stage maxima..., final max]; a stage failure reports the
        step count before the increment, the final one after (timestep.py:219-222)."""
        g = guards if host_vals else guards.cpu().numpy()
        for i, mx in enumerate(g):
            if not np.isfinite(mx) or mx > DIVERGENCE_LIMIT:
                final = i == len(g) - 1
                n = step + 1 if final else step
                raise DivergenceError(f"solution diverged at step {n} (max|u| = {mx:.3e})", step=n)

    def _advance(self, state):
        self._check_ops()
        squeeze = (state.u_device.dim() == 1)
        u = torch.atleast_2d(state.u_device)
        if u.dtype != torch.float64:
            u = u.to(torch.float64)
        u = u.contiguous()
        s = self.pair.s
        guards = torch.zeros(s, dtype=torch.float64, device=self._dev)
        if s == 1:
            unew = self._step_backward_euler(state.t, u, guards)
        elif self.formulation == "stage":
            unew = self._step_stage(state.t, u, guards)
        else:
            unew = self._step_slope(state.t, u, guards)
        return StepperState(state.t + self.dt, unew[0] if squeeze else unew), guards

    # device work of a step, skipped on a dry pass
    def _eval(self, U, **kw):
        if not self._dry:
            self._dd.eval(U, **kw)

    # -- hooks over the DOFs this process owns (sharding.ShardedTimeStepper) ------------
    def _iv(self, v):
        """View of a full (rows, N) vector starting at this process's first
        leaf-interior DOF (what combines over the local interior range read)."""
        a = self._ir[0]
        return v if a == 0 else v[:, a:]

    def _fused_stage_terms(self, fb, terms, r, out, lu, guard, root_pre):
        """hps_solve_stage_terms(_k) when the stage's combination fits it (at
        most 12 terms of one row or k rows, the whole tree); False otherwise."""
        k = self._k
        if not (0 < len(terms) <= 12 and self.ops.fuses_stage_history and
                self.solve_timer is None and self._ir[0] == 0 and
                os.environ.get("HPSB_NO_STAGE_TERMS") != "1"):
            return False
        if any(v.shape[0] not in (1, k) for _, v in terms) or (k > 1 and root_pre is not None):
            return False
        dptr = self._coef_ptr([c for c, _ in terms])
        if not self._dry:
            if k == 1:
                self.ops.solve_stage_terms_device(fb, dptr, [v for _, v in terms], r, out, lu, guard, root_pre)
            else:
                self.ops.solve_stage_terms_k_device(fb, dptr, [v for _, v in terms], r, out, lu, guard)
        return True

    def _coef_ptr(self, vals):
        """Device address of ``vals`` (float64): a slot range of the captured
        step's coefficient table, or a fresh device array when stepping eagerly
        (kept alive until the next step)."""
        sink = _CoefSink.current
        if sink is not None:
            return sink.take([float(v) for v in vals])
        t = torch.tensor([float(v) for v in vals], dtype=torch.float64, device=self._dev)
        keep = getattr(self, "_coef_keep", None)
        if keep is None or keep[0] is not self._step_token:
            keep = self._coef_keep = (self._step_token, [])
        keep[1].append(t)
        return t.data_ptr()

    def _final_combine(self, terms, fb, unew, guard):
        """unew = the final combination, its boundary DOFs set to f(t + dt), and
        the step's guard (timestep.py:263-266): one fused pass."""
        if os.environ.get("HPSB_NO_COMBINE_BND") == "1":
            self._owned_combine(terms, unew)
            self._put_boundary(fb, unew)
            self._owned_maxabs(unew, guard)
            return
        combine_bnd(self._plan, terms, fb, unew, guard)

    def _qg_alias_ok(self):
        """Whether g's result may serve as the QG history entry itself (one
        process: every DOF of it is owned)."""
        return True

    def _root_batch(self):
        return self.ops.fuses_stage_history and self.ops.root_dirichlet_ok and self.solve_timer is None

    def _root_sep_products(self):
        """Rows S_root F_m of a separable f = sum_m tau_m(t) F_m(x) (single-row
        terms, at most 8), cached on the operator set; None when f is not
        separable or HPSB_NO_ROOT_SEP=1.  Computed by the first pass that needs
        them (the coefficient pass that precedes every capture included); never
        launched inside a capture."""
        if os.environ.get("HPSB_NO_ROOT_SEP") == "1":
            return None
        F = self._F
        if F.fn is None or F.sep is None or not (1 <= len(F.sep) <= 8) or any(v.shape[0] != 1 for v in F.sep):
            return None
        cache = getattr(self.ops, "_root_sep", None)
        if cache is not None and cache[0] is F:
            return cache[1]
        if torch.cuda.is_current_stream_capturing():
            return None
        rows = torch.cat(list(F.sep), dim=0).contiguous()
        P = torch.empty((rows.shape[0], self.tree.level_maps[0].n3), dtype=torch.float64, device=self._dev)
        self.ops.root_dirichlet_device(rows, P)
        P = [P[m:m + 1] for m in range(rows.shape[0])]
        self.ops._root_sep = (F, P)
        return P

    def _fused_stage(self, fb, body, out, lu, guard, root_pre=None):
        """Stage solve with the history L u and the guard from the leaf kernel
        of the downward sweep (hps_solve_stage); False when not available."""
        if not self.ops.fuses_stage_history or self.solve_timer is not None:
            return False
        if not self._dry:
            self.ops.solve_stage_device(fb, body, out, lu, guard, root_pre=root_pre)
        return True

    def _eval_lu(self, U, out, guard=None):
        """Stage history L u at the local leaf interiors: the leaf-grid DMMA
        products of the fused stage when the operator set has them, else the
        general leaf evaluation."""
        if self.ops.fuses_stage_history and os.environ.get("HPSB_NO_FD_LU") != "1":
            if not self._dry:
                self.ops.leaf_lu_device(U, out, guard)
            return
        self._eval(U, lu_int=out, guard=guard)

    def _owned_combine(self, terms, out):
        """out = sum c v over every DOF this process owns."""
        combine(terms, out)

    def _owned_maxabs(self, x, guard):
        self._maxabs(x, guard)

    def _reduce_guards(self, g):
        """Guard maxima over every process (identity on one GPU)."""
        return g

    def _maxabs(self, x, guard):
        if not self._dry:
            k, n = x.shape
            _lib.check(_lib.load().hps_maxabs(k, n, x.data_ptr(), x.stride(0), guard.data_ptr(),
                                              current_stream_handle()), "hps_maxabs")

    def _put_boundary(self, fb, u):
        if not self._dry:
            _lib.check(_lib.load().hps_put_boundary(self._plan.handle, u.shape[0], fb.data_ptr(),
                                                    0 if fb.shape[0] == 1 else fb.stride(0),
                                                    u.data_ptr(), u.stride(0), current_stream_handle()),
                       "hps_put_boundary")

    def _solve(self, ops, fb, body, out, jump=None, inv_dt=None):
        if self._dry:
            return out
        tm = self.solve_timer
        if tm is not None:                      # bench hook: CUDA events around each solve
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
        ops.solve_device(fb, body, out, jump=jump, inv_dt=inv_dt)
        if tm is not None:
            e1.record()
            tm.append((e0, e1))
        return out

    def _step_backward_euler(self, t, u, guards, out=None):
        dt, k, N = self.dt, u.shape[0], self.tree.N
        t1 = t + dt
        iv = self._iv
        r = self._buf("r", (k, self._nloc))
        terms = [(1.0, iv(u))] + [(c, iv(v)) for c, v in self._Q.terms(t1, dt)]
        G = self._g(t, u)
        if G is not None:
            terms.append((dt, iv(G)))
        combine(terms, r, n=self._nloc)
        unew = torch.empty((k, N), dtype=torch.float64, device=self._dev) if out is None else out
        self._solve(self.ops, self._bc(t1), r, unew)
        self._owned_maxabs(unew, guards[0])
        return unew

    def _step_stage(self, t, u, guards, out=None):
        """timestep.py:237-266 on the device."""
        pair, dt = self.pair, self.dt
        s, k, N, Lni = pair.s, u.shape[0], self.tree.N, self._nloc
        A, Ah = pair.A, pair.Ahat
        iv = self._iv
        self._step_token = object()          # eager coefficient arrays live until the next step
        Lu = self._buf("Lu", (s, k, Lni))
        nonlin = self.problem.g is not None
        QG = self._buf("QG", (s, k, N)) if (nonlin or (self._Q.fn is not None and self._Q.sep is None)) \
            else None
        QGl = [None] * s                     # the history entries (QG rows, or g's own result tensors)
        qsep = self._Q.sep
        qfac = []                                    # per stage: separable q time factors
        r = self._buf("r", (k, Lni))
        U = [self._buf("u0", (k, N)), self._buf("u1", (k, N))]

        def stage_q_g(i, ti, ui):
            if qsep is not None:
                qfac.append(self._Q.fn.factors(ti))
            if QG is None:
                return
            terms = [] if qsep is not None else self._Q.terms(ti)
            # g alone: written straight into the history row when it runs at a
            # cut of the captured step; otherwise its own fresh result may serve
            # as the row (no copy) -- storage g reuses (u, u_x, an out= buffer)
            # is overwritten by later stages and is copied
            g = self.problem.g
            cut = self._seg is not None and g is not None and not is_pure(g)   # g runs at a graph cut
            G = self._g(ti, ui, out=QG[i] if not terms and cut else None)
            if G is not None:
                terms.append((1.0, G))
            if len(terms) == 1 and terms[0][0] == 1.0 and G is not None:
                if G is QG[i]:
                    QGl[i] = G
                elif self._qg_alias_ok() and getattr(G, "_hb_fresh", False) and G.shape == QG[i].shape \
                        and G.is_contiguous():
                    QGl[i] = G
                else:
                    QGl[i] = QG[i]
                    if not self._dry:
                        QG[i].copy_(G)
            elif terms:
                QGl[i] = QG[i]
                self._owned_combine(terms, QG[i])
            else:
                QGl[i] = QG[i]
                if not self._dry:
                    QG[i].zero_()

        # boundary data of stages 1..s-1 and of t + dt, one launch when f is separable
        bcs = self._F.values([t + pair.c[i] * dt for i in range(1, s)] + [t + dt]) \
            if self._bc_batch else None
        bc_at = lambda i, ti: self._bc(ti) if bcs is None else bcs[i - 1:i]
        # the root's Dirichlet product of every stage solve in one pass over the
        # root operator (k = 1; the fused stage solves then skip it)
        rpre = None
        if bcs is not None and k == 1 and s > 1 and self._root_batch():
            rpre = self._buf("rootpre", (s - 1, self.tree.level_maps[0].n3))
            P = self._root_sep_products()
            if P is not None:
                # separable boundary data: S_root f(t_i) = sum_m tau_m(t_i) (S_root F_m), the
                # products S_root F_m computed once per operator set -- no pass over the
                # root operator per step
                combine_rows([self._F.fn.factors(t + pair.c[i] * dt) for i in range(1, s)], P, rpre)
            elif not self._dry:
                self.ops.root_dirichlet_device(bcs[:s - 1], rpre)
        self._eval_lu(u, Lu[0])
        stage_q_g(0, t + pair.c[0] * dt, u)
        ui = u
        for i in range(1, s):
            ti = t + pair.c[i] * dt
            terms = [(1.0, iv(u))]
            terms += [(dt * A[i, j], Lu[j]) for j in range(i)]
            if QG is not None:
                terms += [(dt * Ah[i, j], iv(QGl[j])) for j in range(i)]
            if qsep is not None:
                for m, phi in enumerate(qsep):
                    terms.append((sum(dt * Ah[i, j] * qfac[j][m] for j in range(i)), iv(phi)))
            ui = U[i & 1]
            bc = bc_at(i, ti)
            rp = None if rpre is None else rpre[i - 1:i]
            # the combination formed by the solve's leaf kernel; solve + history L u_i (not
            # needed after the last stage) + guard in one pass
            if self._fused_stage_terms(bc, terms, r, ui, Lu[i] if i < s - 1 else None, guards[i - 1], rp):
                stage_q_g(i, ti, ui)
                continue
            combine(terms, r, n=Lni)
            if not self._fused_stage(bc, r, ui, Lu[i] if i < s - 1 else None, guards[i - 1], rp):
                self._solve(self.ops, bc, r, ui)
                if i < s - 1:
                    self._eval_lu(ui, Lu[i], guard=guards[i - 1])
                else:
                    self._owned_maxabs(ui, guards[i - 1])
            stage_q_g(i, ti, ui)
        w = pair.bhat - Ah[s - 1]
        terms = [(1.0, ui)]
        if QG is not None:
            terms += [(dt * w[j], QGl[j]) for j in range(s)]
        if qsep is not None:
            for m, phi in enumerate(qsep):
                terms.append((sum(dt * w[j] * qfac[j][m] for j in range(s)), phi))
        # `out` may alias `u`: nothing below reads u
        unew = torch.empty((k, N), dtype=torch.float64, device=self._dev) if out is None else out
        self._final_combine(terms, bc_at(s, t + dt), unew, guards[s - 1])
        return unew

    # -- slope formulations (timestep.py:268-328) ----------------------------------------
    def _slope_assign(self, bc, body, jump, out):
        if jump is not None:
            return self._solve(self.ops_id, bc, body, out, jump=jump, inv_dt=1.0 / self.dt)
        return self._solve(self.ops_id, bc, body, out)

    def _step_slope(self, t, u, guards):
        pair, dt = self.pair, self.dt
        s, k, N, Lni = pair.s, u.shape[0], self.tree.N, self._dd.Lni
        A, Ah = pair.A, pair.Ahat
        nonlinear = not self.problem.is_linear
        dev = self._dev
        jump = None
        if self.penalized:
            jump = self._buf("jump", (k, N))
            self._dd.eval(u, jump=jump)
        Lun = self._buf("Lun", (k, Lni))
        self._dd.eval(u, lu_int=Lun)
        K = torch.empty((s, k, N), dtype=torch.float64, device=dev)
        LK = self._buf("LK", (s, k, Lni))
        r = self._buf("r", (k, Lni))
        zero_bc = torch.zeros((1, self._bnd_pts.shape[0]), dtype=torch.float64, device=dev)
        t0 = t + pair.c[0] * dt
        combine([(1.0, Lun)] + self._Q.terms(t0), r, n=Lni)
        self._slope_assign(self._bc_t(t0), r, jump, K[0])
        self._dd.eval(K[0], lu_int=LK[0])
        if nonlinear:
            Lv = torch.empty((s, k, N), dtype=torch.float64, device=dev)
            Ls = self._buf("Ls", (s, k, Lni))
            gb = self._buf("gbody", (k, N))
            self._g(t0, u, out=gb)
            self._slope_assign(zero_bc, gb, None, Lv[0])
            self._dd.eval(Lv[0], lu_int=Ls[0])
        for i in range(1, s):
            ti = t + pair.c[i] * dt
            terms = [(1.0, Lun)] + [(dt * A[i, j], LK[j]) for j in range(i)] + self._Q.terms(ti)
            if nonlinear:
                terms += [(dt * Ah[i, j], Ls[j]) for j in range(i)]
            combine(terms, r, n=Lni)
            if self.penalized:
                self._solve(self.ops, self._bc_t(ti), r, K[i], jump=jump, inv_dt=1.0 / dt)
            else:
                self._solve(self.ops, self._bc_t(ti), r, K[i])
            need_lk = i < s - 1 or nonlinear
            if need_lk:
                self._dd.eval(K[i], lu_int=LK[i], guard=guards[i - 1])
            else:
                _lib.check(_lib.load().hps_maxabs(k, N, K[i].data_ptr(), N,
                                                  guards[i - 1].data_ptr(),
                                                  current_stream_handle()), "hps_maxabs")
            if nonlinear:
                v = self._buf("v", (k, N))
                combine([(1.0, u)] + [(dt * A[i, j], K[j]) for j in range(i + 1)]
                        + [(dt * Ah[i, j], Lv[j]) for j in range(i)], v)
                self._g(ti, v, out=gb)
                self._slope_assign(zero_bc, gb, None, Lv[i])
                self._dd.eval(Lv[i], lu_int=Ls[i])
        terms = [(1.0, u)] + [(dt * pair.b[j], K[j]) for j in range(s)]
        if nonlinear:
            terms += [(dt * pair.bhat[j], Lv[j]) for j in range(s)]
        unew = torch.empty((k, N), dtype=torch.float64, device=dev)
        combine(terms, unew)
        _lib.check(_lib.load().hps_maxabs(k, N, unew.data_ptr(), N, guards[s - 1].data_ptr(),
                                          current_stream_handle()), "hps_maxabs")
        return unew


def scalar_stability_function(pair, z):
    """Amplification factor of the implicit half on u' = lambda*u."""
    return pair.stability_function(z)
