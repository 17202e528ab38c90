"""Operator coefficients and the per-leaf collocation stencil (host setup).

Convention (reference operators.py:1-16): coefficients hold the elliptic form

    A u = -c11 u_xx - c22 u_yy + c1 u_x + c2 u_y + c u,    L = -A.

Only O(p^4) stencil constants and the coefficient samples are produced here
on the host; the dense leaf blocks, their inverses and every apply happen on
the device (``solver.py``, ``timestep.py``).
"""

import numpy as np

from .chebyshev import cgl_weights, derivative_matrices
from .errors import HpstepError

FIELDS = ("c11", "c22", "c1", "c2", "c")


def _field(v):
    if v is None or callable(v):
        return v
    return float(v)


class OperatorCoefficients:
    """Coefficient fields of ``A``: each a constant, ``None`` or a vectorized
    callable ``f(x, y)`` (reference operators.py:34-100)."""

    def __init__(self, c11, c22=None, c1=None, c2=None, c=None, dim=2):
        self.dim = dim
        self.c11, self.c22 = _field(c11), _field(c22)
        self.c1, self.c2, self.c = _field(c1), _field(c2), _field(c)
        if dim == 1 and (self.c22 is not None or self.c2 is not None):
            raise ValueError("c22/c2 are meaningless for 1D operators")

    @property
    def fields(self):
        return {"c11": self.c11, "c22": self.c22, "c1": self.c1, "c2": self.c2, "c": self.c}

    @property
    def is_constant(self):
        return not any(callable(v) for v in self.fields.values())

    def evaluate(self, points):
        pts = np.atleast_2d(np.asarray(points, dtype=float))
        n = pts.shape[0]
        out = {}
        for k, v in self.fields.items():
            if v is None:
                out[k] = np.zeros(n)
            elif callable(v):
                out[k] = np.broadcast_to(np.asarray(v(*pts.T), dtype=float), (n,)).copy()
            else:
                out[k] = np.full(n, v)
        return out

    def check_ellipticity(self, points):
        vals = self.evaluate(points)
        bad = (vals["c11"] <= 0) | (vals["c22"] <= 0)
        if np.any(bad):
            raise HpstepError(f"operator is not elliptic at {int(bad.sum())} of {bad.size} "
                              "sample points (c11/c22 must be positive)")

    def negated(self):
        def neg(v):
            if v is None:
                return None
            if callable(v):
                return lambda *xy, _f=v: -np.asarray(_f(*xy), dtype=float)
            return -v
        return OperatorCoefficients(c11=neg(self.c11), c22=neg(self.c22), c1=neg(self.c1),
                                    c2=neg(self.c2), c=neg(self.c), dim=self.dim)


class LeafStencil:
    """Grid-only matrices of one leaf in local (interior, edge) order.

    Built from the 1D CGL matrices by index arithmetic: the tensor operator
    ``D1x = kron(d1x, I)`` restricted to the local point set is
    ``d1x[xi, xi'] * [yi == yi']`` (reference operators.py:129-216).
    """

    def __init__(self, tree):
        p = self.p = tree.p
        self.dim = 2
        self.ni, self.nb = tree.ni, tree.nb
        self.m = self.ni + self.nb
        gx, gy = tree.leaf_gx.nodes, tree.leaf_gy.nodes
        w = cgl_weights(p)
        self.d1x, self.d2x = derivative_matrices(gx, w)
        self.d1y, self.d2y = derivative_matrices(gy, w)
        # local point coordinates: interior (x-major), then edges in tensor order
        xi, yi = np.divmod(np.arange(p * p), p)
        inner = (xi % (p - 1) != 0) & (yi % (p - 1) != 0)
        corner = (xi % (p - 1) == 0) & (yi % (p - 1) == 0)
        order = np.concatenate([np.nonzero(inner)[0], np.nonzero(~inner & ~corner)[0]])
        self.xi, self.yi = xi[order], yi[order]
        X, Y = self.xi, self.yi
        same_y = (Y[:, None] == Y[None, :])
        same_x = (X[:, None] == X[None, :])
        self.D1x = np.where(same_y, self.d1x[X[:, None], X[None, :]], 0.0)
        self.D2x = np.where(same_y, self.d2x[X[:, None], X[None, :]], 0.0)
        self.D1y = np.where(same_x, self.d1y[Y[:, None], Y[None, :]], 0.0)
        self.D2y = np.where(same_x, self.d2y[Y[:, None], Y[None, :]], 0.0)
        vert = (X == 0) | (X == p - 1)
        horz = (Y == 0) | (Y == p - 1)
        b = slice(self.ni, self.m)
        self.D_bnd = np.where(vert[b, None], self.D1x[b], self.D1y[b])
        # edge-local tangential derivatives (p-2 interior nodes of the edge)
        self.ex1, self.ex2 = derivative_matrices(gx[1:p - 1])
        self.ey1, self.ey2 = derivative_matrices(gy[1:p - 1])
        self.Ex1, self.Ex2 = self.D1x.copy(), self.D2x.copy()
        self.Ey1, self.Ey2 = self.D1y.copy(), self.D2y.copy()
        for side in (0, p - 1):
            rows = np.nonzero(horz & (Y == side))[0]          # north / south: tangential x
            rows = rows[np.argsort(X[rows], kind="stable")]
            for E, e in ((self.Ex1, self.ex1), (self.Ex2, self.ex2)):
                E[rows, :] = 0.0
                E[np.ix_(rows, rows)] = e
            rows = np.nonzero(vert & (X == side))[0]          # east / west: tangential y
            rows = rows[np.argsort(Y[rows], kind="stable")]
            for E, e in ((self.Ey1, self.ey1), (self.Ey2, self.ey2)):
                E[rows, :] = 0.0
                E[np.ix_(rows, rows)] = e
        self.local_xy = np.column_stack([gx[X], gy[Y]])


class EllipticDiscretization:
    """Per-leaf collocation data of ``A`` on a tree (reference
    operators.py:219-274).  Coefficient samples are taken once on the host
    and uploaded; one sample set serves every leaf for constant coefficients."""

    def __init__(self, tree, coeffs):
        if coeffs.dim != tree.dim:
            raise ValueError(f"operator is {coeffs.dim}D but tree is {tree.dim}D")
        self.tree = tree
        self.coeffs = coeffs
        self.stencil = LeafStencil(tree)
        self.leaf_gidx = np.hstack([tree.leaf_int_gidx, tree.leaf_bnd_gidx])
        self._samples = None
        self._device = {}

    def leaf_points(self, leaf_id):
        a, b = self.tree.leaf_cells[leaf_id]
        lo = np.array([self.tree.bounds[0][0] + a * self.tree.wx,
                       self.tree.bounds[1][0] + b * self.tree.wy])
        return lo[None, :] + self.stencil.local_xy

    def coefficient_samples(self):
        """(Lc, 5, m) samples of (c11, c22, c1, c2, c) at every leaf-local
        point, Lc = 1 for constant coefficients."""
        if self._samples is None:
            st, t = self.stencil, self.tree
            if self.coeffs.is_constant:
                v = self.coeffs.evaluate(self.leaf_points(0))
                self._samples = np.stack([v[f] for f in FIELDS])[None]
            else:
                a, b = t.leaf_cells[:, 0], t.leaf_cells[:, 1]
                X = (t.bounds[0][0] + a * t.wx)[:, None] + st.local_xy[None, :, 0]
                Y = (t.bounds[1][0] + b * t.wy)[:, None] + st.local_xy[None, :, 1]
                v = self.coeffs.evaluate(np.column_stack([X.ravel(), Y.ravel()]))
                self._samples = np.stack([v[f].reshape(t.L, st.m) for f in FIELDS], axis=1)
        return self._samples

    def leaf_interior_rows(self, leaf_id):
        """Host copy of the collocated interior rows (ni x m); diagnostics only.
        Constant coefficients: one cached copy serves every leaf (reference
        operators.py:238-262)."""
        st = self.stencil
        s = self.coefficient_samples()
        if s.shape[0] == 1:
            rows = self._device.get("rows0")
            if rows is None:
                rows = self._device["rows0"] = self._interior_rows(s[0][:, :st.ni])
            return rows
        return self._interior_rows(s[leaf_id][:, :st.ni])

    def _interior_rows(self, v):
        st = self.stencil
        ii = slice(0, st.ni)
        rows = -v[0][:, None] * st.D2x[ii]
        rows = rows - v[1][:, None] * st.D2y[ii]
        if self.coeffs.c1 is not None:
            rows = rows + v[2][:, None] * st.D1x[ii]
        if self.coeffs.c2 is not None:
            rows = rows + v[3][:, None] * st.D1y[ii]
        if self.coeffs.c is not None:
            rows[:, :st.ni] += np.diag(v[4])
        return rows

    def leaf_blocks(self, leaf_id):
        rows = self.leaf_interior_rows(leaf_id)
        return rows[:, :self.stencil.ni], rows[:, self.stencil.ni:]

    # device-side evaluations (apply_lop / gradient / flux_jump) live in
    # timestep.DeviceDiscretization; these host entry points route there.
    def apply_lop(self, u):
        from .timestep import device_discretization
        return device_discretization(self).apply_lop(u)

    def gradient(self, u):
        from .timestep import device_discretization
        return device_discretization(self).gradient(u)

    def flux_jump(self, u):
        from .timestep import device_discretization
        return device_discretization(self).flux_jump(u)


def leaf_matrix(disc, leaf_id):
    """The leaf's full local collocation system (m x m, reference
    operators.py:265-274): the interior rows of ``A``, then identity rows for
    the edge points (Dirichlet data)."""
    st = disc.stencil
    A = np.zeros((st.m, st.m))
    A[:st.ni] = disc.leaf_interior_rows(leaf_id)
    A[st.ni:, st.ni:] = np.eye(st.nb)
    return A


def shift_reaction(coeffs, sigma, dt_gamma):
    """Coefficients of ``sigma*I + dt_gamma*A`` (reference operators.py:103-126)."""
    def scale(v):
        if v is None:
            return None
        if callable(v):
            return lambda *xy, _f=v: dt_gamma * np.asarray(_f(*xy), dtype=float)
        return dt_gamma * v
    c = coeffs.c
    if c is None:
        cn = sigma
    elif callable(c):
        cn = lambda *xy, _f=c: sigma + dt_gamma * np.asarray(_f(*xy), dtype=float)
    else:
        cn = sigma + dt_gamma * c
    return OperatorCoefficients(c11=scale(coeffs.c11), c22=scale(coeffs.c22), c1=scale(coeffs.c1),
                                c2=scale(coeffs.c2), c=cn, dim=coeffs.dim)
