"""CPU oracle for the per-stage HPS solve path of arXiv 2306.02526 (``hpstep``).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
module, and only as the checker (or the timed CPU baseline) -- never as the
product path.  The product (``paper_2306_02526_b200``) must not import it.

This is a numpy/scipy restatement of the reference algorithm, written from the
reference's behaviour, with every piece citing the reference file:line it
follows (paths relative to ``/root/reference/pkg/src/hpstep``).  The dense
arithmetic goes through the same LAPACK entry points the reference uses
(``scipy.linalg.lu_factor`` / ``lu_solve``), so on identical inputs it agrees
with the reference to round-off (pinned by ``tests/test_oracle_golden.py``
against vectors produced by the real reference, ``tests/golden/make_golden.py``).

Scope: 2D domains (the hot path); 1D trees are outside the hot path.
"""

from __future__ import annotations

import math

import numpy as np
import scipy.linalg

PIVOT_RTOL = 1e-13          # linalg.py:17
DIVERGENCE_LIMIT = 1e12     # timestep.py:33


class OracleSingular(Exception):
    """Mirror of SingularMatrixError (errors.py:16-27); ``context`` names the node."""

    def __init__(self, msg, context):
        super().__init__(f"{msg} [{context}]")
        self.context = context


# --------------------------------------------------------------------------
# Chebyshev collocation (chebyshev.py:33-107)
# --------------------------------------------------------------------------

def cgl_nodes(p, a, b):
    """Descending CGL nodes on [a, b] with exact end points (chebyshev.py:33-49)."""
    t = np.cos(np.pi * np.arange(p) / (p - 1))
    t = 0.5 * (t - t[::-1])
    t[0], t[-1] = 1.0, -1.0
    x = 0.5 * (a + b) + 0.5 * (b - a) * t
    x[0], x[-1] = b, a
    return x


def _cgl_weights(p):
    """Closed-form CGL barycentric weights (chebyshev.py:52-58)."""
    w = np.where(np.arange(p) % 2 == 0, 1.0, -1.0)
    w[0] *= 0.5
    w[-1] *= 0.5
    return w


def _bary_weights(x):
    """Generic barycentric weights, log-scaled, unit max (chebyshev.py:61-70)."""
    d = x[:, None] - x[None, :]
    np.fill_diagonal(d, 1.0)
    lw = -np.log(np.abs(d)).sum(axis=1)
    sg = np.sign(d).prod(axis=1)
    w = sg * np.exp(lw - lw.max())
    return w / np.abs(w).max()


def bary_diff(x, order, w=None):
    """Barycentric D1 / D2 with negative-sum diagonals (chebyshev.py:73-96)."""
    if w is None:
        w = _bary_weights(x)
    d = x[:, None] - x[None, :]
    np.fill_diagonal(d, 1.0)
    ratio = w[None, :] / w[:, None]
    D1 = ratio / d
    np.fill_diagonal(D1, 0.0)
    np.fill_diagonal(D1, -D1.sum(axis=1))
    if order == 1:
        return D1
    D2 = 2.0 * (ratio * np.diag(D1)[:, None] - D1) / d
    np.fill_diagonal(D2, 0.0)
    np.fill_diagonal(D2, -D2.sum(axis=1))
    return D2


# --------------------------------------------------------------------------
# Domain tree and global numbering (tree.py:72-404)
# --------------------------------------------------------------------------

class OTree:
    """Binary tree over an n1 x n2 leaf grid with the reference numbering.

    * global order: leaf interiors (DFS leaf order), vertical edges
      ``(i*n2+j)``, horizontal edges ``((n1+1)*n2 + i*(n2+1)+j)``, each q long
      (tree.py:123-156);
    * split: longest physical edge, x on ties, lower half = alpha
      (tree.py:183-205);
    * leaf boundary order: east, (north, south) interleaved, west
      (tree.py:231-243);
    * parent maps: j3 sorted ids, i3a/i3b positions of j3 in each child,
      i1a/i2b the remaining positions in child order (tree.py:258-280).
    """

    def __init__(self, bounds, n1, n2, p):
        (self.x0, self.x1), (self.y0, self.y1) = [tuple(map(float, b)) for b in bounds]
        self.n1, self.n2, self.p = n1, n2, p
        q = self.q = p - 2
        self.ni, self.nb = q * q, 4 * q
        self.wx = (self.x1 - self.x0) / n1
        self.wy = (self.y1 - self.y0) / n2
        self.L = n1 * n2
        self.ebase = self.L * self.ni
        self.N = self.ebase + ((n1 + 1) * n2 + n1 * (n2 + 1)) * q
        self.gx = cgl_nodes(p, 0.0, self.wx)
        self.gy = cgl_nodes(p, 0.0, self.wy)
        self.points = np.zeros((self.N, 2))
        self.mult = np.zeros(self.N, dtype=np.int64)
        # node records: dict(level, cells, children, leaf_id, bnd, j3, i1a, i3a, i2b, i3b)
        self.nodes = []
        self.levels = []
        self.leaves = []
        self._grow((0, n1, 0, n2), 0)
        self.depth = len(self.levels)
        role = np.zeros(self.N, dtype=np.int8)   # 0 interior, 1 interface, 2 boundary
        for i in range(n1 + 1):
            for j in range(n2):
                role[self.vedge(i, j)] = 2 if i in (0, n1) else 1
        for i in range(n1):
            for j in range(n2 + 1):
                role[self.hedge(i, j)] = 2 if j in (0, n2) else 1
        self.role = role
        self.boundary_ids = np.nonzero(role == 2)[0]
        self.interface_ids = np.nonzero(role == 1)[0]
        leaf_nodes = [self.nodes[k] for k in self.leaves]
        self.leaf_int_gidx = np.stack([nd["lid"] * self.ni + np.arange(self.ni) for nd in leaf_nodes])
        self.leaf_bnd_gidx = np.stack([nd["bnd"] for nd in leaf_nodes])
        self.leaf_gidx = np.hstack([self.leaf_int_gidx, self.leaf_bnd_gidx])
        self.leaf_cells = np.array([(nd["cells"][0], nd["cells"][2]) for nd in leaf_nodes])
        # interface sign per leaf boundary slot (tree.py:392-403)
        sg = np.concatenate([np.ones(q), np.tile([1.0, -1.0], q), -np.ones(q)])
        self.leaf_bnd_sign = np.where(role[self.leaf_bnd_gidx] == 1, sg[None, :], 0.0)

    def vedge(self, i, j):
        return self.ebase + (i * self.n2 + j) * self.q + np.arange(self.q)

    def hedge(self, i, j):
        return self.ebase + ((self.n1 + 1) * self.n2 + i * (self.n2 + 1) + j) * self.q \
            + np.arange(self.q)

    def _grow(self, cells, level):
        k = len(self.nodes)
        nd = {"index": k, "level": level, "cells": cells, "children": None, "lid": None}
        self.nodes.append(nd)
        while len(self.levels) <= level:
            self.levels.append([])
        self.levels[level].append(k)
        a0, a1, b0, b1 = cells
        if a1 - a0 == 1 and b1 - b0 == 1:
            self._leaf(nd)
            return k
        if a1 - a0 == 1:
            xsplit = False
        elif b1 - b0 == 1:
            xsplit = True
        else:
            xsplit = (a1 - a0) * self.wx >= (b1 - b0) * self.wy
        if xsplit:
            m = (a0 + a1) // 2
            ca, cb = (a0, m, b0, b1), (m, a1, b0, b1)
        else:
            m = (b0 + b1) // 2
            ca, cb = (a0, a1, b0, m), (a0, a1, m, b1)
        ia = self._grow(ca, level + 1)
        ib = self._grow(cb, level + 1)
        nd["children"] = (ia, ib)
        self._parent(nd)
        return k

    def _leaf(self, nd):
        p, q = self.p, self.q
        nd["lid"] = len(self.leaves)
        self.leaves.append(nd["index"])
        a, b = nd["cells"][0], nd["cells"][2]
        east, west = self.vedge(a + 1, b), self.vedge(a, b)
        north, south = self.hedge(a, b + 1), self.hedge(a, b)
        mid = np.column_stack([north, south]).ravel()
        nd["bnd"] = np.concatenate([east, mid, west])
        gint = nd["lid"] * self.ni + np.arange(self.ni)
        bx = self.x0 + a * self.wx
        by = self.y0 + b * self.wy
        xs = bx + (self.gx - 0.0)
        ys = by + (self.gy - 0.0)
        xi, yi = np.meshgrid(np.arange(p), np.arange(p), indexing="ij")
        xi, yi = xi.ravel(), yi.ravel()
        inner = (xi > 0) & (xi < p - 1) & (yi > 0) & (yi < p - 1)
        corner = ((xi == 0) | (xi == p - 1)) & ((yi == 0) | (yi == p - 1))
        edge = ~inner & ~corner
        pts = np.column_stack([xs[xi], ys[yi]])
        self.points[gint] = pts[inner]
        self.points[nd["bnd"]] = pts[edge]
        self.mult[gint] += 1
        self.mult[nd["bnd"]] += 1

    def _parent(self, nd):
        A = self.nodes[nd["children"][0]]
        B = self.nodes[nd["children"][1]]
        j3 = np.intersect1d(A["bnd"], B["bnd"])
        ina = np.isin(A["bnd"], j3)
        inb = np.isin(B["bnd"], j3)
        pa, pb = np.nonzero(ina)[0], np.nonzero(inb)[0]
        nd["j3"] = j3
        nd["i1a"] = np.nonzero(~ina)[0]
        nd["i2b"] = np.nonzero(~inb)[0]
        nd["i3a"] = pa[np.argsort(A["bnd"][pa])]
        nd["i3b"] = pb[np.argsort(B["bnd"][pb])]
        nd["bnd"] = np.concatenate([A["bnd"][nd["i1a"]], B["bnd"][nd["i2b"]]])

    def parents_root_first(self):
        return [k for lvl in self.levels for k in lvl if self.nodes[k]["children"] is not None]


# --------------------------------------------------------------------------
# Coefficients and the leaf stencil (operators.py:34-274)
# --------------------------------------------------------------------------

FIELDS = ("c11", "c22", "c1", "c2", "c")


class OCoeffs:
    """A u = -c11 u_xx - c22 u_yy + c1 u_x + c2 u_y + c u (operators.py:1-16,34-76).

    Each field: None, a float, or a vectorized callable f(x, y).
    """

    def __init__(self, c11, c22=None, c1=None, c2=None, c=None):
        self.f = {"c11": c11, "c22": c22, "c1": c1, "c2": c2, "c": c}

    @property
    def is_constant(self):
        return not any(callable(v) for v in self.f.values())

    def eval(self, pts):
        n = pts.shape[0]
        out = {}
        for k, v in self.f.items():
            if v is None:
                out[k] = np.zeros(n)
            elif callable(v):
                out[k] = np.broadcast_to(np.asarray(v(pts[:, 0], pts[:, 1]), float), (n,)).copy()
            else:
                out[k] = np.full(n, float(v))
        return out


class OStencil:
    """Leaf-local matrices in (interior, edge) order (operators.py:129-216)."""

    def __init__(self, tree: OTree):
        p = tree.p
        self.ni, self.nb = tree.ni, tree.nb
        self.m = m = tree.ni + tree.nb
        wl = _cgl_weights(p)
        d1x, d2x = bary_diff(tree.gx, 1, wl), bary_diff(tree.gx, 2, wl)
        d1y, d2y = bary_diff(tree.gy, 1, wl), bary_diff(tree.gy, 2, wl)
        I = np.eye(p)
        xi, yi = np.meshgrid(np.arange(p), np.arange(p), indexing="ij")
        xi, yi = xi.ravel(), yi.ravel()
        inner = (xi > 0) & (xi < p - 1) & (yi > 0) & (yi < p - 1)
        corner = ((xi == 0) | (xi == p - 1)) & ((yi == 0) | (yi == p - 1))
        edge = ~inner & ~corner
        flat = np.arange(p * p)
        order = np.concatenate([flat[inner], flat[edge]])
        sel = np.ix_(order, order)
        self.D1x = np.kron(d1x, I)[sel]
        self.D2x = np.kron(d2x, I)[sel]
        self.D1y = np.kron(I, d1y)[sel]
        self.D2y = np.kron(I, d2y)[sel]
        lx, ly = xi[order], yi[order]
        vert = (lx == 0) | (lx == p - 1)
        horz = (ly == 0) | (ly == p - 1)
        bslots = np.arange(self.ni, m)
        self.D_bnd = np.where(vert[bslots, None], self.D1x[bslots], self.D1y[bslots])
        # evaluation operators: tangential rows on edges use edge-local nodes
        ex1, ex2 = bary_diff(tree.gx[1:p - 1], 1), bary_diff(tree.gx[1:p - 1], 2)
        ey1, ey2 = bary_diff(tree.gy[1:p - 1], 1), bary_diff(tree.gy[1:p - 1], 2)
        self.Ex1, self.Ex2 = self.D1x.copy(), self.D2x.copy()
        self.Ey1, self.Ey2 = self.D1y.copy(), self.D2y.copy()
        slots = np.arange(m)
        for ye in (0, p - 1):
            r = slots[horz & (ly == ye)]
            r = r[np.argsort(lx[r])]
            for E, e in ((self.Ex1, ex1), (self.Ex2, ex2)):
                E[r, :] = 0.0
                E[np.ix_(r, r)] = e
        for xe in (0, p - 1):
            r = slots[vert & (lx == xe)]
            r = r[np.argsort(ly[r])]
            for E, e in ((self.Ey1, ey1), (self.Ey2, ey2)):
                E[r, :] = 0.0
                E[np.ix_(r, r)] = e
        self.local_xy = np.column_stack([tree.gx[lx] - 0.0, tree.gy[ly] - 0.0])


class ODisc:
    """Per-leaf collocation rows and leaf-local evaluations (operators.py:219-346)."""

    def __init__(self, tree: OTree, coeffs: OCoeffs):
        self.tree, self.coeffs = tree, coeffs
        self.st = OStencil(tree)
        self._vals = {}
        self._rows = {}

    def leaf_points(self, lid):
        a, b = self.tree.leaf_cells[lid]
        lo = np.array([self.tree.x0 + a * self.tree.wx, self.tree.y0 + b * self.tree.wy])
        return lo[None, :] + self.st.local_xy

    def _key(self, lid):
        return -1 if self.coeffs.is_constant else lid

    def values(self, lid):
        k = self._key(lid)
        if k not in self._vals:
            self._vals[k] = self.coeffs.eval(self.leaf_points(lid))
        return self._vals[k]

    def interior_rows(self, lid):
        """Collocated A at interior points, (ni, m) (operators.py:252-269)."""
        k = self._key(lid)
        if k not in self._rows:
            st, v, ii = self.st, self.values(lid), slice(0, self.st.ni)
            rows = -v["c11"][ii, None] * st.D2x[ii]
            rows = rows - v["c22"][ii, None] * st.D2y[ii]
            if self.coeffs.f["c1"] is not None:
                rows = rows + v["c1"][ii, None] * st.D1x[ii]
            if self.coeffs.f["c2"] is not None:
                rows = rows + v["c2"][ii, None] * st.D1y[ii]
            if self.coeffs.f["c"] is not None:
                rows[:, :st.ni] += np.diag(v["c"][ii])
            self._rows[k] = rows
        return self._rows[k]

    def _stack_vals(self):
        return np.stack([np.column_stack([self.values(l)[f] for f in FIELDS])
                         for l in range(self.tree.L)])

    def _avg(self, vals):
        k = vals.shape[0]
        out = np.empty((k, self.tree.N))
        cols = self.tree.leaf_gidx.ravel()
        for i in range(k):
            out[i] = np.bincount(cols, weights=vals[i].ravel(), minlength=self.tree.N)
        return out / self.tree.mult[None, :]

    def apply_lop(self, u):
        """L = -A leaf-locally with interface averaging (operators.py:276-301)."""
        u = np.asarray(u, float)
        U = np.atleast_2d(u)[:, self.tree.leaf_gidx]
        st, cf = self.st, self.coeffs.f
        V = self._stack_vals()
        out = V[..., 0] * (U @ st.Ex2.T)
        out = out + V[..., 1] * (U @ st.Ey2.T)
        if cf["c1"] is not None:
            out = out - V[..., 2] * (U @ st.Ex1.T)
        if cf["c2"] is not None:
            out = out - V[..., 3] * (U @ st.Ey1.T)
        if cf["c"] is not None:
            out = out - V[..., 4] * U
        r = self._avg(out)
        return r[0] if u.ndim == 1 else r

    def gradient(self, u):
        """Leaf-local (u_x, u_y) with interface averaging (operators.py:303-317)."""
        u = np.asarray(u, float)
        U = np.atleast_2d(u)[:, self.tree.leaf_gidx]
        ux = self._avg(U @ self.st.Ex1.T)
        uy = self._avg(U @ self.st.Ey1.T)
        return (ux[0], uy[0]) if u.ndim == 1 else (ux, uy)

    def flux_jump(self, u):
        """Signed interface flux jumps (operators.py:319-336)."""
        u = np.asarray(u, float)
        U = np.atleast_2d(u)[:, self.tree.leaf_gidx]
        v = (U @ self.st.D_bnd.T) * self.tree.leaf_bnd_sign[None]
        out = np.zeros((v.shape[0], self.tree.N))
        cols = self.tree.leaf_bnd_gidx.ravel()
        for i in range(v.shape[0]):
            out[i] = np.bincount(cols, weights=v[i].ravel(), minlength=self.tree.N)
        return out[0] if u.ndim == 1 else out


# --------------------------------------------------------------------------
# Dense LU with the reference singularity policy (linalg.py:20-48)
# --------------------------------------------------------------------------

class OLU:
    def __init__(self, A, context):
        self.lu, self.piv = scipy.linalg.lu_factor(A, check_finite=False)
        pv = np.abs(np.diag(self.lu))
        pmax = pv.max() if pv.size else 0.0
        if pv.size and (pmax == 0.0 or pv.min() <= PIVOT_RTOL * pmax):
            raise OracleSingular(f"matrix of size {A.shape[0]} is singular", context)
        self.pivots = pv

    def solve(self, B):
        return scipy.linalg.lu_solve((self.lu, self.piv), B, check_finite=False)


# --------------------------------------------------------------------------
# HPS build and solve (solver.py:53-276)
# --------------------------------------------------------------------------

class OHps:
    """Operator set for sigma*I + dt_gamma*A (solver.py:84-158) with solves (:162-276)."""

    def __init__(self, disc: ODisc, sigma=0.0, dt_gamma=1.0, keep_T=False):
        self.disc, self.tree = disc, disc.tree
        self.sigma, self.dt_gamma = float(sigma), float(dt_gamma)
        st, tree = disc.st, disc.tree
        self.D_bi = st.D_bnd[:, :st.ni]
        D_bb = st.D_bnd[:, st.ni:]
        nleaf = 1 if disc.coeffs.is_constant else tree.L
        self.leaf_lu, self.S_leaf, T_leaf = [], [], []
        for lid in range(nleaf):                                   # solver.py:53-64
            rows = disc.interior_rows(lid)
            Aii = self.sigma * np.eye(st.ni) + self.dt_gamma * rows[:, :st.ni]
            Aib = self.dt_gamma * rows[:, st.ni:]
            node = tree.leaves[lid]
            lu = OLU(Aii, f"leaf node {node}")
            S = -lu.solve(Aib)
            self.leaf_lu.append(lu)
            self.S_leaf.append(S)
            T_leaf.append(self.D_bi @ S + D_bb)
        self.merges = {}
        Tcache = {}

        def T_of(k):
            nd = tree.nodes[k]
            if nd["children"] is None:
                return T_leaf[nd["lid"] if nleaf > 1 else 0]
            return Tcache[k]

        for level in range(tree.depth - 2, -1, -1):               # solver.py:137-155
            for k in tree.levels[level]:
                nd = tree.nodes[k]
                if nd["children"] is None:
                    continue
                Ta, Tb = T_of(nd["children"][0]), T_of(nd["children"][1])
                i1a, i3a, i2b, i3b = nd["i1a"], nd["i3a"], nd["i2b"], nd["i3b"]
                X33 = Ta[np.ix_(i3a, i3a)] - Tb[np.ix_(i3b, i3b)]   # solver.py:67-81
                lu = OLU(X33, f"merge node {k}")
                S = lu.solve(np.hstack([-Ta[np.ix_(i3a, i1a)], Tb[np.ix_(i3b, i2b)]]))
                Tst = np.vstack([Ta[np.ix_(i1a, i3a)], Tb[np.ix_(i2b, i3b)]])
                n1, n2 = i1a.size, i2b.size
                T = np.zeros((n1 + n2, n1 + n2))
                T[:n1, :n1] = Ta[np.ix_(i1a, i1a)]
                T[n1:, n1:] = Tb[np.ix_(i2b, i2b)]
                T += Tst @ S
                Tcache[k] = T
                self.merges[k] = (S, lu, Tst)
        self.root_T = Tcache.get(0)
        self.T_leaf = T_leaf if keep_T else None
        self.order = tree.parents_root_first()

    def leaf(self, lid):
        return 0 if len(self.leaf_lu) == 1 else lid

    def boundary_values(self, f):                                  # solver.py:162-174
        tree = self.tree
        f = np.asarray(f, float)
        nbd = tree.boundary_ids.size
        if f.ndim == 0:
            return np.full((1, nbd), float(f))
        if f.shape[-1] == tree.N:
            return np.atleast_2d(f)[:, tree.boundary_ids]
        if f.shape[-1] == nbd:
            return np.atleast_2d(f)
        raise ValueError(f"boundary data must have trailing size {nbd} or {tree.N}")

    def solve(self, f, g=None, jump=None, inv_dt=None):             # solver.py:201-276
        tree, st = self.tree, self.disc.st
        ni, nb, L = st.ni, st.nb, tree.L
        fb = self.boundary_values(f)
        k = fb.shape[0]
        squeeze = (np.asarray(f).ndim <= 1) if g is None else (np.asarray(g).ndim == 1)
        if g is not None:
            G = np.atleast_2d(np.asarray(g, float))
            k = max(k, G.shape[0])
            if fb.shape[0] == 1 and k > 1:
                fb = np.broadcast_to(fb, (k, fb.shape[1]))
        w = None
        H, W3 = {}, {}
        if g is not None:
            gl = G[:, tree.leaf_int_gidx]
            if len(self.leaf_lu) == 1:
                w = self.leaf_lu[0].solve(gl.reshape(k * L, ni).T).T.reshape(k, L, ni)
            else:
                w = np.empty((k, L, ni))
                for l in range(L):
                    w[:, l, :] = self.leaf_lu[l].solve(gl[:, l, :].T).T
            hleaf = np.einsum("bn,kln->klb", self.D_bi, w)
        elif jump is not None:
            hleaf = np.zeros((k, L, nb))
        if g is not None or jump is not None:
            J = None if jump is None else np.atleast_2d(np.asarray(jump, float))

            def h(kk):
                nd = tree.nodes[kk]
                return hleaf[:, nd["lid"], :] if nd["children"] is None else H[kk]

            for kk in reversed(self.order):
                nd = tree.nodes[kk]
                S, lu, Tst = self.merges[kk]
                ha, hb = h(nd["children"][0]), h(nd["children"][1])
                r3 = hb[:, nd["i3b"]] - ha[:, nd["i3a"]]
                if J is not None:
                    r3 = r3 - inv_dt * J[:, nd["j3"]]
                W3[kk] = lu.solve(r3.T).T
                H[kk] = np.concatenate([ha[:, nd["i1a"]], hb[:, nd["i2b"]]], axis=1) \
                    + W3[kk] @ Tst.T
        u = np.zeros((k, tree.N))
        u[:, tree.boundary_ids] = fb
        for kk in self.order:
            nd = tree.nodes[kk]
            S = self.merges[kk][0]
            u3 = u[:, nd["bnd"]] @ S.T
            if kk in W3:
                u3 = u3 + W3[kk]
            u[:, nd["j3"]] = u3
        ub = u[:, tree.leaf_bnd_gidx]
        if len(self.S_leaf) == 1:
            ui = np.einsum("ib,klb->kli", self.S_leaf[0], ub)
        else:
            ui = np.einsum("lib,klb->kli", np.stack(self.S_leaf), ub)
        if w is not None:
            ui = ui + w
        for i in range(ui.shape[0]):
            u[i, tree.leaf_int_gidx.ravel()] = ui[i].ravel()
        return u[0] if squeeze else u

    def solve_homogeneous(self, f):
        return self.solve(f)

    def solve_with_body_load(self, f, g):
        return self.solve(f, g)

    def solve_penalized(self, f, g, jump, dt):
        if dt <= 0:
            raise ValueError(f"time step must be positive, got {dt}")
        return self.solve(f, g, jump, 1.0 / dt)


# --------------------------------------------------------------------------
# IMEX ARK tableaux (tableaux.py:126-231) -- published Kennedy & Carpenter pairs
# --------------------------------------------------------------------------

def ark4_tableau():
    """ARK4(3)6L[2]SA (tableaux.py:126-154)."""
    g = 0.25
    c = [0, 1 / 2, 83 / 250, 31 / 50, 17 / 20, 1]
    A = [[0, 0, 0, 0, 0, 0],
         [g, g, 0, 0, 0, 0],
         [8611 / 62500, -1743 / 31250, g, 0, 0, 0],
         [5012029 / 34652500, -654441 / 2922500, 174375 / 388108, g, 0, 0],
         [15267082809 / 155376265600, -71443401 / 120774400,
          730878875 / 902184768, 2285395 / 8070912, g, 0],
         [82889 / 524892, 0, 15625 / 83664, 69875 / 102672, -2260 / 8211, g]]
    Ah = [[0, 0, 0, 0, 0, 0],
          [1 / 2, 0, 0, 0, 0, 0],
          [13861 / 62500, 6889 / 62500, 0, 0, 0, 0],
          [-116923316275 / 2393684061468, -2731218467317 / 15368042101831,
           9408046702089 / 11113171139209, 0, 0, 0],
          [-451086348788 / 2902428689909, -2682348792572 / 7519795681897,
           12662868775082 / 11960479115383, 3355817975965 / 11060851509271, 0, 0],
          [647845179188 / 3216320057751, 73281519250 / 8382639484533,
           552539513391 / 3454668386233, 3354512671639 / 8306763924573,
           4040 / 17871, 0]]
    A = np.array(A, float)
    return dict(A=A, Ahat=np.array(Ah, float), b=A[-1].copy(), bhat=A[-1].copy(),
                c=np.array(c, float), gamma=g, s=6)


def be_tableau():
    return dict(A=np.array([[1.0]]), Ahat=None, b=np.array([1.0]), bhat=None,
                c=np.array([1.0]), gamma=1.0, s=1)


# --------------------------------------------------------------------------
# Stage-formulation IMEX stepper (timestep.py:36-266)
# --------------------------------------------------------------------------

class OStepper:
    """Stage formulation (timestep.py:237-266) and backward Euler (:231-235).

    ``q(t, pts)``, ``f(t, pts)`` vectorized callables; ``g(t, u, ux, uy)``.
    Records every stage solve output in ``self.stages`` when ``record``.
    """

    def __init__(self, tree, coeffs, tab, dt, q=None, f=None, g=None, ncomp=1, record=False):
        self.tree, self.tab, self.dt = tree, tab, float(dt)
        self.q, self.f, self.g, self.ncomp = q, f, g, ncomp
        self.disc = ODisc(tree, coeffs)
        self.ops = OHps(self.disc, sigma=1.0, dt_gamma=self.dt * tab["gamma"])
        self.bpts = tree.points[tree.boundary_ids]
        self.record = record
        self.stages = []
        self.nstep = 0

    def _stack(self, vals, n):
        if vals is None:
            return np.zeros((self.ncomp, n))
        a = np.asarray(vals, float)
        return a.reshape(self.ncomp, n) if a.ndim > 1 or self.ncomp == 1 \
            else np.broadcast_to(a, (self.ncomp, n))

    def bc(self, t):
        if self.f is None:
            return np.zeros((self.ncomp, self.bpts.shape[0]))
        return self._stack(self.f(t, self.bpts), self.bpts.shape[0])

    def qv(self, t):
        return 0.0 if self.q is None else self._stack(self.q(t, self.tree.points), self.tree.N)

    def gv(self, t, u):
        if self.g is None:
            return 0.0
        return np.asarray(self.g(t, u, *self.disc.gradient(u)), float)

    def guard(self, u):
        mx = np.max(np.abs(u)) if u.size else 0.0
        if not np.isfinite(mx) or mx > DIVERGENCE_LIMIT:
            raise FloatingPointError(f"diverged at step {self.nstep}")

    def step(self, t, u):
        u = np.atleast_2d(np.asarray(u, float))
        tab, dt = self.tab, self.dt
        if tab["s"] == 1:
            t1 = t + dt
            unew = self.ops.solve_with_body_load(self.bc(t1), u + dt * (self.qv(t1) + self.gv(t, u)))
            if self.record:
                self.stages.append(unew.copy())
        else:
            s = tab["s"]
            k, N = u.shape
            Lu = np.empty((s, k, N))
            QG = np.empty((s, k, N))
            Lu[0] = self.disc.apply_lop(u)
            QG[0] = self.qv(t + tab["c"][0] * dt) + self.gv(t + tab["c"][0] * dt, u)
            ui = u
            for i in range(1, s):
                ti = t + tab["c"][i] * dt
                r = u + dt * (np.tensordot(tab["A"][i, :i], Lu[:i], axes=1)
                              + np.tensordot(tab["Ahat"][i, :i], QG[:i], axes=1))
                ui = self.ops.solve_with_body_load(self.bc(ti), r)
                self.guard(ui)
                if self.record:
                    self.stages.append(ui.copy())
                if i < s - 1:
                    Lu[i] = self.disc.apply_lop(ui)
                QG[i] = self.qv(ti) + self.gv(ti, ui)
            unew = ui + dt * np.tensordot(tab["bhat"] - tab["Ahat"][s - 1], QG, axes=1)
            unew[:, self.tree.boundary_ids] = self.bc(t + dt)
        self.nstep += 1
        self.guard(unew)
        return unew

    def run(self, t, u, nsteps):
        squeeze = np.asarray(u).ndim == 1
        for _ in range(nsteps):
            u = self.step(t, u)
            t += self.dt
        return t, (u[0] if squeeze else u)
