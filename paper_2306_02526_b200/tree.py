"""Binary domain tree and global DOF numbering, built level-synchronously.

Same numbering contract as the reference (tree.py:1-13, 123-156, 183-280):

* global vector = leaf interiors (q*q per leaf, leaves in depth-first order,
  x-major tensor order with descending node coordinates), then one block of
  q = p-2 DOFs per vertical edge ``(i*n2+j)``, then per horizontal edge
  ``((n1+1)*n2 + i*(n2+1) + j)``;
* the box is halved along its longer physical edge (x on ties), the lower
  half is alpha;
* leaf boundary order: east edge, (north, south) interleaved, west edge;
* a parent's boundary is ``[alpha_bnd[i1a]; beta_bnd[i2b]]`` and its
  interface ``j3`` is sorted by global id.

Unlike the reference's recursive node-by-node construction, this one works
a whole level at a time with numpy: every node of a level has the same box
shape, so the child-local maps (i1a, i3a, i2b, i3b) are computed once per
level and verified against every node, and the per-node global ids are
produced as ``(nodes, size)`` int arrays that upload directly to the device.
"""

from dataclasses import dataclass

import numpy as np

from .chebyshev import cheb_nodes
from .errors import (InvalidGridError, TreeConsistencyError,
                     UnsupportedConfigurationError, UnsupportedPartitionError)

ROLE_INTERIOR = 0
ROLE_INTERFACE = 1
ROLE_BOUNDARY = 2


def _pow2(n):
    return n >= 1 and (n & (n - 1)) == 0


@dataclass
class LevelMaps:
    """One parent level (root = 0): shapes, uniform maps, per-node ids."""
    count: int
    xsplit: bool
    extent: tuple            # (cells in x, cells in y) of every node box
    origin: np.ndarray       # (count, 2) lower cell corner of every node
    n3: int
    n1a: int
    n2b: int
    nbc: int                 # child boundary size
    i1a: np.ndarray
    i3a: np.ndarray
    i2b: np.ndarray
    i3b: np.ndarray
    gidx_bnd: np.ndarray     # (count, n1a + n2b)
    j3: np.ndarray           # (count, n3)
    node_index: np.ndarray   # (count,) depth-first node index

    @property
    def n12(self):
        return self.n1a + self.n2b


@dataclass
class TreeNode:
    """Per-node view (reference tree.py:32-60), materialised on demand."""
    index: int
    level: int
    cells: tuple
    box: tuple
    parent: int = None
    children: tuple = None
    leaf_id: int = None
    gidx_int: np.ndarray = None
    gidx_bnd: np.ndarray = None
    j1: np.ndarray = None
    j2: np.ndarray = None
    j3: np.ndarray = None
    i1a: np.ndarray = None
    i3a: np.ndarray = None
    i2b: np.ndarray = None
    i3b: np.ndarray = None

    @property
    def is_leaf(self):
        return self.children is None


class DomainTree:
    def __init__(self, bounds, n1, n2, p):
        if p < 4:
            raise InvalidGridError(f"leaf order must be at least 4, got p={p}")
        bounds = tuple(bounds)
        if np.isscalar(bounds[0]):
            raise UnsupportedConfigurationError(
                "the B200 path implements 2D domains; 1D trees are out of scope")
        if n2 is None:
            raise UnsupportedPartitionError("n2 is required for 2D domains")
        if not (_pow2(n1) and _pow2(n2)):
            raise UnsupportedPartitionError(
                f"leaf counts must be powers of two, got n1={n1}, n2={n2}")
        self.dim = 2
        self.bounds = tuple(tuple(float(v) for v in b) for b in bounds)
        self.n1, self.n2, self.p = int(n1), int(n2), int(p)
        q = self.q = p - 2
        self.ni, self.nb = q * q, 4 * q
        self.leaf_count = self.L = n1 * n2
        self.wx = (self.bounds[0][1] - self.bounds[0][0]) / n1
        self.wy = (self.bounds[1][1] - self.bounds[1][0]) / n2
        self._edge_base = self.L * self.ni
        self._hbase = self._edge_base + (n1 + 1) * n2 * q
        self.N = self._edge_base + ((n1 + 1) * n2 + n1 * (n2 + 1)) * q
        self.leaf_gx = cheb_nodes(p, (0.0, self.wx))
        self.leaf_gy = cheb_nodes(p, (0.0, self.wy))
        self._levels_topdown()
        self._leaves()
        self._levels_bottomup()
        self._points_roles()
        self._nodes = None

    # -- geometry of every level ------------------------------------------------
    def _levels_topdown(self):
        org = np.zeros((1, 2), dtype=np.int64)
        ex, ey = self.n1, self.n2
        self._shape = []
        while not (ex == 1 and ey == 1):
            if ex == 1:
                xs = False
            elif ey == 1:
                xs = True
            else:
                xs = ex * self.wx >= ey * self.wy
            self._shape.append((xs, ex, ey, org))
            child = np.repeat(org, 2, axis=0)
            if xs:
                child[1::2, 0] += ex // 2
                ex //= 2
            else:
                child[1::2, 1] += ey // 2
                ey //= 2
            org = child
        self.depth = len(self._shape)          # parent levels
        self.level_count = self.depth + 1
        self.leaf_cells = org                  # (L, 2) in depth-first leaf order
        # depth-first node index of (level d, position i)
        D = self.depth
        size = [2 ** (D - d + 1) - 1 for d in range(D + 1)]
        self._dfs = []
        for d in range(D + 1):
            pos = np.arange(2 ** d, dtype=np.int64)
            idx = np.full(2 ** d, d, dtype=np.int64)
            for k in range(d):
                idx += ((pos >> (d - 1 - k)) & 1) * size[k + 1]
            self._dfs.append(idx)
        self.leaves = self._dfs[D]

    def vedge_ids(self, i, j):
        """(..., q) global ids of vertical edge(s) (i, j)."""
        return self._edge_base + ((np.asarray(i) * self.n2 + np.asarray(j)) * self.q)[..., None] \
            + np.arange(self.q)

    def hedge_ids(self, i, j):
        return self._hbase + ((np.asarray(i) * (self.n2 + 1) + np.asarray(j)) * self.q)[..., None] \
            + np.arange(self.q)

    def _leaves(self):
        a, b = self.leaf_cells[:, 0], self.leaf_cells[:, 1]
        L, q = self.L, self.q
        east, west = self.vedge_ids(a + 1, b), self.vedge_ids(a, b)
        north, south = self.hedge_ids(a, b + 1), self.hedge_ids(a, b)
        mid = np.stack([north, south], axis=2).reshape(L, 2 * q)
        self.leaf_bnd_gidx = np.concatenate([east, mid, west], axis=1)
        self.leaf_int_gidx = np.arange(L * self.ni, dtype=np.int64).reshape(L, self.ni)

    def _levels_bottomup(self):
        q = self.q
        bnd = self.leaf_bnd_gidx
        self.level_maps = [None] * self.depth
        for d in range(self.depth - 1, -1, -1):
            xs, ex, ey, org = self._shape[d]
            A, B = bnd[0::2], bnd[1::2]
            if xs:
                mid = org[:, 0] + ex // 2
                j3 = self.vedge_ids(mid[:, None], org[:, 1][:, None] + np.arange(ey)).reshape(-1, ey * q)
            else:
                mid = org[:, 1] + ey // 2
                j3 = self.hedge_ids(org[:, 0][:, None] + np.arange(ex), mid[:, None]).reshape(-1, ex * q)
            maps = []
            for C in (A, B):
                inn = np.isin(C[0], j3[0])
                pos = np.nonzero(inn)[0]
                i3 = pos[np.argsort(C[0][pos], kind="stable")]
                i1 = np.nonzero(~inn)[0]
                if not np.array_equal(C[:, i3], j3):
                    raise TreeConsistencyError(f"level {d}: interface maps are not uniform")
                maps.append((i1, i3))
            (i1a, i3a), (i2b, i3b) = maps
            if i3a.size != j3.shape[1]:
                raise TreeConsistencyError(f"level {d}: children share {i3a.size} DOFs, "
                                           f"expected {j3.shape[1]}")
            gb = np.concatenate([A[:, i1a], B[:, i2b]], axis=1)
            self.level_maps[d] = LevelMaps(
                count=org.shape[0], xsplit=xs, extent=(ex, ey), origin=org, n3=j3.shape[1],
                n1a=i1a.size, n2b=i2b.size, nbc=A.shape[1], i1a=i1a, i3a=i3a, i2b=i2b, i3b=i3b,
                gidx_bnd=gb, j3=j3, node_index=self._dfs[d])
            bnd = gb

    def _points_roles(self):
        n1, n2, q, p = self.n1, self.n2, self.q, self.p
        (x0, _), (y0, _) = self.bounds
        gx, gy = self.leaf_gx.nodes, self.leaf_gy.nodes
        pts = np.zeros((self.N, 2))
        a, b = self.leaf_cells[:, 0], self.leaf_cells[:, 1]
        bx, by = x0 + a * self.wx, y0 + b * self.wy
        t = np.arange(1, p - 1)
        X = bx[:, None, None] + gx[t][None, :, None] + 0.0 * gy[t][None, None, :]
        Y = by[:, None, None] + gy[t][None, None, :] + 0.0 * gx[t][None, :, None]
        pts[:self._edge_base, 0] = X.reshape(-1)
        pts[:self._edge_base, 1] = Y.reshape(-1)
        # shared edges take the coordinates written by the later (upper) leaf
        # in depth-first order, as the reference's per-leaf writes do
        i = np.arange(n1 + 1)[:, None] + np.zeros(n2, dtype=np.int64)[None, :]
        j = np.arange(n2)[None, :] + np.zeros(n1 + 1, dtype=np.int64)[:, None]
        ids = self.vedge_ids(i, j)
        west_writer = i < n1
        vx = np.where(west_writer, x0 + i * self.wx + gx[p - 1], x0 + (i - 1) * self.wx + gx[0])
        pts[ids, 0] = vx[..., None]
        pts[ids, 1] = (y0 + j * self.wy)[..., None] + gy[t]
        i = np.arange(n1)[:, None] + np.zeros(n2 + 1, dtype=np.int64)[None, :]
        j = np.arange(n2 + 1)[None, :] + np.zeros(n1, dtype=np.int64)[:, None]
        ids = self.hedge_ids(i, j)
        south_writer = j < n2
        hy = np.where(south_writer, y0 + j * self.wy + gy[p - 1], y0 + (j - 1) * self.wy + gy[0])
        pts[ids, 1] = hy[..., None]
        pts[ids, 0] = (x0 + i * self.wx)[..., None] + gx[t]
        self.points = pts
        role = np.zeros(self.N, dtype=np.int8)
        vb = self.vedge_ids(np.array([0, n1])[:, None], np.arange(n2)[None, :])
        vi = self.vedge_ids(np.arange(1, n1)[:, None], np.arange(n2)[None, :])
        hb = self.hedge_ids(np.arange(n1)[:, None], np.array([0, n2])[None, :])
        hi = self.hedge_ids(np.arange(n1)[:, None], np.arange(1, n2)[None, :])
        role[vb.ravel()] = ROLE_BOUNDARY
        role[hb.ravel()] = ROLE_BOUNDARY
        role[vi.ravel()] = ROLE_INTERFACE
        role[hi.ravel()] = ROLE_INTERFACE
        self.role = role
        self.multiplicity = np.where(role == ROLE_INTERFACE, 2, 1).astype(np.int32)
        self.boundary_ids = np.nonzero(role == ROLE_BOUNDARY)[0]
        self.interface_ids = np.nonzero(role == ROLE_INTERFACE)[0]
        self.free_ids = np.nonzero(role != ROLE_BOUNDARY)[0]
        sign = np.concatenate([np.ones(q), np.tile([1.0, -1.0], q), -np.ones(q)])
        self.leaf_bnd_sign = np.where(role[self.leaf_bnd_gidx] == ROLE_INTERFACE, sign[None, :], 0.0)

    # -- reference-compatible node view ---------------------------------------------
    @property
    def nodes(self):
        """Per-node records in depth-first order (built on first access)."""
        if self._nodes is None:
            self._nodes = self._materialise_nodes()
        return self._nodes

    @property
    def levels(self):
        return [list(ix) for ix in self._dfs]

    @property
    def root(self):
        return self.nodes[0]

    def _materialise_nodes(self):
        nodes = [None] * (2 ** (self.depth + 1) - 1)
        (x0, _), (y0, _) = self.bounds
        ext = [(s[1], s[2]) for s in self._shape] + [(1, 1)]
        orgs = [s[3] for s in self._shape] + [self.leaf_cells]
        for d in range(self.depth + 1):
            for pos, idx in enumerate(self._dfs[d]):
                a, b = orgs[d][pos]
                ex, ey = ext[d]
                cells = (int(a), int(a + ex), int(b), int(b + ey))
                box = ((x0 + cells[0] * self.wx, x0 + cells[1] * self.wx),
                       (y0 + cells[2] * self.wy, y0 + cells[3] * self.wy))
                parent = None if d == 0 else int(self._dfs[d - 1][pos // 2])
                nd = TreeNode(index=int(idx), level=d, cells=cells, box=box, parent=parent)
                if d == self.depth:
                    nd.leaf_id = pos
                    nd.gidx_int = self.leaf_int_gidx[pos]
                    nd.gidx_bnd = self.leaf_bnd_gidx[pos]
                else:
                    lm = self.level_maps[d]
                    nd.children = (int(self._dfs[d + 1][2 * pos]), int(self._dfs[d + 1][2 * pos + 1]))
                    nd.i1a, nd.i3a, nd.i2b, nd.i3b = lm.i1a, lm.i3a, lm.i2b, lm.i3b
                    nd.gidx_bnd = lm.gidx_bnd[pos]
                    nd.j1 = nd.gidx_bnd[:lm.n1a]
                    nd.j2 = nd.gidx_bnd[lm.n1a:]
                    nd.j3 = lm.j3[pos]
                nodes[int(idx)] = nd
        return nodes

    def interior_ids(self, node):
        if node.is_leaf:
            return node.gidx_int
        a, b = (self.nodes[c] for c in node.children)
        return np.concatenate([self.interior_ids(a), self.interior_ids(b), node.j3])

    def interface_sets(self, node):
        if node.is_leaf:
            raise TreeConsistencyError(f"node {node.index} is a leaf")
        return node.j1, node.j2, node.j3

    def describe(self):
        (x0, x1), (y0, y1) = self.bounds
        n_int = int(np.sum(self.role == ROLE_INTERIOR))
        lines = [f"DomainTree 2D on [{x0:g}, {x1:g}] x [{y0:g}, {y1:g}], n1={self.n1}, "
                 f"n2={self.n2}, p={self.p}",
                 f"N = {self.N} DOFs: {n_int} interior, {self.interface_ids.size} interface, "
                 f"{self.boundary_ids.size} boundary (leaf corners excluded)",
                 f"leaves = {self.leaf_count}, levels = {self.level_count}, "
                 f"interfaces = {self.leaf_count - 1}"]
        for d in range(self.level_count):
            tag = f", {2 ** d} leaf" if d == self.depth else ""
            lines.append(f"  level {d}: {2 ** d} node(s){tag}")
        return "\n".join(lines)


def build_tree(bounds, n1, n2=None, p=8):
    """Build the domain tree with the reference's global numbering."""
    return DomainTree(bounds, n1, n2, p)
