"""Chebyshev-Gauss-Lobatto collocation constants (host setup, O(p^2)).

Same node convention as the reference (chebyshev.py:33-107): nodes descend
from b to a, exact end points and exact antisymmetry; differentiation
matrices are barycentric with negative-sum diagonals.
"""

from dataclasses import dataclass

import numpy as np

from .errors import InvalidGridError


@dataclass(frozen=True)
class ChebGrid1D:
    p: int
    interval: tuple
    nodes: np.ndarray

    @property
    def a(self):
        return self.interval[0]

    @property
    def b(self):
        return self.interval[1]


def cheb_nodes(p, interval):
    a, b = float(interval[0]), float(interval[1])
    if p < 3:
        raise InvalidGridError(f"need at least 3 collocation points, got p={p}")
    if not a < b:
        raise InvalidGridError(f"empty interval ({a}, {b})")
    s = np.cos(np.pi * np.arange(p) / (p - 1))
    s = 0.5 * (s - s[::-1])
    s[0], s[-1] = 1.0, -1.0
    x = 0.5 * (a + b) + 0.5 * (b - a) * s
    x[0], x[-1] = b, a
    return ChebGrid1D(p=p, interval=(a, b), nodes=x)


def cgl_weights(p):
    w = np.ones(p)
    w[1::2] = -1.0
    w[[0, -1]] *= 0.5
    return w


def generic_weights(x):
    x = np.asarray(x, float)
    gap = np.subtract.outer(x, x)
    np.fill_diagonal(gap, 1.0)
    logs = -np.log(np.abs(gap)).sum(axis=1)
    w = np.sign(gap).prod(axis=1) * np.exp(logs - logs.max())
    return w / np.abs(w).max()


def derivative_matrices(x, w=None):
    """(D1, D2) on nodes ``x`` with barycentric weights ``w``."""
    x = np.asarray(x, float)
    w = generic_weights(x) if w is None else np.asarray(w, float)
    gap = np.subtract.outer(x, x)
    np.fill_diagonal(gap, 1.0)
    ratio = w[None, :] / w[:, None]
    d1 = ratio / gap
    np.fill_diagonal(d1, 0.0)
    np.fill_diagonal(d1, -d1.sum(axis=1))
    d2 = 2.0 * (ratio * np.diag(d1)[:, None] - d1) / gap
    np.fill_diagonal(d2, 0.0)
    np.fill_diagonal(d2, -d2.sum(axis=1))
    return d1, d2


def diff_matrix(grid, order=1):
    d1, d2 = derivative_matrices(grid.nodes, cgl_weights(grid.p))
    if order == 1:
        return d1
    if order == 2:
        return d2
    raise ValueError(f"order must be 1 or 2, got {order}")
