"""Host-side stepping logic that needs no GPU."""
import sys

import numpy as np
import pytest
import torch

from paper_2306_02526_b200 import declare_nonlinear, gradient_use, is_pure
from paper_2306_02526_b200.timestep import _is_fresh


def test_gradient_use_defaults_to_both():
    """The reference always evaluates the gradient (timestep.py:192-196): an
    undeclared g gets both components, whatever it reads (no probing)."""
    for g in (lambda t, u, gx, gy: u - u ** 3,
              lambda t, u, gx, gy: torch.where(u > 5, gx, 0 * u),
              lambda t, u, gx, gy: gx if t > 1 else u):
        assert gradient_use(g) == (True, True)


def test_gradient_use_declaration():
    g = declare_nonlinear(lambda t, u, gx, gy: -u * gx, ux=True, uy=False)
    assert gradient_use(g) == (True, False) and not is_pure(g)
    h = declare_nonlinear(lambda t, u, gx, gy: u - u ** 3, ux=False, uy=False, pure=True)
    assert gradient_use(h) == (False, False) and is_pure(h)
    assert not is_pure(lambda t, u, gx, gy: u)
    with pytest.raises(TypeError):
        declare_nonlinear(len)          # builtins take no attributes


def _refs_after_call(fn, *a):
    r = fn(*a)
    refs = sys.getrefcount(r) - 1           # as _call_g counts them
    return r, refs


def test_fresh_result_detection():
    """Only g's own fresh result may serve as stage-history storage; a g that
    returns its input, a gradient buffer, a persistent out= buffer or a view
    must be copied (history aliasing)."""
    U = torch.randn(1, 64, dtype=torch.float64)
    ux = torch.randn(1, 64, dtype=torch.float64)
    keep = torch.empty(1, 64, dtype=torch.float64)
    cases = {
        "fresh": (lambda t, u, gx, gy: u - u ** 3, True),
        "returns_u": (lambda t, u, gx, gy: u, False),
        "returns_ux": (lambda t, u, gx, gy: gx, False),
        "out_buffer": (lambda t, u, gx, gy: torch.mul(u, u, out=keep), False),
        "view": (lambda t, u, gx, gy: (u * 2).view(1, 64), False),
        "cast": (lambda t, u, gx, gy: (u * 2).float(), True),
    }
    for name, (g, want) in cases.items():
        r, refs = _refs_after_call(g, 0.0, U, ux, ux)
        assert _is_fresh(r, refs) == want, name


def test_field_host_eval_chunks_only_pointwise_callables():
    """Plain (numpy) field callables on large point sets are evaluated in
    chunks on all host cores only if that is bitwise the whole-array call
    (checked on first use); otherwise always as one call (the reference's)."""
    from paper_2306_02526_b200.timestep import _Field
    pts = np.random.default_rng(0).random((200_000, 2))
    fn = lambda t, p: np.sin(2 * np.pi * p[:, 0]) * np.cos(t) + p[:, 1] ** 2
    F = _Field(fn, pts, 1, "cpu")
    a = F.host_eval(0.3)
    assert F._pointwise is True and np.array_equal(a, fn(0.3, pts))
    assert np.array_equal(F.host_eval(0.7), fn(0.7, pts))
    glob = lambda t, p: p[:, 0] / p[:, 0].max()        # depends on every point: not chunkable
    G = _Field(glob, pts, 1, "cpu")
    assert np.array_equal(G.host_eval(0.0), glob(0.0, pts)) and G._pointwise is False
    assert np.array_equal(G.host_eval(1.0), glob(1.0, pts))
    _Field._pool.shutdown()   # no idle threads left behind for the forking tests
    _Field._pool = None

