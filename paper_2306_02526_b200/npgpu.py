"""numpy ufuncs on device tensors, for the reference's plain callables.

The reference's field callables ``F(t, pts)`` and nonlinear terms
``g(t, u, ux, uy)`` are written with numpy (``np.sin(2 * np.pi * pts[:, 0])``).
``DeviceArray`` is a float64 torch tensor that numpy's ufuncs and a few array
functions dispatch to torch (``__array_ufunc__`` / ``__array_function__``), so
such a callable, handed ``DeviceArray`` arguments, runs on the GPU where the
data lives instead of on the host.  Anything outside the mapped subset raises
(numpy then has no implementation) and the caller falls back to the host; the
stepper also checks the device result against the host call once per
callable (``matches_host``) before trusting it.
"""

import numpy as np
import torch

_UFUNCS = {
    np.sin: torch.sin, np.cos: torch.cos, np.tan: torch.tan, np.arcsin: torch.asin, np.arccos: torch.acos,
    np.arctan: torch.atan, np.arctan2: torch.atan2, np.sinh: torch.sinh, np.cosh: torch.cosh,
    np.tanh: torch.tanh, np.exp: torch.exp, np.exp2: torch.exp2, np.expm1: torch.expm1, np.log: torch.log,
    np.log2: torch.log2, np.log10: torch.log10, np.log1p: torch.log1p, np.sqrt: torch.sqrt,
    np.square: torch.square, np.absolute: torch.abs, np.fabs: torch.abs, np.negative: torch.neg,
    np.positive: lambda x: x, np.sign: torch.sign, np.add: torch.add, np.subtract: torch.sub,
    np.multiply: torch.mul, np.true_divide: torch.div, np.power: torch.pow, np.floor: torch.floor,
    np.ceil: torch.ceil, np.trunc: torch.trunc, np.rint: torch.round, np.minimum: torch.minimum,
    np.maximum: torch.maximum, np.fmin: torch.fmin, np.fmax: torch.fmax, np.hypot: torch.hypot,
    np.greater: torch.gt, np.greater_equal: torch.ge, np.less: torch.lt, np.less_equal: torch.le,
    np.equal: torch.eq, np.not_equal: torch.ne, np.logical_and: torch.logical_and,
    np.logical_or: torch.logical_or, np.logical_not: torch.logical_not, np.reciprocal: torch.reciprocal,
}

_FUNCS = {
    np.where: torch.where,
    np.zeros_like: lambda a, dtype=None: torch.zeros_like(a),
    np.ones_like: lambda a, dtype=None: torch.ones_like(a),
    np.full_like: lambda a, v, dtype=None: torch.full_like(a, v),
    np.clip: lambda a, lo, hi: torch.clamp(a, lo, hi),
    np.stack: lambda seq, axis=0: torch.stack(list(seq), dim=axis),
    np.vstack: lambda seq: torch.vstack([torch.atleast_1d(x) for x in seq]),
    np.column_stack: lambda seq: torch.column_stack(list(seq)),
    np.concatenate: lambda seq, axis=0: torch.cat(list(seq), dim=axis),
}


class DeviceArray(torch.Tensor):
    """A float64 tensor that numpy ufuncs (and np.where / *_like / stack /
    concatenate / clip) accept and evaluate with torch on its device."""

    def __array_ufunc__(self, ufunc, method, *inputs, **kwargs):
        f = _UFUNCS.get(ufunc)
        if method != "__call__" or f is None or kwargs:
            return NotImplemented
        dev = self.device
        args = [x if isinstance(x, torch.Tensor) else torch.as_tensor(x, dtype=torch.float64, device=dev)
                for x in inputs]
        return f(*args)

    def __array_function__(self, func, types, args, kwargs):
        f = _FUNCS.get(func)
        if f is None:
            return NotImplemented
        return f(*args, **kwargs)


def wrap(t):
    """``t`` (a float64 tensor) as a DeviceArray view."""
    return t.as_subclass(DeviceArray)


def plain(r):
    """A callable's result as a plain float64 tensor, or None when it is not a
    tensor (a numpy value: the callable did not stay on the device)."""
    if not isinstance(r, torch.Tensor):
        return None
    return r.as_subclass(torch.Tensor).to(torch.float64)


def matches_host(dev_vals, host_vals, rtol=1e-12):
    """Whether a device evaluation agrees with the host (numpy) one to
    rounding: shapes equal after broadcasting, max abs difference within
    rtol * max(1, max |host|)."""
    h = np.asarray(host_vals, dtype=float)
    d = dev_vals.detach().cpu().numpy()
    try:
        d, h = np.broadcast_arrays(d, h)
    except ValueError:
        return False
    if not np.all(np.isfinite(h) == np.isfinite(d)):
        return False
    fin = np.isfinite(h)
    scale = max(1.0, float(np.abs(h[fin]).max())) if fin.any() else 1.0
    return bool(np.all(np.abs(d[fin] - h[fin]) <= rtol * scale))
