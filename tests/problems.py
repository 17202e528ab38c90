"""Problem definitions shared by the tests (numpy callables mirroring
tests/golden/make_golden.py, which built the goldens with the real reference)."""

import numpy as np

UNIT = ((0.0, 1.0), (0.0, 1.0))
TWO_PI = 2 * np.pi


def var_test_fields():
    return dict(c11=lambda x, y: 1 + 0.3 * np.sin(x + y),
                c22=lambda x, y: 1 + 0.2 * np.cos(x - y),
                c1=lambda x, y: np.sin(2 * x), c2=0.5, c=0.3)


def c4_fields():
    a = lambda x, y: 1 + 0.5 * np.sin(TWO_PI * x) * np.cos(TWO_PI * y)
    ax = lambda x, y: np.pi * np.cos(TWO_PI * x) * np.cos(TWO_PI * y)
    ay = lambda x, y: -np.pi * np.sin(TWO_PI * x) * np.sin(TWO_PI * y)
    return dict(c11=a, c22=a, c1=lambda x, y: -(ax(x, y) + 1.0),
                c2=lambda x, y: -(ay(x, y) + 0.5))


def lap_fields():
    return dict(c11=1.0, c22=1.0)


def sine_field(coef, pts):
    x, y = pts[:, 0], pts[:, 1]
    mmax, nmax = coef.shape[-2:]
    sx = np.stack([np.sin(m * np.pi * x) for m in range(1, mmax + 1)])
    sy = np.stack([np.sin(n * np.pi * y) for n in range(1, nmax + 1)])
    if coef.ndim == 2:
        return np.einsum("mn,mp,np->p", coef, sx, sy)
    return np.einsum("kmn,mp,np->kp", coef, sx, sy)


def heat_manufactured():
    phi = lambda pts: np.sin(TWO_PI * pts[:, 0]) * np.sin(TWO_PI * pts[:, 1])
    uex = lambda t, pts: phi(pts) * np.cos(t)
    q = lambda t, pts: phi(pts) * (-np.sin(t) + 8 * np.pi ** 2 * np.cos(t))
    return phi, uex, q


SOLVE_CASES = {
    # name: (fields fn, bounds)
    "lap2x2p10": (lap_fields, UNIT),
    "var4x2p9": (var_test_fields, UNIT),
    "heat4x4p12k3": (lap_fields, UNIT),
    "pen4x4p8": (lap_fields, UNIT),
    "c4var4x4p10": (c4_fields, UNIT),
    "rect4x2p11": (var_test_fields, ((0.0, 2.0), (0.0, 1.0))),
    "heat8x8p16": (lap_fields, UNIT),
}


def rel_l2(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))
