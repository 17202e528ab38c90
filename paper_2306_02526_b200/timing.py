"""Build / solve time scaling of the HPS operator on the GPU (the reference's
``run_timing``, drivers.py:160-204).

For each leaf grid n x n (p x p nodes per leaf) the 2D heat operator
sigma*I + dt*A (A = -Laplacian, the backward-Euler shift) is built on the
device and one body-load solve is timed as the median of ``repeats``
repetitions, on device-resident data, with CUDA events around it -- the
B200 counterpart of the reference's wall-clock table.  Rows keep the
reference's columns (``n_side, N, N_dof, build_seconds,
per_step_solve_seconds, note``) and ``loglog_slope`` fits the growth of the
solve time with the DOF count (the paper's O(N log N) claim, §5.3.1).  The
reference builds its operator from the ``heat2d-homog`` catalogue problem;
here the same heat operator is constructed directly (unit square, c11 = c22 = 1).
"""

import time

import numpy as np

from .device import cuda_device, torch
from .errors import HpstepError
from .operators import EllipticDiscretization, OperatorCoefficients
from .solver import build
from .tree import build_tree

COLUMNS = ["n_side", "N", "N_dof", "build_seconds", "per_step_solve_seconds", "note"]


def _fmt(v):
    if isinstance(v, float):
        return f"{v:.17g}"
    return "" if v is None else str(v)


def write_csv(path, rows, columns=COLUMNS):
    """CSV with 17 significant digits (reference drivers.py:63-73)."""
    with open(path, "w") as fh:
        fh.write(",".join(columns) + "\n")
        for row in rows:
            fh.write(",".join(_fmt(row.get(c)) for c in columns) + "\n")


def run_timing(sizes=(4, 8, 16, 32), p=11, dt=0.01, repeats=3, seed=0, layout=None, out_path=None):
    """Device build and per-step solve times for n x n leaf grids."""
    dev = cuda_device()
    rng = np.random.default_rng(seed)
    coeffs = OperatorCoefficients(c11=1.0, c22=1.0)
    rows = []
    for n in sizes:
        row = {"n_side": int(n), "N": (n * (p - 1) + 1) ** 2, "N_dof": None, "build_seconds": None,
               "per_step_solve_seconds": None, "note": ""}
        try:
            tree = build_tree(((0.0, 1.0), (0.0, 1.0)), n, n, p)
            row["N_dof"] = int(tree.N)
            disc = EllipticDiscretization(tree, coeffs)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            ops = build(tree, coeffs, sigma=1.0, dt_gamma=dt, disc=disc, layout=layout)
            torch.cuda.synchronize()
            row["build_seconds"] = time.perf_counter() - t0
            u = torch.as_tensor(rng.standard_normal((1, tree.N)), device=dev)
            u[:, torch.as_tensor(tree.boundary_ids, device=dev)] = 0.0
            fb = torch.zeros((1, tree.boundary_ids.size), dtype=torch.float64, device=dev)
            out = torch.empty_like(u)
            ops.solve_device(fb, u, out)                       # warm-up
            reps = []
            for _ in range(max(3, repeats)):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                ops.solve_device(fb, u, out)
                e1.record()
                e1.synchronize()
                reps.append(e0.elapsed_time(e1) * 1e-3)
                u, out = out, u
            row["per_step_solve_seconds"] = float(np.median(reps))
            del ops
        except (MemoryError, torch.cuda.OutOfMemoryError, HpstepError) as e:
            if not isinstance(e, (MemoryError, torch.cuda.OutOfMemoryError)) and "memory" not in str(e):
                raise
            row["note"] = "skipped: memory exhausted"
            rows.append(row)
            break
        rows.append(row)
    if out_path:
        write_csv(out_path, rows)
    return rows


def loglog_slope(xs, ys):
    """Least-squares slope of log(y) against log(x) (drivers.py:207-209)."""
    xs, ys = np.log(np.asarray(xs, float)), np.log(np.asarray(ys, float))
    return float(np.polyfit(xs, ys, 1)[0])
