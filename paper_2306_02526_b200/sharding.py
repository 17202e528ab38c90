"""Multi-GPU plumbing for the stage-solve path.

One process per GPU (torchrun), torch.distributed over NCCL for the
plumbing.  Implemented here:

* **ensemble member sharding** (C5, "ensembles shard by member"): an
  ``ncomp = k`` problem is split into contiguous member blocks, rank r
  stepping members ``[start_r, stop_r)`` with its own replica of the shared
  operator set -- no per-stage communication; results are gathered once;
* **replicas** (the single-problem configs in round 1): every rank runs the
  whole problem; throughput is aggregated, timing is the max over ranks.

Subtree sharding of one problem across GPUs (level log2(P) subtrees per
rank with an exchange of subtree-root fluxes / boundary values per stage) is
the next step; see DESIGN.md.
"""

import numpy as np

from .timestep import ParabolicProblem, SeparableField


def member_slice(k, rank, world):
    """Contiguous member block of ``rank`` (sizes differ by at most one)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of {world}")
    base, extra = divmod(k, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def _rows(fn, start, stop, k):
    if fn is None:
        return None

    def sliced(*args):
        v = np.asarray(fn(*args), dtype=float)
        if v.ndim > 1 and v.shape[0] == k:
            return v[start:stop]
        return v  # broadcast field (same for every member)
    return sliced


def shard_problem(problem, rank, world):
    """The sub-problem of members ``member_slice(ncomp, rank, world)``.

    Field callables returning ``(ncomp, n)`` are sliced; broadcast fields and
    ``g`` (pointwise per member) are shared unchanged.
    """
    k = problem.ncomp
    start, stop = member_slice(k, rank, world)

    def field(f):
        if isinstance(f, SeparableField):
            return SeparableField([(_rows(phi, start, stop, k), s) for phi, s in f.terms])
        return _rows(f, start, stop, k)

    return ParabolicProblem(coeffs=problem.coeffs, q=field(problem.q), g=problem.g,
                            f=field(problem.f), f_t=field(problem.f_t), u0=_rows(problem.u0, start, stop, k),
                            time_independent_bc=problem.time_independent_bc, ncomp=stop - start,
                            name=f"{problem.name}[{start}:{stop}]")


def max_over_ranks(value, device=None):
    """Max of a scalar over all ranks (identity without a process group)."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def gather_members(u_local, k, device=None):
    """All-gather per-rank member blocks (rows) into the full (k, N) array."""
    import torch
    import torch.distributed as dist
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return u_local
    world, rank = dist.get_world_size(), dist.get_rank()
    n = u_local.shape[-1]
    sizes = [member_slice(k, r, world) for r in range(world)]
    mx = max(b - a for a, b in sizes)
    buf = torch.zeros((mx, n), dtype=u_local.dtype, device=device if device is not None else u_local.device)
    buf[:u_local.shape[0]] = u_local
    parts = [torch.empty_like(buf) for _ in range(world)]
    dist.all_gather(parts, buf)
    return torch.cat([p[:b - a] for p, (a, b) in zip(parts, sizes)], dim=0)
