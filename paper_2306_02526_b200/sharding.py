"""Multi-GPU plumbing for the stage-solve path.

One process per GPU (torchrun), torch.distributed over NCCL for the
plumbing.  Implemented here:

* **subtree sharding** of one problem (C2-C4): the tree is cut below parent
  level lstar = log2(P) into P subtrees ("parts"); rank r steps the leaves and
  levels >= lstar of its parts.  Per stage solve the ranks exchange only the
  level-lstar fluxes (an all-gather of P x n12 doubles), every rank then runs
  the few top levels itself (up and down, so no scatter is needed) and
  finishes its own subtrees.  The stage right-hand side is leaf-local: the
  interior history ``L u`` needs no exchange; the interface-averaged gradient
  that feeds a nonlinear g is completed on the top-level interfaces by one
  all-reduce of the partial sums (each abutting leaf adds half);
* **ensemble member sharding** (C5, "ensembles shard by member"): an
  ``ncomp = k`` problem is split into contiguous member blocks, rank r
  stepping members ``[start_r, stop_r)`` with its own replica of the shared
  operator set -- no per-stage communication; results are gathered once;
* **replicas** (bench option): every rank runs the whole problem.

Everything that talks to torch.distributed works on any backend (NCCL on the
GPUs; gloo for the CPU tests, staging CUDA tensors through the host).
"""

import os

import numpy as np

from .errors import UnsupportedConfigurationError
from .timestep import ParabolicProblem, SeparableField, TimeStepper, _call_g, gradient_use, is_pure


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


# ---------------------------------------------------------------------------
# subtree sharding of one problem
# ---------------------------------------------------------------------------

class SubtreePartition:
    """The P-part subtree partition of a tree (host numpy only).

    Part g = the subtree of node g on parent level lstar = log2(P); parts are
    Morton-contiguous, so part g owns the leaves ``[g*L/P, (g+1)*L/P)`` and
    the nodes ``[g*c/P, (g+1)*c/P)`` of every level >= lstar (the tree is
    built depth first, reference tree.py:161-181)."""

    def __init__(self, tree, nparts):
        nparts = int(nparts)
        lstar = nparts.bit_length() - 1
        if nparts < 1 or (1 << lstar) != nparts or (nparts > 1 and lstar >= tree.depth):
            raise UnsupportedConfigurationError(
                f"subtree partition needs a power-of-two part count below 2^depth "
                f"(depth {tree.depth}), got {nparts}")
        self.tree, self.nparts, self.lstar = tree, nparts, lstar
        self.lpp = tree.L // nparts
        lms = tree.level_maps
        # interfaces the TOP phase computes on every rank
        top = [np.asarray(lms[d].j3).ravel() for d in range(lstar)]
        self.top_ids = np.sort(np.concatenate(top)) if top else np.zeros(0, dtype=np.int64)

    def owner_parts(self, rank, world):
        """Contiguous parts of ``rank`` (P must be a multiple of the world size)."""
        if self.nparts % world:
            raise UnsupportedConfigurationError(
                f"{self.nparts} parts cannot be split over {world} ranks")
        m = self.nparts // world
        return rank * m, (rank + 1) * m

    def leaves(self, part0, part1):
        """(leaf0, nleaf) of a part range."""
        return part0 * self.lpp, (part1 - part0) * self.lpp

    def interior_range(self, part0, part1):
        l0, nl = self.leaves(part0, part1)
        return l0 * self.tree.ni, (l0 + nl) * self.tree.ni

    def inner_ids(self, part0, part1):
        """Interface DOFs eliminated inside the parts (j3 of their nodes on levels >= lstar)."""
        lms = self.tree.level_maps
        out = []
        for d in range(self.lstar, self.tree.depth):
            per = lms[d].count // self.nparts
            out.append(np.asarray(lms[d].j3)[part0 * per:part1 * per].ravel())
        return np.sort(np.concatenate(out)) if out else np.zeros(0, dtype=np.int64)

    def owned_ids(self, part0, part1, with_top):
        """Every DOF the parts' solve writes (+ the top interfaces and the
        Dirichlet boundary when ``with_top``): a partition of [0, N) over the
        ranks when exactly one rank passes with_top."""
        a, b = self.interior_range(part0, part1)
        ids = [np.arange(a, b), self.inner_ids(part0, part1)]
        if with_top:
            ids += [self.top_ids, np.asarray(self.tree.boundary_ids)]
        return np.sort(np.concatenate(ids))


def _dist():
    import torch.distributed as dist
    return dist if dist.is_available() and dist.is_initialized() else None


def _force():
    """HPSB_FORCE_COLLECTIVES=1: issue the collectives even on a one-rank
    group (tests of the collective / graph-capture paths on one GPU)."""
    return os.environ.get("HPSB_FORCE_COLLECTIVES") == "1"


def _solo(dist, group):
    return dist is None or (dist.get_world_size(group) == 1 and not _force())


def _staged(t, group):
    """gloo collectives run on host tensors: stage CUDA tensors through the CPU."""
    dist = _dist()
    return t.is_cuda and dist.get_backend(group) == "gloo"


def exchange_fluxes(block, part0, part1, group=None):
    """All-gather of the level-lstar fluxes: ``block`` (k, P, n12) holds this
    rank's parts [part0, part1) on entry and every part on exit."""
    import torch
    dist = _dist()
    if _solo(dist, group):
        return block
    world = dist.get_world_size(group)
    k, P, n12 = block.shape
    m = part1 - part0
    staged = _staged(block, group)
    src = block[:, part0:part1].contiguous()
    if staged:
        src = src.cpu()
    out = torch.empty(world * src.numel(), dtype=src.dtype, device=src.device)
    dist.all_gather_into_tensor(out, src.reshape(-1), group=group)
    # (world, k, m, n12) -> (k, world*m, n12)
    full = out.view(world, k, m, n12).permute(1, 0, 2, 3).reshape(k, world * m, n12)
    block.copy_(full if not staged else full.to(block.device))
    return block


def complete_edges(vecs, top_ids, group=None):
    """Finish interface-averaged leaf outputs on the top-level interfaces:
    each rank holds the half-contributions of its own leaves there; the sum
    over ranks adds exactly the two halves (and zeros), the same two-addend
    sum the single-GPU kernel forms."""
    import torch
    dist = _dist()
    if _solo(dist, group) or top_ids.numel() == 0:
        return vecs
    buf = torch.stack([v[:, top_ids] for v in vecs])
    staged = _staged(buf, group)
    work = buf.cpu() if staged else buf
    dist.all_reduce(work, op=dist.ReduceOp.SUM, group=group)
    if staged:
        buf.copy_(work)
    for v, b in zip(vecs, buf):
        v[:, top_ids] = b
    return vecs


def allreduce_sum(tensors, group=None):
    """Sum each tensor over the ranks in place (one collective on a flat
    buffer; gloo stages through the host)."""
    import torch
    dist = _dist()
    if _solo(dist, group) or not tensors:
        return tensors
    flat = torch.cat([t.reshape(-1) for t in tensors])
    staged = _staged(flat, group)
    work = flat.cpu() if staged else flat
    dist.all_reduce(work, op=dist.ReduceOp.SUM, group=group)
    if staged:
        flat.copy_(work)
    o = 0
    for t in tensors:
        n = t.numel()
        t.copy_(flat[o:o + n].view(t.shape))
        o += n
    return tensors


def gather_owned(u, owned_ids, group=None):
    """Full (k, N) vector on every rank from each rank's owned DOFs (the owned
    sets partition [0, N); a sum with zeros elsewhere is exact)."""
    import torch
    dist = _dist()
    if dist is None or dist.get_world_size(group) == 1:
        return u
    contrib = torch.zeros_like(u)
    contrib[:, owned_ids] = u[:, owned_ids]
    staged = _staged(contrib, group)
    work = contrib.cpu() if staged else contrib
    dist.all_reduce(work, op=dist.ReduceOp.SUM, group=group)
    return work.to(u.device) if staged else work


def reduce_max(t, group=None):
    dist = _dist()
    if dist is None or dist.get_world_size(group) == 1:
        return t
    staged = _staged(t, group)
    work = t.cpu() if staged else t.clone()
    dist.all_reduce(work, op=dist.ReduceOp.MAX, group=group)
    return work.to(t.device) if staged else work


class ShardedTimeStepper(TimeStepper):
    """The stage-formulation (and backward-Euler) stepper of one problem
    sharded by subtrees over the ranks of a process group, one GPU each
    (SURVEY.md 8(e)); same constructor and ``step`` / ``run`` /
    ``initial_state`` as :class:`TimeStepper`.

    Rank r owns parts ``SubtreePartition.owner_parts(r, world)`` (``nparts``
    defaults to the world size; more parts than ranks is allowed).  Per stage
    it assembles the body load on its own leaf interiors, runs the UP phase of
    its parts, all-gathers the level-lstar fluxes, runs the top levels and
    then the DOWN phase of its parts.  Vectors are global length N on every
    rank; a rank's copy is exact on the DOFs it owns, the top interfaces and
    the Dirichlet boundary, which is everything its own leaves read.  States
    returned by ``step`` / ``run`` are gathered (exact everywhere)."""

    def __init__(self, tree, problem, tableau, dt, nparts=None, group=None, disc=None, threads=None,
                 layout=None):
        dist = _dist()
        self._group = group
        self._world = 1 if dist is None else dist.get_world_size(group)
        self._rank = 0 if dist is None else dist.get_rank(group)
        self._multi = self._world > 1 or _force()      # collectives are issued
        nparts = self._world if nparts is None else int(nparts)
        self._partition = SubtreePartition(tree, nparts)
        self._nparts = nparts
        self._parts = self._partition.owner_parts(self._rank, self._world)
        super().__init__(tree, problem, tableau, dt, formulation="stage", disc=disc, threads=threads,
                         layout=layout)
        import torch
        P = self._partition
        self._leaves = P.leaves(*self._parts)
        self._ir = P.interior_range(*self._parts)
        self._nloc = self._ir[1] - self._ir[0]
        self._edges = (tree.L * tree.ni, tree.N)
        self._top_ids = torch.as_tensor(P.top_ids, dtype=torch.long, device=self._dev)
        self._owned = torch.as_tensor(P.owned_ids(*self._parts, with_top=self._rank == 0), dtype=torch.long,
                                      device=self._dev)

    # buffers start at zero: DOFs other ranks own are never written here and
    # must stay finite for the (range-wise) combinations and guards
    def _buf(self, name, shape):
        import torch
        b = self._bufs.get(name)
        if b is None or tuple(b.shape) != tuple(shape):
            b = torch.zeros(shape, dtype=torch.float64, device=self._dev)
            self._bufs[name] = b
        return b

    def _eval_lu(self, U, out, guard=None):
        self._eval(U, lu_int=out, guard=guard, leaves=self._leaves)

    def _fused_stage(self, fb, body, out, lu, guard, root_pre=None):
        return False                      # the sharded solve runs in phases with an exchange

    def _root_batch(self):
        return False

    def _qg_alias_ok(self):
        return False                      # only the owned DOFs of the history are written

    def _final_combine(self, terms, fb, unew, guard):
        self._owned_combine(terms, unew)
        self._put_boundary(fb, unew)
        self._owned_maxabs(unew, guard)

    def _fused_stage_terms(self, fb, terms, r, out, lu, guard, root_pre):
        return False

    def _ranges(self):
        return (self._ir, self._edges)

    def _owned_combine(self, terms, out):
        from .timestep import combine
        for a, b in self._ranges():
            combine([(c, v[:, a:b] if v.shape[0] > 0 else v) for c, v in terms], out[:, a:b])

    def _owned_maxabs(self, x, guard):
        for a, b in self._ranges():
            self._maxabs(x[:, a:b], guard)

    def _reduce_guards(self, g):
        return reduce_max(g, self._group)

    def _g(self, t, U, out=None):
        """g over the owned DOFs with the gradient completed on the top interfaces."""
        if self.problem.g is None:
            return None
        ux, uy = self._buf("gx", U.shape), self._buf("gy", U.shape)
        res = out if out is not None else self._buf("gval", U.shape)
        if self._dry:
            return res
        g = self.problem.g
        if any(gradient_use(g)):
            self._dd.eval(U, ux=ux, uy=uy, leaves=self._leaves)
            if self._multi:
                self._collective(lambda: complete_edges([ux, uy], self._top_ids, self._group))

        def fill(tt):
            for a, b in self._ranges():
                res[:, a:b].copy_(_call_g(g, tt, U[:, a:b], ux[:, a:b], uy[:, a:b]))
        if self._seg is not None and not is_pure(g):   # cut: g runs at every replay
            self._eager(lambda tc=t: fill(self._replay_t + tc))
        else:
            fill(t)
        return res

    def _solve(self, ops, fb, body, out, jump=None, inv_dt=None):
        from . import _lib
        if self._dry:
            return out
        if jump is not None:
            raise UnsupportedConfigurationError("the sharded stepper has no penalized solve")
        tm = self.solve_timer
        if tm is not None:
            import torch
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
        p0, p1 = self._parts
        ops.solve_phase(_lib.HPS_PHASE_UP, p0, p1, fb, body, out)
        if self._multi:
            block = ops.plan.flux_block(out.shape[0])
            self._collective(lambda: exchange_fluxes(block, p0, p1, self._group))
        if self._top_rows(ops):
            self._top_row_sharded(ops, fb, out)
            ops.solve_phase(_lib.HPS_PHASE_DOWN, p0, p1, fb, body, out)
        else:
            ops.solve_phase(_lib.HPS_PHASE_TOP | _lib.HPS_PHASE_DOWN, p0, p1, fb, body, out)
        if tm is not None:
            e1.record()
            tm.append((e0, e1))
        return out

    # -- collectives inside the captured step ----------------------------------------------
    def _collective(self, fn):
        """A collective of the stage solve.  With NCCL it is captured into the
        step's CUDA graph with the kernels around it (NCCL collectives are
        graph-capturable; no host round trip per collective at replay);
        HPSB_GRAPH_COLLECTIVES=0, or a host-staged backend (gloo), cuts the
        graph there instead and issues it eagerly between the segments."""
        dist = _dist()
        captured = (self._seg is not None and dist is not None and dist.get_backend(self._group) == "nccl"
                    and os.environ.get("HPSB_GRAPH_COLLECTIVES", "1") != "0")
        if captured:
            fn()
        else:
            self._eager(fn)

    # -- row-sharded top levels -------------------------------------------
    def _top_rows(self, ops):
        """Whether the levels above lstar run row-sharded over the ranks
        (HPSB_TOP_ROWS=1/0 forces it): each rank then streams 1/world of their
        operators at the price of 2 lstar - 1 small all-reduces per solve.
        That pays for per-node operators (C4: the replicated top levels
        stream ~0.4 ms of operators per solve at 8 ranks); the shared layout's
        top levels are latency-bound and run replicated."""
        e = os.environ.get("HPSB_TOP_ROWS")
        if e is not None:
            return e == "1" and ops.plan.lstar > 0
        return ops.plan.lstar > 0 and ops.layout == "per_node" and self._world > 1

    def _top_row_sharded(self, ops, fb, out):
        """Levels lstar-1 .. 0 up, then 0 .. lstar-1 down, each rank applying
        its share of every level's operator rows; one all-reduce (sum) per
        level completes the level's w3 / fluxes (up) or interface values
        (down) on every rank."""
        import torch
        k, plan, world, rank = out.shape[0], ops.plan, self._world, self._rank
        lms = self.tree.level_maps
        self._put_boundary(fb, out)                        # the Dirichlet data (what TOP wrote)
        for d in reversed(range(plan.lstar)):
            ops.top_level(d, False, rank, world, out)
            if self._multi:
                blocks = [b for b in plan.level_blocks(k, d) if b is not None]
                self._collective(lambda blocks=blocks: allreduce_sum(blocks, self._group))
        for d in range(plan.lstar):
            lm = lms[d]
            stage = self._buf(f"top_stage{d}", (k, lm.count * lm.n3))
            ops.top_level(d, True, rank, world, out, stage)
            if self._multi:
                self._collective(lambda stage=stage: allreduce_sum([stage], self._group))
            idx = self._bufs.get(f"top_j3_{d}")
            if idx is None:
                idx = self._bufs[f"top_j3_{d}"] = torch.as_tensor(np.asarray(lm.j3).ravel(), dtype=torch.long,
                                                                  device=self._dev)
            out.index_copy_(1, idx, stage)

    def gather(self, state):
        """The state with every DOF exact on every rank."""
        from .timestep import StepperState
        u = state.u_device
        squeeze = u.dim() == 1
        U = u.reshape(1, -1) if squeeze else u
        full = gather_owned(U, self._owned, self._group)
        return StepperState(state.t, full[0] if squeeze else full)

    def step(self, state):
        return self.gather(super().step(state))

    def run(self, state, nsteps, check_every=32):
        return self.gather(super().run(state, nsteps, check_every))
