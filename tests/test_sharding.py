"""Multi-process (gloo, world size 2, CPU) coverage of the multi-GPU host
logic: member partition, sharded problem fields, max-over-ranks timing and
the member all-gather."""

import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2306_02526_b200.sharding import member_slice


def test_member_slices_partition_the_ensemble():
    for k in (1, 4, 7, 64):
        for world in (1, 2, 3, 8):
            spans = [member_slice(k, r, world) for r in range(world)]
            assert spans[0][0] == 0 and spans[-1][1] == k
            assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
            sizes = [b - a for a, b in spans]
            assert max(sizes) - min(sizes) <= 1
    with pytest.raises(ValueError):
        member_slice(4, 2, 2)


def test_shard_problem_slices_member_fields():
    import paper_2306_02526_b200 as hb
    from paper_2306_02526_b200.sharding import shard_problem
    pts = np.random.default_rng(0).uniform(size=(10, 2))
    coef = np.arange(5.0)[:, None] * np.ones((5, 10))
    prob = hb.ParabolicProblem(coeffs=hb.OperatorCoefficients(c11=1.0, c22=1.0),
                               q=hb.SeparableField.product(lambda p: coef + p[:, 0]),
                               u0=lambda p: np.zeros((5, p.shape[0])) + np.arange(5.0)[:, None],
                               g=lambda t, u, ux, uy: u, ncomp=5, time_independent_bc=True)
    sub = shard_problem(prob, 1, 2)          # members 3, 4
    assert sub.ncomp == 2
    assert np.array_equal(sub.u0(pts)[:, 0], [3.0, 4.0])
    assert np.allclose(sub.q(0.0, pts), (coef + pts[:, 0])[3:])
    assert sub.g is prob.g


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    import torch
    import torch.distributed as dist
    from paper_2306_02526_b200.sharding import gather_members, max_over_ranks
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        k, n = 5, 3
        a, b = member_slice(k, rank, world)
        local = torch.arange(a * n, b * n, dtype=torch.float64).reshape(b - a, n)
        full = gather_members(local, k)
        t = max_over_ranks(10.0 + rank)
        out[rank] = (full.numpy().tolist(), t)
    finally:
        dist.destroy_process_group()


def test_gloo_two_ranks_gather_and_max():
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, port, out), nprocs=world, join=True)
    for r in range(world):
        full, t = out[r]
        assert np.array_equal(np.array(full), np.arange(15.0).reshape(5, 3))
        assert t == 11.0


# ---------------------------------------------------------------------------
# subtree sharding: the partition, the per-stage flux
# all-gather, the top-interface gradient completion and the final gather,
# driven by a partitioned restatement of the oracle solve on 2 gloo ranks
# ---------------------------------------------------------------------------

def _partition_solve(ops, part, p0, p1, f, G, exchange, gather, rows=None):
    """The oracle solve (oracle/hps_oracle.py OHps.solve) split like
    hps_solve_phase: UP over the parts' leaves and levels >= lstar, the flux
    exchange, TOP, DOWN over the parts."""
    tree, st = ops.tree, ops.disc.st
    ni, ls, P = st.ni, part.lstar, part.nparts
    k = G.shape[0]
    fb = np.broadcast_to(ops.boundary_values(f), (k, tree.boundary_ids.size))
    lid0, nl = part.leaves(p0, p1)
    own_leaves = range(lid0, lid0 + nl)
    lu = ops.leaf_lu[0]
    w, hleaf = {}, {}
    for l in own_leaves:
        w[l] = lu.solve(G[:, tree.leaf_int_gidx[l]].T).T
        hleaf[l] = w[l] @ ops.D_bi.T
    H, W3 = {}, {}

    def h(kk):
        nd = tree.nodes[kk]
        return hleaf[nd["lid"]] if nd["children"] is None else H[kk]

    def up(kk):
        nd = tree.nodes[kk]
        S, f3, Tst = ops.merges[kk]
        ha, hb = h(nd["children"][0]), h(nd["children"][1])
        W3[kk] = f3.solve((hb[:, nd["i3b"]] - ha[:, nd["i3a"]]).T).T
        H[kk] = np.concatenate([ha[:, nd["i1a"]], hb[:, nd["i2b"]]], axis=1) + W3[kk] @ Tst.T

    def own_nodes(d):
        lvl = [kk for kk in tree.levels[d] if tree.nodes[kk]["children"] is not None]
        per = len(lvl) // P
        return lvl[p0 * per:p1 * per]

    for d in range(tree.depth - 2, ls - 1, -1):      # UP: the parts' levels, deepest first
        for kk in own_nodes(d):
            up(kk)
    top_nodes = tree.levels[ls]
    n12 = tree.nodes[top_nodes[0]]["bnd"].size
    block = np.zeros((k, P, n12))
    for g in range(p0, p1):
        block[:, g] = H[top_nodes[g]]
    block = exchange(block, p0, p1)                  # every part's level-lstar flux
    for g in range(P):
        H[top_nodes[g]] = block[:, g]
    u = np.zeros((k, tree.N))
    u[:, tree.boundary_ids] = fb

    def down(kk):
        nd = tree.nodes[kk]
        u[:, nd["j3"]] = u[:, nd["bnd"]] @ ops.merges[kk][0].T + W3[kk]

    if rows is None:
        for d in range(ls - 1, -1, -1):              # TOP, every level on every rank
            for kk in tree.levels[d]:
                up(kk)
        for d in range(ls):
            for kk in tree.levels[d]:
                down(kk)
    else:
        # TOP row-sharded (hps_top_level): rank r keeps its contiguous share of
        # the level's row space (node-major, R rows per node), zeros elsewhere,
        # and one sum over the ranks per level completes it
        rank, world, allreduce = rows

        def share(nrows):
            m = np.zeros(nrows, dtype=bool)
            m[nrows * rank // world:nrows * (rank + 1) // world] = True
            return m

        for d in range(ls - 1, -1, -1):
            nodes = tree.levels[d]
            for kk in nodes:
                up(kk)
            n3 = W3[nodes[0]].shape[1]
            nh = H[nodes[0]].shape[1] if d > 0 else 0
            R = n3 + nh
            mask = share(len(nodes) * R).reshape(len(nodes), R)
            blk = np.zeros((k, len(nodes), R))
            for j, kk in enumerate(nodes):
                blk[:, j, :n3] = W3[kk]
                if nh:
                    base = np.concatenate([h(tree.nodes[kk]["children"][0])[:, tree.nodes[kk]["i1a"]],
                                           h(tree.nodes[kk]["children"][1])[:, tree.nodes[kk]["i2b"]]], axis=1)
                    blk[:, j, n3:] = H[kk] - base      # the rank's rows of Tstack X33^-1 r3
            blk = allreduce(np.where(mask[None], blk, 0.0))
            for j, kk in enumerate(nodes):
                W3[kk] = blk[:, j, :n3]
                if nh:
                    base = np.concatenate([h(tree.nodes[kk]["children"][0])[:, tree.nodes[kk]["i1a"]],
                                           h(tree.nodes[kk]["children"][1])[:, tree.nodes[kk]["i2b"]]], axis=1)
                    H[kk] = base + blk[:, j, n3:]
        for d in range(ls):
            nodes = tree.levels[d]
            n3 = W3[nodes[0]].shape[1]
            mask = share(len(nodes) * n3).reshape(len(nodes), n3)
            stage = np.zeros((k, len(nodes), n3))
            for j, kk in enumerate(nodes):
                nd = tree.nodes[kk]
                stage[:, j] = u[:, nd["bnd"]] @ ops.merges[kk][0].T + W3[kk]
            stage = allreduce(np.where(mask[None], stage, 0.0))
            for j, kk in enumerate(nodes):
                u[:, tree.nodes[kk]["j3"]] = stage[:, j]
    for d in range(ls, tree.depth - 1):              # DOWN
        for kk in own_nodes(d):
            down(kk)
    for l in own_leaves:
        u[:, tree.leaf_int_gidx[l]] = u[:, tree.leaf_bnd_gidx[l]] @ ops.S_leaf[0].T + w[l]
    return gather(u)


def _subtree_worker(rank, world, port, nparts, out):
    import torch
    import torch.distributed as dist
    from oracle import hps_oracle as O
    from paper_2306_02526_b200.sharding import (SubtreePartition, allreduce_sum, complete_edges,
                                                exchange_fluxes, gather_owned)
    from paper_2306_02526_b200.tree import build_tree
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        n, p, k = 8, 8, 2
        ot = O.OTree(((0.0, 1.0), (0.0, 1.0)), n, n, p)
        ops = O.OHps(O.ODisc(ot, O.OCoeffs(1.0, 1.0)), sigma=1.0, dt_gamma=0.01)
        part = SubtreePartition(build_tree(((0.0, 1.0), (0.0, 1.0)), n, n, p), nparts)
        p0, p1 = part.owner_parts(rank, world)
        rng = np.random.default_rng(5)
        G = rng.standard_normal((k, ot.N))
        f = rng.standard_normal(ot.boundary_ids.size)
        owned = torch.as_tensor(part.owned_ids(p0, p1, with_top=rank == 0))

        def exchange(block, a, b):
            t = torch.from_numpy(np.ascontiguousarray(block))
            return exchange_fluxes(t, a, b).numpy()

        def gather(u):
            return gather_owned(torch.from_numpy(u), owned).numpy()

        u = _partition_solve(ops, part, p0, p1, f, G, exchange, gather)
        ref = ops.solve(np.broadcast_to(f, (k, f.size)), G)

        def allreduce(a):
            t = torch.from_numpy(np.ascontiguousarray(a))
            allreduce_sum([t])
            return t.numpy()

        u_rows = _partition_solve(ops, part, p0, p1, f, G, exchange, gather, rows=(rank, world, allreduce))
        # gradient partial sums of the own leaves, completed on the top interfaces
        uu = rng.standard_normal((1, ot.N))
        lid0, nl = part.leaves(p0, p1)
        gi = ot.leaf_gidx[lid0:lid0 + nl]
        vals = uu[:, gi] @ ops.disc.st.Ex1.T
        part_ux = np.bincount(gi.ravel(), weights=vals[0].ravel(), minlength=ot.N) / np.maximum(ot.mult, 1)
        ux = torch.from_numpy(part_ux[None].copy())
        complete_edges([ux], torch.as_tensor(part.top_ids))
        full_ux = ops.disc.gradient(uu[0])[0]
        check = np.concatenate([part.owned_ids(p0, p1, with_top=False), part.top_ids])
        out[rank] = dict(err=float(np.abs(u - ref).max() / np.abs(ref).max()),
                         err_rows=float(np.abs(u_rows - ref).max() / np.abs(ref).max()),
                         gerr=float(np.abs(ux.numpy()[0, check] - full_ux[check]).max()),
                         owned=part.owned_ids(p0, p1, with_top=rank == 0).tolist())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("nparts", [2, 4])
def test_gloo_two_ranks_subtree_partitioned_solve(nparts):
    world = 2
    port = _free_port()
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_subtree_worker, args=(world, port, nparts, out), nprocs=world, join=True)
    owned = []
    for r in range(world):
        assert out[r]["err"] < 1e-13
        assert out[r]["err_rows"] < 1e-13      # row-sharded top levels
        assert out[r]["gerr"] < 1e-13
        owned += out[r]["owned"]
    # the ranks' owned DOFs partition the global vector
    from paper_2306_02526_b200.tree import build_tree
    N = build_tree(((0.0, 1.0), (0.0, 1.0)), 8, 8, 8).N
    assert sorted(owned) == list(range(N))


def test_subtree_partition_ranges():
    from paper_2306_02526_b200.sharding import SubtreePartition
    from paper_2306_02526_b200.tree import build_tree
    from paper_2306_02526_b200.errors import UnsupportedConfigurationError
    tree = build_tree(((0.0, 1.0), (0.0, 1.0)), 8, 8, 6)
    part = SubtreePartition(tree, 4)
    assert part.lstar == 2 and part.lpp == 16
    assert part.owner_parts(1, 2) == (2, 4)
    assert part.leaves(2, 4) == (32, 32)
    assert part.interior_range(0, 1) == (0, 16 * tree.ni)
    # top interfaces = j3 of the two top parent levels
    lms = tree.level_maps
    assert part.top_ids.size == lms[0].n3 + 2 * lms[1].n3
    allids = np.concatenate([part.owned_ids(g, g + 1, with_top=g == 0) for g in range(4)])
    assert np.array_equal(np.sort(allids), np.arange(tree.N))
    for bad in (3, 128):
        with pytest.raises(UnsupportedConfigurationError):
            SubtreePartition(tree, bad)
    with pytest.raises(UnsupportedConfigurationError):
        part.owner_parts(0, 3)
