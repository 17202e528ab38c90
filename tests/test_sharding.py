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
