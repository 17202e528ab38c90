"""Subtree-partitioned solves and the subtree-sharded stepper on the device
(SURVEY.md 8(e)).  Needs a B200.  The multi-GPU exchange itself is covered
on the CPU (tests/test_sharding.py, gloo); here the part-restricted kernels
run on one GPU: every part of a plan partitioned into P subtrees solved
phase by phase must reproduce the reference goldens, and the sharded stepper
(one rank owning every part, or two gloo ranks sharing the GPU) must track
the single-GPU stepper."""

import os
import socket

import numpy as np
import pytest

from tests.problems import SOLVE_CASES, UNIT, c4_fields, heat_manufactured, rel_l2, sine_field

pytestmark = pytest.mark.gpu

TOL = 1e-10


def _ops(z, name, layout, nparts, keep_dtn=False):
    import paper_2306_02526_b200 as hb
    fields, bounds = SOLVE_CASES[name]
    n1, n2, p = (int(v) for v in z["shape"])
    tree = hb.build_tree(bounds, n1, n2, p)
    ops = hb.build(tree, hb.OperatorCoefficients(**fields()), sigma=float(z["sigma"]),
                   dt_gamma=float(z["dt_gamma"]), keep_dtn=keep_dtn, layout=layout, nparts=nparts)
    return tree, ops


CASES = [("heat8x8p16", 2), ("heat8x8p16", 8), ("c4var4x4p10", 4), ("heat4x4p12k3", 2),
         ("var4x2p9", 2)]


@pytest.mark.parametrize("layout", ["per_node", "shared"])
@pytest.mark.parametrize("name,nparts", CASES)
def test_partitioned_plan_solves_match_reference(golden, name, nparts, layout):
    import torch
    from paper_2306_02526_b200 import _lib
    z = golden("solve_" + name)
    tree, ops = _ops(z, name, layout, nparts, keep_dtn=True)
    assert ops.plan.nparts == nparts
    # whole solve through hps_solve on the partitioned operator set
    u = ops.solve_with_body_load(z["f"], z["g"])
    assert rel_l2(u, z["u"]) < TOL
    assert rel_l2(ops.solve_homogeneous(z["f"]), z["u_hom"]) < TOL
    # hooks read per-part panels
    if "root_S" in z:
        assert rel_l2(ops.merge_operators(0).S, z["root_S"]) < TOL
    assert rel_l2(ops.leaf_operators(tree.L - 1).T, ops.leaf_operators(tree.L - 1).T) == 0.0
    # phase by phase, one part at a time
    G = torch.as_tensor(np.atleast_2d(z["g"]), device="cuda").contiguous()
    k = G.shape[0]
    fb = ops._boundary_values(z["f"], G.device)
    out = torch.zeros((k, tree.N), dtype=torch.float64, device="cuda")
    lpp = tree.L // nparts
    for g in range(nparts):
        body = G[:, g * lpp * tree.ni:]
        ops.solve_phase(_lib.HPS_PHASE_UP, g, g + 1, fb, body, out)
    ops.solve_phase(_lib.HPS_PHASE_TOP, 0, nparts, fb, G, out)
    for g in range(nparts):
        ops.solve_phase(_lib.HPS_PHASE_DOWN, g, g + 1, fb, G[:, g * lpp * tree.ni:], out)
    ph = out.cpu().numpy()
    ph = ph[0] if np.ndim(z["u"]) == 1 else ph
    assert rel_l2(ph, z["u"]) < TOL
    assert np.abs(ph - u).max() <= 1e-13 * np.abs(u).max()


def test_partitioned_plan_rejects_bad_part_counts():
    import paper_2306_02526_b200 as hb
    from paper_2306_02526_b200.errors import HpstepError
    tree = hb.build_tree(UNIT, 4, 4, 8)
    for bad in (3, 16):
        with pytest.raises(HpstepError):
            hb.build(tree, hb.OperatorCoefficients(c11=1.0, c22=1.0), sigma=1.0, dt_gamma=0.01, nparts=bad)


def _heat(hb, n, p):
    tree = hb.build_tree(UNIT, n, n, p)
    phi, uex, q = heat_manufactured()
    prob = hb.ParabolicProblem(coeffs=hb.OperatorCoefficients(c11=1.0, c22=1.0),
                               q=hb.SeparableField.product(phi, lambda t: -np.sin(t) + 8 * np.pi ** 2 * np.cos(t)),
                               f=hb.SeparableField.product(phi, np.cos), u0=lambda pts: uex(0.0, pts))
    return tree, prob


def _burgers(hb, n, p, modes):
    tree = hb.build_tree(UNIT, n, n, p)
    prob = hb.ParabolicProblem(coeffs=hb.OperatorCoefficients(**c4_fields()),
                               g=lambda t, u, ux, uy: -u * ux,
                               u0=lambda pts: sine_field(modes, pts), time_independent_bc=True)
    return tree, prob


def _modes():
    return np.random.default_rng(3).uniform(-1, 1, size=(4, 4))


@pytest.mark.parametrize("kind,nparts,graph", [("heat", 2, True), ("heat", 4, False), ("burgers", 2, True),
                                              ("burgers", 4, False)])
def test_sharded_stepper_single_rank_matches_stepper(kind, nparts, graph, monkeypatch):
    import paper_2306_02526_b200 as hb
    from paper_2306_02526_b200.sharding import ShardedTimeStepper
    tree, prob = _heat(hb, 8, 12) if kind == "heat" else _burgers(hb, 8, 10, _modes())
    dt = 1e-3 if kind == "heat" else 2e-3
    if not graph:
        monkeypatch.setenv("HPSB_NO_GRAPH", "1")
    ref = hb.TimeStepper(tree, prob, "ARK4", dt=dt).run(hb.TimeStepper(tree, prob, "ARK4", dt=dt).initial_state(), 6)
    sh = ShardedTimeStepper(tree, prob, "ARK4", dt=dt, nparts=nparts)
    s = sh.run(sh.initial_state(), 6)
    assert abs(s.t - ref.t) < 1e-14
    assert rel_l2(s.u, ref.u) < 1e-12


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _two_rank_worker(rank, world, port, kind, out):
    import torch.distributed as dist
    import paper_2306_02526_b200 as hb
    from paper_2306_02526_b200.sharding import ShardedTimeStepper
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        tree, prob = _heat(hb, 8, 12) if kind == "heat" else _burgers(hb, 8, 10, _modes())
        dt = 1e-3 if kind == "heat" else 2e-3
        sh = ShardedTimeStepper(tree, prob, "ARK4", dt=dt)
        s = sh.run(sh.initial_state(), 4)
        out[rank] = s.u.tolist()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("kind", ["heat", "burgers"])
def test_sharded_stepper_two_gloo_ranks_match_stepper(kind):
    """Two ranks (gloo, host-staged exchange) sharing the one GPU: no kernel
    waits on another rank, the exchanges are host collectives between launches."""
    import torch.multiprocessing as mp
    import paper_2306_02526_b200 as hb
    tree, prob = _heat(hb, 8, 12) if kind == "heat" else _burgers(hb, 8, 10, _modes())
    dt = 1e-3 if kind == "heat" else 2e-3
    st = hb.TimeStepper(tree, prob, "ARK4", dt=dt)
    ref = st.run(st.initial_state(), 4).u
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_two_rank_worker, args=(2, _free_port(), kind, out), nprocs=2, join=True)
    for r in range(2):
        assert rel_l2(np.array(out[r]), ref) < 1e-12


def test_sharded_backward_euler_matches_stepper():
    import paper_2306_02526_b200 as hb
    from paper_2306_02526_b200.sharding import ShardedTimeStepper
    tree, prob = _heat(hb, 8, 12)
    ref = hb.TimeStepper(tree, prob, "BE", dt=1e-2)
    r = ref.run(ref.initial_state(), 4)
    sh = ShardedTimeStepper(tree, prob, "BE", dt=1e-2, nparts=4)
    s = sh.run(sh.initial_state(), 4)
    assert rel_l2(s.u, r.u) < 1e-12


@pytest.mark.parametrize("layout", ["per_node", "shared"])
@pytest.mark.parametrize("name,nparts", [("heat8x8p16", 8), ("c4var4x4p10", 4), ("heat4x4p12k3", 2)])
@pytest.mark.parametrize("nranks", [1, 3])
def test_row_sharded_top_levels_match_reference(golden, name, nparts, layout, nranks):
    """The top levels (< lstar) row-sharded over `nranks` ranks (hps_top_level),
    the ranks' shares run one after another on this GPU and summed on the
    host side -- what the per-level all-reduce does -- then the parts' DOWN
    phases: the reference solution."""
    import torch
    from paper_2306_02526_b200 import _lib
    z = golden("solve_" + name)
    tree, ops = _ops(z, name, layout, nparts)
    plan = ops.plan
    G = torch.as_tensor(np.atleast_2d(z["g"]), device="cuda").contiguous()
    k = G.shape[0]
    fb = ops._boundary_values(z["f"], G.device)
    out = torch.zeros((k, tree.N), dtype=torch.float64, device="cuda")
    lpp = tree.L // nparts
    for g in range(nparts):
        ops.solve_phase(_lib.HPS_PHASE_UP, g, g + 1, fb, G[:, g * lpp * tree.ni:], out)
    bid = torch.as_tensor(tree.boundary_ids, device="cuda")
    out[:, bid] = fb.expand(k, -1) if fb.shape[0] == 1 else fb
    for d in reversed(range(plan.lstar)):
        acc = None
        for r in range(nranks):
            ops.top_level(d, False, r, nranks, out)
            blocks = [b.clone() for b in plan.level_blocks(k, d) if b is not None]
            acc = blocks if acc is None else [a + b for a, b in zip(acc, blocks)]
        for b, a in zip([b for b in plan.level_blocks(k, d) if b is not None], acc):
            b.copy_(a)
    for d in range(plan.lstar):
        lm = tree.level_maps[d]
        tot = torch.zeros((k, lm.count * lm.n3), dtype=torch.float64, device="cuda")
        for r in range(nranks):
            stage = torch.empty_like(tot)
            ops.top_level(d, True, r, nranks, out, stage)
            tot += stage
        out[:, torch.as_tensor(np.asarray(lm.j3).ravel(), device="cuda")] = tot
    for g in range(nparts):
        ops.solve_phase(_lib.HPS_PHASE_DOWN, g, g + 1, fb, G[:, g * lpp * tree.ni:], out)
    ph = out.cpu().numpy()
    ph = ph[0] if np.ndim(z["u"]) == 1 else ph
    assert rel_l2(ph, z["u"]) < TOL


@pytest.mark.parametrize("layout", ["per_node", "shared"])
def test_sharded_stepper_row_sharded_top_single_rank(layout, monkeypatch):
    import paper_2306_02526_b200 as hb
    from paper_2306_02526_b200.sharding import ShardedTimeStepper
    monkeypatch.setenv("HPSB_TOP_ROWS", "1")
    tree, prob = _heat(hb, 8, 12)
    ref = hb.TimeStepper(tree, prob, "ARK4", dt=1e-3, layout=layout)
    r = ref.run(ref.initial_state(), 5)
    sh = ShardedTimeStepper(tree, prob, "ARK4", dt=1e-3, nparts=4, layout=layout)
    s = sh.run(sh.initial_state(), 5)
    assert rel_l2(s.u, r.u) < 1e-12


def _two_rank_rows_worker(rank, world, port, out):
    os.environ["HPSB_TOP_ROWS"] = "1"
    _two_rank_worker(rank, world, port, "burgers", out)


def test_sharded_stepper_row_sharded_top_two_gloo_ranks():
    """Row-sharded top levels over two gloo ranks sharing the GPU (per-level
    host-staged all-reduces between launches; no kernel waits on another rank)."""
    import torch.multiprocessing as mp
    import paper_2306_02526_b200 as hb
    tree, prob = _burgers(hb, 8, 10, _modes())
    st = hb.TimeStepper(tree, prob, "ARK4", dt=2e-3)
    ref = st.run(st.initial_state(), 4).u
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_two_rank_rows_worker, args=(2, _free_port(), out), nprocs=2, join=True)
    for r in range(2):
        assert rel_l2(np.array(out[r]), ref) < 1e-12


def _nccl_one_rank_worker(rank, world, port, mode, out):
    """One NCCL rank on this GPU with the collectives forced (a one-rank group
    makes them no-op copies, but they are issued and captured like at N > 1)."""
    import torch
    import torch.distributed as dist
    import paper_2306_02526_b200 as hb
    from paper_2306_02526_b200.sharding import ShardedTimeStepper
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), HPSB_FORCE_COLLECTIVES="1")
    if mode == "cut":
        os.environ["HPSB_GRAPH_COLLECTIVES"] = "0"
    if mode == "rows":
        os.environ["HPSB_TOP_ROWS"] = "1"
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", 0))
    try:
        tree, prob = _burgers(hb, 8, 10, _modes())
        sh = ShardedTimeStepper(tree, prob, "ARK4", dt=2e-3, nparts=4)
        s = sh.run(sh.initial_state(), 4)
        out["u"] = s.u.tolist()
        out["graph"] = sh._graph is not None
        out["segments"] = len(sh._graph["graph"].parts) if sh._graph is not None else -1
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["captured", "cut", "rows"])
def test_sharded_stepper_nccl_collectives_in_graph(mode):
    """The stage solve's collectives issued through NCCL: captured into the
    step's CUDA graph (default; one graph segment per step besides the cuts
    around g), or cut out of it (HPSB_GRAPH_COLLECTIVES=0); same trajectory
    as the single-GPU stepper."""
    import torch.multiprocessing as mp
    import paper_2306_02526_b200 as hb
    tree, prob = _burgers(hb, 8, 10, _modes())
    st = hb.TimeStepper(tree, prob, "ARK4", dt=2e-3)
    ref = st.run(st.initial_state(), 4).u
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_nccl_one_rank_worker, args=(1, _free_port(), mode, out), nprocs=1, join=True)
    assert out["graph"]
    assert rel_l2(np.array(out["u"]), ref) < 1e-12
    if mode == "cut":
        assert out["segments"] > 6          # cut at every collective (and around g)
