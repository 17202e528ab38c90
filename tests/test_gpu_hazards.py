"""Round-1 correctness hazards, checked on the device against the CPU oracle:

* a nonlinear term whose result storage is reused (g returning u, u_x, or a
  persistent out= buffer) must not corrupt the ARK4 stage history
  (reference timestep.py:262 copies into QG[i]);
* a g that reads the gradient only under a data or time condition receives
  the real gradient every call (reference timestep.py:192-196 always
  evaluates it);
* concurrent solves on two streams (each its own workspace), also beside a
  kernel that holds SMs, give bitwise the serial results and cannot hang the
  dataflow kernel (reference solver.py:84-89: solves are concurrent-safe).
Needs a B200."""

import numpy as np
import pytest

from tests.problems import UNIT, rel_l2, sine_field

pytestmark = pytest.mark.gpu

TOL = 1e-10


def _hb():
    import paper_2306_02526_b200 as hb
    return hb


def _pair(name):
    """(device g on torch tensors, oracle g on numpy arrays) for each case."""
    import torch
    keep = {}

    def out_buffer(t, u, ux, uy):
        b = keep.get("b")
        if b is None or b.shape != u.shape:
            b = keep["b"] = torch.empty_like(u)
        return torch.mul(u, 0.5 - u * u, out=b)

    cases = {
        "returns_u": (lambda t, u, ux, uy: u, lambda t, u, ux, uy: u),
        "returns_ux": (lambda t, u, ux, uy: ux, lambda t, u, ux, uy: ux),
        "out_buffer": (out_buffer, lambda t, u, ux, uy: u * (0.5 - u * u)),
        "data_conditional_grad": (lambda t, u, ux, uy: torch.where(u > 0.3, ux, torch.zeros_like(u)),
                                  lambda t, u, ux, uy: np.where(u > 0.3, ux, 0.0)),
        "time_conditional_grad": (lambda t, u, ux, uy: (u * uy if t > 0.015 else u * 0.5),
                                  lambda t, u, ux, uy: (u * uy if t > 0.015 else u * 0.5)),
    }
    return cases[name]


@pytest.mark.parametrize("name", ["returns_u", "returns_ux", "out_buffer", "data_conditional_grad",
                                  "time_conditional_grad"])
@pytest.mark.parametrize("graph", [True, False])
def test_nonlinear_term_storage_and_gradient(name, graph, monkeypatch):
    from oracle import hps_oracle as O  # checker only
    hb = _hb()
    if not graph:
        monkeypatch.setenv("HPSB_NO_GRAPH", "1")
    gd, go = _pair(name)
    modes = np.random.default_rng(7).uniform(-1, 1, (4, 3))
    u0 = lambda pts: sine_field(modes, pts)
    dt, n, p, steps = 5e-3, 4, 10, 6
    tree = hb.build_tree(UNIT, n, n, p)
    prob = hb.ParabolicProblem(coeffs=hb.OperatorCoefficients(c11=0.05, c22=0.05), g=gd, u0=u0,
                               time_independent_bc=True)
    st = hb.TimeStepper(tree, prob, "ARK4", dt=dt)
    s = st.run(st.initial_state(), steps)
    ot = O.OTree(UNIT, n, n, p)
    ost = O.OStepper(ot, O.OCoeffs(c11=0.05, c22=0.05), O.ark4_tableau(), dt, g=go)
    _, ref = ost.run(0.0, u0(ot.points), steps)
    assert rel_l2(s.u, ref) < TOL, name


def test_concurrent_stream_solves_match_serial():
    """Two streams solving at once (own workspaces), and a solve beside a
    long kernel on a third stream that occupies SMs: bitwise the serial
    results, no hang (the dataflow kernel's tasks only wait on lower tickets)."""
    import torch
    hb = _hb()
    tree = hb.build_tree(UNIT, 32, 32, 12)
    ops = hb.build(tree, hb.OperatorCoefficients(c11=1.0, c22=1.0), sigma=1.0, dt_gamma=1e-4)
    rng = np.random.default_rng(3)
    dev = torch.device("cuda")
    fb = [torch.as_tensor(rng.standard_normal((1, tree.boundary_ids.size)), device=dev) for _ in range(2)]
    body = [torch.as_tensor(rng.standard_normal((1, tree.N)), device=dev) for _ in range(2)]
    ref = [ops.solve_device(fb[i], body[i], torch.empty((1, tree.N), dtype=torch.float64, device=dev))
           for i in range(2)]
    torch.cuda.synchronize()
    streams = [torch.cuda.Stream() for _ in range(3)]
    hog_a = torch.randn(8192, 8192, device=dev)
    for _ in range(3):
        outs = [torch.empty((1, tree.N), dtype=torch.float64, device=dev) for _ in range(2)]
        with torch.cuda.stream(streams[2]):
            hog = hog_a @ hog_a          # holds SMs while the solves launch
        for rep in range(4):
            for i in range(2):
                with torch.cuda.stream(streams[i]):
                    ops.solve_device(fb[i], body[i], outs[i])
        torch.cuda.synchronize()
        for i in range(2):
            assert torch.equal(outs[i], ref[i])
    del hog
    # the public API from two host threads at once (one stream each)
    import threading
    res = [None, None]

    def work(i):
        with torch.cuda.stream(streams[i]):
            res[i] = ops.solve_with_body_load(fb[i][0].cpu().numpy(), body[i][0].cpu().numpy())

    th = [threading.Thread(target=work, args=(i,)) for i in range(2)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for i in range(2):
        assert np.array_equal(res[i], ref[i][0].cpu().numpy())


def test_streams_get_distinct_workspaces():
    import torch
    hb = _hb()
    from paper_2306_02526_b200.solver import device_plan, graph_workspace
    tree = hb.build_tree(UNIT, 4, 4, 8)
    plan = device_plan(tree)
    a = plan.workspace(1)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        b = plan.workspace(1)
    with graph_workspace("x"):
        c = plan.workspace(1)
    assert len({a.data_ptr(), b.data_ptr(), c.data_ptr()}) == 3
    assert plan.workspace(1).data_ptr() == a.data_ptr()
