"""Device time stepping and leaf evaluations against vectors produced by the
real reference (tests/golden/make_golden.py).  Needs a B200."""

import numpy as np
import pytest

from tests.problems import (UNIT, c4_fields, heat_manufactured, lap_fields, rel_l2, sine_field,
                            var_test_fields)

pytestmark = pytest.mark.gpu

TOL = 1e-10   # north-star parity bar (relative L2, per stage and at the final time)


def _hb():
    import paper_2306_02526_b200 as hb
    return hb


def test_leaf_evaluations_match_reference(golden):
    hb = _hb()
    z = golden("evals_var4x2p9")
    tree = hb.build_tree(UNIT, 4, 2, 9)
    disc = hb.EllipticDiscretization(tree, hb.OperatorCoefficients(**var_test_fields()))
    assert rel_l2(disc.apply_lop(z["u"]), z["lu"]) < 1e-13
    lu1 = disc.apply_lop(z["u"][0])
    assert lu1.shape == z["lu1"].shape and rel_l2(lu1, z["lu1"]) < 1e-13
    ux, uy = disc.gradient(z["u"])
    assert rel_l2(ux, z["ux"]) < 1e-13 and rel_l2(uy, z["uy"]) < 1e-13
    assert rel_l2(disc.flux_jump(z["u"]), z["jump"]) < 1e-13


def _c1_stepper(hb, separable, layout=None):
    tree = hb.build_tree(UNIT, 8, 8, 12)
    phi, uex, q = heat_manufactured()
    if separable:
        qf = hb.SeparableField.product(phi, lambda t: -np.sin(t) + 8 * np.pi ** 2 * np.cos(t))
        ff = hb.SeparableField.product(phi, np.cos)
    else:
        qf, ff = q, uex
    prob = hb.ParabolicProblem(coeffs=hb.OperatorCoefficients(c11=1.0, c22=1.0), q=qf, f=ff,
                               u0=lambda pts: uex(0.0, pts))
    return tree, hb.TimeStepper(tree, prob, "ARK4", dt=1e-3, layout=layout), uex


@pytest.mark.parametrize("separable,layout", [(True, "shared"), (False, "shared"), (True, "per_node")])
def test_c1_heat_matches_reference(golden, separable, layout, monkeypatch):
    hb = _hb()
    z = golden("step_c1")
    tree, st, uex = _c1_stepper(hb, separable, layout)
    monkeypatch.setenv("HPSB_NO_GRAPH", "1")      # eager first step: record every stage solve
    stages = []
    orig = st.ops.solve_device

    def rec(fb, body, out, **kw):
        r = orig(fb, body, out, **kw)
        stages.append(out[0].cpu().numpy().copy())
        return r

    orig_stage = st.ops.solve_stage_device

    def rec_stage(fb, body, out, lu, guard, **kw):
        r = orig_stage(fb, body, out, lu, guard, **kw)
        stages.append(out[0].cpu().numpy().copy())
        return r

    orig_terms = st.ops.solve_stage_terms_device

    def rec_terms(fb, dptr, vecs, rout, out, lu, guard, *a, **kw):
        r = orig_terms(fb, dptr, vecs, rout, out, lu, guard, *a, **kw)
        stages.append(out[0].cpu().numpy().copy())
        return r

    st.ops.solve_device = rec
    st.ops.solve_stage_device = rec_stage
    st.ops.solve_stage_terms_device = rec_terms
    s = st.step(st.initial_state())
    st.ops.solve_device = orig
    st.ops.solve_stage_device = orig_stage
    st.ops.solve_stage_terms_device = orig_terms
    monkeypatch.delenv("HPSB_NO_GRAPH")           # the rest runs as replays of a captured step
    for i, (a, b) in enumerate(zip(stages, z["stages"])):
        assert rel_l2(a, b) < TOL, f"stage {i + 1}"
    assert isinstance(s.u, np.ndarray) and s.u.shape == (tree.N,)
    assert rel_l2(s.u, z["u1"]) < TOL
    s = st.run(s, 9)
    assert rel_l2(s.u, z["u10"]) < TOL
    s = st.run(s, 90)
    assert abs(s.t - float(z["t100"])) < 1e-12
    assert rel_l2(s.u, z["u100"]) < TOL
    assert np.abs(s.u - uex(s.t, tree.points)).max() < 1e-10


def test_allen_cahn_matches_reference(golden):
    hb = _hb()
    z = golden("step_allen_cahn")
    tree = hb.build_tree(UNIT, 8, 8, 12)
    prob = hb.ParabolicProblem(coeffs=hb.OperatorCoefficients(c11=0.01, c22=0.01),
                               g=lambda t, u, ux, uy: u - u ** 3,
                               u0=lambda pts: sine_field(z["modes"], pts), time_independent_bc=True)
    st = hb.TimeStepper(tree, prob, "ARK4", dt=float(z["dt"]))
    s = st.step(st.initial_state())
    assert rel_l2(s.u, z["u1"]) < TOL
    s = st.run(s, 9)
    assert rel_l2(s.u, z["u10"]) < TOL


def test_burgers_variable_coefficients_matches_reference(golden):
    hb = _hb()
    z = golden("step_burgers_var")
    tree = hb.build_tree(UNIT, 8, 8, 10)
    prob = hb.ParabolicProblem(coeffs=hb.OperatorCoefficients(**c4_fields()),
                               g=lambda t, u, ux, uy: -u * ux,
                               u0=lambda pts: sine_field(z["modes"], pts), time_independent_bc=True)
    st = hb.TimeStepper(tree, prob, "ARK4", dt=float(z["dt"]))
    s = st.step(st.initial_state())
    assert rel_l2(s.u, z["u1"]) < TOL
    s = st.run(s, 4)
    assert rel_l2(s.u, z["u5"]) < TOL


@pytest.mark.parametrize("separable", [True, False])
def test_ensemble_matches_reference(golden, separable):
    hb = _hb()
    z = golden("step_ensemble")
    coef = z["modes"]
    tree = hb.build_tree(UNIT, 4, 4, 10)
    qf = (hb.SeparableField.product(lambda pts: sine_field(coef, pts)) if separable
          else (lambda t, pts: sine_field(coef, pts)))
    prob = hb.ParabolicProblem(coeffs=hb.OperatorCoefficients(**lap_fields()), q=qf,
                               u0=lambda pts: np.zeros((4, pts.shape[0])),
                               time_independent_bc=True, ncomp=4)
    st = hb.TimeStepper(tree, prob, "ARK4", dt=float(z["dt"]))
    s = st.run(st.initial_state(), 3)
    assert s.u.shape == (4, tree.N)
    assert rel_l2(s.u, z["u3"]) < TOL


def test_backward_euler_matches_reference(golden):
    hb = _hb()
    z = golden("step_be")
    tree = hb.build_tree(UNIT, 4, 4, 10)
    phi, uex, q = heat_manufactured()
    prob = hb.ParabolicProblem(coeffs=hb.OperatorCoefficients(**lap_fields()), q=q, f=uex,
                               u0=lambda pts: uex(0.0, pts))
    st = hb.TimeStepper(tree, prob, "BE", dt=float(z["dt"]))
    s = st.run(st.initial_state(), 3)
    assert rel_l2(s.u, z["u3"]) < TOL


@pytest.mark.parametrize("form", ["slope", "slope-penalized"])
def test_slope_formulations_match_reference(golden, form):
    hb = _hb()
    z = golden("step_slope")
    tree = hb.build_tree(UNIT, 4, 4, 10)
    phi, uex, q = heat_manufactured()
    prob = hb.ParabolicProblem(coeffs=hb.OperatorCoefficients(**lap_fields()), q=q, f=uex,
                               f_t=lambda t, pts: -phi(pts) * np.sin(t),
                               u0=lambda pts: uex(0.0, pts))
    st = hb.TimeStepper(tree, prob, "ARK4", dt=1e-3, formulation=form)
    s = st.run(st.initial_state(), 3)
    assert rel_l2(s.u, z[form.replace("-", "_")]) < TOL


def test_nonlinear_penalized_slope_matches_reference(golden):
    hb = _hb()
    z = golden("step_slope")
    tree = hb.build_tree(UNIT, 4, 4, 10)
    prob = hb.ParabolicProblem(coeffs=hb.OperatorCoefficients(c11=0.01, c22=0.01),
                               g=lambda t, u, ux, uy: u - u ** 3,
                               u0=lambda pts: sine_field(z["modes"], pts), time_independent_bc=True)
    st = hb.TimeStepper(tree, prob, "ARK4", dt=1e-2, formulation="slope-penalized")
    s = st.run(st.initial_state(), 3)
    assert rel_l2(s.u, z["ac_pen"]) < TOL


def test_divergence_guard_reports_step():
    hb = _hb()
    tree = hb.build_tree(UNIT, 2, 2, 8)
    # explosive reaction: u_t = Lu + 1e4 u^2 blows up within a few steps
    prob = hb.ParabolicProblem(coeffs=hb.OperatorCoefficients(c11=1.0, c22=1.0),
                               g=lambda t, u, ux, uy: 1e4 * u * u,
                               u0=lambda pts: 10.0 + 0 * pts[:, 0], time_independent_bc=True,
                               f=lambda t, pts: 10.0 + 0 * pts[:, 0])
    st = hb.TimeStepper(tree, prob, "ARK4", dt=1e-2)
    with pytest.raises(hb.DivergenceError) as e:
        st.run(st.initial_state(), 50)
    assert e.value.step is not None and e.value.step <= 50


def test_mismatched_shift_is_rejected():
    hb = _hb()
    tree = hb.build_tree(UNIT, 2, 2, 8)
    prob = hb.ParabolicProblem(coeffs=hb.OperatorCoefficients(c11=1.0, c22=1.0),
                               u0=lambda pts: 0 * pts[:, 0])
    st = hb.TimeStepper(tree, prob, "ARK4", dt=1e-2)
    st.dt = 2e-2
    with pytest.raises(hb.UnsupportedConfigurationError):
        st.step(st.initial_state())
    st.set_dt(5e-3)
    st.step(st.initial_state())


@pytest.mark.parametrize("layout", ["shared", "per_node"])
def test_graph_replay_matches_eager_stepping(monkeypatch, layout):
    """A captured step replayed with per-step coefficient tables gives the
    same trajectory as eager launches (same kernels, same coefficients)."""
    hb = _hb()
    tree, st_g, uex = _c1_stepper(hb, True, layout)
    s_g = st_g.run(st_g.initial_state(), 12, check_every=5)
    assert st_g._graph is not None
    monkeypatch.setenv("HPSB_NO_GRAPH", "1")
    tree, st_e, _ = _c1_stepper(hb, True, layout)
    s_e = st_e.run(st_e.initial_state(), 12)
    assert abs(s_g.t - s_e.t) < 1e-15
    assert rel_l2(s_g.u, s_e.u) < 1e-15
    assert st_g._step_count == st_e._step_count == 12


def test_graph_replay_nonlinear_and_backward_euler(golden):
    hb = _hb()
    z = golden("step_allen_cahn")
    tree = hb.build_tree(UNIT, 8, 8, 12)
    prob = hb.ParabolicProblem(coeffs=hb.OperatorCoefficients(c11=0.01, c22=0.01),
                               g=lambda t, u, ux, uy: u - u ** 3,
                               u0=lambda pts: sine_field(z["modes"], pts), time_independent_bc=True)
    st = hb.TimeStepper(tree, prob, "ARK4", dt=float(z["dt"]))
    s = st.run(st.initial_state(), 10)          # 1 eager probe step, 9 replays
    assert st._graph is not None
    assert rel_l2(s.u, z["u10"]) < TOL
    zb = golden("step_be")
    tree = hb.build_tree(UNIT, 4, 4, 10)
    phi, uex, q = heat_manufactured()
    prob = hb.ParabolicProblem(coeffs=hb.OperatorCoefficients(**lap_fields()),
                               q=hb.SeparableField.product(phi, lambda t: -np.sin(t) + 8 * np.pi ** 2 * np.cos(t)),
                               f=hb.SeparableField.product(phi, np.cos), u0=lambda pts: uex(0.0, pts))
    st = hb.TimeStepper(tree, prob, "BE", dt=float(zb["dt"]))
    s = st.run(st.initial_state(), 3)
    assert st._graph is not None
    assert rel_l2(s.u, zb["u3"]) < TOL


@pytest.mark.parametrize("key,tab,form,dt", [("ark4", "ARK4", "stage", 1e-2), ("ark4_slope", "ARK4", "slope", 1e-2),
                                             ("be_var", "BE", "stage", 5e-2)])
def test_step_map_assembly_matches_reference(golden, key, tab, form, dt):
    """stability.py:59-85 on the device: 64 basis fields per multi-rhs step."""
    hb = _hb()
    from paper_2306_02526_b200.stability import analyze, assemble_step_map
    z = golden("stability_4x4p6")
    tree = hb.build_tree(UNIT, 4, 4, 6)
    coeffs = hb.OperatorCoefficients(**(var_test_fields() if key == "be_var" else lap_fields()))
    prob = hb.ParabolicProblem(coeffs=coeffs, u0=lambda pts: np.zeros(pts.shape[0]), time_independent_bc=True)
    M = assemble_step_map(tree, prob, tab, dt, formulation=form)
    assert rel_l2(M, z[key + "_M"]) < TOL
    spec = analyze(M, dt=dt, scheme=tab, formulation=form)
    assert abs(spec.spectral_radius - float(z[key + "_rho"])) < 1e-10
    assert spec.zero_count == int(z[key + "_zeros"])
    with pytest.raises(hb.UnsupportedConfigurationError):
        assemble_step_map(tree, hb.ParabolicProblem(coeffs=coeffs, g=lambda t, u, ux, uy: u), tab, dt)


@pytest.mark.parametrize("p", [10, 12, 16])
def test_gradient_kernel_matches_oracle(p):
    """The register-row gradient kernel (stage.cu k_leaf_grad) against the
    oracle's interface-averaged gradient (operators.py:303-317)."""
    hb = _hb()
    from oracle import hps_oracle as O
    tree = hb.build_tree(UNIT, 4, 4, p)
    disc = hb.EllipticDiscretization(tree, hb.OperatorCoefficients(**var_test_fields()))
    od = O.ODisc(O.OTree(UNIT, 4, 4, p), O.OCoeffs(**var_test_fields()))
    u = np.random.default_rng(p).standard_normal((3, tree.N))
    ux, uy = disc.gradient(u)
    rx, ry = od.gradient(u)
    assert rel_l2(ux, rx) < 1e-13 and rel_l2(uy, ry) < 1e-13


def test_step_host_overlapped_copies_match_step():
    """TimeStepper.step_host (host state in, host result out, copies on their
    own streams) gives the same states as step()."""
    import torch
    hb = _hb()
    tree, st, uex = _c1_stepper(hb, True)
    s0 = st.initial_state()
    u0 = torch.as_tensor(np.asarray(s0.u), dtype=torch.float64).pin_memory()
    ref = st.step(hb.StepperState(0.0, u0.clone())).u
    outs = [torch.empty_like(u0).pin_memory() for _ in range(3)]
    for o in outs:
        st.step_host(0.0, u0, o)
    st.sync_host()
    for o in outs:
        assert np.array_equal(o.numpy(), ref)


@pytest.mark.parametrize("graph", [True, False])
def test_ark5_matches_reference(golden, graph, monkeypatch):
    """ARK5(4)8L[2]SA (reference tableaux.py:157-221): 7 implicit stages per
    step, stage right-hand sides of up to 15 terms (past the fused
    stage-terms kernel's 12: the combination fallback), the root Dirichlet
    product of 8 boundary-data rows per step; per stage and per step."""
    hb = _hb()
    z = golden("step_ark5")
    if not graph:
        monkeypatch.setenv("HPSB_NO_GRAPH", "1")
    tree = hb.build_tree(UNIT, 4, 4, 10)
    phi, uex, q = heat_manufactured()
    prob = hb.ParabolicProblem(coeffs=hb.OperatorCoefficients(**lap_fields()),
                               q=hb.SeparableField.product(phi, lambda t: -np.sin(t) + 8 * np.pi ** 2 * np.cos(t)),
                               f=hb.SeparableField.product(phi, np.cos), u0=lambda pts: uex(0.0, pts))
    st = hb.TimeStepper(tree, prob, "ARK5", dt=float(z["dt"]))
    assert st.pair.s == 8
    s = st.step(st.initial_state())
    assert rel_l2(s.u, z["u1"]) < TOL
    s = st.run(s, 4)
    assert rel_l2(s.u, z["u5"]) < TOL
    prob = hb.ParabolicProblem(coeffs=hb.OperatorCoefficients(c11=0.01, c22=0.01),
                               g=lambda t, u, ux, uy: u - u ** 3,
                               u0=lambda pts: sine_field(z["ac_modes"], pts), time_independent_bc=True)
    st = hb.TimeStepper(tree, prob, "ARK5", dt=float(z["ac_dt"]))
    s = st.run(st.initial_state(), 3)
    assert rel_l2(s.u, z["ac_u3"]) < TOL


def test_ark5_stages_match_reference(golden, monkeypatch):
    hb = _hb()
    z = golden("step_ark5")
    monkeypatch.setenv("HPSB_NO_GRAPH", "1")
    from tests.test_gpu_scale import _record_stages
    tree = hb.build_tree(UNIT, 4, 4, 10)
    phi, uex, q = heat_manufactured()
    prob = hb.ParabolicProblem(coeffs=hb.OperatorCoefficients(**lap_fields()), q=q, f=uex,
                               u0=lambda pts: uex(0.0, pts))
    st = hb.TimeStepper(tree, prob, "ARK5", dt=float(z["dt"]))
    stages = []
    restore = _record_stages(st, stages)
    s = st.step(st.initial_state())
    restore()
    assert len(stages) == 7
    for i, (a, b) in enumerate(zip(stages, z["stages"])):
        assert rel_l2(a[0], b) < TOL, f"stage {i + 1}"
    assert rel_l2(s.u, z["u1"]) < TOL


def test_plain_numpy_fields_and_g_run_on_device_arrays():
    """The reference caller's plain numpy callables (q, f, an undeclared g)
    run on the GPU through npgpu.DeviceArray once they matched the host call;
    the trajectory equals the one with SeparableField / declared g, and a
    callable outside the mapped numpy subset still runs (on the host)."""
    import numpy as np
    import paper_2306_02526_b200 as hb
    from paper_2306_02526_b200.timestep import _Field
    pts = np.random.default_rng(1).random((5000, 2))
    fn = lambda t, p: np.where(p[:, 0] > 0.5, np.sin(2 * np.pi * p[:, 1]), np.exp(-p[:, 0])) * np.cos(t)
    F = _Field(fn, pts, 1, "cuda")
    v = F.eval_now(0.4)
    assert F._device_ok is True and v.is_cuda
    assert np.abs(v.cpu().numpy()[0] - fn(0.4, pts)).max() < 1e-14
    h = lambda t, p: np.linalg.norm(p, axis=1) * t        # not mapped: host
    H = _Field(h, pts, 1, "cuda")
    assert np.array_equal(H.eval_now(0.4).cpu().numpy()[0], h(0.4, pts)) and H._device_ok is False

    tree = hb.build_tree(((0.0, 1.0), (0.0, 1.0)), 8, 8, 10)
    phi = lambda p: np.sin(2 * np.pi * p[:, 0]) * np.sin(2 * np.pi * p[:, 1])
    def run(plain):
        if plain:
            q = lambda t, p: phi(p) * (-np.sin(t) + 8 * np.pi ** 2 * np.cos(t))
            f = lambda t, p: phi(p) * np.cos(t)
            g = lambda t, u, ux, uy: -0.1 * np.sin(u)
        else:
            q = hb.SeparableField.product(phi, lambda t: -np.sin(t) + 8 * np.pi ** 2 * np.cos(t))
            f = hb.SeparableField.product(phi, np.cos)
            g = hb.declare_nonlinear(lambda t, u, ux, uy: -0.1 * torch_sin(u), ux=False, uy=False, pure=True)
        prob = hb.ParabolicProblem(coeffs=hb.OperatorCoefficients(c11=1.0, c22=1.0), q=q, f=f, g=g, u0=phi)
        st = hb.TimeStepper(tree, prob, "ARK4", dt=1e-3)
        return st.run(st.initial_state(), 3).u, st
    import torch
    torch_sin = torch.sin
    a, _ = run(False)
    b, st = run(True)
    assert np.abs(a - b).max() <= 1e-13 * np.abs(a).max()
    assert getattr(st.problem.g, "_hb_npdev", None) is True


@pytest.mark.parametrize("root_sep", [True, False])
def test_nonzero_separable_boundary_data_matches_oracle(root_sep, monkeypatch):
    """Two-term separable Dirichlet data that does not vanish on the boundary
    (the manufactured heat problems' data does): the root Dirichlet products
    from the per-operator-set rows S_root F_m (root_sep) and from a pass over
    the root operator per step, eager and captured, against the oracle
    stepper (reference timestep.py:237-266, solver.py:259-265)."""
    hb = _hb()
    from oracle import hps_oracle as O
    if not root_sep:
        monkeypatch.setenv("HPSB_NO_ROOT_SEP", "1")
    x, y = (lambda p: p[:, 0]), (lambda p: p[:, 1])
    phi1 = lambda p: np.sin(x(p) + 2 * y(p)) + 2.0
    phi2 = lambda p: x(p) * y(p) + np.cos(3 * x(p))
    emt = lambda t: np.exp(-t)
    # u = cos(t) phi1 + exp(-t) phi2;  q = u_t - lap u
    f = hb.SeparableField([(phi1, np.cos), (phi2, emt)])
    q = hb.SeparableField([(lambda p: -phi1(p), np.sin),
                           (lambda p: -phi2(p) + 9 * np.cos(3 * x(p)), emt),
                           (lambda p: 5 * np.sin(x(p) + 2 * y(p)), np.cos)])
    uex = lambda t, p: np.cos(t) * phi1(p) + emt(t) * phi2(p)
    n, p_, dt, nsteps = 8, 10, 2e-3, 4
    tree = hb.build_tree(UNIT, n, n, p_)
    prob = hb.ParabolicProblem(coeffs=hb.OperatorCoefficients(c11=1.0, c22=1.0), q=q, f=f,
                               u0=lambda pts: uex(0.0, pts))
    ot = O.OTree(UNIT, n, n, p_)
    ost = O.OStepper(ot, O.OCoeffs(c11=1.0, c22=1.0), O.ark4_tableau(), dt, q=q, f=f)
    _, uref = ost.run(0.0, uex(0.0, ot.points), nsteps)
    st = hb.TimeStepper(tree, prob, "ARK4", dt=dt)
    s = st.run(st.initial_state(), nsteps)              # 1 eager step, then replays of the captured step
    assert st._graph is not None
    assert (getattr(st.ops, "_root_sep", None) is not None) == root_sep
    assert rel_l2(s.u, uref) < TOL
    assert rel_l2(s.u, uex(nsteps * dt, tree.points)) < 1e-6      # and the manufactured solution
    monkeypatch.setenv("HPSB_NO_GRAPH", "1")
    st2 = hb.TimeStepper(tree, prob, "ARK4", dt=dt)
    s2 = st2.run(st2.initial_state(), nsteps)
    assert rel_l2(s2.u, uref) < TOL


def test_stage_history_by_leaf_grid_products_switch():
    """HPSB_LU_PRODUCTS=1 (read once per process): the fused stage's history
    L u_i by the two leaf-grid products instead of the interior equation --
    two ARK4 steps of the manufactured heat problem against the oracle in a
    fresh process (reference timestep.py:259-261)."""
    import os
    import subprocess
    import sys
    code = (
        "import numpy as np, paper_2306_02526_b200 as hb\n"
        "from oracle import hps_oracle as O\n"
        "unit = ((0.0, 1.0), (0.0, 1.0))\n"
        "phi = lambda p: np.sin(2 * np.pi * p[:, 0]) * np.sin(2 * np.pi * p[:, 1]) + p[:, 0]\n"
        "tau = lambda t: -np.sin(t) + 8 * np.pi ** 2 * np.cos(t)\n"
        "tree = hb.build_tree(unit, 8, 8, 12)\n"
        "prob = hb.ParabolicProblem(coeffs=hb.OperatorCoefficients(c11=1.0, c22=1.0),\n"
        "    q=hb.SeparableField.product(phi, tau), f=hb.SeparableField.product(phi, np.cos), u0=phi)\n"
        "st = hb.TimeStepper(tree, prob, 'ARK4', dt=1e-3)\n"
        "s = st.run(st.initial_state(), 3)\n"
        "ot = O.OTree(unit, 8, 8, 12)\n"
        "ost = O.OStepper(ot, O.OCoeffs(c11=1.0, c22=1.0), O.ark4_tableau(), 1e-3,\n"
        "    q=lambda t, p: phi(p) * tau(t), f=lambda t, p: phi(p) * np.cos(t))\n"
        "_, uref = ost.run(0.0, phi(ot.points), 3)\n"
        "err = np.linalg.norm(s.u - uref) / np.linalg.norm(uref)\n"
        "assert err < 1e-10, err\n"
        "print('ok', err)\n")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, HPSB_LU_PRODUCTS="1")
    env["PYTHONPATH"] = root + os.pathsep + env.get("PYTHONPATH", "")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0 and "ok" in r.stdout, (r.stdout[-500:], r.stderr[-2000:])


@pytest.mark.parametrize("p", [7, 9, 11, 13, 15])
def test_fused_stage_odd_leaf_orders_match_oracle(p):
    """Odd interior orders q = p - 2 (unvectorised stores of u_int / L u in the
    leaf kernel, q + 2 not a multiple of 4): three ARK4 steps with nonzero
    boundary data against the oracle (reference timestep.py:237-266)."""
    hb = _hb()
    from oracle import hps_oracle as O
    phi = lambda pts: np.cos(pts[:, 0] + 0.5) * np.cosh(0.7 * pts[:, 1])
    tau = lambda t: 1.0 + 0.3 * np.sin(5 * t)
    f = hb.SeparableField.product(phi, tau)
    q = hb.SeparableField([(phi, lambda t: 1.5 * np.cos(5 * t)), (lambda pts: 0.51 * phi(pts), tau)])
    n, dt = 4, 1e-3
    tree = hb.build_tree(UNIT, n, n, p)
    prob = hb.ParabolicProblem(coeffs=hb.OperatorCoefficients(c11=1.0, c22=1.0), q=q, f=f, u0=phi)
    st = hb.TimeStepper(tree, prob, "ARK4", dt=dt)
    s = st.run(st.initial_state(), 3)
    ot = O.OTree(UNIT, n, n, p)
    ost = O.OStepper(ot, O.OCoeffs(c11=1.0, c22=1.0), O.ark4_tableau(), dt, q=q, f=f)
    _, uref = ost.run(0.0, phi(ot.points), 3)
    assert rel_l2(s.u, uref) < TOL
