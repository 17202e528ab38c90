"""Device solve / build parity against the reference goldens (needs a B200)."""

import numpy as np
import pytest

from tests.problems import SOLVE_CASES, rel_l2

pytestmark = pytest.mark.gpu

TOL = 1e-10   # north-star parity bar: relative L2 per solve


def _ops(z, name, keep_dtn=True, layout=None):
    import paper_2306_02526_b200 as hb
    fields, bounds = SOLVE_CASES[name]
    n1, n2, p = (int(v) for v in z["shape"])
    tree = hb.build_tree(bounds, n1, n2, p)
    coeffs = hb.OperatorCoefficients(**fields())
    ops = hb.build(tree, coeffs, sigma=float(z["sigma"]), dt_gamma=float(z["dt_gamma"]),
                   keep_dtn=keep_dtn, layout=layout)
    return tree, ops


@pytest.mark.parametrize("layout", ["per_node", "shared"])
@pytest.mark.parametrize("name", sorted(SOLVE_CASES))
def test_device_solve_matches_reference(golden, name, layout):
    z = golden("solve_" + name)
    tree, ops = _ops(z, name, layout=layout)
    u = ops.solve_with_body_load(z["f"], z["g"])
    assert u.shape == z["u"].shape
    assert rel_l2(u, z["u"]) < TOL
    uh = ops.solve_homogeneous(z["f"])
    assert rel_l2(uh, z["u_hom"]) < TOL
    if "u_pen" in z:
        up = ops.solve_penalized(z["f"], z["g"], z["jump"], float(z["dt_pen"]))
        assert rel_l2(up, z["u_pen"]) < TOL


@pytest.mark.parametrize("layout", ["per_node", "shared"])
@pytest.mark.parametrize("name", sorted(SOLVE_CASES))
def test_device_build_matches_reference(golden, name, layout):
    z = golden("solve_" + name)
    tree, ops = _ops(z, name, layout=layout)
    lo = ops.leaf_operators(0)
    assert rel_l2(lo.S, z["S_leaf0"]) < TOL
    assert rel_l2(lo.T, z["T_leaf0"]) < TOL
    if "root_S" in z:
        mo = ops.merge_operators(0)
        assert rel_l2(mo.S, z["root_S"]) < TOL
        assert rel_l2(mo.Tstack, z["root_Tstack"]) < TOL
        assert rel_l2(mo.T, z["root_T"]) < TOL


def test_device_solve_torch_inputs_stay_on_device(golden):
    import torch
    z = golden("solve_lap2x2p10")
    tree, ops = _ops(z, "lap2x2p10", keep_dtn=False)
    f = torch.as_tensor(z["f"], device="cuda")
    g = torch.as_tensor(z["g"], device="cuda")
    u = ops.solve_with_body_load(f, g)
    assert u.is_cuda and u.shape == (tree.N,)
    assert rel_l2(u.cpu().numpy(), z["u"]) < TOL


def test_device_singular_leaf_names_node():
    import paper_2306_02526_b200 as hb
    tree = hb.build_tree(((0.0, 1.0), (0.0, 1.0)), 1, 1, 8)
    zero = hb.OperatorCoefficients(c11=0.0, c22=0.0)
    with pytest.raises(hb.SingularMatrixError) as exc:
        hb.build(tree, zero, sigma=0.0, dt_gamma=1.0)
    assert "leaf node" in str(exc.value)


@pytest.mark.parametrize("layout", ["per_node", "shared"])
def test_device_solve_is_bitwise_reproducible_and_multi_rhs_consistent(golden, layout):
    """test_solver.py:255-273: repeated solves are bitwise equal; a stacked
    multi-RHS solve equals the loop of single solves to 1e-14."""
    z = golden("solve_heat4x4p12k3")
    tree, ops = _ops(z, "heat4x4p12k3", keep_dtn=False, layout=layout)
    a = ops.solve_with_body_load(z["f"], z["g"])
    b = ops.solve_with_body_load(z["f"], z["g"])
    assert np.array_equal(a, b)
    loop = np.stack([ops.solve_with_body_load(z["f"][i], z["g"][i]) for i in range(3)])
    assert rel_l2(a, loop) < 1e-14


@pytest.mark.parametrize("layout", ["per_node", "shared"])
def test_operator_set_save_load_roundtrip(golden, tmp_path, layout):
    """solver.py:294-337: a dumped operator set reloads without a build, solves
    bitwise identically, and refuses a mismatched configuration."""
    import paper_2306_02526_b200 as hb
    z = golden("solve_c4var4x4p10" if layout == "per_node" else "solve_heat4x4p12k3")
    name = "c4var4x4p10" if layout == "per_node" else "heat4x4p12k3"
    tree, ops = _ops(z, name, keep_dtn=False, layout=layout)
    path = tmp_path / "ops.bin"
    ops.save(str(path))
    ops2 = hb.HpsOperatorSet.load(str(path), ops.disc, ops.sigma, ops.dt_gamma)
    a = ops.solve_with_body_load(z["f"], z["g"])
    b = ops2.solve_with_body_load(z["f"], z["g"])
    assert np.array_equal(a, b)
    assert rel_l2(b, z["u"]) < TOL
    with pytest.raises(hb.HpstepError):
        hb.HpsOperatorSet.load(str(path), ops.disc, ops.sigma, 2 * ops.dt_gamma)


@pytest.mark.parametrize("layout,nparts", [("shared", 1), ("per_node", 1), ("shared", 2)])
def test_many_rhs_solve_matches_oracle(layout, nparts):
    """k = 20 right-hand sides: on shared operators every level (fused ones
    included) runs as one tensor-core GEMM over (node, rhs) rows."""
    import paper_2306_02526_b200 as hb
    from oracle import hps_oracle as O
    n, p, k = 8, 12, 20
    tree = hb.build_tree(((0.0, 1.0), (0.0, 1.0)), n, n, p)
    ops = hb.build(tree, hb.OperatorCoefficients(c11=1.0, c22=1.0), sigma=1.0, dt_gamma=1e-3, layout=layout,
                   nparts=nparts)
    ot = O.OTree(((0.0, 1.0), (0.0, 1.0)), n, n, p)
    oops = O.OHps(O.ODisc(ot, O.OCoeffs(1.0, 1.0)), sigma=1.0, dt_gamma=1e-3)
    rng = np.random.default_rng(9)
    g = rng.standard_normal((k, tree.N))
    f = rng.standard_normal((k, tree.boundary_ids.size))
    u = ops.solve_with_body_load(f, g)
    ref = oops.solve(f, g)
    assert rel_l2(u, ref) < TOL
    single = ops.solve_with_body_load(f[3], g[3])
    assert rel_l2(single, ref[3]) < TOL


@pytest.mark.parametrize("p", [10, 12, 16])
def test_fused_stage_matches_solve_then_eval(p):
    """hps_solve_stage (solve + interior L u + guard from the leaf kernel of the
    down sweep) equals hps_solve followed by hps_leaf_eval."""
    import torch
    import paper_2306_02526_b200 as hb
    from paper_2306_02526_b200.timestep import device_discretization
    tree = hb.build_tree(((0.0, 1.0), (0.0, 1.0)), 8, 8, p)
    coeffs = hb.OperatorCoefficients(c11=1.0, c22=0.7, c1=0.3, c2=-0.2, c=0.1)
    disc = hb.EllipticDiscretization(tree, coeffs)
    ops = hb.HpsOperatorSet(disc, sigma=1.0, dt_gamma=1e-3, layout="shared")
    assert ops.fuses_stage_history
    k = 2
    rng = np.random.default_rng(p)
    body = torch.as_tensor(rng.standard_normal((k, tree.N)), device="cuda")
    fb = torch.as_tensor(rng.standard_normal((k, tree.boundary_ids.size)), device="cuda")
    u1 = torch.empty((k, tree.N), dtype=torch.float64, device="cuda")
    u2 = torch.empty_like(u1)
    lu1 = torch.empty((k, tree.L * tree.ni), dtype=torch.float64, device="cuda")
    lu2 = torch.empty_like(lu1)
    g1 = torch.zeros(1, dtype=torch.float64, device="cuda")
    g2 = torch.zeros(1, dtype=torch.float64, device="cuda")
    ops.solve_stage_device(fb, body, u1, lu1, g1)
    ops.solve_device(fb, body, u2)
    device_discretization(disc).eval(u2, lu_int=lu2, guard=g2)
    assert torch.equal(u1, u2)
    assert rel_l2(lu1.cpu().numpy(), lu2.cpu().numpy()) < 1e-13
    assert g1.item() == g2.item() and g1.item() > 0


@pytest.mark.gpu
@pytest.mark.parametrize("p", [10, 12, 16])
def test_leaf_lu_matches_leaf_eval(p):
    """hps_leaf_lu (the explicit stage's L u_n by the leaf-grid DMMA products)
    equals the general leaf evaluation at the interiors, on a full range and a
    leaf sub-range, with the same guard."""
    import torch
    import paper_2306_02526_b200 as hb
    from paper_2306_02526_b200.timestep import device_discretization
    tree = hb.build_tree(((0.0, 1.0), (0.0, 1.0)), 8, 8, p)
    coeffs = hb.OperatorCoefficients(c11=1.0, c22=0.7, c1=0.3, c2=-0.2, c=0.1)
    disc = hb.EllipticDiscretization(tree, coeffs)
    ops = hb.HpsOperatorSet(disc, sigma=1.0, dt_gamma=1e-3, layout="shared")
    assert ops.fuses_stage_history
    k = 2
    rng = np.random.default_rng(100 + p)
    u = torch.as_tensor(rng.standard_normal((k, tree.N)), device="cuda")
    lu1 = torch.empty((k, tree.L * tree.ni), dtype=torch.float64, device="cuda")
    lu2 = torch.empty_like(lu1)
    g1 = torch.zeros(1, dtype=torch.float64, device="cuda")
    g2 = torch.zeros(1, dtype=torch.float64, device="cuda")
    ops.leaf_lu_device(u, lu1, g1)
    device_discretization(disc).eval(u, lu_int=lu2, guard=g2)
    assert rel_l2(lu1.cpu().numpy(), lu2.cpu().numpy()) < 1e-13
    assert g1.item() == g2.item() == float(u.abs().max())
    # leaf sub-range: rows start at the first leaf's interior, nothing else written
    leaf0, nleaf = 5, 17
    lu3 = torch.full_like(lu1, 7.0)
    ops.leaf_lu_device(u, lu3[:, leaf0 * tree.ni:], leaves=(leaf0, nleaf))
    a, b = leaf0 * tree.ni, (leaf0 + nleaf) * tree.ni
    assert rel_l2(lu3[:, a:b].cpu().numpy(), lu2[:, a:b].cpu().numpy()) < 1e-13
    assert torch.all(lu3[:, :a] == 7.0) and torch.all(lu3[:, b:] == 7.0)


@pytest.mark.parametrize("n", [8, 32])
def test_root_dirichlet_product_in_stage_solve(n):
    """The root's Dirichlet product batched over several boundary-data rows
    (hps_root_dirichlet) and handed to the fused stage solve (root_pre) gives
    the solve without it (round-off: the root's sums are grouped differently)."""
    import torch
    import paper_2306_02526_b200 as hb
    tree = hb.build_tree(((0.0, 1.0), (0.0, 1.0)), n, n, 16)
    disc = hb.EllipticDiscretization(tree, hb.OperatorCoefficients(c11=1.0, c22=1.0))
    ops = hb.HpsOperatorSet(disc, sigma=1.0, dt_gamma=2.5e-4, layout="shared")
    assert ops.root_dirichlet_ok
    rng = np.random.default_rng(7 + n)
    fb = torch.as_tensor(rng.standard_normal((3, tree.boundary_ids.size)), device="cuda")
    body = torch.as_tensor(rng.standard_normal((1, tree.N)), device="cuda")
    rp = torch.empty((3, tree.level_maps[0].n3), dtype=torch.float64, device="cuda")
    ops.root_dirichlet_device(fb, rp)
    for s_ in range(3):
        u1 = torch.zeros((1, tree.N), dtype=torch.float64, device="cuda")
        u2 = torch.zeros_like(u1)
        lu1 = torch.empty((1, tree.L * tree.ni), dtype=torch.float64, device="cuda")
        lu2 = torch.empty_like(lu1)
        g1 = torch.zeros(1, dtype=torch.float64, device="cuda")
        g2 = torch.zeros(1, dtype=torch.float64, device="cuda")
        ops.solve_stage_device(fb[s_:s_ + 1], body, u1, lu1, g1, root_pre=rp[s_:s_ + 1])
        ops.solve_stage_device(fb[s_:s_ + 1], body, u2, lu2, g2)
        assert rel_l2(u1.cpu().numpy(), u2.cpu().numpy()) < 1e-14
        assert rel_l2(lu1.cpu().numpy(), lu2.cpu().numpy()) < 1e-12
        assert abs(g1.item() - g2.item()) <= 1e-13 * g2.item()


@pytest.mark.parametrize("p", [12, 16])
def test_stage_terms_match_combine_then_stage(p):
    """hps_solve_stage_terms (the body load formed from its terms by the up
    sweep's leaf kernel and written out) equals hps_combine + hps_solve_stage:
    the same body load bitwise (same fma order), the same solution."""
    import torch
    import paper_2306_02526_b200 as hb
    from paper_2306_02526_b200.timestep import combine
    tree = hb.build_tree(((0.0, 1.0), (0.0, 1.0)), 16, 16, p)
    disc = hb.EllipticDiscretization(tree, hb.OperatorCoefficients(c11=1.0, c22=1.0))
    ops = hb.HpsOperatorSet(disc, sigma=1.0, dt_gamma=2.5e-4, layout="shared")
    rng = np.random.default_rng(p)
    Lni = tree.L * tree.ni
    vecs = [torch.as_tensor(rng.standard_normal((1, Lni)), device="cuda") for _ in range(7)]
    coefs = [1.0, -0.3, 2.5e-4, 0.125, -7.0, 1e-3, 0.5]
    dc = torch.tensor(coefs, dtype=torch.float64, device="cuda")
    fb = torch.as_tensor(rng.standard_normal((1, tree.boundary_ids.size)), device="cuda")
    for nt in (1, 2, 7):
        r1 = torch.empty((1, Lni), dtype=torch.float64, device="cuda")
        u1 = torch.zeros((1, tree.N), dtype=torch.float64, device="cuda")
        u2 = torch.zeros_like(u1)
        lu1, lu2 = torch.empty_like(r1), torch.empty_like(r1)
        g1 = torch.zeros(1, dtype=torch.float64, device="cuda")
        g2 = torch.zeros(1, dtype=torch.float64, device="cuda")
        ops.solve_stage_terms_device(fb, dc.data_ptr(), vecs[:nt], r1, u1, lu1, g1)
        r2 = combine(list(zip(coefs[:nt], vecs[:nt])), torch.empty_like(r1))
        ops.solve_stage_device(fb, r2, u2, lu2, g2)
        assert torch.equal(r1, r2), nt
        assert torch.equal(u1, u2), nt
        assert torch.equal(lu1, lu2) and g1.item() == g2.item(), nt


def test_combine_bnd_matches_combine_put_maxabs():
    """hps_combine_bnd (final combination + Dirichlet data + guard, one pass)
    equals hps_combine, hps_put_boundary and hps_maxabs in sequence."""
    import torch
    import paper_2306_02526_b200 as hb
    from paper_2306_02526_b200 import _lib
    from paper_2306_02526_b200.device import current_stream_handle
    from paper_2306_02526_b200.solver import device_plan
    from paper_2306_02526_b200.timestep import combine, combine_bnd
    tree = hb.build_tree(((0.0, 1.0), (0.0, 1.0)), 8, 4, 12)
    plan = device_plan(tree)
    rng = np.random.default_rng(3)
    k, N = 2, tree.N
    v = [torch.as_tensor(rng.standard_normal((k, N)), device="cuda") for _ in range(3)]
    v.append(torch.as_tensor(rng.standard_normal((1, N)), device="cuda"))
    terms = [(1.0, v[0]), (-0.5, v[1]), (0.25, v[2]), (3.0, v[3])]
    fb = torch.as_tensor(rng.standard_normal((k, tree.boundary_ids.size)), device="cuda")
    out1 = torch.empty((k, N), dtype=torch.float64, device="cuda")
    g1 = torch.zeros(1, dtype=torch.float64, device="cuda")
    combine_bnd(plan, terms, fb, out1, g1)
    out2 = combine(terms, torch.empty_like(out1))
    lib = _lib.load()
    _lib.check(lib.hps_put_boundary(plan.handle, k, fb.data_ptr(), fb.stride(0), out2.data_ptr(), out2.stride(0),
                                    current_stream_handle()), "put")
    g2 = torch.zeros(1, dtype=torch.float64, device="cuda")
    _lib.check(lib.hps_maxabs(k, N, out2.data_ptr(), out2.stride(0), g2.data_ptr(), current_stream_handle()), "max")
    assert torch.equal(out1, out2)
    assert g1.item() == g2.item() == float(out2.abs().max())


def test_timing_harness_rows(tmp_path):
    """run_timing (drivers.py:160-204) on the device: one row per size with
    the reference's columns, build and median solve times, CSV written."""
    from paper_2306_02526_b200.timing import COLUMNS, run_timing
    path = tmp_path / "timing.csv"
    rows = run_timing(sizes=(2, 4), p=11, out_path=str(path))
    assert [r["n_side"] for r in rows] == [2, 4]
    for r in rows:
        assert r["N"] == (r["n_side"] * 10 + 1) ** 2
        assert r["build_seconds"] > 0 and r["per_step_solve_seconds"] > 0
    assert path.read_text().splitlines()[0] == ",".join(COLUMNS)


@pytest.mark.parametrize("p", list(range(6, 17)))
def test_tensor_leaf_solve_every_order(p):
    """The tensor-product (Kronecker-sum) leaf kernels take every leaf order
    p = 6..16 (q = p - 2 interior points): plain solves and one fused ARK4
    step agree with the CPU oracle to the north-star tolerance."""
    import paper_2306_02526_b200 as hb
    from oracle import hps_oracle as O
    unit = ((0.0, 1.0), (0.0, 1.0))
    rng = np.random.default_rng(p)
    tree = hb.build_tree(unit, 4, 4, p)
    ops = hb.build(tree, hb.OperatorCoefficients(c11=1.0, c22=0.5, c1=0.3), sigma=1.0, dt_gamma=2e-3)
    assert ops.leaf_solve == "tensor", p
    f = rng.standard_normal(tree.boundary_ids.size)
    g = rng.standard_normal(tree.N)
    ot = O.OTree(unit, 4, 4, p)
    ref = O.OHps(O.ODisc(ot, O.OCoeffs(c11=1.0, c22=0.5, c1=0.3)), 1.0, 2e-3).solve_with_body_load(f, g)
    assert rel_l2(ops.solve_with_body_load(f, g), ref) < TOL, p
    two_pi = 2 * np.pi
    phi = lambda pts: np.sin(two_pi * pts[:, 0]) * np.sin(two_pi * pts[:, 1])
    prob = hb.ParabolicProblem(coeffs=hb.OperatorCoefficients(c11=1.0, c22=1.0),
                               q=hb.SeparableField.product(phi, lambda t: -np.sin(t) + 8 * np.pi ** 2 * np.cos(t)),
                               f=hb.SeparableField.product(phi, np.cos), u0=phi)
    st = hb.TimeStepper(tree, prob, "ARK4", dt=1e-3)
    assert st.ops.leaf_solve == "tensor", p
    s = st.run(st.initial_state(), 2)
    ost = O.OStepper(ot, O.OCoeffs(c11=1.0, c22=1.0), O.ark4_tableau(), 1e-3,
                     q=lambda t, pts: phi(pts) * (-np.sin(t) + 8 * np.pi ** 2 * np.cos(t)),
                     f=lambda t, pts: phi(pts) * np.cos(t))
    _, uref = ost.run(0.0, phi(ot.points), 2)
    assert rel_l2(s.u, uref) < TOL, p


def test_level_pairs_match_unpaired_solve_and_oracle(tmp_path):
    """The dataflow kernel's level pairs (mega.cu: a pair's child level from the
    parent's boundary values through a composite operator) against the CPU
    oracle (reference solver.py:258-268) and against the same solve with
    HPSB_NO_MEGA_PAIRS=1 in a fresh process (the switch is read once)."""
    import os
    import subprocess
    import sys

    import paper_2306_02526_b200 as hb
    from oracle import hps_oracle as O
    from paper_2306_02526_b200 import _lib

    n, p = 32, 8
    unit = ((0.0, 1.0), (0.0, 1.0))
    rng = np.random.default_rng(7)
    tree = hb.build_tree(unit, n, n, p)
    ops = hb.build(tree, hb.OperatorCoefficients(c11=1.0, c22=0.7, c=0.3), sigma=1.0, dt_gamma=2e-3)
    assert _lib.load().hps_ops_level_pairs(ops.handle) > 0, "no level pairs prepared for a 32 x 32 tree"
    f = rng.standard_normal(tree.boundary_ids.size)
    g = rng.standard_normal(tree.N)
    u = ops.solve_with_body_load(f, g)
    ot = O.OTree(unit, n, n, p)
    ref = O.OHps(O.ODisc(ot, O.OCoeffs(c11=1.0, c22=0.7, c=0.3)), 1.0, 2e-3).solve_with_body_load(f, g)
    assert rel_l2(u, ref) < 1e-10
    np.save(tmp_path / "f.npy", f)
    np.save(tmp_path / "g.npy", g)
    code = (
        "import numpy as np, paper_2306_02526_b200 as hb\n"
        "from paper_2306_02526_b200 import _lib\n"
        f"tree = hb.build_tree((({unit[0][0]}, {unit[0][1]}), ({unit[1][0]}, {unit[1][1]})), {n}, {n}, {p})\n"
        "ops = hb.build(tree, hb.OperatorCoefficients(c11=1.0, c22=0.7, c=0.3), sigma=1.0, dt_gamma=2e-3)\n"
        "assert _lib.load().hps_ops_level_pairs(ops.handle) == 0\n"
        f"u = ops.solve_with_body_load(np.load(r'{tmp_path / 'f.npy'}'), np.load(r'{tmp_path / 'g.npy'}'))\n"
        f"np.save(r'{tmp_path / 'u.npy'}', u)\n")
    env = dict(os.environ, HPSB_NO_MEGA_PAIRS="1")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env["PYTHONPATH"] = root + os.pathsep + env.get("PYTHONPATH", "")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    u0 = np.load(tmp_path / "u.npy")
    assert rel_l2(u, u0) < 1e-12
    assert not np.array_equal(u, u0), "the paired and unpaired solves agree bitwise: pairs not taken"
