"""Pin the CPU oracle against vectors produced by the real reference
(tests/golden/make_golden.py).  CPU only."""

import numpy as np
import pytest

from oracle import hps_oracle as O
from tests.problems import (SOLVE_CASES, UNIT, c4_fields, heat_manufactured,
                            lap_fields, rel_l2, sine_field)

TREES = ["2x2p6", "4x2p9", "4x4p7", "8x8p12", "rect4x2p8", "rect2x4p8"]


@pytest.mark.parametrize("name", TREES)
def test_oracle_tree_matches_reference(golden, name):
    z = golden("tree_" + name)
    n1, n2, p = z["shape"]
    t = O.OTree(z["bounds"], int(n1), int(n2), int(p))
    assert t.N == int(z["N"])
    assert np.array_equal(t.points, z["points"])
    assert np.array_equal(t.boundary_ids, z["boundary_ids"])
    assert np.array_equal(t.interface_ids, z["interface_ids"])
    assert np.array_equal(t.mult, z["multiplicity"])
    assert np.array_equal(t.leaf_int_gidx, z["leaf_int_gidx"])
    assert np.array_equal(t.leaf_bnd_gidx, z["leaf_bnd_gidx"])
    assert np.array_equal(t.leaf_bnd_sign, z["leaf_bnd_sign"])
    parents = t.parents_root_first()
    assert np.array_equal(parents, z["parents"])
    for key in ("j3", "i1a", "i3a", "i2b", "i3b"):
        got = np.concatenate([t.nodes[k][key] for k in parents])
        assert np.array_equal(got, z[key]), key
    got = np.concatenate([t.nodes[k]["bnd"] for k in parents])
    assert np.array_equal(got, z["gidx_bnd"])


@pytest.mark.parametrize("name", sorted(SOLVE_CASES))
def test_oracle_solve_matches_reference(golden, name):
    z = golden("solve_" + name)
    fields, bounds = SOLVE_CASES[name]
    n1, n2, p = (int(v) for v in z["shape"])
    tree = O.OTree(bounds, n1, n2, p)
    disc = O.ODisc(tree, O.OCoeffs(**fields()))
    ops = O.OHps(disc, float(z["sigma"]), float(z["dt_gamma"]), keep_T=True)
    assert rel_l2(ops.S_leaf[0], z["S_leaf0"]) < 1e-13
    assert rel_l2(ops.T_leaf[0], z["T_leaf0"]) < 1e-13
    if "root_S" in z:
        S, _, Tst = ops.merges[0]
        assert rel_l2(S, z["root_S"]) < 1e-13
        assert rel_l2(Tst, z["root_Tstack"]) < 1e-13
        assert rel_l2(ops.root_T, z["root_T"]) < 1e-13
    assert rel_l2(ops.solve_with_body_load(z["f"], z["g"]), z["u"]) < 1e-13
    assert rel_l2(ops.solve_homogeneous(z["f"]), z["u_hom"]) < 1e-13
    if "u_pen" in z:
        u = ops.solve_penalized(z["f"], z["g"], z["jump"], float(z["dt_pen"]))
        assert rel_l2(u, z["u_pen"]) < 1e-13


def test_oracle_singular_leaf_names_node():
    tree = O.OTree(UNIT, 1, 1, 8)
    disc = O.ODisc(tree, O.OCoeffs(c11=0.0, c22=0.0))
    with pytest.raises(O.OracleSingular) as e:
        O.OHps(disc, 0.0, 1.0)
    assert "leaf node" in str(e.value)


def test_oracle_c1_stepping_matches_reference(golden):
    z = golden("step_c1")
    tree = O.OTree(UNIT, 8, 8, 12)
    phi, uex, q = heat_manufactured()
    st = O.OStepper(tree, O.OCoeffs(**lap_fields()), O.ark4_tableau(), 1e-3, q=q, f=uex,
                    record=True)
    u0 = uex(0.0, tree.points)
    t, u = st.run(0.0, u0, 1)
    stages = np.array([s[0] for s in st.stages])
    assert rel_l2(stages, z["stages"]) < 1e-13
    assert rel_l2(u, z["u1"]) < 1e-13
    t, u = st.run(t, u, 9)
    assert rel_l2(u, z["u10"]) < 1e-12
    t, u = st.run(t, u, 90)
    assert rel_l2(u, z["u100"]) < 1e-12
    assert np.abs(u - uex(t, tree.points)).max() < 1e-10


def test_oracle_allen_cahn_matches_reference(golden):
    z = golden("step_allen_cahn")
    tree = O.OTree(UNIT, 8, 8, 12)
    st = O.OStepper(tree, O.OCoeffs(c11=0.01, c22=0.01), O.ark4_tableau(), float(z["dt"]),
                    g=lambda t, u, ux, uy: u - u ** 3)
    t, u = st.run(0.0, sine_field(z["modes"], tree.points), 1)
    assert rel_l2(u, z["u1"]) < 1e-13
    t, u = st.run(t, u, 9)
    assert rel_l2(u, z["u10"]) < 1e-12


def test_oracle_burgers_var_matches_reference(golden):
    z = golden("step_burgers_var")
    tree = O.OTree(UNIT, 8, 8, 10)
    st = O.OStepper(tree, O.OCoeffs(**c4_fields()), O.ark4_tableau(), float(z["dt"]),
                    g=lambda t, u, ux, uy: -u * ux)
    t, u = st.run(0.0, sine_field(z["modes"], tree.points), 1)
    assert rel_l2(u, z["u1"]) < 1e-13
    t, u = st.run(t, u, 4)
    assert rel_l2(u, z["u5"]) < 1e-12


def test_oracle_ensemble_matches_reference(golden):
    z = golden("step_ensemble")
    tree = O.OTree(UNIT, 4, 4, 10)
    coef = z["modes"]
    st = O.OStepper(tree, O.OCoeffs(**lap_fields()), O.ark4_tableau(), float(z["dt"]),
                    q=lambda t, pts: sine_field(coef, pts), ncomp=4)
    t, u = st.run(0.0, np.zeros((4, tree.N)), 3)
    assert rel_l2(u, z["u3"]) < 1e-13


def test_oracle_backward_euler_matches_reference(golden):
    z = golden("step_be")
    tree = O.OTree(UNIT, 4, 4, 10)
    phi, uex, q = heat_manufactured()
    st = O.OStepper(tree, O.OCoeffs(**lap_fields()), O.be_tableau(), float(z["dt"]), q=q, f=uex)
    t, u = st.run(0.0, uex(0.0, tree.points), 3)
    assert rel_l2(u, z["u3"]) < 1e-13


def test_oracle_leaf_evaluations_match_reference(golden):
    from tests.problems import var_test_fields
    z = golden("evals_var4x2p9")
    tree = O.OTree(UNIT, 4, 2, 9)
    disc = O.ODisc(tree, O.OCoeffs(**var_test_fields()))
    assert rel_l2(disc.apply_lop(z["u"]), z["lu"]) < 1e-13
    assert rel_l2(disc.apply_lop(z["u"][0]), z["lu1"]) < 1e-13
    ux, uy = disc.gradient(z["u"])
    assert rel_l2(ux, z["ux"]) < 1e-13 and rel_l2(uy, z["uy"]) < 1e-13
    assert rel_l2(disc.flux_jump(z["u"]), z["jump"]) < 1e-13


def _golden_tableau(z):
    return dict(A=z["A"], Ahat=z["Ahat"], b=z["b"], bhat=z["b"], c=z["c"], gamma=float(z["gamma"]),
                s=int(z["b"].size))


def test_ark5_tableau_matches_reference(golden):
    """The drop-in's ARK5(4)8L[2]SA arrays are bitwise the reference's
    (tableaux.py:157-221); alias and registry as the reference."""
    from paper_2306_02526_b200.tableaux import available_tableaux, load_tableau
    z = golden("step_ark5")
    p = load_tableau("ARK5")
    assert p.name == "ARK5(4)8L[2]SA" and p.s == 8 and p.order == 5 and p.embedded_order == 4
    for key in ("A", "Ahat", "b", "c", "b_emb"):
        assert np.array_equal(getattr(p, key), z[key]), key
    assert np.array_equal(p.bhat, z["b"]) and p.gamma == float(z["gamma"])
    assert "ARK5(4)8L[2]SA" in available_tableaux()


def test_oracle_ark5_stepping_matches_reference(golden):
    """The oracle's stage stepper with the 8-stage pair (every stage has more
    than the 6-stage pair's terms) against the reference run."""
    z = golden("step_ark5")
    tab = _golden_tableau(z)
    phi, uex, q = heat_manufactured()
    tree = O.OTree(UNIT, 4, 4, 10)
    st = O.OStepper(tree, O.OCoeffs(c11=1.0, c22=1.0), tab, float(z["dt"]), q=q, f=uex, record=True)
    t, u = st.run(0.0, uex(0.0, tree.points), 1)
    for i, (a, b) in enumerate(zip(st.stages, z["stages"])):
        assert rel_l2(a[0], b) < 1e-13, f"stage {i + 1}"
    assert rel_l2(u, z["u1"]) < 1e-13
    t, u = st.run(t, u, 4)
    assert rel_l2(u, z["u5"]) < 1e-13
    ac = O.OStepper(tree, O.OCoeffs(c11=0.01, c22=0.01), tab, float(z["ac_dt"]),
                    g=lambda t, u, ux, uy: u - u ** 3)
    _, a3 = ac.run(0.0, sine_field(z["ac_modes"], tree.points), 3)
    assert rel_l2(a3, z["ac_u3"]) < 1e-13
