"""Generate golden vectors from the REAL reference (``hpstep`` under /root/reference).

Run in the build container only (the reference does not travel to the GPU box):

    python tests/golden/make_golden.py

Writes ``tests/golden/*.npz``.  Every case is seeded and small enough for the
reference to finish in seconds; the fixtures pin the CPU oracle
(``oracle/hps_oracle.py``) and the device path (``-m gpu`` tests).
"""

import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
sys.path.insert(0, REF)

from hpstep.operators import EllipticDiscretization, OperatorCoefficients  # noqa: E402
from hpstep.solver import build  # noqa: E402
from hpstep.timestep import ParabolicProblem, TimeStepper  # noqa: E402
from hpstep.tree import build_tree  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
UNIT = ((0.0, 1.0), (0.0, 1.0))
TWO_PI = 2 * np.pi


def save(name, **arrs):
    path = os.path.join(HERE, name + ".npz")
    np.savez_compressed(path, **arrs)
    print(f"wrote {path} ({os.path.getsize(path) / 1024:.1f} KiB)")


# ---------------------------------------------------------------------------
# problem definitions shared with tests (numpy callables)
# ---------------------------------------------------------------------------

def coeffs_var_test():
    """test_solver.py:198-213 variable-coefficient case."""
    return OperatorCoefficients(
        c11=lambda x, y: 1 + 0.3 * np.sin(x + y),
        c22=lambda x, y: 1 + 0.2 * np.cos(x - y),
        c1=lambda x, y: np.sin(2 * x), c2=0.5, c=0.3, dim=2)


def coeffs_c4():
    """C4: L = div(a grad u) + b.grad u, a = 1 + 0.5 sin2pix cos2piy, b = (1, 0.5)."""
    a = lambda x, y: 1 + 0.5 * np.sin(TWO_PI * x) * np.cos(TWO_PI * y)
    ax = lambda x, y: np.pi * np.cos(TWO_PI * x) * np.cos(TWO_PI * y)
    ay = lambda x, y: -np.pi * np.sin(TWO_PI * x) * np.sin(TWO_PI * y)
    return OperatorCoefficients(c11=a, c22=a, c1=lambda x, y: -(ax(x, y) + 1.0),
                                c2=lambda x, y: -(ay(x, y) + 0.5), dim=2)


def sine_modes(seed, mmax=8, nmax=4, k=None):
    rng = np.random.default_rng(seed)
    shape = (mmax, nmax) if k is None else (k, mmax, nmax)
    return rng.uniform(-1.0, 1.0, size=shape)


def sine_field(coef, pts):
    x, y = pts[:, 0], pts[:, 1]
    mmax, nmax = coef.shape[-2:]
    sx = np.stack([np.sin(m * np.pi * x) for m in range(1, mmax + 1)])
    sy = np.stack([np.sin(n * np.pi * y) for n in range(1, nmax + 1)])
    if coef.ndim == 2:
        return np.einsum("mn,mp,np->p", coef, sx, sy)
    return np.einsum("kmn,mp,np->kp", coef, sx, sy)


def heat_manufactured():
    """C1/C2: u* = sin2pix sin2piy cos t, q = sin2pix sin2piy (-sin t + 8pi^2 cos t)."""
    phi = lambda pts: np.sin(TWO_PI * pts[:, 0]) * np.sin(TWO_PI * pts[:, 1])
    uex = lambda t, pts: phi(pts) * np.cos(t)
    q = lambda t, pts: phi(pts) * (-np.sin(t) + 8 * np.pi ** 2 * np.cos(t))
    return phi, uex, q


# ---------------------------------------------------------------------------

def tree_case(name, bounds, n1, n2, p):
    tree = build_tree(bounds, n1, n2, p)
    parents = [i for lvl in tree.levels for i in lvl if not tree.nodes[i].is_leaf]
    cat = lambda key: np.concatenate([getattr(tree.nodes[i], key) for i in parents])
    cnt = lambda key: np.array([getattr(tree.nodes[i], key).size for i in parents])
    save(f"tree_{name}", N=tree.N, points=tree.points, boundary_ids=tree.boundary_ids,
         interface_ids=tree.interface_ids, multiplicity=tree.multiplicity,
         leaf_int_gidx=tree.leaf_int_gidx, leaf_bnd_gidx=tree.leaf_bnd_gidx,
         leaf_bnd_sign=tree.leaf_bnd_sign,
         parents=np.array(parents), parent_level=np.array([tree.nodes[i].level for i in parents]),
         j3=cat("j3"), j3_n=cnt("j3"), i1a=cat("i1a"), i1a_n=cnt("i1a"),
         i3a=cat("i3a"), i2b=cat("i2b"), i2b_n=cnt("i2b"), i3b=cat("i3b"),
         gidx_bnd=cat("gidx_bnd"), gidx_bnd_n=cnt("gidx_bnd"),
         bounds=np.array(bounds, float), shape=np.array([n1, n2, p]))


def solve_case(name, coeffs_fn, bounds, n1, n2, p, sigma, dtg, seed, k=1, penal=False,
               keep_ops=True):
    tree = build_tree(bounds, n1, n2, p)
    coeffs = coeffs_fn()
    disc = EllipticDiscretization(tree, coeffs)
    ops = build(tree, coeffs, sigma=sigma, dt_gamma=dtg, disc=disc, keep_dtn=True)
    rng = np.random.default_rng(seed)
    nbd = tree.boundary_ids.size
    shp = (lambda n: (n,)) if k == 1 else (lambda n: (k, n))
    f = rng.standard_normal(shp(nbd))
    g = rng.standard_normal(shp(tree.N))
    out = dict(f=f, g=g, u=ops.solve_with_body_load(f, g), u_hom=ops.solve_homogeneous(f),
               sigma=sigma, dt_gamma=dtg, bounds=np.array(bounds, float),
               shape=np.array([n1, n2, p]), S_leaf0=np.array(ops.S_leaf[0]),
               T_leaf0=np.array(ops.T_leaf[0]))
    if keep_ops and tree.leaf_count > 1:
        mo = ops.merge_operators(0)
        out.update(root_S=mo.S, root_Tstack=mo.Tstack, root_T=mo.T)
    if penal:
        jump = np.zeros(shp(tree.N))
        ids = tree.interface_ids
        jump[..., ids] = rng.standard_normal(shp(ids.size))
        out.update(jump=jump, dt_pen=0.37, u_pen=ops.solve_penalized(f, g, jump, 0.37))
    save(f"solve_{name}", **out)


def c1_case():
    """C1: 8x8 p=12 heat, ARK4, dt=1e-3; stages of step 1, u after 1, 10, 100 steps."""
    tree = build_tree(UNIT, 8, 8, 12)
    phi, uex, q = heat_manufactured()
    prob = ParabolicProblem(coeffs=OperatorCoefficients(c11=1.0, c22=1.0, dim=2), q=q,
                            f=uex, u0=lambda pts: uex(0.0, pts))
    st = TimeStepper(tree, prob, "ARK4", dt=1e-3)
    stages = []
    orig = st.ops.solve_with_body_load

    def rec(f, g):
        u = orig(f, g)
        stages.append(np.array(u))
        return u

    st.ops.solve_with_body_load = rec
    s = st.step(st.initial_state())
    st.ops.solve_with_body_load = orig
    u1 = s.u.copy()
    s = st.run(s, 9)
    u10 = s.u.copy()
    s = st.run(s, 90)
    err = np.abs(s.u - uex(s.t, tree.points)).max()
    print(f"C1 t={s.t} max err vs exact {err:.3e}")
    save("step_c1", stages=np.array(stages)[:, 0] if np.array(stages).ndim == 3 else np.array(stages),
         u1=u1, u10=u10, u100=s.u, t100=s.t, err100=err)


def allen_cahn_case():
    """C3 recipe at 8x8 p=12: eps=0.01, g = u - u^3, 32 sine modes seed 0, dt=1e-2."""
    tree = build_tree(UNIT, 8, 8, 12)
    coef = sine_modes(0)
    prob = ParabolicProblem(coeffs=OperatorCoefficients(c11=0.01, c22=0.01, dim=2),
                            g=lambda t, u, ux, uy: u - u ** 3,
                            u0=lambda pts: sine_field(coef, pts), time_independent_bc=True)
    st = TimeStepper(tree, prob, "ARK4", dt=1e-2)
    s = st.step(st.initial_state())
    u1 = s.u.copy()
    s = st.run(s, 9)
    save("step_allen_cahn", modes=coef, u1=u1, u10=s.u, dt=1e-2)


def burgers_var_case():
    """C4 recipe at 8x8 p=10: variable coefficients + g = -u u_x, dt=1e-4."""
    tree = build_tree(UNIT, 8, 8, 10)
    coef = sine_modes(1)
    prob = ParabolicProblem(coeffs=coeffs_c4(), g=lambda t, u, ux, uy: -u * ux,
                            u0=lambda pts: sine_field(coef, pts), time_independent_bc=True)
    st = TimeStepper(tree, prob, "ARK4", dt=1e-4)
    s = st.step(st.initial_state())
    u1 = s.u.copy()
    s = st.run(s, 4)
    save("step_burgers_var", modes=coef, u1=u1, u5=s.u, dt=1e-4)


def ensemble_case():
    """C5 recipe at 4x4 p=10, k=4 members: q_k sine modes (seed 2), u0=0, dt=1e-3."""
    tree = build_tree(UNIT, 4, 4, 10)
    coef = sine_modes(2, k=4)
    prob = ParabolicProblem(coeffs=OperatorCoefficients(c11=1.0, c22=1.0, dim=2),
                            q=lambda t, pts: sine_field(coef, pts),
                            u0=lambda pts: np.zeros((4, pts.shape[0])),
                            time_independent_bc=True, ncomp=4)
    st = TimeStepper(tree, prob, "ARK4", dt=1e-3)
    s = st.run(st.initial_state(), 3)
    save("step_ensemble", modes=coef, u3=s.u, dt=1e-3)


def ark5_case():
    """ARK5(4)8L[2]SA (reference tableaux.py:157-221): its coefficient arrays;
    the C1 heat recipe at 4x4 p=10 (stages of step 1, u after 1 and 5 steps)
    and the Allen-Cahn recipe at 4x4 p=10 (u after 3 steps)."""
    from hpstep.tableaux import load_tableau
    tab = load_tableau("ARK5")
    tree = build_tree(UNIT, 4, 4, 10)
    phi, uex, q = heat_manufactured()
    prob = ParabolicProblem(coeffs=OperatorCoefficients(c11=1.0, c22=1.0, dim=2), q=q,
                            f=uex, u0=lambda pts: uex(0.0, pts))
    st = TimeStepper(tree, prob, "ARK5", dt=2e-3)
    stages = []
    orig = st.ops.solve_with_body_load

    def rec(f, g):
        u = orig(f, g)
        stages.append(np.array(u))
        return u

    st.ops.solve_with_body_load = rec
    s = st.step(st.initial_state())
    st.ops.solve_with_body_load = orig
    u1 = s.u.copy()
    s = st.run(s, 4)
    coef = sine_modes(0)
    ac = ParabolicProblem(coeffs=OperatorCoefficients(c11=0.01, c22=0.01, dim=2),
                          g=lambda t, u, ux, uy: u - u ** 3,
                          u0=lambda pts: sine_field(coef, pts), time_independent_bc=True)
    sa = TimeStepper(tree, ac, "ARK5", dt=1e-2)
    a3 = sa.run(sa.initial_state(), 3)
    save("step_ark5", A=tab.A, Ahat=tab.Ahat, b=tab.b, c=tab.c, b_emb=tab.b_emb, gamma=tab.gamma,
         stages=np.array(stages)[:, 0], u1=u1, u5=s.u, dt=2e-3, ac_modes=coef, ac_u3=a3.u, ac_dt=1e-2)


def be_case():
    tree = build_tree(UNIT, 4, 4, 10)
    phi, uex, q = heat_manufactured()
    prob = ParabolicProblem(coeffs=OperatorCoefficients(c11=1.0, c22=1.0, dim=2), q=q,
                            f=uex, u0=lambda pts: uex(0.0, pts))
    st = TimeStepper(tree, prob, "BE", dt=1e-2)
    s = st.run(st.initial_state(), 3)
    save("step_be", u3=s.u, dt=1e-2)


def evals_case():
    """apply_lop / gradient / flux_jump (operators.py:276-336), variable
    coefficients on a 4x2 p=9 tree, k=2 stacked seeded fields."""
    tree = build_tree(UNIT, 4, 2, 9)
    disc = EllipticDiscretization(tree, coeffs_var_test())
    rng = np.random.default_rng(31)
    u = rng.standard_normal((2, tree.N))
    ux, uy = disc.gradient(u)
    save("evals_var4x2p9", u=u, lu=disc.apply_lop(u), ux=ux, uy=uy, jump=disc.flux_jump(u),
         lu1=disc.apply_lop(u[0]))


def slope_cases():
    """Slope / penalized-slope formulations (timestep.py:268-328) at 4x4 p=10:
    linear heat with time-dependent BC (f_t given) and nonlinear Allen-Cahn."""
    tree = build_tree(UNIT, 4, 4, 10)
    phi, uex, q = heat_manufactured()
    ut = lambda t, pts: -phi(pts) * np.sin(t)
    lap = OperatorCoefficients(c11=1.0, c22=1.0, dim=2)
    out = {}
    for form in ("slope", "slope-penalized"):
        prob = ParabolicProblem(coeffs=lap, q=q, f=uex, f_t=ut, u0=lambda pts: uex(0.0, pts))
        st = TimeStepper(tree, prob, "ARK4", dt=1e-3, formulation=form)
        s = st.run(st.initial_state(), 3)
        out[form.replace("-", "_")] = s.u.copy()
    coef = sine_modes(3)
    prob = ParabolicProblem(coeffs=OperatorCoefficients(c11=0.01, c22=0.01, dim=2),
                            g=lambda t, u, ux, uy: u - u ** 3,
                            u0=lambda pts: sine_field(coef, pts), time_independent_bc=True)
    st = TimeStepper(tree, prob, "ARK4", dt=1e-2, formulation="slope-penalized")
    s = st.run(st.initial_state(), 3)
    save("step_slope", modes=coef, **out, ac_pen=s.u.copy())


def stability_case():
    """Step-map assembly (stability.py:57-85) and its spectrum at 4x4 p=6,
    homogeneous heat (and variable coefficients for BE): ARK4 stage / slope, BE."""
    from hpstep.stability import analyze, assemble_step_map
    tree = build_tree(UNIT, 4, 4, 6)
    out = {}
    for key, coeffs, tab, form, dt in (("ark4", OperatorCoefficients(c11=1.0, c22=1.0, dim=2), "ARK4", "stage", 1e-2),
                                       ("ark4_slope", OperatorCoefficients(c11=1.0, c22=1.0, dim=2), "ARK4", "slope",
                                        1e-2),
                                       ("be_var", coeffs_var_test(), "BE", "stage", 5e-2)):
        prob = ParabolicProblem(coeffs=coeffs, u0=lambda pts: np.zeros(pts.shape[0]), time_independent_bc=True)
        M = assemble_step_map(tree, prob, tab, dt, formulation=form)
        spec = analyze(M, dt=dt, scheme=tab, formulation=form)
        out[key + "_M"] = M
        out[key + "_eig"] = spec.eigenvalues
        out[key + "_rho"] = spec.spectral_radius
        out[key + "_zeros"] = spec.zero_count
    save("stability_4x4p6", **out)


def main():
    if "--only" in sys.argv:
        for name in sys.argv[sys.argv.index("--only") + 1:]:
            globals()[name]()
        return
    tree_case("2x2p6", UNIT, 2, 2, 6)
    tree_case("4x2p9", UNIT, 4, 2, 9)
    tree_case("4x4p7", UNIT, 4, 4, 7)
    tree_case("8x8p12", UNIT, 8, 8, 12)
    tree_case("rect4x2p8", ((0.0, 2.0), (0.0, 1.0)), 4, 2, 8)
    tree_case("rect2x4p8", ((0.0, 3.0), (-1.0, 1.0)), 2, 4, 8)
    lap = lambda: OperatorCoefficients(c11=1.0, c22=1.0, dim=2)
    solve_case("lap2x2p10", lap, UNIT, 2, 2, 10, 0.0, 1.0, 3)
    solve_case("var4x2p9", coeffs_var_test, UNIT, 4, 2, 9, 0.0, 1.0, 2)
    solve_case("heat4x4p12k3", lap, UNIT, 4, 4, 12, 1.0, 2.5e-4, 7, k=3)
    solve_case("pen4x4p8", lap, UNIT, 4, 4, 8, 1.0, 0.01, 5, penal=True)
    solve_case("c4var4x4p10", coeffs_c4, UNIT, 4, 4, 10, 1.0, 2.5e-6, 9)
    solve_case("rect4x2p11", coeffs_var_test, ((0.0, 2.0), (0.0, 1.0)), 4, 2, 11, 1.0, 0.05, 4)
    solve_case("heat8x8p16", lap, UNIT, 8, 8, 16, 1.0, 2.5e-5, 11, keep_ops=False)
    c1_case()
    allen_cahn_case()
    burgers_var_case()
    ensemble_case()
    be_case()
    ark5_case()
    stability_case()
    evals_case()
    slope_cases()


if __name__ == "__main__":
    main()
