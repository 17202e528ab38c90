"""Product host logic (no GPU): tree numbering and stencil against the reference
goldens and the oracle; the C-ABI library loads and exports every symbol."""

import ctypes
import os
import re

import numpy as np
import pytest

from oracle import hps_oracle as O

TREES = ["2x2p6", "4x2p9", "4x4p7", "8x8p12", "rect4x2p8", "rect2x4p8"]
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("name", TREES)
def test_product_tree_matches_reference(golden, name):
    from paper_2306_02526_b200.tree import build_tree
    z = golden("tree_" + name)
    n1, n2, p = (int(v) for v in z["shape"])
    t = build_tree(z["bounds"], n1, n2, p)
    assert t.N == int(z["N"])
    assert np.array_equal(t.points, z["points"])
    for key in ("boundary_ids", "interface_ids", "multiplicity", "leaf_int_gidx",
                "leaf_bnd_gidx", "leaf_bnd_sign"):
        assert np.array_equal(getattr(t, key), z[key]), key
    parents = [k for lvl in t.levels for k in lvl if not t.nodes[k].is_leaf]
    assert np.array_equal(parents, z["parents"])
    for key in ("j3", "i1a", "i3a", "i2b", "i3b", "gidx_bnd"):
        got = np.concatenate([getattr(t.nodes[k], key) for k in parents])
        assert np.array_equal(got, z[key]), key


@pytest.mark.parametrize("name", TREES)
def test_product_stencil_matches_oracle(golden, name):
    from paper_2306_02526_b200.operators import LeafStencil
    from paper_2306_02526_b200.tree import build_tree
    z = golden("tree_" + name)
    n1, n2, p = (int(v) for v in z["shape"])
    st = LeafStencil(build_tree(z["bounds"], n1, n2, p))
    ost = O.OStencil(O.OTree(z["bounds"], n1, n2, p))
    for key in ("D1x", "D2x", "D1y", "D2y", "D_bnd", "Ex1", "Ex2", "Ey1", "Ey2", "local_xy"):
        assert np.array_equal(getattr(st, key), getattr(ost, key)), key


def test_level_maps_uniform_and_shapes_large():
    """C2-shaped tree: closed-form level shapes and uniform maps."""
    from paper_2306_02526_b200.tree import build_tree
    t = build_tree(((0.0, 1.0), (0.0, 1.0)), 128, 128, 16)
    assert t.N == 3673600 and t.depth == 14
    q = 14
    for d, lm in enumerate(t.level_maps):
        m = 128 >> (d // 2)
        if d % 2 == 0:
            assert (lm.n3, lm.n12) == (m * q, 4 * m * q)
        else:
            assert (lm.n3, lm.n12) == (m * q // 2, 3 * m * q)
        assert lm.gidx_bnd.shape == (2 ** d, lm.n12)


def test_library_exports_every_header_symbol():
    from paper_2306_02526_b200 import _lib
    lib = _lib.load()
    hdr = open(os.path.join(ROOT, "include", "hpstep_b200.h")).read()
    names = set(re.findall(r"\b(hps_[a-z_]+)\s*\(", hdr))
    assert names, "no declarations parsed"
    for n in sorted(names):
        assert hasattr(lib, n), n
    assert names <= set(_lib.SIGNATURES), names - set(_lib.SIGNATURES)
    assert lib.hps_version() == 1


def test_product_has_no_cpu_fallback():
    """The product package never imports the oracle, and fails loudly without a GPU."""
    import paper_2306_02526_b200 as hb
    pkg = os.path.dirname(hb.__file__)
    for fn in os.listdir(pkg):
        if fn.endswith(".py"):
            src = open(os.path.join(pkg, fn)).read()
            assert "oracle" not in src.replace("the oracle", ""), fn
    import torch
    if not torch.cuda.is_available():
        t = hb.build_tree(((0.0, 1.0), (0.0, 1.0)), 2, 2, 6)
        with pytest.raises(hb.HpstepError):
            hb.build(t, hb.OperatorCoefficients(c11=1.0, c22=1.0))


@pytest.mark.parametrize("p", [10, 12, 16])
@pytest.mark.parametrize("dtg", [2.5e-5, 1e-2, 1.0])
def test_tensor_leaf_factors_reproduce_dense_interior_solve(p, dtg):
    """The Kronecker-sum factorisation used by the tensor-product leaf solve
    (csrc/leaf_fd.cu) reproduces (sigma I + dtg A_ii)^-1 r and D_bi w."""
    import paper_2306_02526_b200 as hb
    from paper_2306_02526_b200.solver import tensor_leaf_factors
    tree = hb.build_tree(((0.0, 1.0), (0.0, 1.0)), 2, 2, p)
    disc = hb.EllipticDiscretization(tree, hb.OperatorCoefficients(c11=1.0, c22=0.7, c1=0.4, c2=-0.2, c=0.3))
    q, ni = tree.q, tree.ni
    fd = tensor_leaf_factors(disc, 1.0, dtg)
    assert fd is not None and fd.size == 5 * q * q + 8 * q + 513
    Aii, Aib = disc.leaf_blocks(0)
    r = np.random.default_rng(1).standard_normal(ni)
    w_ref = np.linalg.solve(np.eye(ni) + dtg * Aii, r)
    M = fd[:5 * ni].reshape(5, q, q)
    W = M[2] @ (((M[0] @ r.reshape(q, q)) @ M[1]) * M[4]) @ M[3]
    assert np.linalg.norm(W.ravel() - w_ref) / np.linalg.norm(w_ref) < 1e-13
    E = fd[5 * ni:5 * ni + 4 * q].reshape(4, q)
    h = np.concatenate([E[0] @ W,                                    # east: d/dx, rows yi
                        np.stack([W @ E[2], W @ E[3]], 1).ravel(),   # north/south interleaved
                        E[1] @ W])                                   # west
    D_bi = disc.stencil.D_bnd[:, :ni]
    assert np.allclose(h, D_bi @ W.ravel(), rtol=1e-12, atol=1e-12 * np.abs(h).max())
    # interior -> boundary couplings used by the down sweep: dtg A_ib u_b
    B = fd[5 * ni + 4 * q:5 * ni + 8 * q].reshape(4, q)
    ub = np.random.default_rng(2).standard_normal(4 * q)
    x, y = np.divmod(np.arange(ni), q)
    cpl = B[0][x] * ub[y] + B[1][x] * ub[3 * q + y] + B[2][y] * ub[q + 2 * x] + B[3][y] * ub[q + 2 * x + 1]
    ref = dtg * (Aib @ ub)
    assert np.allclose(cpl, ref, rtol=1e-12, atol=1e-12 * np.abs(ref).max())
    # stage history on the leaf grid: Mx G + G My^T - c G = L u at the interiors
    o = 5 * ni + 8 * q
    Mx, My, c0 = fd[o:o + 256].reshape(16, 16), fd[o + 256:o + 512].reshape(16, 16), fd[o + 512]
    ui = np.random.default_rng(3).standard_normal(ni)
    G = np.zeros((16, 16))
    G[1:p - 1, 1:p - 1] = ui.reshape(q, q)
    G[0, 1:p - 1], G[p - 1, 1:p - 1] = ub[:q], ub[3 * q:]
    G[1:p - 1, 0], G[1:p - 1, p - 1] = ub[q:3 * q:2], ub[q + 1:3 * q:2]
    lop = (Mx @ G + G @ My.T - c0 * G)[1:p - 1, 1:p - 1].ravel()
    ref = -(Aii @ ui + Aib @ ub)          # L = -A at the interior points
    assert np.allclose(lop, ref, rtol=1e-11, atol=1e-11 * np.abs(ref).max())


def test_tensor_leaf_factors_only_for_constant_coefficients():
    import paper_2306_02526_b200 as hb
    from paper_2306_02526_b200.solver import tensor_leaf_factors
    tree = hb.build_tree(((0.0, 1.0), (0.0, 1.0)), 2, 2, 10)
    disc = hb.EllipticDiscretization(tree, hb.OperatorCoefficients(c11=lambda x, y: 1 + x, c22=1.0))
    assert tensor_leaf_factors(disc, 1.0, 0.1) is None
    for p, ok in ((5, False), (6, True), (9, True), (16, True), (17, False)):  # kernels for q = p - 2 in [4, 14]
        tree = hb.build_tree(((0.0, 1.0), (0.0, 1.0)), 2, 2, p)
        disc = hb.EllipticDiscretization(tree, hb.OperatorCoefficients(c11=1.0, c22=1.0))
        assert (tensor_leaf_factors(disc, 1.0, 0.1) is not None) == ok, p


def test_step_map_analysis_matches_reference(golden):
    """stability.analyze on the reference's assembled maps reproduces the
    reference's spectrum, spectral radius and zero count (host only)."""
    from paper_2306_02526_b200.stability import analyze, spectrum_csv_lines
    z = golden("stability_4x4p6")
    for key in ("ark4", "ark4_slope", "be_var"):
        spec = analyze(z[key + "_M"], dt=0.01, scheme="ARK4")
        assert abs(spec.spectral_radius - float(z[key + "_rho"])) < 1e-12
        assert spec.zero_count == int(z[key + "_zeros"])
        assert np.allclose(np.sort_complex(spec.eigenvalues), np.sort_complex(z[key + "_eig"]), atol=1e-10)
    lines = spectrum_csv_lines(spec)
    assert lines[1] == "re,im,modulus" and len(lines) == 2 + spec.eigenvalues.size


def test_loglog_slope():
    from paper_2306_02526_b200.timing import loglog_slope
    xs = np.array([1e3, 1e4, 1e5, 1e6])
    assert abs(loglog_slope(xs, 3.0 * xs ** 1.1) - 1.1) < 1e-12
