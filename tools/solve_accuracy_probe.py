"""Single stage-solve accuracy of the device path against the CPU oracle on
the C2 recipe's body load at n x n leaves, per switch (run each variant in
its own process: the switches are read once)."""
import json, os, subprocess, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench

n = int(sys.argv[1]) if len(sys.argv) > 1 else 64
mode = sys.argv[2] if len(sys.argv) > 2 else "driver"
cfg = dict(bench.CONFIGS["C2"], n=n)
dtg = cfg["dt"] * 0.25
path = f"/tmp/acc_{n}.npz"
if mode == "oracle":
    from oracle import hps_oracle as O
    ot = O.OTree(((0.0, 1.0), (0.0, 1.0)), n, n, cfg["p"])
    oh = O.OHps(O.ODisc(ot, O.OCoeffs(c11=1.0, c22=1.0)), 1.0, dtg)
    x, y = ot.points[:, 0], ot.points[:, 1]
    body = bench.phi(ot.points) * (1 + 0.3 * np.cos(3 * x) * np.sin(5 * y))
    fb = bench.phi(ot.points)[ot.boundary_ids] * 0 + np.sin(7 * x[ot.boundary_ids]) * 1e-3
    u = oh.solve_with_body_load(fb, body)
    np.savez(path, body=body, fb=fb, u=u)
elif mode == "gpu":
    import paper_2306_02526_b200 as hb
    z = np.load(path)
    tree = hb.build_tree(((0.0, 1.0), (0.0, 1.0)), n, n, cfg["p"])
    ops = hb.build(tree, hb.OperatorCoefficients(c11=1.0, c22=1.0), sigma=1.0, dt_gamma=dtg,
                   layout=os.environ.get("PROBE_LAYOUT"))
    u = ops.solve_with_body_load(z["fb"], z["body"])
    d = u - z["u"]
    L = tree.L * tree.ni
    print(json.dumps({"env": os.environ.get("PROBE_ENV", ""), "rel_l2": float(np.linalg.norm(d) / np.linalg.norm(z["u"])),
                      "max_rel": float(np.abs(d).max() / np.abs(z["u"]).max()),
                      "max_rel_interior": float(np.abs(d[:L]).max() / np.abs(z["u"]).max()),
                      "max_rel_edges": float(np.abs(d[L:]).max() / np.abs(z["u"]).max())}))
else:
    subprocess.run([sys.executable, __file__, str(n), "oracle"], check=True)
    variants = os.environ.get("PROBE_VARIANTS", "").split(",") if os.environ.get("PROBE_VARIANTS") else ["", "HPSB_NO_FD=1", "HPSB_NO_MEGA=1", "HPSB_NO_ROOT_PAIR=1", "PROBE_LAYOUT=per_node",
                "HPSB_NO_SUB_SH=1", "HPSB_NO_VN=1", "HPSB_NO_FD=1 HPSB_NO_MEGA=1 PROBE_LAYOUT=per_node"]
    for v in variants:
        env = dict(os.environ)
        for kv in v.split():
            a, b = kv.split("=")
            env[a] = b
        env["PROBE_ENV"] = v
        subprocess.run([sys.executable, __file__, str(n), "gpu"], env=env)
