"""Drift of the GPU stepper from the CPU oracle over several steps of the C2
recipe at n x n leaves, per switch (each variant in its own process).

    python tools/drift_probe.py N STEPS [VAR1,VAR2,...]   (VAR = "K=V K=V")"""
import json, os, subprocess, sys
import numpy as np
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
cfg = dict(bench.CONFIGS["C2"], n=n)
path = f"/tmp/drift_{n}_{steps}.npz"
mode = os.environ.get("DRIFT_MODE", "driver")
if mode == "oracle":
    tree, ost, u = bench.oracle_stepper(cfg, n)
    t, us = 0.0, []
    for i in range(steps):
        t, u = ost.run(t, u, 1)
        us.append(u.copy())
    np.savez(path, us=np.array(us), pts=tree.points)
elif mode == "gpu":
    import paper_2306_02526_b200 as hb
    z = np.load(path)
    tree = hb.build_tree(((0.0, 1.0), (0.0, 1.0)), n, n, cfg["p"])
    st = hb.TimeStepper(tree, hb.ParabolicProblem(**bench.make_problem(hb, cfg)), "ARK4", dt=cfg["dt"])
    s = st.initial_state()
    out = []
    for i in range(steps):
        s = st.step(s)
        g, u = np.asarray(s.u), z["us"][i]
        ex = bench.phi(z["pts"]) * np.cos(s.t)
        out.append((float(np.linalg.norm(g - u) / np.linalg.norm(u)), float(np.abs(g - ex).max() / np.abs(ex).max()),
                    float(np.abs(u - ex).max() / np.abs(ex).max())))
    print(json.dumps({"env": os.environ.get("PROBE_ENV", ""), "gpu_oracle_relL2": [o[0] for o in out][-1],
                      "per_step_growth": (out[-1][0] - out[0][0]) / max(1, steps - 1),
                      "gpu_exact": out[-1][1], "oracle_exact": out[-1][2]}), flush=True)
else:
    env = dict(os.environ, DRIFT_MODE="oracle")
    subprocess.run([sys.executable, __file__, str(n), str(steps)], env=env, check=True)
    variants = sys.argv[3].split(",") if len(sys.argv) > 3 else [""]
    for v in variants:
        env = dict(os.environ, DRIFT_MODE="gpu", PROBE_ENV=v)
        for kv in v.split():
            a, b = kv.split("=")
            env[a] = b
        subprocess.run([sys.executable, __file__, str(n), str(steps)], env=env)
