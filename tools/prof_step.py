"""Profiling driver: build a config, warm up, then run ``--steps`` ARK4 steps
between cudaProfilerStart/Stop (use ncu --profile-from-start off)."""

import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2306_02526_b200 as hb  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--steps", type=int, default=1)
    ap.add_argument("--warmup", type=int, default=2)
    ap.add_argument("--solve-only", action="store_true")
    ap.add_argument("--layout", default=None)
    a = ap.parse_args()
    cfg = bench.CONFIGS[a.config]
    tree = hb.build_tree(((0.0, 1.0), (0.0, 1.0)), cfg["n"], cfg["n"], cfg["p"])
    prob = hb.ParabolicProblem(**bench.make_problem(hb, cfg))
    st = hb.TimeStepper(tree, prob, "ARK4", dt=cfg["dt"], layout=a.layout)
    s = st.initial_state()
    s = hb.StepperState(s.t, s.u_device)
    s = st.run(s, a.warmup)
    torch.cuda.synchronize()
    if a.solve_only:
        k = cfg["k"]
        fb = torch.zeros((1, tree.boundary_ids.size), dtype=torch.float64, device="cuda")
        body = torch.randn((k, tree.N), dtype=torch.float64, device="cuda")
        out = torch.empty_like(body)
        st.ops.solve_device(fb, body, out)
        torch.cuda.synchronize()
        torch.cuda.cudart().cudaProfilerStart()
        for _ in range(a.steps):
            st.ops.solve_device(fb, body, out)
    else:
        torch.cuda.cudart().cudaProfilerStart()
        s = st.run(s, a.steps)
    torch.cuda.synchronize()
    torch.cuda.cudart().cudaProfilerStop()
    print("done", s.t)


if __name__ == "__main__":
    main()
