"""Break down the e2e step time: H2D, step, D2H on C2."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2306_02526_b200 as hb  # noqa: E402

cfg = bench.CONFIGS["C2"]
tree = hb.build_tree(((0.0, 1.0), (0.0, 1.0)), cfg["n"], cfg["n"], cfg["p"])
st = hb.TimeStepper(tree, hb.ParabolicProblem(**bench.make_problem(hb, cfg)), "ARK4", dt=cfg["dt"])
s = st.initial_state()
d = s.u_device
uh = torch.empty(tree.N, dtype=torch.float64).pin_memory()
uh.copy_(d.cpu())
out = torch.empty(tree.N, dtype=torch.float64).pin_memory()
print("pinned", uh.is_pinned(), out.is_pinned())
for it in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    x = uh.to("cuda", non_blocking=True)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    s2 = st.step(hb.StepperState(0.0, x))
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    out.copy_(s2.u_device, non_blocking=True)
    torch.cuda.synchronize()
    t3 = time.perf_counter()
    s3 = st.step(hb.StepperState(0.0, uh))
    out.copy_(s3.u_device, non_blocking=True)
    torch.cuda.synchronize()
    t4 = time.perf_counter()
    print(f"h2d {1e3*(t1-t0):.2f} ms  step {1e3*(t2-t1):.2f} ms  d2h {1e3*(t3-t2):.2f} ms  api-e2e {1e3*(t4-t3):.2f} ms")
