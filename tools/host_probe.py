"""Host cost of graph stepping: time of the per-step coefficient (dry) pass
and wall vs device time of run() for a config."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2306_02526_b200 as hb  # noqa: E402

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
tree = hb.build_tree(((0.0, 1.0), (0.0, 1.0)), cfg["n"], cfg["n"], cfg["p"])
prob = hb.ParabolicProblem(**bench.make_problem(hb, cfg))
st = hb.TimeStepper(tree, prob, "ARK4", dt=cfg["dt"])
s = st.run(st.initial_state(), 3)
s = hb.StepperState(s.t, s.u_device)
G = st._graph
t0 = time.perf_counter()
for _ in range(50):
    st._dry_coefs(s.t, G["gin"], G["guards"])
print("dry pass ms", (time.perf_counter() - t0) / 50 * 1e3)
for n in (5, 20):
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    e0.record()
    s = st.run(s, n)
    e1.record()
    torch.cuda.synchronize()
    print(n, "steps: wall ms/step", (time.perf_counter() - t0) / n * 1e3, "device ms/step", e0.elapsed_time(e1) / n)
