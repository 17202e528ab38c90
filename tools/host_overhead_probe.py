"""Host cost of one replayed step (dry coefficient pass + copies + replay
launch) against its device time: is the stepper host-bound?"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_2306_02526_b200 as hb

cfg = bench.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
tree = hb.build_tree(((0.0, 1.0), (0.0, 1.0)), cfg["n"], cfg["n"], cfg["p"])
st = hb.TimeStepper(tree, hb.ParabolicProblem(**bench.make_problem(hb, cfg)), "ARK4", dt=cfg["dt"])
s = st.run(st.initial_state(), 3)
s = hb.StepperState(s.t, s.u_device)
torch.cuda.synchronize()
n = 50
t0 = time.perf_counter()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
s = st.run(s, n, check_every=n)
e1.record()
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"{cfg['name']}: host enqueue {1e3 * (t1 - t0) / n:.3f} ms/step, device {e0.elapsed_time(e1) / n:.3f} ms/step, "
      f"wall {1e3 * (t2 - t0) / n:.3f} ms/step")
# dry pass alone
G = st._graph
t0 = time.perf_counter()
for _ in range(n):
    st._dry_coefs(s.t, G["gin"], G["guards"])
print(f"dry coefficient pass {1e3 * (time.perf_counter() - t0) / n:.3f} ms")
