"""Per-kernel CUDA-event durations of an ARK4 step of the C2 recipe at several
tree sizes (n x n leaves, p = 16): the intercept of each kernel's time against
the leaf count is its launch / prologue / tail cost, the slope its throughput."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2306_02526_b200 as hb  # noqa: E402
from paper_2306_02526_b200 import _lib  # noqa: E402


def main():
    lib = _lib.load()
    cfg = dict(bench.CONFIGS["C2"])
    for n in [int(x) for x in (sys.argv[1:] or ["32", "64", "128", "256"])]:
        tree = hb.build_tree(((0.0, 1.0), (0.0, 1.0)), n, n, cfg["p"])
        prob = hb.ParabolicProblem(**bench.make_problem(hb, cfg))
        st = hb.TimeStepper(tree, prob, "ARK4", dt=cfg["dt"])
        s = st.initial_state()
        s = hb.StepperState(s.t, s.u_device)
        s, _ = st._advance(s)
        torch.cuda.synchronize()
        _lib.kernel_times()
        lib.hps_ktimer_enable(1)
        for _ in range(3):
            s, _ = st._advance(s)
        lib.hps_ktimer_enable(0)
        kt = _lib.kernel_times()
        print(f"n={n} leaves={n * n} " + " ".join(f"{k[:22]}={1e3 * ms / c:.1f}" for k, (ms, c) in
                                                   sorted(kt.items(), key=lambda kv: -kv[1][0])[:8]), flush=True)
        del st, s
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
