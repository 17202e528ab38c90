"""Per-rank cost of a subtree-sharded run, measured on ONE GPU.

For P in --parts, builds the config with a P-part plan and times (CUDA
events, graph-replayed) what rank 0 of a P-GPU run executes per stage solve:
UP over its part, the replicated TOP levels, DOWN over its part -- i.e. the
sharded solve minus the flux all-gather (P x n12 doubles, latency only) --
plus the whole ARK4 step of rank 0 (its leaf evaluations / combinations and
the three solve phases per stage).  The single-GPU solve / step are printed
beside it.  Numbers are device times, not a multi-GPU measurement."""

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import paper_2306_02526_b200 as hb  # noqa: E402
from paper_2306_02526_b200 import _lib  # noqa: E402
from paper_2306_02526_b200.sharding import ShardedTimeStepper  # noqa: E402


def graph_time(fn, reps=20):
    from paper_2306_02526_b200.solver import graph_workspace
    with graph_workspace("probe"):      # the graph's workspace, allocated by the warm call
        fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            fn()
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2")
    ap.add_argument("--parts", default="2,4,8")
    ap.add_argument("--layout", default=None)
    ap.add_argument("--steps", type=int, default=5)
    a = ap.parse_args()
    cfg = bench.CONFIGS[a.config]
    tree = hb.build_tree(((0.0, 1.0), (0.0, 1.0)), cfg["n"], cfg["n"], cfg["p"])
    prob = hb.ParabolicProblem(**bench.make_problem(hb, cfg))
    k = cfg["k"]
    res = {"config": a.config}
    st = hb.TimeStepper(tree, prob, "ARK4", dt=cfg["dt"], layout=a.layout)
    s = st.run(st.initial_state(), 2)
    body = torch.randn((k, tree.N), dtype=torch.float64, device="cuda")
    out = torch.empty_like(body)
    fb = torch.zeros((1, tree.boundary_ids.size), dtype=torch.float64, device="cuda")
    res["solve_ms_1gpu"] = graph_time(lambda: st.ops.solve_device(fb, body, out))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s = hb.StepperState(s.t, s.u_device)
    e0.record()
    s = st.run(s, a.steps)
    e1.record()
    torch.cuda.synchronize()
    res["step_ms_1gpu"] = e0.elapsed_time(e1) / a.steps
    del st
    for P in [int(x) for x in a.parts.split(",")]:
        sh = ShardedTimeStepper(tree, prob, "ARK4", dt=cfg["dt"], nparts=P, layout=a.layout)
        ops = sh.ops
        # what rank 0 of P ranks owns
        part = sh._partition
        sh._parts = (0, 1)
        sh._leaves = part.leaves(0, 1)
        sh._ir = part.interior_range(0, 1)
        sh._nloc = sh._ir[1] - sh._ir[0]
        up = lambda: ops.solve_phase(_lib.HPS_PHASE_UP, 0, 1, fb, body, out)
        top = lambda: ops.solve_phase(_lib.HPS_PHASE_TOP, 0, 1, fb, body, out)
        down = lambda: ops.solve_phase(_lib.HPS_PHASE_DOWN, 0, 1, fb, body, out)
        ls = ops.plan.lstar
        stages = [torch.zeros((k, tree.level_maps[d].count * tree.level_maps[d].n3), dtype=torch.float64,
                              device="cuda") for d in range(ls)]

        def top_rows():   # rank 0's share of the row-sharded top levels (the all-reduces excluded)
            for d in reversed(range(ls)):
                ops.top_level(d, False, 0, P, out)
            for d in range(ls):
                ops.top_level(d, True, 0, P, out, stages[d])
        r = {"up_ms": graph_time(up), "top_ms": graph_time(top), "down_ms": graph_time(down),
             "top_rows_ms": graph_time(top_rows), "top_allreduces": 2 * ls - 1,
             "full_solve_partitioned_plan_ms": graph_time(lambda: ops.solve_device(fb, body, out))}
        r["rank_solve_ms"] = r["up_ms"] + r["top_ms"] + r["down_ms"]
        r["rank_solve_rows_ms"] = r["up_ms"] + r["top_rows_ms"] + r["down_ms"]
        s2 = sh.run(sh.initial_state(), 2)          # numerically meaningless (one part), timing only
        s2 = hb.StepperState(s2.t, s2.u_device)
        e0.record()
        s2 = sh.run(s2, a.steps)
        e1.record()
        torch.cuda.synchronize()
        r["rank_step_ms"] = e0.elapsed_time(e1) / a.steps
        r["speedup_solve"] = res["solve_ms_1gpu"] / r["rank_solve_ms"]
        r["speedup_solve_rows"] = res["solve_ms_1gpu"] / r["rank_solve_rows_ms"]
        r["speedup_step"] = res["step_ms_1gpu"] / r["rank_step_ms"]
        res[f"P{P}"] = r
        del sh
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
