"""The paper's solve-time scaling (§5.3.1) at B200 scale: run_timing over
n = 4 .. 512 leaves per side, p = 11, both operator layouts; writes the CSVs
and the log-log slopes of solve time vs DOFs."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2306_02526_b200.timing import loglog_slope, run_timing  # noqa: E402

out = {}
for layout in ("shared", "per_node"):
    rows = run_timing(sizes=(4, 8, 16, 32, 64, 128, 256, 512), p=11, layout=layout,
                      out_path=os.path.join(ROOT, "gpurun_out", f"timing_{layout}.csv"))
    ok = [r for r in rows if r["per_step_solve_seconds"]]
    big = [r for r in ok if r["N_dof"] >= 1e5]
    out[layout] = dict(rows=rows, slope_all=loglog_slope([r["N_dof"] for r in ok], [r["per_step_solve_seconds"] for r in ok]),
                       slope_large=loglog_slope([r["N_dof"] for r in big], [r["per_step_solve_seconds"] for r in big]) if len(big) > 1 else None)
print(json.dumps(out, indent=1))
