import sys; sys.path.insert(0, '/root/repo')
import numpy as np, torch
import paper_2306_02526_b200 as hb
n = int(sys.argv[1]) if len(sys.argv) > 1 else 8
tree = hb.build_tree(((0.0, 1.0), (0.0, 1.0)), n, n, 16)
ops = hb.build(tree, hb.OperatorCoefficients(c11=1.0, c22=1.0), sigma=1.0, dt_gamma=1e-3, layout="shared")
rng = np.random.default_rng(0)
u = ops.solve_with_body_load(rng.standard_normal(tree.boundary_ids.size), rng.standard_normal(tree.N))
torch.cuda.synchronize(); print("ok", np.linalg.norm(u))
