"""Host plan statistics of a bench config (depth, evaluations, RP pairs, beta bytes):
python tools/plan_stats.py cfg4"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2112_06316_b200 as P
from bench import CONFIGS, make_mesh

name = sys.argv[1] if len(sys.argv) > 1 else "cfg4"
splits, nu, k, gamma, desc = CONFIGS[name]
t = time.perf_counter()
mesh = make_mesh(name, P)
hp = P.HostPlan(mesh, P.SolveConfig(k=k, gamma=gamma))
pr = hp.proximity()
npairs = len(pr["target"])
print(f"{name}: N={mesh.size()} depth={hp.depth} plan {time.perf_counter() - t:.1f}s pairs={npairs} "
      f"({npairs / mesh.size():.2f}/target) beta={npairs * 256 * 32 / 1e9:.1f} GB far_nodes={len(pr['far_nodes'])}",
      flush=True)
for d in range(3, hp.depth + 1):
    print(d, hp.level_cones(d)["seg_box"].shape[0], hp.evaluations(d, 0), hp.evaluations(d, 1), flush=True)
