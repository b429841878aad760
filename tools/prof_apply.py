"""Profiling driver: build one operator and run a few device-resident applies.
Usage: python tools/prof_apply.py [cfg1|cfg2] [applies]"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2112_06316_b200 as P
from bench import CONFIGS, make_mesh

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
applies = int(sys.argv[2]) if len(sys.argv) > 2 else 2
splits, nu, k, gamma, desc = CONFIGS[name]
t = time.perf_counter()
mesh = make_mesh(name, P)
op = P.CombinedOperator(mesh, P.SolveConfig(k=k, gamma=gamma))
print(f"setup {time.perf_counter() - t:.1f}s N={mesh.size()} breakdown {op.setup_times()}", flush=True)
op.upload_density(P.random_density(mesh.size(), 1))
ms = op.time_applies(applies, flush_l2=False)
print(f"{name}: {ms:.3f} ms/apply over {applies}; phases {op.time_phases()}", flush=True)
