"""Operator construction at a bench config (beta tables computed on the GPU) for profiling."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2112_06316_b200 as P
from bench import CONFIGS, make_mesh

name = sys.argv[1] if len(sys.argv) > 1 else "cfg1"
splits, nu, k, gamma, desc = CONFIGS[name]
mesh = make_mesh(name, P)
t = time.perf_counter()
op = P.CombinedOperator(mesh, P.SolveConfig(k=k, gamma=gamma))
print(f"{name}: setup {time.perf_counter() - t:.2f}s {op.setup_times()}", flush=True)
