"""Operator setup time per phase at a bench config: python tools/setup_times.py cfg2"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2112_06316_b200 as P
from bench import CONFIGS, make_mesh

name = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
splits, nu, k, gamma, desc = CONFIGS[name]
t = time.perf_counter()
mesh = make_mesh(name, P)
t1 = time.perf_counter()
op = P.CombinedOperator(mesh, P.SolveConfig(k=k, gamma=gamma))
t2 = time.perf_counter()
print(f"{name}: mesh {t1 - t:.2f}s operator {t2 - t1:.2f}s phases {op.setup_times()}", flush=True)
