"""Bitwise comparison of two library builds on a few spheres:
   IFGF_B200_LIB=<a.so> python tools/bitwise_vs.py save a; IFGF_B200_LIB=<b.so> python tools/bitwise_vs.py save b;
   python tools/bitwise_vs.py cmp a b"""
import os, sys, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
CASES = [(1, 6, 2 * np.pi), (2, 8, 4 * np.pi), (3, 8, 8 * np.pi)]
out = os.path.join(os.environ.get("GRAFT_REPO_ROOT", "."), "gpurun_out")
if sys.argv[1] == "save":
    import paper_2112_06316_b200 as P
    for i, (s, nu, k) in enumerate(CASES):
        pm = P.SurfaceMesh.sphere(1.0, s, nu, nu)
        S, D = P.CombinedOperator(pm, P.SolveConfig(k=k)).layer_potentials(P.random_density(pm.size(), 3))
        np.save(f"{out}/bw_{sys.argv[2]}_{i}.npy", np.stack([S, D]))
else:
    for i in range(len(CASES)):
        a, b = np.load(f"{out}/bw_{sys.argv[2]}_{i}.npy"), np.load(f"{out}/bw_{sys.argv[3]}_{i}.npy")
        print(i, "bitwise" if np.array_equal(a, b) else f"differs, max rel {np.max(np.abs(a - b)) / np.max(np.abs(a)):.2e}")
