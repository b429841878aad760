import os, sys, numpy as np
sys.path.insert(0, '/root/repo')
import paper_2112_06316_b200 as P
splits, nu, k = int(sys.argv[1]), int(sys.argv[2]), float(sys.argv[3])
pm = P.SurfaceMesh.sphere(1.0, splits, nu, nu)
phi = P.random_density(pm.size(), 5)
res = {}
for m in sys.argv[4:]:
    os.environ["IFGF_PARENT_MERGE"] = m
    S, D = P.CombinedOperator(pm, P.SolveConfig(k=k)).layer_potentials(phi)
    res[m] = (S, D)
    np.save(f'/root/repo/gpurun_out/dbg_{os.environ.get("TAGV","cur")}_{m}.npy', np.stack([S, D]))
base = res[sys.argv[4]]
for m, (S, D) in res.items():
    print(m, 'S diff', np.abs(S - base[0]).max(), (S != base[0]).sum(), 'D diff', np.abs(D - base[1]).max(), (D != base[1]).sum(), flush=True)
