"""Component-wise GPU-vs-reference errors (diagnostic, not a test)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2112_06316_b200 as P
from oracle import ref as R

def rl(a, b):
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / nb) if nb > 0 else float(np.linalg.norm(a))

for (splits, nu, k, gamma) in [(1, 6, 2*np.pi, -1.0), (2, 16, 4*np.pi, 4*np.pi)]:
    pm = P.SurfaceMesh.sphere(1.0, splits, nu, nu)
    rm = R.RefMesh.sphere(1.0, splits, nu, nu)
    t = time.time(); op = P.CombinedOperator(pm, P.SolveConfig(k=k, gamma=gamma)); tg = time.time() - t
    t = time.time(); ro = R.RefOperator(rm, k, gamma=gamma); tr = time.time() - t
    print(f"== N={pm.size()} k={k:.3f}: setup gpu {tg:.2f}s ref {tr:.2f}s", flush=True)
    phi = P.random_density(pm.size(), 1)
    nd = pm.nodes(); a = phi * nd['jac'] * nd['weight']
    S, D = op.ifgf_apply(a); Sr, Dr = ro.ifgf_apply(a)
    print("ifgf S", rl(S, Sr), "D", rl(D, Dr))
    pipes = [1, 2, 3]
    perm = ro.perm()
    lf = op.level_d_fill(a[perm], pipes); lr = ro.level_d_fill(a[perm], pipes)
    print("level_d_fill", rl(lf, lr))
    off, bs, bd = op.beta(); roff, rbs, rbd = ro.beta()
    print("beta S", rl(bs, rbs), "D", rl(bd, rbd), "max abs diff", np.abs(bs - rbs).max(), np.abs(bd-rbd).max())
    rs, rd = op.rp_singular_apply(phi); rrs, rrd = ro.rp_apply(phi)
    print("rp S", rl(rs, rrs), "D", rl(rd, rrd))
    LS, LD = op.layer_potentials(phi); LSr, LDr = ro.layer_potentials(phi)
    print("layer S", rl(LS, LSr), "D", rl(LD, LDr))
    nearS = LS - S - rs; nearSr = LSr - Sr - rrs
    nearD = LD - D - rd; nearDr = LDr - Dr - rrd
    print("near S", rl(nearS, nearSr), "D", rl(nearD, nearDr))
    out = op.apply(phi); outr = ro.apply(phi)
    print("apply", rl(out, outr))
    op.set_beta(roff, rbs, rbd)
    out2 = op.apply(phi)
    print("apply with reference beta", rl(out2, outr), flush=True)
