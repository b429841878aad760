"""Generates the golden fixtures under tests/golden/ from the REFERENCE itself.

Run in the build container (where /root/reference exists and oracle/_ref is built):
    python tests/golden/make_golden.py
Each case stores the seeded density and the reference's outputs of
CombinedOperator::apply / layer_potentials / apply_direct, ifgf_apply (a = phi J w), the
RP singular apply, plus plan counts, so the CPU oracle restatement and the B200 path are
pinned against the reference without rebuilding it.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle import ref as R  # noqa: E402

CASES = {
    # name: (radius, splits, nu, k, gamma, strategy)
    "s1n6_k2pi_hybrid": (1.0, 1, 6, 2 * np.pi, -1.0, "hybrid"),
    "s1n6_k2pi_w4": (1.0, 1, 6, 2 * np.pi, -1.0, "w4"),
    "s0n4_k2pi_hybrid": (1.0, 0, 4, 2 * np.pi, -1.0, "hybrid"),
    "s2n6_k4pi_hybrid": (1.0, 2, 6, 4 * np.pi, -1.0, "hybrid"),
}


def make(name, radius, splits, nu, k, gamma, strategy):
    rm = R.RefMesh.sphere(radius, splits, nu, nu)
    ro = R.RefOperator(rm, k, gamma=gamma, strategy=strategy)
    phi = R.random_density(rm.n, 1)
    out = ro.apply(phi)
    S, D = ro.layer_potentials(phi)
    direct = ro.apply_direct(phi)
    a = phi * rm.jac * rm.weight
    fS, fD = ro.ifgf_apply(a)
    rS, rD = ro.rp_apply(phi)
    segs = [len(ro.level_cones(d)["seg_box"]) for d in range(3, ro.depth + 1)]
    pr = ro.proximity()
    np.savez_compressed(os.path.join(HERE, f"{name}.npz"), phi=phi, out=out, S=S, D=D, direct=direct,
                        ifgf_S=fS, ifgf_D=fD, rp_S=rS, rp_D=rD, perm=ro.perm(), depth=ro.depth,
                        gamma=ro.gamma, strategy=ro.strategy, segments=np.array(segs, dtype=np.int64),
                        npairs=len(pr["target"]), nfar=len(pr["far_nodes"]),
                        params=np.array([radius, splits, nu, k, gamma]), strategy_name=strategy)
    print(name, rm.n, "depth", ro.depth, "segments", segs, "pairs", len(pr["target"]))


if __name__ == "__main__":
    for nm, c in CASES.items():
        make(nm, *c)
