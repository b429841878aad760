"""Generates tests/golden/<cfg>_large.npz from the REFERENCE itself for the configs whose
outputs are too large to store (see large_check.py for what is stored and why).

Run in the build container (where /root/reference exists and oracle/_ref is built):
    python tests/golden/make_large.py cfg3            # ~1 h on 8 cores, ~45 GB RAM
    python tests/golden/make_large.py cfg2 --tag val  # validation of the procedure

Steps (all reference code, oracle/ref_driver.cpp `ref_plan_*`):
  build_octree, compute_relations, plan_cones, classify_targets (solver.cpp:47-51);
  ifgf_apply + the level-D near loop (layer_potentials minus its RP term);
  beta_precompute + rp_singular_apply on the RP sub-sample's pairs.
Then, separately, the product's CPU planner (device = -1) for its per-level decision hashes.
"""
import argparse
import json
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, HERE)
import large_check as LC  # noqa: E402
from bench import CONFIGS, make_mesh  # noqa: E402
from oracle import ref as R  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("cfg")
    ap.add_argument("--tag", default="large")
    ap.add_argument("--skip-product", action="store_true")
    args = ap.parse_args()
    splits, nu, k, gamma, desc = CONFIGS[args.cfg]
    rm = make_mesh(args.cfg, R)
    n = rm.n
    phi = R.random_density(n, 1)
    t0 = time.time()
    rp = R.RefPlan(rm, k, gamma=gamma)
    print(f"[{args.cfg}] N={n} depth={rp.depth} setup {rp.setup_seconds} ({time.time() - t0:.0f} s)", flush=True)
    seg_hash = rp.segment_hashes()
    seg_count = rp.segment_counts()
    S, D, secs = rp.ifgf_near(phi)
    print(f"[{args.cfg}] ifgf+near {secs}", flush=True)
    sample = LC.sample_targets(n)
    rp_idx = LC.rp_sample_targets(sample)
    rpS, rpD, rp_pairs, rp_sec = rp.rp_sample(phi, rp_idx)
    print(f"[{args.cfg}] rp sample: {len(rp_idx)} targets, {rp_pairs} pairs, {rp_sec:.1f} s", flush=True)
    fix = dict(
        cfg=args.cfg, n=n, k=k, gamma=rp.gamma, depth=rp.depth, phi_head=phi[:8].copy(),
        sample_idx=sample, S_sample=S[sample], D_sample=D[sample],
        projS=LC.projections(S), projD=LC.projections(D),
        normS=np.linalg.norm(S), normD=np.linalg.norm(D),
        rp_idx=rp_idx, rpS=rpS, rpD=rpD, rp_pairs=rp_pairs,
        seg_levels=np.array(sorted(seg_hash), dtype=np.int64),
        seg_hash=np.array([seg_hash[d] for d in sorted(seg_hash)], dtype=np.uint64),
        seg_count=np.array([seg_count[d] for d in sorted(seg_count)], dtype=np.int64),
        perm_hash=np.uint64(rp.perm_hash()), npairs=rp.npairs(),
        ref_seconds=json.dumps(dict(rp.setup_seconds, **secs, rp_sample=rp_sec, threads=os.cpu_count())),
    )
    del S, D, rp
    if not args.skip_product:
        import paper_2112_06316_b200 as P

        t0 = time.time()
        pm = make_mesh(args.cfg, P)
        hp = P.HostPlan(pm, P.SolveConfig(k=k, gamma=gamma, device=-1))
        fix["product_cpu_decision_hash"] = np.array([hp.decision_hash(d) for d in range(3, hp.depth + 1)],
                                                    dtype=np.uint64)
        fix["product_cpu_segments"] = np.array([len(hp.level_cones(d)["seg_box"]) for d in range(3, hp.depth + 1)],
                                               dtype=np.int64)
        print(f"[{args.cfg}] product CPU planner {time.time() - t0:.0f} s", flush=True)
    path = os.path.join(HERE, f"{args.cfg}_{args.tag}.npz")
    np.savez_compressed(path, **fix)
    print("wrote", path, os.path.getsize(path))


if __name__ == "__main__":
    main()
