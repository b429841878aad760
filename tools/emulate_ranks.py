"""Multi-GPU configs on ONE B200, rank by rank: the per-rank operators of a
world-W run (per-rank plans, target-sharded beta tables) are built one after the other, each
times its own apply (far field of its sources onto all targets + near field / RP / combine of
its targets) and reports its partial results; the host then sums what the NCCL reduce-
scatter would sum. Nothing waits on another rank: each rank's kernels run alone.

  python tools/emulate_ranks.py cfg4 2 [--steps 5]

Output (one JSON line): per-rank setup / device ms per apply, the emulated W-GPU apply time
(max over ranks; the exchange — 2 x 16 N bytes reduce-scattered and 16 N all-gathered over
NVLink — is NOT included and is estimated separately), and, when tests/golden/<cfg>_large.npz
exists, parity of the assembled S, D (no RP), RP sample and out against the reference.
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests", "golden"))
import paper_2112_06316_b200 as P  # noqa: E402
from bench import CONFIGS, make_mesh  # noqa: E402


def emulate(cfg_name, world, steps=5, log=sys.stderr):
    class A:  # noqa: N801
        pass

    args = A()
    args.cfg, args.world, args.steps = cfg_name, world, steps
    splits, nu, k, gamma, desc = CONFIGS[args.cfg]
    mesh = make_mesh(args.cfg, P)
    n = mesh.size()
    phi = P.random_density(n, 1)
    nd = mesh.nodes()
    a = phi * nd["jac"] * nd["weight"]
    W = args.world
    S_far = np.zeros(n, complex)
    D_far = np.zeros(n, complex)
    ranks = []
    parts = []
    for r in range(W):
        t0 = time.perf_counter()
        cfg = P.SolveConfig(k=k, gamma=gamma, part_rank=r, part_world=W)
        plan = P.HostPlan(mesh, cfg)
        perm = plan.perm().astype(np.int64)
        gam = plan.gamma
        op = P.CombinedOperator(mesh, cfg, plan=plan, compute_beta=False)
        del plan
        b = op.partition(W)
        op.set_partition(int(b[r]), int(b[r + 1]))
        op.compute_beta()  # owned targets' pairs only
        setup = time.perf_counter() - t0
        op.upload_density(phi)
        op.time_applies(3, flush_l2=False)
        each = op.time_applies_each(args.steps, flush_l2=False)
        phases = op.time_phases()
        S_r, D_r = op.ifgf_apply(a)          # this rank's sources -> all targets
        S_lp, D_lp = op.layer_potentials(phi)  # owned targets: own far part + near + RP
        rS, rD = op.rp_singular_apply(phi)    # owned targets
        out_r = op.apply(phi)                 # owned targets: own far part + near + RP, combined
        lo, hi = int(b[r]), int(b[r + 1])
        owned = perm[lo:hi]                   # original indices of the owned Morton range
        S_far += S_r
        D_far += D_r
        parts.append((owned, S_r, D_r, S_lp, D_lp, rS, rD, out_r))
        ranks.append({"rank": r, "owned": hi - lo, "setup_s": setup, "setup_breakdown_s": op.setup_times(),
                      "ms_per_apply": float(np.mean(each)), "ms_best": float(np.min(each)), "phases_ms": phases,
                      "kernels_per_apply": op.kernels_per_apply()})
        if log:
            print(json.dumps(ranks[-1]), file=log, flush=True)
        del op
    S = np.zeros(n, complex)
    D = np.zeros(n, complex)
    RS = np.zeros(n, complex)
    RD = np.zeros(n, complex)
    out = np.zeros(n, complex)
    for owned, S_r, D_r, S_lp, D_lp, rS, rD, out_r in parts:
        # what the reduce-scatter adds: the other ranks' far partials at the owned targets
        S[owned] = S_lp[owned] + (S_far[owned] - S_r[owned])
        D[owned] = D_lp[owned] + (D_far[owned] - D_r[owned])
        RS[owned] = rS[owned]
        RD[owned] = rD[owned]
        out[owned] = out_r[owned] + (D_far[owned] - D_r[owned]) - 1j * gam * (S_far[owned] - S_r[owned])
    ms = max(x["ms_per_apply"] for x in ranks)
    res = {"cfg": args.cfg, "N": n, "world": W, "emulated": "ranks run one after the other on one B200",
           "ms_per_apply_max_over_ranks": ms, "points_per_s_emulated": n / (ms * 1e-3),
           "exchange_bytes": {"reduce_scatter": 32 * n, "all_gather": 16 * n,
                              "est_ms_nvlink_900GBps": (32 * n + 16 * n) / 900e9 * 1e3},
           "gamma": gam, "ranks": ranks}
    fix_path = os.path.join(ROOT, "tests", "golden", f"{args.cfg}_large.npz")
    if os.path.exists(fix_path):
        import large_check as LC

        fix = np.load(fix_path)
        res["parity"] = {"S_D_noRP": LC.compare(fix, S - RS, D - RD)}
        idx = fix["rp_idx"]
        res["parity"]["rp_sample"] = LC.compare_rp(fix, RS[idx], RD[idx])
        pos = np.searchsorted(fix["sample_idx"], idx)
        want = 0.5 * phi[idx] + (fix["D_sample"][pos] + fix["rpD"]) - 1j * gam * (fix["S_sample"][pos] + fix["rpS"])
        res["parity"]["out_rel_l2_rp_sample"] = float(np.linalg.norm(out[idx] - want) / np.linalg.norm(want))
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("cfg")
    ap.add_argument("world", type=int)
    ap.add_argument("--steps", type=int, default=5)
    args = ap.parse_args()
    print(json.dumps(emulate(args.cfg, args.world, args.steps)))


if __name__ == "__main__":
    main()
