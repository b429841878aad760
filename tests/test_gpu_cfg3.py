"""Parity at the headline single-GPU config, cfg3 (64-wavelength sphere, N = 6,291,456),
against the reference fixture tests/golden/cfg3_large.npz (made from oracle/_ref by
tests/golden/make_large.py; what it holds and why: tests/golden/large_check.py).

* S and D without the RP term over all N (64 random projections -> estimated rel-L2) and
  exactly on 65,536 sampled targets: <= 1e-10 (north_star);
* the RP term of 16,384 targets against the reference's own beta_precompute +
  rp_singular_apply on those targets' pairs;
* out = 1/2 phi + D - i gamma S on those targets;
* the plan: Morton permutation, per-level relevant segments (the reference's plan_cones)
  and pair count equal; the GPU decider's per-evaluation decisions hash-equal to the
  product's CPU planner (glibc acos/atan2) at this size.
"""
import os
import sys

import numpy as np
import pytest

import paper_2112_06316_b200 as P

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "golden"))
import large_check as LC  # noqa: E402

FIX = os.path.join(HERE, "golden", "cfg3_large.npz")
TOL = 1e-10


@pytest.fixture(scope="module")
def cfg3():
    if not os.path.exists(FIX):
        pytest.skip("cfg3 fixture not generated (tests/golden/make_large.py cfg3)")
    fix = np.load(FIX)
    mesh = P.SurfaceMesh.sphere(1.0, 6, 16, 16)
    cfg = P.SolveConfig(k=float(fix["k"]))
    plan = P.HostPlan(mesh, cfg)  # GPU decider
    op = P.CombinedOperator(mesh, cfg, plan=plan)
    phi = P.random_density(mesh.size(), 1)
    assert np.array_equal(phi[:8], fix["phi_head"])
    return fix, mesh, plan, op, phi


def test_cfg3_plan_matches_reference(cfg3):
    fix, mesh, plan, op, phi = cfg3
    assert plan.depth == int(fix["depth"])
    assert abs(plan.gamma - float(fix["gamma"])) == 0.0
    assert LC.seq_hash(plan.perm()) == int(fix["perm_hash"])
    levels = list(fix["seg_levels"])
    for i, d in enumerate(levels):
        L = plan.level_cones(int(d))
        assert len(L["seg_box"]) == int(fix["seg_count"][i]), d
        assert LC.segment_hash(L["seg_box"], L["seg_gamma"]) == int(fix["seg_hash"][i]), d
    assert len(plan.proximity()["target"]) == int(fix["npairs"])


def test_cfg3_gpu_decisions_equal_cpu_planner(cfg3):
    fix, mesh, plan, op, phi = cfg3
    if "product_cpu_decision_hash" not in fix:
        pytest.skip("fixture made without the CPU-planner hashes")
    got = [plan.decision_hash(d) for d in range(3, plan.depth + 1)]
    assert got == [int(x) for x in fix["product_cpu_decision_hash"]]


def test_cfg3_layer_potentials_and_rp(cfg3):
    fix, mesh, plan, op, phi = cfg3
    S, D = op.layer_potentials(phi)
    rS, rD = op.rp_singular_apply(phi)
    res = LC.compare(fix, S - rS, D - rD)
    print(res)
    for name in ("S", "D"):
        assert res[name]["rel_l2_est_full"] <= TOL, res
        assert res[name]["rel_l2_sample"] <= TOL, res
        assert res[name]["rel_norm_diff"] <= TOL, res
    idx = fix["rp_idx"]
    rp = LC.compare_rp(fix, rS[idx], rD[idx])
    print(rp)
    assert rp["S"]["rel_l2_sample"] <= TOL and rp["D"]["rel_l2_sample"] <= TOL
    out = op.apply(phi)
    pos = np.searchsorted(fix["sample_idx"], idx)
    g = float(fix["gamma"])
    want = 0.5 * phi[idx] + (fix["D_sample"][pos] + fix["rpD"]) - 1j * g * (fix["S_sample"][pos] + fix["rpS"])
    e = float(np.linalg.norm(out[idx] - want) / np.linalg.norm(want))
    print(f"cfg3 out (RP-sampled targets) rel-L2 {e:.3e}")
    assert e <= TOL
