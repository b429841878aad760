"""The large-config reference fixtures (tests/golden/<cfg>_large.npz, made from oracle/_ref by
tests/golden/make_large.py) and their size-independent checks (large_check.py), on CPU:

* the fixture belongs to this repository's inputs: same seeded density head, the reference's
  per-level segment counts equal the product CPU planner's (recorded when it was made);
* the projection estimator measures relative L2 over ALL targets: on a perturbed copy of the
  reference's sample it reproduces the exact error to within its statistical spread;
* the sequence hashes match a direct evaluation (oracle/ref_driver.cpp ref_plan_*_hash);
* when the reference library is built here, its cfg1 plan hashes equal the product's.
"""
import glob
import os
import sys

import numpy as np
import pytest

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "golden"))
import large_check as LC  # noqa: E402

import paper_2112_06316_b200 as P  # noqa: E402

FIXTURES = sorted(glob.glob(os.path.join(HERE, "golden", "*_large.npz")))


@pytest.mark.parametrize("path", FIXTURES, ids=[os.path.basename(p) for p in FIXTURES])
def test_fixture_consistent(path):
    f = np.load(path)
    n = int(f["n"])
    assert np.array_equal(P.random_density(8, 1), f["phi_head"])
    assert len(f["sample_idx"]) == LC.SAMPLE and np.all(np.diff(f["sample_idx"]) > 0)
    assert np.array_equal(f["sample_idx"], LC.sample_targets(n))
    assert np.array_equal(f["rp_idx"], LC.rp_sample_targets(f["sample_idx"]))
    assert len(f["projS"]) == LC.K_PROJ and np.isfinite(f["normS"]) and np.isfinite(f["normD"])
    if "product_cpu_segments" in f:
        assert np.array_equal(f["seg_count"], f["product_cpu_segments"])  # reference plan == product plan


def test_projection_estimator_tracks_full_rel_l2():
    rng = np.random.default_rng(3)
    n = 200_000
    S = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    D = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    idx = LC.sample_targets(n, 4096)
    fix = {"projS": LC.projections(S), "projD": LC.projections(D), "normS": np.linalg.norm(S),
           "normD": np.linalg.norm(D), "sample_idx": idx, "S_sample": S[idx], "D_sample": D[idx]}
    for eps, frac in ((1e-12, 1.0), (1e-8, 0.01)):  # spread-out and localised errors
        e = np.zeros(n, complex)
        m = rng.random(n) < frac
        e[m] = eps * (rng.standard_normal(m.sum()) + 1j * rng.standard_normal(m.sum()))
        true = np.linalg.norm(e) / np.linalg.norm(S)
        est = LC.compare(fix, S + e, D)["S"]["rel_l2_est_full"]
        assert 0.6 * true <= est <= 1.5 * true, (eps, frac, est, true)
        assert LC.compare(fix, S, D + e)["D"]["rel_l2_est_full"] > 0


def test_sequence_hash_definition():
    v = np.array([5, 1 << 40, 7], dtype=np.uint64)
    M = (1 << 64) - 1

    def sm(x):
        x = (x + 0x9E3779B97F4A7C15) & M
        z = x
        z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M
        z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M
        return z ^ (z >> 31)

    want = sum(sm((int(x) + sm(i)) & M) for i, x in enumerate(v)) & M
    assert LC.seq_hash(v) == want


def test_plan_hashes_match_reference_cfg1(ref):
    from bench import CONFIGS, make_mesh

    splits, nu, k, gamma, _ = CONFIGS["cfg1"]
    rp = ref.RefPlan(make_mesh("cfg1", ref), k, gamma=gamma)
    hp = P.HostPlan(make_mesh("cfg1", P), P.SolveConfig(k=k, gamma=gamma, device=-1))
    assert rp.perm_hash() == LC.seq_hash(hp.perm())
    for d, h in rp.segment_hashes().items():
        L = hp.level_cones(d)
        assert LC.segment_hash(L["seg_box"], L["seg_gamma"]) == h
