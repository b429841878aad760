"""Host setup parity: the product's geometry, octree, relations, cone plan (relevant
segments and every segment decision) and proximity pairs are bit-identical to the
reference's (any discrete mismatch costs ~1e-6)."""
import numpy as np
import pytest

import paper_2112_06316_b200 as P

PLAN_CASES = [
    # (radius, splits, nu, k, gamma, strategy)
    (1.0, 1, 6, 2 * np.pi, -1.0, "hybrid"),
    (1.0, 1, 6, 2 * np.pi, -1.0, "w4"),
    (1.0, 2, 6, 4 * np.pi, -1.0, "hybrid"),
    (0.5, 1, 6, 4 * np.pi, -1.0, "hybrid"),
    (1.0, 0, 4, 2 * np.pi, -1.0, "hybrid"),
    (1.0, 1, 8, 6 * np.pi, 3.5, "w2w3"),
]
_S = {"hybrid": P.DlStrategy.Hybrid, "w4": P.DlStrategy.W4, "w2w3": P.DlStrategy.W2W3}


@pytest.mark.parametrize("splits,nu", [(0, 4), (1, 6), (2, 16), (0, 12)])
def test_sphere_generator_bitwise(ref, splits, nu):
    pm = P.SurfaceMesh.sphere(1.0, splits, nu, nu)
    rm = ref.RefMesh.sphere(1.0, splits, nu, nu)
    nd = pm.nodes()
    for key in ("pos", "normal", "jac", "weight", "pu", "pv", "patch_of"):
        assert np.array_equal(nd[key], getattr(rm, key)), key
    for q in (0, len(rm.patches) - 1):
        pq = pm.patch(q)
        rq = rm.patches[q]
        assert (pq["du"], pq["dv"], pq["orient"]) == (rq.du, rq.dv, rq.orient)
        assert np.array_equal(pq["coeff"], rq.coeff)
        assert np.array_equal(pq["coeff_u"], rq.coeff_u)


def test_spheroid_generator_bitwise(ref):
    pm = P.SurfaceMesh.spheroid(0, 8, 8, 10.0, 2.0, 2.0)
    rm = ref.RefMesh.spheroid(0, 8, 8, 10.0, 2.0, 2.0)
    nd = pm.nodes()
    for key in ("pos", "normal", "jac", "weight"):
        assert np.array_equal(nd[key], getattr(rm, key)), key


def test_random_density_matches_reference_harness(ref):
    assert np.array_equal(P.random_density(1000, 1), ref.random_density(1000, 1))
    assert np.array_equal(P.random_density(17, 12345), ref.random_density(17, 12345))


@pytest.mark.parametrize("case", PLAN_CASES)
def test_plan_bitwise(ref, case):
    radius, splits, nu, k, gamma, strat = case
    pm = P.SurfaceMesh.sphere(radius, splits, nu, nu)
    rm = ref.RefMesh.sphere(radius, splits, nu, nu)
    hp = P.HostPlan(pm, P.SolveConfig(k=k, gamma=gamma, dl_strategy=_S[strat]))
    ro = ref.RefOperator(rm, k, gamma=gamma, strategy=strat, n_beta=8)  # beta size irrelevant here
    assert hp.depth == ro.depth
    assert hp.gamma == ro.gamma
    assert int(hp.strategy) == ro.strategy
    assert np.array_equal(hp.perm(), ro.perm())
    a, b = hp.tree_geom(), ro.tree_geom()
    assert np.array_equal(a[0], b[0]) and a[1] == b[1]
    for d in range(1, hp.depth + 1):
        x, y = hp.boxes(d), ro.boxes(d)
        for key in x:
            assert np.array_equal(x[key], y[key]), (d, key)
        for which in (0, 1):
            for u, v in zip(hp.relation(d, which), ro.relation(d, which)):
                assert np.array_equal(u, v), (d, which)
        if d >= 3:
            A, B = hp.level_cones(d), ro.level_cones(d)
            assert (A["ns"], A["nc"], A["ds"], A["dth"], A["dph"]) == (B["ns"], B["nc"], B["ds"], B["dth"], B["dph"])
            assert np.array_equal(A["seg_box"], B["seg_box"]) and np.array_equal(A["seg_gamma"], B["seg_gamma"])
    A, B = hp.proximity(), ro.proximity()
    for key in A:
        assert np.array_equal(A[key], B[key]), key


def test_plan_matches_golden_counts():
    import glob
    import os

    for f in sorted(glob.glob(os.path.join(os.path.dirname(__file__), "golden", "*.npz"))):
        g = np.load(f)
        if "params" not in g:  # the large-config fixtures: tests/test_large_fixtures.py
            continue
        radius, splits, nu, k, gamma = g["params"]
        strat = str(g["strategy_name"])
        pm = P.SurfaceMesh.sphere(float(radius), int(splits), int(nu), int(nu))
        hp = P.HostPlan(pm, P.SolveConfig(k=float(k), gamma=float(gamma), dl_strategy=_S[strat]))
        assert hp.depth == int(g["depth"])
        assert np.array_equal(hp.perm(), g["perm"])
        assert [len(hp.level_cones(d)["seg_box"]) for d in range(3, hp.depth + 1)] == list(g["segments"])
        assert len(hp.proximity()["target"]) == int(g["npairs"])
        assert hp.gamma == float(g["gamma"])


def test_beta_fingerprint_matches_reference(ref):
    pm = P.SurfaceMesh.sphere(1.0, 1, 6, 6)
    rm = ref.RefMesh.sphere(1.0, 1, 6, 6)
    hp = P.HostPlan(pm, P.SolveConfig(k=2 * np.pi))
    ro = ref.RefOperator(rm, 2 * np.pi)
    assert hp.beta_fingerprint() == ro.beta_fingerprint()


def test_diagnostics_text():
    pm = P.SurfaceMesh.sphere(1.0, 2, 16, 16)
    hp = P.HostPlan(pm, P.SolveConfig(k=4 * np.pi, gamma=4 * np.pi))
    txt = hp.diagnostics()
    assert "level 4: boxes=272 segments=9424 interp_points=706800 ns=2 nc=4" in txt
    assert "level 3: boxes=56 segments=4432" in txt
    assert hp.evaluations(4, 0) == 1071192 and hp.evaluations(4, 1) == 1646400


def test_per_rank_plans_partition_the_full_plan():
    # a per-rank plan keeps exactly the full plan's relevant segments of the boxes holding its
    # sources (same evaluations reach them), so the ranks' segment sets cover the full plan
    pm = P.SurfaceMesh.sphere(1.0, 2, 10, 10)
    k = 8 * np.pi
    full = P.HostPlan(pm, P.SolveConfig(k=k, device=-1))
    world = 3
    parts = [P.HostPlan(pm, P.SolveConfig(k=k, device=-1, part_rank=r, part_world=world)) for r in range(world)]
    for d in range(3, full.depth + 1):
        F = full.level_cones(d)
        fset = set(zip(F["seg_box"].tolist(), F["seg_gamma"].tolist()))
        union = set()
        for hp in parts:
            A = hp.level_cones(d)
            aset = set(zip(A["seg_box"].tolist(), A["seg_gamma"].tolist()))
            assert aset <= fset, d
            union |= aset
        assert union == fset, d
    # the plan-free partition is leaf aligned, covers all points and is the same on every rank
    n = pm.size()
    from paper_2112_06316_b200.distributed import plan_partition
    bounds = [plan_partition(hp, world) for hp in parts]
    assert all(np.array_equal(bounds[0], x) for x in bounds)
    assert bounds[0][0] == 0 and bounds[0][-1] == n
    with pytest.raises(P.InvalidArgument):
        plan_partition(parts[0], world + 1)


@pytest.mark.parametrize("splits,nu,k", [(1, 6, 4 * np.pi), (1, 8, 8 * np.pi), (2, 4, 8 * np.pi)])
def test_pair_accounting_each_pair_at_one_level(splits, nu, k):
    # every (target, source) pair is covered exactly once: by the leaf neighbour scope (near
    # field, self pairs included) or by one cousin list at one level (the reference's
    # "pair accounting: each far pair at exactly one level", test_ifgf.cpp:197-233)
    mesh = P.SurfaceMesh.sphere(1.0, splits, nu, nu)
    hp = P.HostPlan(mesh, P.SolveConfig(k=k))
    assert hp.depth >= 4
    n = mesh.size()
    count = np.zeros((n, n), dtype=np.int32)  # Morton x Morton
    for d in range(3, hp.depth + 1):
        bx = hp.boxes(d)
        kinds = [1] if d < hp.depth else [0, 1]  # neighbours only at the leaf level
        for which in kinds:
            ptr, idx = hp.relation(d, which)
            for b in range(len(ptr) - 1):
                b0, b1 = bx["begin"][b], bx["end"][b]
                for j in idx[ptr[b]:ptr[b + 1]]:
                    count[b0:b1, bx["begin"][j]:bx["end"][j]] += 1
    assert count.min() == 1 and count.max() == 1
