"""Parity of the kernel variants the default cases do not reach: non-default interpolation
orders (generic leaf / cousin / parent kernels), forced parent-fill geometry templates,
the per-lane cousin kernel, and a stretched spheroid (cfg4's geometry class: elongated
patches, different pipe plans per level)."""
import os

import numpy as np
import pytest

import paper_2112_06316_b200 as P

pytestmark = pytest.mark.gpu

TOL = 1e-10


def rel_l2(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.mark.parametrize("ps,pang", [(2, 4), (4, 6), (3, 7)])
def test_nondefault_orders(ref, ps, pang):
    pm = P.SurfaceMesh.sphere(1.0, 1, 6, 6)
    rm = ref.RefMesh.sphere(1.0, 1, 6, 6)
    k = 2 * np.pi
    op = P.CombinedOperator(pm, P.SolveConfig(k=k, cone=P.ConeConfig(ps=ps, pang=pang)))
    ro = ref.RefOperator(rm, k, ps=ps, pang=pang)
    phi = P.random_density(pm.size(), 1)
    assert rel_l2(op.apply(phi), ro.apply(phi)) <= TOL


@pytest.mark.parametrize("env,value", [("IFGF_PARENT_TEMPLATES", "force"), ("IFGF_PARENT_TEMPLATES", "0"),
                                       ("IFGF_COUSIN_TC", "0"), ("IFGF_PARENT_CB", "1"),
                                       ("IFGF_PARENT_CB", "force"), ("IFGF_SIDE_STREAM", "1"),
                                       ("IFGF_SIDE_STREAM", "rp")])
@pytest.mark.parametrize("splits,nu,k", [(2, 6, 4 * np.pi), (2, 16, 4 * np.pi), (3, 6, 8 * np.pi)])
def test_kernel_variants(ref, monkeypatch, env, value, splits, nu, k):
    monkeypatch.setenv(env, value)  # read when the operator (and its kernels) are set up
    pm = P.SurfaceMesh.sphere(1.0, splits, nu, nu)
    rm = ref.RefMesh.sphere(1.0, splits, nu, nu)
    op = P.CombinedOperator(pm, P.SolveConfig(k=k))
    ro = ref.RefOperator(rm, k)
    phi = P.random_density(pm.size(), 2)
    assert rel_l2(op.apply(phi), ro.apply(phi)) <= TOL


@pytest.mark.parametrize("strategy", ["hybrid", "w4", "w2w3"])
def test_parent_cell_batched_equals_per_segment(monkeypatch, strategy):
    # the cell-batched parent fill (parent_cb.cu: segments of one cone cell as GEMMs against
    # their children's blocks) against the per-segment kernel, on every pipe combination the
    # strategies produce (S only, D only, both), with extra evaluations routed through its
    # one-by-one exception path; equal to rounding
    pm = P.SurfaceMesh.sphere(1.0, 3, 8, 8)
    k = 8 * np.pi
    st = {"hybrid": P.DlStrategy.Hybrid, "w4": P.DlStrategy.W4, "w2w3": P.DlStrategy.W2W3}[strategy]
    nd = pm.nodes()
    a = P.random_density(pm.size(), 6) * nd["jac"] * nd["weight"]
    res = {}
    for mode, extra in (("0", None), ("force", None), ("force", "7")):
        monkeypatch.setenv("IFGF_PARENT_CB", mode)
        if extra:
            monkeypatch.setenv("IFGF_PARENT_CB_EXC_EVERY", extra)
        else:
            monkeypatch.delenv("IFGF_PARENT_CB_EXC_EVERY", raising=False)
        op = P.CombinedOperator(pm, P.SolveConfig(k=k, dl_strategy=st))
        res[(mode, extra)] = [op.ifgf_apply(a, s, d) for s, d in ((True, True), (True, False), (False, True))]
    base = res[("0", None)]
    for key in (("force", None), ("force", "7")):
        for (S0, D0), (S1, D1), which in zip(base, res[key], ("both", "S", "D")):
            if which != "D":
                assert rel_l2(S1, S0) <= 1e-13, (key, which)
            if which != "S":
                assert rel_l2(D1, D0) <= 1e-13, (key, which)


@pytest.mark.parametrize("splits,nu,k", [(2, 6, 4 * np.pi), (3, 8, 8 * np.pi), (2, 16, 4 * np.pi)])
def test_near_variants_bitwise(monkeypatch, splits, nu, k):
    # the near field's single-target warp kernels visit the same sources in the same order
    # with the same lane assignment: per-apply screening, precomputed near lists and patch
    # runs give bitwise the same near field / apply. The default target-pair lists (one
    # source row for two targets) assign lanes differently: equal to rounding.
    pm = P.SurfaceMesh.sphere(1.0, splits, nu, nu)
    phi = P.random_density(pm.size(), 4)
    res = {}
    for mode in ("screen", "lists", "runs", "pairs"):
        monkeypatch.setenv("IFGF_NEAR", mode)
        res[mode] = P.CombinedOperator(pm, P.SolveConfig(k=k)).layer_potentials(phi)
    monkeypatch.delenv("IFGF_NEAR")
    res["default"] = P.CombinedOperator(pm, P.SolveConfig(k=k)).layer_potentials(phi)
    for mode in ("lists", "runs"):
        for a, b in zip(res["screen"], res[mode]):
            assert np.array_equal(a, b), mode
    for mode in ("pairs", "default"):
        for a, b in zip(res["screen"], res[mode]):
            assert rel_l2(b, a) <= 1e-14, mode
    for a, b in zip(res["pairs"], res["default"]):
        assert np.array_equal(a, b)


@pytest.mark.parametrize("splits,nu,k", [(2, 6, 4 * np.pi), (3, 8, 8 * np.pi)])
def test_parent_merge_bitwise(monkeypatch, splits, nu, k):
    # merged parent work items (IFGF_PARENT_MERGE segments per warp) share DMMA tiles between
    # segments but add into every node accumulator in the same order: bitwise equal output
    pm = P.SurfaceMesh.sphere(1.0, splits, nu, nu)
    phi = P.random_density(pm.size(), 5)
    out = []
    for m in ("1", "2"):
        monkeypatch.setenv("IFGF_PARENT_MERGE", m)
        out.append(P.CombinedOperator(pm, P.SolveConfig(k=k)).layer_potentials(phi))
    for o in out[1:]:
        assert np.array_equal(o[0], out[0][0]) and np.array_equal(o[1], out[0][1])


@pytest.mark.parametrize("axes,k,nu", [((4.0, 1.0, 1.0), 2 * np.pi, 8), ((2.5, 0.6, 1.2), 3 * np.pi, 8),
                                       ((40.0, 4.0, 4.0), np.pi / 4, 16)])
def test_spheroid_parity(ref, axes, k, nu):
    # the last case is cfg4's (40, 4, 4) spheroid (10:1 patches) at 1/8 of its wavenumber
    pm = P.SurfaceMesh.spheroid(2, nu, nu, *axes)
    rm = ref.RefMesh.spheroid(2, nu, nu, *axes)
    op = P.CombinedOperator(pm, P.SolveConfig(k=k))
    ro = ref.RefOperator(rm, k)
    phi = P.random_density(pm.size(), 3)
    S, D = op.layer_potentials(phi)
    rS, rD = ro.layer_potentials(phi)
    assert rel_l2(S, rS) <= TOL and rel_l2(D, rD) <= TOL
    assert rel_l2(op.apply(phi), ro.apply(phi)) <= TOL


@pytest.mark.parametrize("mesh", ["sphere", "spheroid"])
def test_gpu_closest_points_bitwise(ref, mesh):
    # pair classification with the golden-section searches batched on the GPU equals the
    # host restatement and the reference bit for bit (pairs, ubar/vbar, far lists)
    if mesh == "sphere":
        pm, rm, k = P.SurfaceMesh.sphere(1.0, 2, 16, 16), ref.RefMesh.sphere(1.0, 2, 16, 16), 4 * np.pi
    else:
        pm, rm, k = P.SurfaceMesh.spheroid(2, 8, 8, 4.0, 1.0, 1.0), ref.RefMesh.spheroid(2, 8, 8, 4.0, 1.0, 1.0), 2 * np.pi
    gpu = P.HostPlan(pm, P.SolveConfig(k=k, device=0)).proximity()
    cpu = P.HostPlan(pm, P.SolveConfig(k=k, device=-1)).proximity()
    theirs = ref.RefOperator(rm, k, n_beta=8).proximity()
    for key in theirs:
        assert np.array_equal(gpu[key], theirs[key]), key
        assert np.array_equal(cpu[key], theirs[key]), key


@pytest.mark.parametrize("mesh", ["sphere", "spheroid", "cfg1", "cfg4_small"])
def test_gpu_cone_decisions_bitwise(ref, mesh):
    # segment decisions batched on the GPU (uncertain ones redone on the host with glibc)
    # give the reference's relevant segments, cousin / parent ordinals and groups bit for bit
    if mesh == "sphere":
        pm, rm, k = P.SurfaceMesh.sphere(1.0, 2, 10, 10), ref.RefMesh.sphere(1.0, 2, 10, 10), 8 * np.pi
    elif mesh == "spheroid":
        pm, rm, k = P.SurfaceMesh.spheroid(2, 8, 8, 4.0, 1.0, 1.0), ref.RefMesh.spheroid(2, 8, 8, 4.0, 1.0, 1.0), 2 * np.pi
    elif mesh == "cfg4_small":  # cfg4's (40, 4, 4) spheroid, 10:1 patches, at 1/8 the wavenumber
        pm = P.SurfaceMesh.spheroid(2, 16, 16, 40.0, 4.0, 4.0)
        rm = ref.RefMesh.spheroid(2, 16, 16, 40.0, 4.0, 4.0)
        k = np.pi / 4
    else:
        pm, rm, k = P.SurfaceMesh.sphere(1.0, 2, 16, 16), ref.RefMesh.sphere(1.0, 2, 16, 16), 4 * np.pi
    gpu = P.HostPlan(pm, P.SolveConfig(k=k, device=0))
    cpu = P.HostPlan(pm, P.SolveConfig(k=k, device=-1))
    ro = ref.RefOperator(rm, k, n_beta=8)
    assert gpu.depth == cpu.depth == ro.depth
    for d in range(3, gpu.depth + 1):
        A, B, C = gpu.level_cones(d), cpu.level_cones(d), ro.level_cones(d)
        for key in ("seg_box", "seg_gamma"):
            assert np.array_equal(A[key], C[key]) and np.array_equal(B[key], C[key]), (d, key)
        for which in (0, 1):
            assert gpu.evaluations(d, which) == cpu.evaluations(d, which)
        assert gpu.decision_hash(d) == cpu.decision_hash(d), d
    assert gpu.diagnostics() == cpu.diagnostics()


@pytest.mark.parametrize("splits,nu,k", [(0, 4, 2 * np.pi), (0, 6, np.pi), (1, 4, 4.0)])
def test_tiny_meshes_without_far_levels(ref, splits, nu, k):
    # depth < 3: no cone levels at all, the apply is near field + RP only (solver.cpp:78-147);
    # the smallest geometries the reference accepts
    pm = P.SurfaceMesh.sphere(1.0, splits, nu, nu)
    rm = ref.RefMesh.sphere(1.0, splits, nu, nu)
    op = P.CombinedOperator(pm, P.SolveConfig(k=k))
    ro = ref.RefOperator(rm, k)
    phi = P.random_density(pm.size(), 6)
    assert rel_l2(op.apply(phi), ro.apply(phi)) <= TOL
    S, D = op.layer_potentials(phi)
    rS, rD = ro.layer_potentials(phi)
    assert rel_l2(S, rS) <= TOL and rel_l2(D, rD) <= TOL


@pytest.mark.parametrize("kw", [
    dict(n_c0=3, n_s0=2),
    dict(finest_box_lambda=0.25),
    dict(finest_box_lambda=1.0),
    dict(n_beta=48, cov_d=4),
    dict(n_beta=128, cov_d=8),
])
def test_configuration_knobs(ref, kw):
    # ConeConfig / SolveConfig / RpConfig knobs (ifgf.hpp:12-17, solver.hpp:32-45,
    # rp.hpp:14-19) against the reference built with the same values
    pm = P.SurfaceMesh.sphere(1.0, 2, 8, 8)
    rm = ref.RefMesh.sphere(1.0, 2, 8, 8)
    k = 4 * np.pi
    cone = P.ConeConfig(n_c0=kw.get("n_c0", 2), n_s0=kw.get("n_s0", 1))
    rp = P.RpConfig(n_beta=kw.get("n_beta", 96), cov_d=kw.get("cov_d", 6))
    cfg = P.SolveConfig(k=k, cone=cone, rp=rp, finest_box_lambda=kw.get("finest_box_lambda", 0.5))
    op = P.CombinedOperator(pm, cfg)
    ro = ref.RefOperator(rm, k, n_c0=kw.get("n_c0", 0), n_s0=kw.get("n_s0", 0),
                         finest_box_lambda=kw.get("finest_box_lambda", 0.0), n_beta=kw.get("n_beta", 0),
                         cov_d=kw.get("cov_d", 0))
    phi = P.random_density(pm.size(), 8)
    assert rel_l2(op.apply(phi), ro.apply(phi)) <= TOL


@pytest.mark.parametrize("nu,nv", [(6, 9), (12, 5)])
def test_rectangular_patch_grids(ref, nu, nv):
    # nu != nv node grids per patch (geometry.hpp:16-34): RP coefficient transforms, beta
    # table extents and the leaf / near field all see rectangular patches
    pm = P.SurfaceMesh.sphere(1.0, 1, nu, nv)
    rm = ref.RefMesh.sphere(1.0, 1, nu, nv)
    k = 3 * np.pi
    op = P.CombinedOperator(pm, P.SolveConfig(k=k))
    ro = ref.RefOperator(rm, k)
    phi = P.random_density(pm.size(), 10)
    assert rel_l2(op.apply(phi), ro.apply(phi)) <= TOL


def test_largest_patch_resolution(ref):
    # 48 x 48 nodes per patch, the reference's limit (geometry.cpp:33): the paper's smallest
    # sphere (6 x 48^2 = 13,824 unknowns, 4 lambda); beta rows of 2,304 entries per pair
    pm = P.SurfaceMesh.sphere(1.0, 0, 48, 48)
    rm = ref.RefMesh.sphere(1.0, 0, 48, 48)
    k = 4 * np.pi
    op = P.CombinedOperator(pm, P.SolveConfig(k=k))
    ro = ref.RefOperator(rm, k)
    phi = P.random_density(pm.size(), 12)
    assert rel_l2(op.apply(phi), ro.apply(phi)) <= TOL
