"""Multi-GPU algorithm emulated rank by rank on one B200: the sum over
ranks of the owned-source far fields equals the full far field, and the owned-target
outputs assembled over ranks equal the single-GPU apply — exactly what the NCCL
reduce / broadcast steps compute, with the collectives replaced by host sums."""
import numpy as np
import pytest

import paper_2112_06316_b200 as P

pytestmark = pytest.mark.gpu


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.mark.parametrize("world", [2, 3, 8])
def test_partitioned_apply_equals_full(world):
    mesh = P.SurfaceMesh.sphere(1.0, 2, 16, 16)  # cfg1 sphere, depth 4
    k = 4 * np.pi
    op = P.CombinedOperator(mesh, P.SolveConfig(k=k, gamma=k))
    n = mesh.size()
    phi = P.random_density(n, 1)
    full = op.apply(phi)
    nd = mesh.nodes()
    a = phi * nd["jac"] * nd["weight"]
    S_full, D_full = op.ifgf_apply(a)
    bounds = op.partition(world)
    assert bounds[0] == 0 and bounds[-1] == n and np.all(np.diff(bounds.astype(np.int64)) >= 0)
    S = np.zeros(n, complex)
    D = np.zeros(n, complex)
    for r in range(world):
        op.set_partition(int(bounds[r]), int(bounds[r + 1]))
        s, d = op.ifgf_apply(a)
        S += s
        D += d
    assert rel(S, S_full) <= 1e-13 and rel(D, D_full) <= 1e-13
    out = np.zeros(n, complex)
    owner_count = np.zeros(n, int)
    for r in range(world):
        op.set_partition(int(bounds[r]), int(bounds[r + 1]))
        o = op.finish_owned(phi, S, D)
        owner_count += (o != 0)
        out += o
    assert np.all(owner_count == 1)  # every target finished by exactly one rank
    assert rel(out, full) <= 1e-13
    op.set_partition(0, n)
    assert np.array_equal(op.apply(phi), full)


@pytest.mark.parametrize("world", [2, 3])
def test_target_sharded_beta(world):
    # SURVEY.md §8(e) "partition beta by target": each rank's operator holds only the owned
    # targets' beta tables (built after the partition), and the owned outputs assembled over
    # ranks still equal the single-GPU apply
    mesh = P.SurfaceMesh.sphere(1.0, 2, 16, 16)
    k = 4 * np.pi
    cfg = P.SolveConfig(k=k, gamma=k)
    full_op = P.CombinedOperator(mesh, cfg)
    n = mesh.size()
    phi = P.random_density(n, 3)
    full = full_op.apply(phi)
    nd = mesh.nodes()
    S, D = full_op.ifgf_apply(phi * nd["jac"] * nd["weight"])
    bounds = full_op.partition(world)
    out = np.zeros(n, complex)
    for r in range(world):
        op = P.CombinedOperator(mesh, cfg, compute_beta=False)
        op.set_partition(int(bounds[r]), int(bounds[r + 1]))
        op.compute_beta()  # owned pairs only
        out += op.finish_owned(phi, S, D)
        with pytest.raises(P.InvalidArgument):
            op.beta()  # no full tables on a sharded operator
    assert rel(out, full) <= 1e-13


@pytest.mark.parametrize("world", [2, 4])
def test_per_rank_plans(world):
    # per-rank plans (SolveConfig.part_rank / part_world): each holds only the boxes with its
    # sources; the ranks' far fields sum to the full far field and the owned outputs
    # assemble the single-GPU apply
    mesh = P.SurfaceMesh.sphere(1.0, 2, 16, 16)
    k = 4 * np.pi
    full_op = P.CombinedOperator(mesh, P.SolveConfig(k=k, gamma=k))
    n = mesh.size()
    phi = P.random_density(n, 5)
    full = full_op.apply(phi)
    nd = mesh.nodes()
    a = phi * nd["jac"] * nd["weight"]
    S_full, D_full = full_op.ifgf_apply(a)
    S = np.zeros(n, complex)
    D = np.zeros(n, complex)
    out = np.zeros(n, complex)
    segs = 0
    full_plan = P.HostPlan(mesh, P.SolveConfig(k=k, gamma=k))
    for r in range(world):
        cfg = P.SolveConfig(k=k, gamma=k, part_rank=r, part_world=world)
        plan = P.HostPlan(mesh, cfg)
        segs += sum(len(plan.level_cones(d)["seg_box"]) for d in range(3, plan.depth + 1))
        op = P.CombinedOperator(mesh, cfg, plan=plan, compute_beta=False)
        bounds = op.partition(world)
        op.set_partition(int(bounds[r]), int(bounds[r + 1]))
        op.compute_beta()
        s, d = op.ifgf_apply(a)
        S += s
        D += d
    assert rel(S, S_full) <= 1e-13 and rel(D, D_full) <= 1e-13
    # pruning: the ranks together hold about one plan's worth of segments, not world plans
    full_segs = sum(len(full_plan.level_cones(d)["seg_box"]) for d in range(3, full_plan.depth + 1))
    assert segs < 1.6 * full_segs
    # owned outputs from the per-rank operators
    for r in range(world):
        cfg = P.SolveConfig(k=k, gamma=k, part_rank=r, part_world=world)
        op = P.CombinedOperator(mesh, cfg, compute_beta=False)
        bounds = op.partition(world)
        op.set_partition(int(bounds[r]), int(bounds[r + 1]))
        op.compute_beta()
        out += op.finish_owned(phi, S_full, D_full)
    assert rel(out, full) <= 1e-13
