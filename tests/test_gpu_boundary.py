"""Boundary behaviour of the operator API that the reference's callers rely on: argument
checks (InvalidArgument instead of out-of-bounds access), the beta-table cache of
SolveConfig::beta_cache_path (solver.cpp:64-74), target-sharded tables invalidated by a
partition change, and the multi-batch beta path (> 2^17 pairs) against the reference's own
beta_precompute (rp.cpp:309-395)."""
import os
import tempfile

import numpy as np
import pytest

import paper_2112_06316_b200 as P

pytestmark = pytest.mark.gpu


def rel_l2(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.fixture(scope="module")
def small():
    mesh = P.SurfaceMesh.sphere(1.0, 2, 6, 6)
    k = 4 * np.pi
    op = P.CombinedOperator(mesh, P.SolveConfig(k=k))
    return mesh, k, op


def test_apply_into_rejects_bad_buffers(small):
    mesh, k, op = small
    n = mesh.size()
    phi = P.random_density(n, 1)
    out = np.empty(n, np.complex128)
    op.apply_into(phi, out)
    assert np.array_equal(out, op.apply(phi))
    bad = [
        (phi.astype(np.complex64), out),          # dtype
        (phi[:-1], out),                           # short
        (np.repeat(phi, 2)[::2], out),             # strided view
        (phi, np.empty(n - 1, np.complex128)),     # short out
        (phi, np.empty((n, 1), np.complex128)),    # shape
    ]
    ro = np.empty(n, np.complex128)
    ro.flags.writeable = False
    bad.append((phi, ro))
    for a, b in bad:
        with pytest.raises(P.InvalidArgument):
            op.apply_into(a, b)


def test_beta_cache_path_written_then_reused(small):
    mesh, k, op = small
    phi = P.random_density(mesh.size(), 2)
    with tempfile.TemporaryDirectory() as d:
        path = os.path.join(d, "beta.bin")
        a = P.CombinedOperator(mesh, P.SolveConfig(k=k, beta_cache_path=path))
        assert not a.beta_cache_hit and os.path.exists(path)
        b = P.CombinedOperator(mesh, P.SolveConfig(k=k, beta_cache_path=path))
        assert b.beta_cache_hit
        assert np.array_equal(a.apply(phi), b.apply(phi))
        # a mismatching cache (other wavenumber) is ignored and overwritten, as the reference
        c = P.CombinedOperator(mesh, P.SolveConfig(k=1.5 * k, beta_cache_path=path))
        assert not c.beta_cache_hit


def test_partition_change_invalidates_sharded_beta(small):
    mesh, k, _ = small
    n = mesh.size()
    op = P.CombinedOperator(mesh, P.SolveConfig(k=k), compute_beta=False)
    b = op.partition(2)
    op.set_partition(int(b[0]), int(b[1]))
    op.compute_beta()  # tables of the owned targets only
    phi = P.random_density(n, 3)
    op.apply(phi)
    op.set_partition(0, n)  # other targets now owned: the sharded tables must not be used
    with pytest.raises(P.InternalError, match="another Morton range"):
        op.apply(phi)
    op.compute_beta()
    full = P.CombinedOperator(mesh, P.SolveConfig(k=k))
    assert np.array_equal(op.apply(phi), full.apply(phi))


def test_per_rank_plan_rejects_foreign_range():
    mesh = P.SurfaceMesh.sphere(1.0, 2, 6, 6)
    cfg = P.SolveConfig(k=4 * np.pi, part_rank=0, part_world=2)
    op = P.CombinedOperator(mesh, cfg, compute_beta=False)
    b = op.partition(2)
    op.set_partition(int(b[0]), int(b[1]))
    with pytest.raises(P.InvalidArgument, match="per-rank plan"):
        op.set_partition(int(b[1]), int(b[2]))


@pytest.mark.slow
def test_beta_multibatch_matches_reference(ref):
    # 1,536 patches of 8 x 8 nodes: more than 2^17 singular pairs, so the GPU tables are built
    # in several batches (graded rules refilled per batch); compared with the reference's own
    # beta_precompute, not with a cache of the product's tables
    splits, nu, k = 4, 8, 8 * np.pi
    pm = P.SurfaceMesh.sphere(1.0, splits, nu, nu)
    op = P.CombinedOperator(pm, P.SolveConfig(k=k))
    off, bs, bd = op.beta()
    npairs = len(off) - 1
    assert npairs > (1 << 17), npairs
    ro = ref.RefOperator(ref.RefMesh.sphere(1.0, splits, nu, nu), k)
    roff, rbs, rbd = ro.beta()
    assert np.array_equal(off, roff)
    eS, eD = rel_l2(bs, rbs), rel_l2(bd, rbd)
    # per batch, so a batch-boundary error cannot hide in the global norm
    batch = 1 << 17
    worst = 0.0
    for p0 in range(0, npairs, batch):
        a, b = int(off[p0]), int(off[min(npairs, p0 + batch)])
        worst = max(worst, rel_l2(bs[a:b], rbs[a:b]), rel_l2(bd[a:b], rbd[a:b]))
    print(f"pairs={npairs} beta rel-L2 S={eS:.3e} D={eD:.3e} worst batch {worst:.3e}")
    assert eS <= 1e-12 and eD <= 1e-12 and worst <= 1e-12
    phi = P.random_density(pm.size(), 1)
    S, D = op.rp_singular_apply(phi)
    Sr, Dr = ro.rp_apply(phi)
    assert rel_l2(S, Sr) <= 1e-10 and rel_l2(D, Dr) <= 1e-10
