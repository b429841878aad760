"""Fields after the solve (postprocess.cpp): GPU far/near-field sums vs
the reference's own far_field / near_field on the same density, and the physics check of a
solved sphere against the Mie series (eps_far equal to the reference's)."""
import numpy as np
import pytest

import paper_2112_06316_b200 as P

pytestmark = pytest.mark.gpu


def _ref_far(ref, rm, dens, gamma, k, n_phi, n_theta):
    dirs = np.zeros(3 * n_phi * n_theta)
    vals = np.zeros(2 * n_phi * n_theta)
    d = np.ascontiguousarray(dens, dtype=np.complex128).view(np.float64)
    assert ref.lib().ref_far_field(rm.h, ref._p(d), gamma, k, n_phi, n_theta, ref._p(dirs), ref._p(vals)) == 0
    return dirs.reshape(-1, 3), vals.view(np.complex128)


def test_far_field_matches_reference(ref):
    k = 2 * np.pi * 1.5
    pm = P.SurfaceMesh.sphere(1.0, 1, 8, 8)
    rm = ref.RefMesh.sphere(1.0, 1, 8, 8)
    dens = P.random_density(pm.size(), 7)
    g = P.far_field(pm, dens, 3.0, k, 9, 17)
    dirs, vals = _ref_far(ref, rm, dens, 3.0, k, 9, 17)
    assert np.allclose(g.directions, dirs, rtol=0, atol=1e-15)
    assert np.max(np.abs(g.values - vals)) <= 1e-12 * np.max(np.abs(vals))
    assert g.direction(2, 3).shape == (3,)


def test_near_field_matches_reference(ref):
    k = 2 * np.pi
    pm = P.SurfaceMesh.sphere(1.0, 1, 8, 8)
    rm = ref.RefMesh.sphere(1.0, 1, 8, 8)
    dens = P.random_density(pm.size(), 11)
    rng = np.random.default_rng(5)
    dirs = rng.normal(size=(40, 3))
    dirs /= np.linalg.norm(dirs, axis=1)[:, None]
    radii = np.concatenate([np.linspace(1.2, 3.0, 30), [0.3, 0.5, 0.9, 1.0005, 1.01, 1.05, 0.0, 2.0, 1.5, 4.0]])
    pts = dirs * radii[:, None]
    nf = P.near_field(pm, dens, 4.0, k, P.IncidentField(theta=0.4, phi=2.1), pts, 0.02)
    sc = np.zeros(2 * len(pts))
    tot = np.zeros(2 * len(pts))
    flg = np.zeros(len(pts), dtype=np.uint8)
    d = np.ascontiguousarray(dens).view(np.float64)
    import ctypes as C

    assert ref.lib().ref_near_field(rm.h, ref._p(d), 4.0, k, 0.4, 2.1, ref._p(np.ascontiguousarray(pts)), len(pts),
                                    0.02, ref._p(sc), ref._p(tot), flg.ctypes.data_as(C.POINTER(C.c_ubyte))) == 0
    sc = sc.view(np.complex128)
    tot = tot.view(np.complex128)
    far = radii > 1.05
    assert np.max(np.abs(nf.scattered[far] - sc[far])) <= 1e-12 * np.max(np.abs(sc[far]))
    assert np.max(np.abs(nf.total[far] - tot[far])) <= 1e-12 * np.max(np.abs(tot[far]))
    assert np.array_equal(nf.flagged, flg)  # interior / close points flagged identically
    assert nf.flagged[radii < 0.95].all() and not nf.flagged[radii > 1.1].any()


def test_solved_sphere_far_field_against_mie(ref):
    # 2-lambda sphere, plane wave along -z (solver.hpp default phi = pi): eps_far vs Mie
    radius, k = 1.0, 2 * np.pi
    pm = P.SurfaceMesh.sphere(radius, 2, 10, 10)
    op = P.CombinedOperator(pm, P.SolveConfig(k=k))
    inc = P.IncidentField(theta=0.0, phi=np.pi)
    res = P.solve(op, inc, tol=1e-8, max_iter=200)
    assert res.converged
    g = P.far_field(pm, res.solution, op.gamma, k, 21, 41)
    d = [np.cos(inc.theta) * np.sin(inc.phi), np.sin(inc.theta) * np.sin(inc.phi), np.cos(inc.phi)]
    mie = P.mie_far_field(radius, k, d, g.directions)
    eps, skipped = P.eps_far(mie, g.values)
    assert skipped == 0 and eps < 1e-3
    # the reference's own solve + far field reaches the same accuracy
    rm = ref.RefMesh.sphere(radius, 2, 10, 10)
    dens = np.zeros(2 * pm.size())
    hist = np.zeros(200)
    it = ref.lib().ref_solve(rm.h, k, -1.0, inc.theta, inc.phi, 1e-8, 200, 0, 0, ref._p(dens), ref._p(hist), 200)
    assert it == res.iterations
    _, rvals = _ref_far(ref, rm, dens.view(np.complex128), op.gamma, k, 21, 41)
    eps_ref, _ = P.eps_far(mie, rvals)
    assert abs(eps - eps_ref) <= 1e-6 * max(eps_ref, 1e-12) + 1e-9


def test_point_source_solve_and_exterior_cancellation(ref):
    # IncidentField::Kind::PointSources (solver.hpp:17-26): GMRES matches the reference's
    # iterations, and for sources INSIDE the sound-soft sphere the exterior total field
    # vanishes (scattered = -incident), a check of the whole solve + near-field chain
    k = 2 * np.pi
    pm = P.SurfaceMesh.sphere(1.0, 2, 10, 10)
    op = P.CombinedOperator(pm, P.SolveConfig(k=k))
    src = np.array([[0.1, -0.2, 0.15], [-0.3, 0.05, 0.0]])
    inc = P.IncidentField(sources=src)
    res = P.solve(op, inc, tol=1e-8, max_iter=200)
    assert res.converged
    rm = ref.RefMesh.sphere(1.0, 2, 10, 10)
    dens = np.zeros(2 * pm.size())
    hist = np.zeros(200)
    it = ref.lib().ref_solve_sources(rm.h, k, -1.0, ref._p(np.ascontiguousarray(src)), len(src), 1e-8, 200, 0,
                                     ref._p(dens), ref._p(hist), 200)
    assert it == res.iterations
    assert np.allclose(res.residual_history, hist[:it], rtol=1e-7, atol=0)
    rng = np.random.default_rng(9)
    d = rng.normal(size=(50, 3))
    pts = d / np.linalg.norm(d, axis=1)[:, None] * rng.uniform(1.5, 3.0, size=(50, 1))
    nf = P.near_field(pm, res.solution, op.gamma, k, inc, pts, 0.05)
    assert not nf.flagged.any()
    u_inc = nf.total - nf.scattered
    assert np.max(np.abs(nf.total)) <= 1e-4 * np.max(np.abs(u_inc))


def test_rp_regular_apply_matches_reference(ref):
    # regular Fejer-rule S and D at off-surface targets (rp.hpp:78-82), accumulated into the
    # outputs; a target on a node is InvalidArgument like the reference
    k = 3 * np.pi
    pm = P.SurfaceMesh.sphere(1.0, 1, 8, 8)
    rm = ref.RefMesh.sphere(1.0, 1, 8, 8)
    dens = P.random_density(pm.size(), 4)
    rng = np.random.default_rng(2)
    d = rng.normal(size=(60, 3))
    t = d / np.linalg.norm(d, axis=1)[:, None] * rng.uniform(0.2, 3.0, size=(60, 1))
    S0 = np.full(60, 0.5 + 0.25j)
    S, D = P.rp_regular_apply(pm, dens, t, k, out_single=S0.copy())
    rs = np.zeros(120)
    rd = np.zeros(120)
    dd = np.ascontiguousarray(dens).view(np.float64)
    assert ref.lib().ref_rp_regular_apply(rm.h, ref._p(dd), ref._p(np.ascontiguousarray(t)), 60, k, ref._p(rs),
                                          ref._p(rd)) == 0
    rs = rs.view(np.complex128)
    rd = rd.view(np.complex128)
    assert np.max(np.abs(S - S0 - rs)) <= 1e-12 * np.max(np.abs(rs))
    assert np.max(np.abs(D - rd)) <= 1e-12 * np.max(np.abs(rd))
    with pytest.raises(P.InvalidArgument):
        P.rp_regular_apply(pm, dens, pm.nodes()["pos"][:2], k)
