"""Host side of the field evaluation (postprocess.hpp): the Mie series and the eps
metric, against the reference's own implementations (no GPU needed)."""
import numpy as np
import pytest

import paper_2112_06316_b200 as P

def test_mie_far_field_matches_reference(ref):
    # host utility (postprocess.cpp:176-205): our partial-wave sum vs the reference's
    rng = np.random.default_rng(3)
    dirs = rng.normal(size=(64, 3))
    for kr, extra in ((2 * np.pi, 0), (16 * np.pi, 5), (0.3, 0)):
        ours = P.mie_far_field(1.0, kr, [0.2, -0.3, 1.0], dirs, extra)
        theirs = np.zeros(2 * len(dirs))
        assert ref.lib().ref_mie_far_field(1.0, kr, np.array([0.2, -0.3, 1.0]).ctypes.data_as(ref.d_p),
                                           np.ascontiguousarray(dirs).ctypes.data_as(ref.d_p), len(dirs), extra,
                                           theirs.ctypes.data_as(ref.d_p)) == 0
        theirs = theirs.view(np.complex128)
        assert np.max(np.abs(ours - theirs)) <= 1e-13 * np.max(np.abs(theirs))


def test_eps_metric_semantics():
    # max | |ref| - |apx| | / |ref| over nonzero references; zero references counted
    eps, skipped = P.eps_far(np.array([1.0, 0.0, 2j]), np.array([1.1, 5.0, -2j]))
    assert skipped == 1 and abs(eps - 0.1) < 1e-15
    with pytest.raises(P.InvalidArgument):
        P.eps_near(np.array([1.0]), np.array([1.0, 2.0]))


def test_incident_trace_kinds():
    # incident_at (solver.cpp:25-35): plane wave along (cos t sin p, sin t sin p, cos p) and
    # the point-source sum of e^{ikr}/r; a source on a node is InvalidArgument
    mesh = P.SurfaceMesh.sphere(1.0, 1, 6, 6)
    pos = mesh.nodes()["pos"]
    k = 3.0
    inc = P.IncidentField(theta=0.3, phi=2.0)
    d = inc.wave_direction()
    assert np.allclose(P.incident_trace(inc, mesh, k), np.exp(1j * k * pos @ d), rtol=0, atol=1e-14)
    src = np.array([[0.1, 0.2, -0.1], [0.0, -0.3, 0.2]])
    r = np.linalg.norm(pos[:, None, :] - src[None], axis=2)
    want = (np.exp(1j * k * r) / r).sum(axis=1)
    assert np.allclose(P.incident_trace(P.IncidentField(sources=src), mesh, k), want, rtol=1e-14, atol=0)
    with pytest.raises(P.InvalidArgument):
        P.incident_trace(P.IncidentField(sources=pos[:1]), mesh, k)


def test_closest_point_and_graded_rules_bitwise(ref):
    # proximity building blocks (rp.hpp:44-57) equal the reference's bit for bit
    pm = P.SurfaceMesh.sphere(1.0, 1, 8, 8)
    rm = ref.RefMesh.sphere(1.0, 1, 8, 8)
    rng = np.random.default_rng(1)
    for _ in range(20):
        q = int(rng.integers(0, 24))
        x = rng.normal(size=3)
        x *= rng.uniform(0.9, 1.3) / np.linalg.norm(x)
        u0, v0 = rng.uniform(-1, 1, size=2)
        ours = P.closest_point(pm, q, x, u0, v0)
        theirs = np.zeros(3)
        assert ref.lib().ref_closest_point(rm.h, q, ref._p(np.ascontiguousarray(x)), u0, v0, ref._p(theirs)) == 0
        assert ours == tuple(theirs)
    def same(a, b):  # bitwise, or both refused (NaN)
        return a == b or (np.isnan(a) and np.isnan(b))

    for d in (2, 4, 6, 9):
        for tau in np.linspace(0, 2 * np.pi, 17):
            for alpha in (-0.7, 0.0, 0.3, 1.0, 1.5):
                assert same(P.cov_xi(alpha, tau, d), ref.lib().ref_graded(2, alpha, tau, d))
                assert same(P.cov_xi_deriv(alpha, tau, d), ref.lib().ref_graded(3, alpha, tau, d))
            assert same(P.cov_w(tau, d), ref.lib().ref_graded(0, 0.0, tau, d))
            assert same(P.cov_w_deriv(tau, d), ref.lib().ref_graded(1, 0.0, tau, d))
    with pytest.raises(P.InvalidArgument):
        P.closest_point(pm, 99, [1.0, 0.0, 0.0], 0.0, 0.0)
