"""Fields after the solve — mirror of the reference's postprocess.hpp.

far_field / near_field run their dense sums on the GPU over the oversampled surface
quadrature (csrc/cuda/fields.cu); mie_far_field and the eps metrics are host utilities.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from ._lib import InvalidArgument, check, lib
from .operator import IncidentField, SurfaceMesh, _cvec, _ptr


@dataclass
class FarFieldGrid:  # postprocess.hpp:14-22
    n_phi: int
    n_theta: int
    directions: np.ndarray  # (n_phi * n_theta, 3), phi (polar) index fastest
    values: np.ndarray      # complex

    def direction(self, m: int, n: int) -> np.ndarray:
        return self.directions[m + self.n_phi * n]


@dataclass
class NearFieldGrid:  # postprocess.hpp:24-32
    points: np.ndarray
    scattered: np.ndarray
    total: np.ndarray
    flagged: np.ndarray
    nx: int = 0
    ny: int = 0


def far_field(mesh: SurfaceMesh, density, gamma: float, k: float, n_phi: int, n_theta: int,
              device: int = 0) -> FarFieldGrid:
    """u_inf(xhat) = (1/4pi) Int {-ik <xhat,nu> - i gamma} e^{-ik xhat.y} phi dS
    (postprocess.cpp:83-104)."""
    phi = _cvec(density, mesh.size())
    n = int(n_phi) * int(n_theta)
    dirs = np.zeros((max(n, 0), 3))
    vals = np.zeros(max(n, 0), dtype=np.complex128)
    check(lib().ifgf_far_field(mesh._h, _ptr(phi), gamma, k, n_phi, n_theta, device, _ptr(dirs), _ptr(vals)),
          "far_field")
    return FarFieldGrid(int(n_phi), int(n_theta), dirs, vals)


def near_field(mesh: SurfaceMesh, density, gamma: float, k: float, incident: IncidentField, points,
               flag_distance: float, device: int = 0, sources=None) -> NearFieldGrid:
    """scattered = D[phi] - i gamma S[phi] at off-surface points, total = scattered + u^i
    (postprocess.cpp:106-139); `sources` switches the incidence to point sources."""
    phi = _cvec(density, mesh.size())
    pts = np.ascontiguousarray(points, dtype=np.float64).reshape(-1, 3)
    if sources is None and incident.sources is not None:
        sources = incident.sources
    src = np.ascontiguousarray(sources if sources is not None else np.zeros((0, 3)), dtype=np.float64).reshape(-1, 3)
    npts = pts.shape[0]
    sc = np.zeros(npts, dtype=np.complex128)
    tot = np.zeros(npts, dtype=np.complex128)
    flg = np.zeros(npts, dtype=np.uint8)
    check(lib().ifgf_near_field(mesh._h, _ptr(phi), gamma, k, incident.theta, incident.phi, _ptr(src),
                                src.shape[0], _ptr(pts), npts, flag_distance, device, _ptr(sc), _ptr(tot),
                                flg.ctypes.data_as(C.POINTER(C.c_uint8))), "near_field")
    return NearFieldGrid(pts, sc, tot, flg)


def rp_regular_apply(mesh: SurfaceMesh, density, targets, k: float, out_single=None, out_dbl=None,
                     device: int = 0):
    """S and D of the density at off-surface targets by the nodal Fejér rule (rp.hpp:78-82),
    added into out_single / out_dbl (new zero arrays when not given); returns both."""
    phi = _cvec(density, mesh.size())
    t = np.ascontiguousarray(targets, dtype=np.float64).reshape(-1, 3)
    S = np.zeros(t.shape[0], dtype=np.complex128) if out_single is None else _cvec(out_single, t.shape[0])
    D = np.zeros(t.shape[0], dtype=np.complex128) if out_dbl is None else _cvec(out_dbl, t.shape[0])
    check(lib().ifgf_rp_regular_apply(mesh._h, _ptr(phi), _ptr(t), t.shape[0], k, device, _ptr(S), _ptr(D)),
          "rp_regular_apply")
    return S, D


def mie_far_field(radius: float, k: float, direction, eval_directions, extra_terms: int = 0) -> np.ndarray:
    """Sound-soft sphere far field for plane-wave incidence along `direction`
    (postprocess.cpp:176-205)."""
    d = np.ascontiguousarray(direction, dtype=np.float64).reshape(3)
    e = np.ascontiguousarray(eval_directions, dtype=np.float64).reshape(-1, 3)
    out = np.zeros(e.shape[0], dtype=np.complex128)
    check(lib().ifgf_mie_far_field(radius, k, _ptr(d), _ptr(e), e.shape[0], extra_terms, _ptr(out)),
          "mie_far_field")
    return out


def _eps(reference, approx):
    r = _cvec(reference)
    a = _cvec(approx)
    if r.shape != a.shape:
        raise InvalidArgument("eps metric: grid size mismatch")
    eps = C.c_double()
    skipped = C.c_int()
    check(lib().ifgf_eps_metric(_ptr(r), _ptr(a), r.shape[0], C.byref(eps), C.byref(skipped)), "eps metric")
    return eps.value, skipped.value


def eps_far(reference, approx):
    """max | |ref| - |apx| | / |ref| over nonzero references; returns (eps, skipped)."""
    return _eps(reference, approx)


def eps_near(reference, approx):
    return _eps(reference, approx)
