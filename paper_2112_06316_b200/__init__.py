"""B200-native combined-field operator apply of the IFGF/RP-accelerated CFIE solver
(arXiv 2112.06316): host setup in C++, hot path in hand-written sm_100a CUDA, behind the
C-ABI of include/ifgf_b200.h. This package is the Python mirror of the reference's C++
operator API (solver.hpp / geometry.hpp / ifgf.hpp / rp.hpp)."""
from ._lib import (ConvergenceFailure, DegenerateGeometry, DeviceError, IfgfError, InternalError,
                   InvalidArgument, ParseError, lib)
from .operator import (CombinedOperator, closest_point, cov_w, cov_w_deriv, cov_xi, cov_xi_deriv, ConeConfig, DlStrategy, Factor, GmresResult, HostPlan,
                       IncidentField, RpConfig, SolveConfig, SurfaceMesh, gmres_solve, incident_trace, nccl_unique_id,
                       random_density, solve)
from .postprocess import (FarFieldGrid, NearFieldGrid, eps_far, eps_near, far_field, mie_far_field,
                          near_field, rp_regular_apply)

__all__ = [
    "CombinedOperator", "closest_point", "cov_w", "cov_w_deriv", "cov_xi", "cov_xi_deriv", "ConeConfig", "DlStrategy", "Factor", "GmresResult", "HostPlan", "IncidentField",
    "RpConfig", "SolveConfig", "SurfaceMesh", "gmres_solve", "incident_trace", "nccl_unique_id", "random_density", "solve", "lib",
    "IfgfError", "InvalidArgument", "ParseError", "DegenerateGeometry", "ConvergenceFailure",
    "InternalError", "DeviceError", "FarFieldGrid", "NearFieldGrid", "far_field", "near_field",
    "mie_far_field", "eps_far", "eps_near", "rp_regular_apply",
]
