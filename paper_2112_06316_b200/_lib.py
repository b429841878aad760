"""ctypes binding of lib/libifgf_b200.so (the C-ABI declared in include/ifgf_b200.h).

The shared library is the product: host setup in C++ plus the sm_100a kernels. There is
no Python or CPU fallback for any compute entry point — if the library is missing this
module raises at import of the first handle.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("IFGF_B200_LIB") or os.path.join(HERE, "lib", "libifgf_b200.so")
HEADER = os.path.join(os.path.dirname(HERE), "include", "ifgf_b200.h")

d_p = C.POINTER(C.c_double)
i32_p = C.POINTER(C.c_int32)
u32_p = C.POINTER(C.c_uint32)
u64_p = C.POINTER(C.c_uint64)
vp = C.c_void_p


class IfgfConfig(C.Structure):
    _fields_ = [
        ("k", C.c_double),
        ("gamma", C.c_double),
        ("strategy", C.c_int32),
        ("finest_box_lambda", C.c_double),
        ("n_c0", C.c_int32),
        ("n_s0", C.c_int32),
        ("ps", C.c_int32),
        ("pang", C.c_int32),
        ("delta_rel", C.c_double),
        ("delta_abs", C.c_double),
        ("n_beta", C.c_int32),
        ("cov_d", C.c_int32),
        ("workers", C.c_int32),
        ("device", C.c_int32),
        ("part_rank", C.c_int32),
        ("part_world", C.c_int32),
        ("beta_cache_path", C.c_char_p),
    ]


_SIGS = {
    "ifgf_last_error": (C.c_char_p, []),
    "ifgf_config_default": (None, [C.POINTER(IfgfConfig)]),
    "ifgf_version": (C.c_int, []),
    "ifgf_surface_sphere": (C.c_int, [C.c_double, C.c_int, C.c_int, C.c_int, C.POINTER(vp)]),
    "ifgf_surface_spheroid": (C.c_int, [C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, C.c_double,
                                        C.POINTER(vp)]),
    "ifgf_surface_from_series": (C.c_int, [C.c_int, i32_p, d_p, d_p, C.POINTER(vp)]),
    "ifgf_surface_import": (C.c_int, [C.c_int, i32_p, d_p, d_p, d_p, d_p, d_p, C.c_int64, d_p, d_p, d_p,
                                      d_p, d_p, d_p, C.POINTER(vp)]),
    "ifgf_surface_size": (C.c_int64, [vp]),
    "ifgf_surface_npatches": (C.c_int, [vp]),
    "ifgf_surface_diameter": (C.c_double, [vp]),
    "ifgf_surface_nodes": (C.c_int, [vp, d_p, d_p, d_p, d_p, d_p, d_p, i32_p]),
    "ifgf_surface_patch": (C.c_int, [vp, C.c_int, i32_p, d_p, d_p, d_p, d_p]),
    "ifgf_surface_free": (None, [vp]),
    "ifgf_random_density": (C.c_int, [C.c_int64, C.c_uint64, d_p]),
    "ifgf_plan_create": (C.c_int, [vp, C.POINTER(IfgfConfig), C.POINTER(vp)]),
    "ifgf_plan_free": (None, [vp]),
    "ifgf_plan_depth": (C.c_int, [vp]),
    "ifgf_plan_gamma": (C.c_double, [vp]),
    "ifgf_plan_strategy": (C.c_int, [vp]),
    "ifgf_plan_setup_seconds": (C.c_double, [vp]),
    "ifgf_plan_perm": (C.c_int, [vp, u32_p]),
    "ifgf_plan_tree_geom": (C.c_int, [vp, d_p, d_p]),
    "ifgf_plan_nboxes": (C.c_int64, [vp, C.c_int]),
    "ifgf_plan_boxes": (C.c_int, [vp, C.c_int, u64_p, i32_p, u32_p, u32_p, i32_p, i32_p]),
    "ifgf_plan_relation": (C.c_int64, [vp, C.c_int, C.c_int, i32_p, i32_p]),
    "ifgf_plan_level": (C.c_int64, [vp, C.c_int, i32_p, d_p, i32_p, i32_p]),
    "ifgf_plan_evaluations": (C.c_int64, [vp, C.c_int, C.c_int]),
    "ifgf_plan_npairs": (C.c_int64, [vp]),
    "ifgf_plan_tile_stats": (C.c_int, [vp, C.c_int, C.POINTER(C.c_int64)]),
    "ifgf_plan_cousin_tile_stats": (C.c_int, [vp, C.c_int, C.c_int, C.POINTER(C.c_int64)]),
    "ifgf_plan_nfar": (C.c_int64, [vp]),
    "ifgf_plan_pairs": (C.c_int, [vp, u32_p, i32_p, d_p, d_p, u32_p, u32_p, u32_p, u32_p]),
    "ifgf_plan_beta_fingerprint": (C.c_uint64, [vp]),
    "ifgf_plan_diagnostics": (C.c_int, [vp, C.c_char_p, C.c_size_t]),
    "ifgf_plan_work": (C.c_int, [vp, d_p]),
    "ifgf_plan_decision_hash": (C.c_uint64, [vp, C.c_int]),
    "ifgf_operator_work": (C.c_int, [vp, d_p]),
    "ifgf_operator_create": (C.c_int, [vp, C.POINTER(IfgfConfig), C.POINTER(vp)]),
    "ifgf_operator_from_plan": (C.c_int, [vp, C.c_int, C.c_int, C.POINTER(vp)]),
    "ifgf_operator_free": (None, [vp]),
    "ifgf_operator_size": (C.c_int64, [vp]),
    "ifgf_operator_gamma": (C.c_double, [vp]),
    "ifgf_operator_setup_times": (C.c_int, [vp, d_p]),
    "ifgf_operator_apply": (C.c_int, [vp, d_p, d_p]),
    "ifgf_operator_layer_potentials": (C.c_int, [vp, d_p, d_p, d_p]),
    "ifgf_operator_apply_device": (C.c_int, [vp, vp, vp]),
    "ifgf_operator_apply_direct": (C.c_int, [vp, d_p, d_p]),
    "ifgf_operator_ifgf_apply": (C.c_int, [vp, d_p, C.c_int, C.c_int, C.c_int, d_p, d_p]),
    "ifgf_operator_level_d_fill": (C.c_int64, [vp, d_p, i32_p, C.c_int, d_p, C.c_int64]),
    "ifgf_operator_rp_apply": (C.c_int, [vp, d_p, d_p, d_p]),
    "ifgf_operator_beta_entries": (C.c_int64, [vp]),
    "ifgf_operator_npairs": (C.c_int64, [vp]),
    "ifgf_operator_set_beta": (C.c_int, [vp, u64_p, d_p, d_p]),
    "ifgf_operator_get_beta": (C.c_int, [vp, u64_p, d_p, d_p]),
    "ifgf_operator_save_beta_cache": (C.c_int, [vp, C.c_char_p]),
    "ifgf_operator_load_beta_cache": (C.c_int, [vp, C.c_char_p]),
    "ifgf_operator_beta_cache_hit": (C.c_int, [vp]),
    "ifgf_operator_upload_density": (C.c_int, [vp, d_p]),
    "ifgf_operator_time_applies": (C.c_int, [vp, C.c_int, C.c_int, d_p]),
    "ifgf_operator_time_phases": (C.c_int, [vp, d_p]),
    "ifgf_operator_time_applies_each": (C.c_int, [vp, C.c_int, C.c_int, d_p]),
    "ifgf_operator_kernels_per_apply": (C.c_int, [vp]),
    "ifgf_operator_device_phi": (vp, [vp]),
    "ifgf_operator_device_out": (vp, [vp]),
    "ifgf_nccl_unique_id": (C.c_int, [vp]),
    "ifgf_operator_set_comm": (C.c_int, [vp, C.c_int, C.c_int, vp]),
    "ifgf_operator_partition": (C.c_int, [vp, C.c_int, u32_p]),
    "ifgf_plan_partition": (C.c_int, [vp, C.c_int, u32_p]),
    "ifgf_operator_set_partition": (C.c_int, [vp, C.c_uint32, C.c_uint32]),
    "ifgf_operator_compute_beta": (C.c_int, [vp]),
    "ifgf_operator_finish_owned": (C.c_int, [vp, d_p, d_p, d_p, d_p]),
    "ifgf_gmres_solve": (C.c_int, [vp, d_p, C.c_double, C.c_int, C.c_int, d_p, d_p, C.c_int,
                                   C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "ifgf_solve": (C.c_int, [vp, C.c_double, C.c_double, C.c_double, C.c_int, C.c_int, d_p, d_p, C.c_int,
                             C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "ifgf_solve_incident": (C.c_int, [vp, C.c_double, C.c_double, d_p, C.c_int64, C.c_double, C.c_int, C.c_int, d_p,
                                      d_p, C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    "ifgf_incident_trace": (C.c_int, [vp, C.c_double, C.c_double, C.c_double, d_p, C.c_int64, d_p]),
    "ifgf_far_field": (C.c_int, [vp, d_p, C.c_double, C.c_double, C.c_int, C.c_int, C.c_int, d_p, d_p]),
    "ifgf_near_field": (C.c_int, [vp, d_p, C.c_double, C.c_double, C.c_double, C.c_double, d_p, C.c_int64, d_p,
                                  C.c_int64, C.c_double, C.c_int, d_p, d_p, C.POINTER(C.c_uint8)]),
    "ifgf_closest_point": (C.c_int, [vp, C.c_int, d_p, C.c_double, C.c_double, d_p]),
    "ifgf_graded": (C.c_double, [C.c_int, C.c_double, C.c_double, C.c_int]),
    "ifgf_rp_regular_apply": (C.c_int, [vp, d_p, d_p, C.c_int64, C.c_double, C.c_int, d_p, d_p]),
    "ifgf_mie_far_field": (C.c_int, [C.c_double, C.c_double, d_p, d_p, C.c_int64, C.c_int, d_p]),
    "ifgf_eps_metric": (C.c_int, [d_p, d_p, C.c_int64, d_p, C.POINTER(C.c_int)]),
}

_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
                "(there is no CPU fallback for the operator)")
        L = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def exported_symbols():
    return list(_SIGS)


class IfgfError(RuntimeError):
    """Base of the mirrored reference exception taxonomy (common.hpp:40-66)."""

    status = 0


class InvalidArgument(IfgfError, ValueError):
    status = 1


class ParseError(IfgfError):
    status = 2


class DegenerateGeometry(IfgfError):
    status = 3


class ConvergenceFailure(IfgfError):
    status = 4


class InternalError(IfgfError):
    status = 5


class DeviceError(IfgfError):
    status = 6


_BY_STATUS = {c.status: c for c in (InvalidArgument, ParseError, DegenerateGeometry, ConvergenceFailure,
                                    InternalError, DeviceError)}


def check(rc, what=""):
    if rc == 0:
        return
    msg = lib().ifgf_last_error().decode(errors="replace")
    cls = _BY_STATUS.get(abs(int(rc)), IfgfError)
    raise cls(f"{what}: {msg}" if what else msg)
