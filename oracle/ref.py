"""TEST INFRASTRUCTURE ONLY: ctypes binding of oracle/_ref/libifgf_ref.so.

The library is the UNMODIFIED reference (/root/reference/proj/src/*.cpp) plus the
extern "C" shim oracle/ref_driver.cpp, built by oracle/Makefile. Only tests/,
__graft_entry__.smoke() and bench.py's CPU-baseline / reference legs may use it; the
product path (paper_2112_06316_b200) never imports this module.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_ref", "libifgf_ref.so")

_lib = None

d_p = C.POINTER(C.c_double)
i_p = C.POINTER(C.c_int)
i32_p = C.POINTER(C.c_int32)
u32_p = C.POINTER(C.c_uint32)
u64_p = C.POINTER(C.c_uint64)


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        if not available():
            raise RuntimeError(f"reference oracle not built: {LIB_PATH} (run `make -C oracle`)")
        L = C.CDLL(LIB_PATH)
        vp = C.c_void_p
        sig = {
            "ref_last_error": (C.c_char_p, []),
            "ref_mesh_sphere": (vp, [C.c_double, C.c_int, C.c_int, C.c_int]),
            "ref_mesh_spheroid": (vp, [C.c_int, C.c_int, C.c_int, C.c_double, C.c_double, C.c_double]),
            "ref_mesh_free": (None, [vp]),
            "ref_mesh_size": (C.c_long, [vp]),
            "ref_mesh_npatches": (C.c_int, [vp]),
            "ref_mesh_diameter": (C.c_double, [vp]),
            "ref_mesh_nodes": (None, [vp, d_p, d_p, d_p, d_p, d_p, d_p, i_p]),
            "ref_mesh_patch_dims": (None, [vp, C.c_int, i_p, d_p]),
            "ref_mesh_patch_coeffs": (None, [vp, C.c_int, d_p, d_p, d_p]),
            "ref_random_density": (None, [C.c_long, C.c_ulonglong, d_p]),
            "ref_op_create": (vp, [vp, C.c_double, C.c_double, C.c_int, C.c_int, C.c_char_p,
                                   C.c_int, C.c_int, C.c_int, C.c_int, C.c_double, C.c_int, C.c_int]),
            "ref_op_free": (None, [vp]),
            "ref_op_gamma": (C.c_double, [vp]),
            "ref_op_setup_seconds": (C.c_double, [vp]),
            "ref_op_beta_cache_hit": (C.c_int, [vp]),
            "ref_op_strategy": (C.c_int, [vp]),
            "ref_op_apply": (C.c_int, [vp, d_p, d_p]),
            "ref_op_layer_potentials": (C.c_int, [vp, d_p, d_p, d_p]),
            "ref_op_apply_direct": (C.c_int, [vp, d_p, d_p]),
            "ref_op_ifgf_apply": (C.c_int, [vp, d_p, C.c_int, C.c_int, C.c_int, C.c_int, d_p, d_p]),
            "ref_op_rp_apply": (C.c_int, [vp, d_p, d_p, d_p]),
            "ref_op_level_d_fill": (C.c_long, [vp, d_p, i_p, C.c_int, d_p]),
            "ref_op_depth": (C.c_int, [vp]),
            "ref_op_tree_geom": (None, [vp, d_p, d_p]),
            "ref_op_perm": (None, [vp, u32_p]),
            "ref_op_leaf_of_point": (None, [vp, i32_p]),
            "ref_op_nboxes": (C.c_long, [vp, C.c_int]),
            "ref_op_boxes": (None, [vp, C.c_int, u64_p, i32_p, u32_p, u32_p, i32_p, i32_p]),
            "ref_op_relation": (C.c_long, [vp, C.c_int, C.c_int, i32_p, i32_p]),
            "ref_op_level_cones": (C.c_long, [vp, C.c_int, i_p, d_p]),
            "ref_op_level_segs": (None, [vp, C.c_int, i32_p, i32_p]),
            "ref_op_npairs": (C.c_long, [vp]),
            "ref_op_nfar": (C.c_long, [vp]),
            "ref_op_pairs": (None, [vp, u32_p, i32_p, d_p, d_p, u32_p, u32_p, u32_p, u32_p]),
            "ref_op_delta": (None, [vp, d_p]),
            "ref_op_beta_size": (C.c_long, [vp]),
            "ref_op_beta": (None, [vp, u64_p, d_p, d_p]),
            "ref_op_beta_fingerprint": (C.c_ulonglong, [vp]),
            "ref_op_save_beta_cache": (C.c_int, [vp, C.c_char_p]),
            "ref_op_time_apply": (C.c_double, [vp, d_p, d_p]),
            "ref_solve": (C.c_int, [vp, C.c_double, C.c_double, C.c_double, C.c_double, C.c_double,
                                    C.c_int, C.c_int, C.c_int, d_p, d_p, C.c_int]),
            "ref_solve_sources": (C.c_int, [vp, C.c_double, C.c_double, d_p, C.c_long, C.c_double, C.c_int, C.c_int,
                                            d_p, d_p, C.c_int]),
            "ref_closest_point": (C.c_int, [vp, C.c_int, d_p, C.c_double, C.c_double, d_p]),
            "ref_graded": (C.c_double, [C.c_int, C.c_double, C.c_double, C.c_int]),
            "ref_rp_regular_apply": (C.c_int, [vp, d_p, d_p, C.c_long, C.c_double, d_p, d_p]),
            "ref_far_field": (C.c_int, [vp, d_p, C.c_double, C.c_double, C.c_int, C.c_int, d_p, d_p]),
            "ref_near_field": (C.c_int, [vp, d_p, C.c_double, C.c_double, C.c_double, C.c_double, d_p, C.c_long,
                                         C.c_double, d_p, d_p, C.POINTER(C.c_ubyte)]),
            "ref_mie_far_field": (C.c_int, [C.c_double, C.c_double, d_p, d_p, C.c_long, C.c_int, d_p]),
            "ref_plan_create": (vp, [vp, C.c_double, C.c_double, C.c_int, d_p]),
            "ref_plan_free": (None, [vp]),
            "ref_plan_gamma": (C.c_double, [vp]),
            "ref_plan_depth": (C.c_int, [vp]),
            "ref_plan_npairs": (C.c_long, [vp]),
            "ref_plan_nfar": (C.c_long, [vp]),
            "ref_plan_nsegs": (C.c_long, [vp, C.c_int]),
            "ref_plan_segment_hash": (C.c_ulonglong, [vp, C.c_int]),
            "ref_plan_perm_hash": (C.c_ulonglong, [vp]),
            "ref_plan_ifgf_near": (C.c_int, [vp, d_p, d_p, d_p, d_p]),
            "ref_plan_rp_sample": (C.c_int, [vp, d_p, C.POINTER(C.c_long), C.c_long, d_p, d_p,
                                             C.POINTER(C.c_long), d_p]),
        }
        for name, (res, args) in sig.items():
            f = getattr(L, name)
            f.restype = res
            f.argtypes = args
        _lib = L
    return _lib


def _p(a, t=d_p):
    return a.ctypes.data_as(t)


def _err(msg):
    return RuntimeError(f"{msg}: {lib().ref_last_error().decode()}")


@dataclass
class RefPatch:
    nu: int
    nv: int
    du: int
    dv: int
    orient: float
    coeff: np.ndarray  # (3, du*dv), u fastest
    coeff_u: np.ndarray
    coeff_v: np.ndarray


class RefMesh:
    """A reference SurfaceMesh (geometry.hpp:36-57) held by the reference library."""

    def __init__(self, handle):
        if not handle:
            raise _err("reference mesh construction failed")
        self.h = handle
        L = lib()
        n = L.ref_mesh_size(handle)
        self.n = n
        self.pos = np.zeros((n, 3))
        self.normal = np.zeros((n, 3))
        self.jac = np.zeros(n)
        self.weight = np.zeros(n)
        self.pu = np.zeros(n)
        self.pv = np.zeros(n)
        self.patch_of = np.zeros(n, dtype=np.int32)
        L.ref_mesh_nodes(handle, _p(self.pos), _p(self.normal), _p(self.jac), _p(self.weight),
                         _p(self.pu), _p(self.pv), _p(self.patch_of, i_p))
        self.patches = []
        for q in range(L.ref_mesh_npatches(handle)):
            dims = np.zeros(4, dtype=np.int32)
            orient = C.c_double()
            L.ref_mesh_patch_dims(handle, q, _p(dims, i_p), C.byref(orient))
            nu, nv, du, dv = (int(x) for x in dims)
            c = np.zeros((3, du * dv))
            cu = np.zeros((3, du * dv))
            cv = np.zeros((3, du * dv))
            L.ref_mesh_patch_coeffs(handle, q, _p(c), _p(cu), _p(cv))
            self.patches.append(RefPatch(nu, nv, du, dv, orient.value, c, cu, cv))

    @classmethod
    def sphere(cls, radius, splits, nu, nv):
        return cls(lib().ref_mesh_sphere(radius, splits, nu, nv))

    @classmethod
    def spheroid(cls, splits, nu, nv, ax, ay, az):
        return cls(lib().ref_mesh_spheroid(splits, nu, nv, ax, ay, az))

    def diameter(self):
        return lib().ref_mesh_diameter(self.h)

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.ref_mesh_free(self.h)
            self.h = None


def random_density(n, seed):
    out = np.zeros(2 * n)
    lib().ref_random_density(n, seed, _p(out))
    return out.view(np.complex128)


def _c(v):
    v = np.ascontiguousarray(v, dtype=np.complex128)
    return v.view(np.float64), v


STRATEGY = {"w4": 0, "w2w3": 1, "hybrid": 2}


class RefOperator:
    """The reference CombinedOperator (solver.hpp:50-84) behind the shim."""

    def __init__(self, mesh: RefMesh, k, gamma=-1.0, strategy="hybrid", workers=0, beta_cache="",
                 ps=0, pang=0, n_c0=0, n_s0=0, finest_box_lambda=0.0, n_beta=0, cov_d=0):
        self.mesh = mesh
        self.n = mesh.n
        self.k = k
        self.h = lib().ref_op_create(mesh.h, k, gamma, STRATEGY[strategy], workers,
                                     beta_cache.encode(), ps, pang, n_c0, n_s0,
                                     finest_box_lambda, n_beta, cov_d)
        if not self.h:
            raise _err("reference CombinedOperator construction failed")

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.ref_op_free(self.h)
            self.h = None

    @property
    def gamma(self):
        return lib().ref_op_gamma(self.h)

    @property
    def setup_seconds(self):
        return lib().ref_op_setup_seconds(self.h)

    @property
    def strategy(self):
        return lib().ref_op_strategy(self.h)

    def _call2(self, fn, phi):
        f, keep = _c(phi)
        out = np.zeros(2 * self.n)
        rc = fn(self.h, _p(f), _p(out))
        if rc:
            raise _err(f"{fn.__name__} rc={rc}")
        return out.view(np.complex128)

    def apply(self, phi):
        return self._call2(lib().ref_op_apply, phi)

    def apply_direct(self, phi):
        return self._call2(lib().ref_op_apply_direct, phi)

    def time_apply(self, phi):
        f, keep = _c(phi)
        return lib().ref_op_time_apply(self.h, _p(f), None)

    def layer_potentials(self, phi):
        f, keep = _c(phi)
        S = np.zeros(2 * self.n)
        D = np.zeros(2 * self.n)
        rc = lib().ref_op_layer_potentials(self.h, _p(f), _p(S), _p(D))
        if rc:
            raise _err("layer_potentials")
        return S.view(np.complex128), D.view(np.complex128)

    def ifgf_apply(self, a, single=True, dbl=True, strategy=None, workers=0):
        f, keep = _c(a)
        S = np.zeros(2 * self.n)
        D = np.zeros(2 * self.n)
        st = -1 if strategy is None else STRATEGY[strategy]
        rc = lib().ref_op_ifgf_apply(self.h, _p(f), int(single), int(dbl), st, workers, _p(S), _p(D))
        if rc:
            raise _err("ifgf_apply")
        return S.view(np.complex128), D.view(np.complex128)

    def rp_apply(self, phi):
        f, keep = _c(phi)
        S = np.zeros(2 * self.n)
        D = np.zeros(2 * self.n)
        rc = lib().ref_op_rp_apply(self.h, _p(f), _p(S), _p(D))
        if rc:
            raise _err("rp_apply")
        return S.view(np.complex128), D.view(np.complex128)

    def level_d_fill(self, a_perm, pipes):
        f, keep = _c(a_perm)
        pp = np.asarray(pipes, dtype=np.int32)
        size = lib().ref_op_level_d_fill(self.h, _p(f), _p(pp, i_p), len(pp), None)
        out = np.zeros(2 * size)
        got = lib().ref_op_level_d_fill(self.h, _p(f), _p(pp, i_p), len(pp), _p(out))
        if got < 0:
            raise _err("level_d_fill")
        return out.view(np.complex128)

    # ------------------------------------------------------------ plan export
    @property
    def depth(self):
        return lib().ref_op_depth(self.h)

    def perm(self):
        p = np.zeros(self.n, dtype=np.uint32)
        lib().ref_op_perm(self.h, _p(p, u32_p))
        return p

    def tree_geom(self):
        rm = np.zeros(3)
        side = C.c_double()
        lib().ref_op_tree_geom(self.h, _p(rm), C.byref(side))
        return rm, side.value

    def boxes(self, d):
        nb = lib().ref_op_nboxes(self.h, d)
        key = np.zeros(nb, dtype=np.uint64)
        coords = np.zeros((nb, 3), dtype=np.int32)
        begin = np.zeros(nb, dtype=np.uint32)
        end = np.zeros(nb, dtype=np.uint32)
        parent = np.zeros(nb, dtype=np.int32)
        children = np.zeros((nb, 8), dtype=np.int32)
        lib().ref_op_boxes(self.h, d, _p(key, u64_p), _p(coords, i32_p), _p(begin, u32_p),
                           _p(end, u32_p), _p(parent, i32_p), _p(children, i32_p))
        return dict(key=key, coords=coords, begin=begin, end=end, parent=parent, children=children)

    def relation(self, d, which):
        nb = lib().ref_op_nboxes(self.h, d)
        total = lib().ref_op_relation(self.h, d, which, None, None)
        ptr = np.zeros(nb + 1, dtype=np.int32)
        idx = np.zeros(max(total, 1), dtype=np.int32)
        lib().ref_op_relation(self.h, d, which, _p(ptr, i32_p), _p(idx, i32_p))
        return ptr, idx[:total]

    def level_cones(self, d):
        params = np.zeros(4, dtype=np.int32)
        deltas = np.zeros(3)
        nseg = lib().ref_op_level_cones(self.h, d, _p(params, i_p), _p(deltas))
        box = np.zeros(nseg, dtype=np.int32)
        gamma = np.zeros(nseg, dtype=np.int32)
        lib().ref_op_level_segs(self.h, d, _p(box, i32_p), _p(gamma, i32_p))
        return dict(ns=int(params[0]), nc=int(params[1]), ps=int(params[2]), pang=int(params[3]),
                    ds=deltas[0], dth=deltas[1], dph=deltas[2], seg_box=box, seg_gamma=gamma)

    def proximity(self):
        L = lib()
        npairs = L.ref_op_npairs(self.h)
        nfar = L.ref_op_nfar(self.h)
        target = np.zeros(npairs, dtype=np.uint32)
        patch = np.zeros(npairs, dtype=np.int32)
        ubar = np.zeros(npairs)
        vbar = np.zeros(npairs)
        fb = np.zeros(npairs, dtype=np.uint32)
        fe = np.zeros(npairs, dtype=np.uint32)
        tpb = np.zeros(self.n + 1, dtype=np.uint32)
        far = np.zeros(max(nfar, 1), dtype=np.uint32)
        L.ref_op_pairs(self.h, _p(target, u32_p), _p(patch, i32_p), _p(ubar), _p(vbar),
                       _p(fb, u32_p), _p(fe, u32_p), _p(tpb, u32_p), _p(far, u32_p))
        return dict(target=target, patch=patch, ubar=ubar, vbar=vbar, far_begin=fb, far_end=fe,
                    target_pair_begin=tpb, far_nodes=far[:nfar])

    def beta(self):
        L = lib()
        npairs = L.ref_op_npairs(self.h)
        size = L.ref_op_beta_size(self.h)
        off = np.zeros(npairs + 1, dtype=np.uint64)
        bs = np.zeros(2 * size)
        bd = np.zeros(2 * size)
        L.ref_op_beta(self.h, _p(off, u64_p), _p(bs), _p(bd))
        return off, bs.view(np.complex128), bd.view(np.complex128)

    def beta_fingerprint(self):
        return lib().ref_op_beta_fingerprint(self.h)

    def save_beta_cache(self, path):
        if lib().ref_op_save_beta_cache(self.h, path.encode()):
            raise _err("save_beta_cache")


class RefPlan:
    """The reference's setup WITHOUT the beta tables (build_octree, compute_relations,
    plan_cones, classify_targets; solver.cpp:47-51) for the configs whose tables do not fit
    here (cfg3: 101 GB). ifgf_near() = layer_potentials without its RP term (ifgf_apply +
    a restated solver.cpp:100-144 loop over the reference's green/dlayer_kernel);
    rp_sample() = the reference's beta_precompute + rp_singular_apply on the given targets'
    pairs only."""

    def __init__(self, mesh: RefMesh, k, gamma=-1.0, workers=0):
        self.mesh = mesh
        self.n = mesh.n
        self.k = k
        t = np.zeros(3)
        self.h = lib().ref_plan_create(mesh.h, k, gamma, workers, _p(t))
        if not self.h:
            raise _err("reference plan construction failed")
        self.setup_seconds = {"tree": float(t[0]), "plan_cones": float(t[1]), "classify_targets": float(t[2])}

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.ref_plan_free(self.h)
            self.h = None

    @property
    def gamma(self):
        return lib().ref_plan_gamma(self.h)

    @property
    def depth(self):
        return lib().ref_plan_depth(self.h)

    def segment_hashes(self):
        return {d: int(lib().ref_plan_segment_hash(self.h, d)) for d in range(3, self.depth + 1)}

    def segment_counts(self):
        return {d: int(lib().ref_plan_nsegs(self.h, d)) for d in range(3, self.depth + 1)}

    def perm_hash(self):
        return int(lib().ref_plan_perm_hash(self.h))

    def npairs(self):
        return int(lib().ref_plan_npairs(self.h))

    def ifgf_near(self, phi):
        """(S, D, seconds{ifgf_apply, near}) without the RP term"""
        f, keep = _c(phi)
        S = np.zeros(2 * self.n)
        D = np.zeros(2 * self.n)
        t = np.zeros(2)
        rc = lib().ref_plan_ifgf_near(self.h, _p(f), _p(S), _p(D), _p(t))
        if rc:
            raise _err("ifgf_near")
        return S.view(np.complex128), D.view(np.complex128), {"ifgf_apply": float(t[0]), "near": float(t[1])}

    def rp_sample(self, phi, targets):
        """RP (S, D) at the ascending original-index targets, npairs, seconds"""
        f, keep = _c(phi)
        tg = np.ascontiguousarray(targets, dtype=np.int64)
        S = np.zeros(2 * len(tg))
        D = np.zeros(2 * len(tg))
        npairs = C.c_long(0)
        sec = np.zeros(1)
        rc = lib().ref_plan_rp_sample(self.h, _p(f), tg.ctypes.data_as(C.POINTER(C.c_long)), len(tg), _p(S), _p(D),
                                      C.byref(npairs), _p(sec))
        if rc:
            raise _err("rp_sample")
        return S.view(np.complex128), D.view(np.complex128), int(npairs.value), float(sec[0])
