"""Python mirror of the reference operator API over the C-ABI.

Names, argument meaning and error behaviour follow /root/reference/proj/include/ifgf/
(solver.hpp:32-112, geometry.hpp:36-73, ifgf.hpp:12-118, rp.hpp:14-100) so the parity
tests read like the reference's own doctest suites. Complex vectors are numpy complex128
in original node order.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from enum import IntEnum

import numpy as np

from . import _lib
from ._lib import IfgfConfig, check, d_p, i32_p, lib, u32_p, u64_p


class DlStrategy(IntEnum):
    W4 = 0
    W2W3 = 1
    Hybrid = 2


class Factor(IntEnum):
    W1 = 1
    W2 = 2
    W3 = 3
    W4 = 4


@dataclass
class ConeConfig:  # ifgf.hpp:12-17
    n_c0: int = 2
    n_s0: int = 1
    ps: int = 3
    pang: int = 5


@dataclass
class RpConfig:  # rp.hpp:14-19
    delta_rel: float = 1.0
    delta_abs: float = -1.0
    n_beta: int = 96
    cov_d: int = 6


@dataclass
class SolveConfig:  # solver.hpp:32-45 (+ device)
    k: float = 0.0
    gamma: float = -1.0
    tol: float = 1e-4
    max_iter: int = 300
    restart: int = 0
    finest_box_lambda: float = 0.5
    cone: ConeConfig = field(default_factory=ConeConfig)
    dl_strategy: DlStrategy = DlStrategy.Hybrid
    rp: RpConfig = field(default_factory=RpConfig)
    workers: int = 0
    device: int = 0
    # per-rank plan of a multi-GPU run: only boxes with sources of this rank's Morton range
    part_rank: int = 0
    part_world: int = 1
    beta_cache_path: str = ""  # solver.hpp:44: load the "rpbeta v1" cache or compute + save

    def to_c(self) -> IfgfConfig:
        c = IfgfConfig()
        lib().ifgf_config_default(C.byref(c))
        c.k = self.k
        c.gamma = self.gamma
        c.strategy = int(self.dl_strategy)
        c.finest_box_lambda = self.finest_box_lambda
        c.n_c0, c.n_s0, c.ps, c.pang = self.cone.n_c0, self.cone.n_s0, self.cone.ps, self.cone.pang
        c.delta_rel, c.delta_abs = self.rp.delta_rel, self.rp.delta_abs
        c.n_beta, c.cov_d = self.rp.n_beta, self.rp.cov_d
        c.workers = self.workers
        c.device = self.device
        c.part_rank = self.part_rank
        c.part_world = self.part_world
        c.beta_cache_path = self.beta_cache_path.encode() if self.beta_cache_path else None
        return c


def _ptr(a, t=d_p):
    return a.ctypes.data_as(t)


def _cvec(v, n=None):
    v = np.ascontiguousarray(v, dtype=np.complex128)
    if n is not None and v.shape != (n,):
        raise _lib.InvalidArgument(f"size mismatch: expected {n} complex values, got {v.shape}")
    return v


def nccl_unique_id() -> bytes:
    """128-byte ncclUniqueId for set_comm (rank 0 creates it, the others receive it)"""
    buf = C.create_string_buffer(128)
    check(lib().ifgf_nccl_unique_id(buf), "nccl_unique_id")
    return buf.raw


def closest_point(mesh: "SurfaceMesh", q: int, x, u0: float, v0: float):
    """(u, v, dist) of the closest point of patch q to x (rp.hpp:49-51)."""
    out = np.zeros(3)
    check(lib().ifgf_closest_point(mesh._h, int(q), _ptr(np.ascontiguousarray(x, dtype=np.float64)), u0, v0,
                                   _ptr(out)), "closest_point")
    return float(out[0]), float(out[1]), float(out[2])


def cov_w(tau: float, d: int) -> float:  # rp.hpp:53-57, graded change of variables
    return float(lib().ifgf_graded(0, 0.0, tau, d))


def cov_w_deriv(tau: float, d: int) -> float:
    return float(lib().ifgf_graded(1, 0.0, tau, d))


def cov_xi(alpha: float, tau: float, d: int) -> float:
    return float(lib().ifgf_graded(2, alpha, tau, d))


def cov_xi_deriv(alpha: float, tau: float, d: int) -> float:
    return float(lib().ifgf_graded(3, alpha, tau, d))


def random_density(n: int, seed: int) -> np.ndarray:
    """U(-1,1) + i U(-1,1) from std::mt19937_64(seed), in the reference harness's draw order."""
    out = np.zeros(n, dtype=np.complex128)
    check(lib().ifgf_random_density(n, seed, _ptr(out)), "random_density")
    return out


class SurfaceMesh:
    """Patches + flat per-node arrays (geometry.hpp:36-57), owned by the C library."""

    def __init__(self, handle):
        self._h = handle

    @classmethod
    def _make(cls, fn, *args):
        h = C.c_void_p()
        check(fn(*args, C.byref(h)), fn.__name__)
        return cls(h)

    @classmethod
    def sphere(cls, radius: float, splits: int, nu: int, nv: int) -> "SurfaceMesh":  # build_sphere
        return cls._make(lib().ifgf_surface_sphere, radius, splits, nu, nv)

    @classmethod
    def spheroid(cls, splits, nu, nv, ax, ay, az) -> "SurfaceMesh":
        return cls._make(lib().ifgf_surface_spheroid, splits, nu, nv, ax, ay, az)

    @classmethod
    def from_series(cls, dims, coeff, interior=(0.0, 0.0, 0.0)) -> "SurfaceMesh":  # assemble_mesh
        dims = np.ascontiguousarray(dims, dtype=np.int32).reshape(-1)
        coeff = np.ascontiguousarray(coeff, dtype=np.float64).reshape(-1)
        inter = np.asarray(interior, dtype=np.float64)
        return cls._make(lib().ifgf_surface_from_series, len(dims) // 4, _ptr(dims, i32_p), _ptr(coeff),
                         _ptr(inter))

    @classmethod
    def import_arrays(cls, dims, orient, coeff, coeff_u, coeff_v, interior, pos, normal, jac, weight, pu,
                      pv) -> "SurfaceMesh":
        dims = np.ascontiguousarray(dims, dtype=np.int32).reshape(-1)
        arrs = [np.ascontiguousarray(a, dtype=np.float64).reshape(-1)
                for a in (orient, coeff, coeff_u, coeff_v, interior, pos, normal, jac, weight, pu, pv)]
        n = len(arrs[7])
        return cls._make(lib().ifgf_surface_import, len(dims) // 4, _ptr(dims, i32_p), *(_ptr(a) for a in arrs[:5]),
                         n, *(_ptr(a) for a in arrs[5:]))

    def __del__(self):
        if getattr(self, "_h", None) and _lib._lib is not None:
            _lib._lib.ifgf_surface_free(self._h)
            self._h = None

    def size(self) -> int:
        return int(lib().ifgf_surface_size(self._h))

    def npatches(self) -> int:
        return int(lib().ifgf_surface_npatches(self._h))

    def diameter(self) -> float:
        return float(lib().ifgf_surface_diameter(self._h))

    def nodes(self) -> dict:
        n = self.size()
        out = dict(pos=np.zeros((n, 3)), normal=np.zeros((n, 3)), jac=np.zeros(n), weight=np.zeros(n),
                   pu=np.zeros(n), pv=np.zeros(n), patch_of=np.zeros(n, dtype=np.int32))
        check(lib().ifgf_surface_nodes(self._h, _ptr(out["pos"]), _ptr(out["normal"]), _ptr(out["jac"]),
                                       _ptr(out["weight"]), _ptr(out["pu"]), _ptr(out["pv"]),
                                       _ptr(out["patch_of"], i32_p)), "surface_nodes")
        return out

    def patch(self, q: int) -> dict:
        dims = np.zeros(4, dtype=np.int32)
        orient = C.c_double()
        check(lib().ifgf_surface_patch(self._h, q, _ptr(dims, i32_p), C.byref(orient), None, None, None), "patch")
        m = int(dims[2]) * int(dims[3])
        c, cu, cv = np.zeros(3 * m), np.zeros(3 * m), np.zeros(3 * m)
        check(lib().ifgf_surface_patch(self._h, q, None, None, _ptr(c), _ptr(cu), _ptr(cv)), "patch")
        return dict(nu=int(dims[0]), nv=int(dims[1]), du=int(dims[2]), dv=int(dims[3]), orient=orient.value,
                    coeff=c.reshape(3, m), coeff_u=cu.reshape(3, m), coeff_v=cv.reshape(3, m))


class HostPlan:
    """CPU-side setup (octree, relations, cone plan, proximity) — the CombinedOperator ctor
    minus the device upload (solver.cpp:43-62). Exposed for plan-parity tests."""

    def __init__(self, mesh: SurfaceMesh, cfg: SolveConfig):
        self.mesh = mesh
        self.cfg = cfg
        h = C.c_void_p()
        c = cfg.to_c()
        check(lib().ifgf_plan_create(mesh._h, C.byref(c), C.byref(h)), "plan_create")
        self._h = h
        self.n = mesh.size()

    def __del__(self):
        if getattr(self, "_h", None) and _lib._lib is not None:
            _lib._lib.ifgf_plan_free(self._h)
            self._h = None

    @property
    def depth(self):
        return lib().ifgf_plan_depth(self._h)

    @property
    def gamma(self):
        return lib().ifgf_plan_gamma(self._h)

    @property
    def strategy(self):
        return DlStrategy(lib().ifgf_plan_strategy(self._h))

    @property
    def setup_seconds(self):
        return lib().ifgf_plan_setup_seconds(self._h)

    def perm(self):
        p = np.zeros(self.n, dtype=np.uint32)
        check(lib().ifgf_plan_perm(self._h, _ptr(p, u32_p)))
        return p

    def tree_geom(self):
        rm = np.zeros(3)
        side = C.c_double()
        check(lib().ifgf_plan_tree_geom(self._h, _ptr(rm), C.byref(side)))
        return rm, side.value

    def boxes(self, d):
        nb = lib().ifgf_plan_nboxes(self._h, d)
        key = np.zeros(nb, dtype=np.uint64)
        cell = np.zeros((nb, 3), dtype=np.int32)
        beg = np.zeros(nb, dtype=np.uint32)
        end = np.zeros(nb, dtype=np.uint32)
        par = np.zeros(nb, dtype=np.int32)
        ch = np.zeros((nb, 8), dtype=np.int32)
        check(lib().ifgf_plan_boxes(self._h, d, _ptr(key, u64_p), _ptr(cell, i32_p), _ptr(beg, u32_p),
                                    _ptr(end, u32_p), _ptr(par, i32_p), _ptr(ch, i32_p)))
        return dict(key=key, coords=cell, begin=beg, end=end, parent=par, children=ch)

    def relation(self, d, which):
        nb = lib().ifgf_plan_nboxes(self._h, d)
        total = lib().ifgf_plan_relation(self._h, d, which, None, None)
        ptr = np.zeros(nb + 1, dtype=np.int32)
        idx = np.zeros(max(total, 1), dtype=np.int32)
        lib().ifgf_plan_relation(self._h, d, which, _ptr(ptr, i32_p), _ptr(idx, i32_p))
        return ptr, idx[:total]

    def level_cones(self, d):
        params = np.zeros(4, dtype=np.int32)
        deltas = np.zeros(3)
        nseg = lib().ifgf_plan_level(self._h, d, _ptr(params, i32_p), _ptr(deltas), None, None)
        box = np.zeros(max(nseg, 1), dtype=np.int32)
        gam = np.zeros(max(nseg, 1), dtype=np.int32)
        lib().ifgf_plan_level(self._h, d, None, None, _ptr(box, i32_p), _ptr(gam, i32_p))
        return dict(ns=int(params[0]), nc=int(params[1]), ps=int(params[2]), pang=int(params[3]),
                    ds=deltas[0], dth=deltas[1], dph=deltas[2], seg_box=box[:nseg], seg_gamma=gam[:nseg])

    def evaluations(self, d, which):
        return int(lib().ifgf_plan_evaluations(self._h, d, which))

    def decision_hash(self, d):
        """FNV-1a of level d's per-evaluation segment ordinals and parent groups."""
        return int(lib().ifgf_plan_decision_hash(self._h, d))

    def proximity(self):
        L = lib()
        npairs = L.ifgf_plan_npairs(self._h)
        nfar = L.ifgf_plan_nfar(self._h)
        out = dict(target=np.zeros(npairs, dtype=np.uint32), patch=np.zeros(npairs, dtype=np.int32),
                   ubar=np.zeros(npairs), vbar=np.zeros(npairs), far_begin=np.zeros(npairs, dtype=np.uint32),
                   far_end=np.zeros(npairs, dtype=np.uint32),
                   target_pair_begin=np.zeros(self.n + 1, dtype=np.uint32),
                   far_nodes=np.zeros(max(nfar, 1), dtype=np.uint32))
        check(L.ifgf_plan_pairs(self._h, _ptr(out["target"], u32_p), _ptr(out["patch"], i32_p),
                                _ptr(out["ubar"]), _ptr(out["vbar"]), _ptr(out["far_begin"], u32_p),
                                _ptr(out["far_end"], u32_p), _ptr(out["target_pair_begin"], u32_p),
                                _ptr(out["far_nodes"], u32_p)))
        out["far_nodes"] = out["far_nodes"][:nfar]
        return out

    def beta_fingerprint(self):
        return int(lib().ifgf_plan_beta_fingerprint(self._h))

    def diagnostics(self) -> str:
        buf = C.create_string_buffer(1 << 16)
        check(lib().ifgf_plan_diagnostics(self._h, buf, len(buf)))
        return buf.value.decode()


class CombinedOperator:
    """B200 combined-field operator 1/2 I + D - i gamma S (solver.hpp:47-84).

    The constructor does the reference-identical host setup, uploads the plan to HBM and
    computes the RP beta tables on the GPU. The mesh must outlive the operator, as in the
    reference (solver.hpp:73)."""

    def __init__(self, mesh: SurfaceMesh, cfg: SolveConfig, plan: HostPlan | None = None,
                 compute_beta: bool = True):
        self.mesh = mesh
        self.cfg = cfg
        h = C.c_void_p()
        if plan is None:
            if not compute_beta:
                plan = HostPlan(mesh, cfg)
            else:
                c = cfg.to_c()
                check(lib().ifgf_operator_create(mesh._h, C.byref(c), C.byref(h)), "CombinedOperator")
        if plan is not None:
            check(lib().ifgf_operator_from_plan(plan._h, cfg.device, int(compute_beta), C.byref(h)),
                  "CombinedOperator")
        self._h = h
        self.n = int(lib().ifgf_operator_size(h))

    def __del__(self):
        if getattr(self, "_h", None) and _lib._lib is not None:
            _lib._lib.ifgf_operator_free(self._h)
            self._h = None

    @property
    def gamma(self) -> float:
        return float(lib().ifgf_operator_gamma(self._h))

    @property
    def k(self) -> float:
        return self.cfg.k

    def apply(self, density) -> np.ndarray:
        phi = _cvec(density, self.n)
        out = np.empty(self.n, dtype=np.complex128)
        check(lib().ifgf_operator_apply(self._h, _ptr(phi), _ptr(out)), "apply")
        return out

    def apply_into(self, phi: np.ndarray, out: np.ndarray) -> None:
        """apply() into caller-owned (e.g. pinned) buffers, no allocation or copy. Both must be
        C-contiguous complex128 of shape (n,) and out writeable (InvalidArgument otherwise, as
        the reference's size checks, solver.cpp:82)."""
        for name, v in (("phi", phi), ("out", out)):
            if not isinstance(v, np.ndarray) or v.dtype != np.complex128 or v.shape != (self.n,) \
                    or not v.flags.c_contiguous:
                raise _lib.InvalidArgument(f"apply_into: {name} must be a C-contiguous complex128 array of shape ({self.n},)")
        if not out.flags.writeable:
            raise _lib.InvalidArgument("apply_into: out is not writeable")
        check(lib().ifgf_operator_apply(self._h, _ptr(phi), _ptr(out)), "apply")

    @property
    def beta_cache_hit(self) -> bool:
        """the tables came from cfg.beta_cache_path (CombinedOperator::beta_cache_was_reused)"""
        return lib().ifgf_operator_beta_cache_hit(self._h) == 1

    def layer_potentials(self, density):
        phi = _cvec(density, self.n)
        S = np.empty(self.n, dtype=np.complex128)
        D = np.empty(self.n, dtype=np.complex128)
        check(lib().ifgf_operator_layer_potentials(self._h, _ptr(phi), _ptr(S), _ptr(D)), "layer_potentials")
        return S, D

    def apply_direct(self, density) -> np.ndarray:
        phi = _cvec(density, self.n)
        out = np.empty(self.n, dtype=np.complex128)
        check(lib().ifgf_operator_apply_direct(self._h, _ptr(phi), _ptr(out)), "apply_direct")
        return out

    def ifgf_apply(self, a, single_layer=True, double_layer=True, strategy: DlStrategy | None = None):
        av = _cvec(a, self.n)
        S = np.zeros(self.n, dtype=np.complex128)
        D = np.zeros(self.n, dtype=np.complex128)
        st = -1 if strategy is None else int(strategy)
        check(lib().ifgf_operator_ifgf_apply(self._h, _ptr(av), int(single_layer), int(double_layer), st,
                                             _ptr(S), _ptr(D)), "ifgf_apply")
        return S, D

    def level_d_fill(self, a_perm, pipes) -> np.ndarray:
        av = _cvec(a_perm, self.n)
        pp = np.ascontiguousarray([int(p) for p in pipes], dtype=np.int32)
        n = lib().ifgf_operator_level_d_fill(self._h, _ptr(av), _ptr(pp, i32_p), len(pp), None, 0)
        if n < 0:
            check(-n, "level_d_fill")
        out = np.zeros(n, dtype=np.complex128)
        got = lib().ifgf_operator_level_d_fill(self._h, _ptr(av), _ptr(pp, i32_p), len(pp), _ptr(out), n)
        if got < 0:
            check(-got, "level_d_fill")
        return out

    def rp_singular_apply(self, density):
        phi = _cvec(density, self.n)
        S = np.zeros(self.n, dtype=np.complex128)
        D = np.zeros(self.n, dtype=np.complex128)
        check(lib().ifgf_operator_rp_apply(self._h, _ptr(phi), _ptr(S), _ptr(D)), "rp_apply")
        return S, D

    def beta(self):
        m = int(lib().ifgf_operator_beta_entries(self._h))
        npairs = int(lib().ifgf_operator_npairs(self._h))
        bs = np.zeros(m, dtype=np.complex128)
        bd = np.zeros(m, dtype=np.complex128)
        off = np.zeros(npairs + 1, dtype=np.uint64)
        check(lib().ifgf_operator_get_beta(self._h, _ptr(off, u64_p), _ptr(bs), _ptr(bd)), "get_beta")
        return off, bs, bd

    def set_beta(self, offset, bs, bd):
        off = np.ascontiguousarray(offset, dtype=np.uint64)
        s = _cvec(bs)
        d = _cvec(bd)
        check(lib().ifgf_operator_set_beta(self._h, _ptr(off, u64_p), _ptr(s), _ptr(d)), "set_beta")

    def compute_beta(self):
        """(Re)compute the beta tables on the GPU: all pairs, or after set_partition /
        set_comm only the owned targets' pairs (target-sharded)."""
        check(lib().ifgf_operator_compute_beta(self._h), "compute_beta")

    def save_beta_cache(self, path: str):
        check(lib().ifgf_operator_save_beta_cache(self._h, path.encode()), "save_beta_cache")

    def load_beta_cache(self, path: str) -> bool:
        rc = lib().ifgf_operator_load_beta_cache(self._h, path.encode())
        if rc < 0:
            check(-rc, "load_beta_cache")
        return rc == 1

    # ---- measurement helpers
    def upload_density(self, density):
        phi = _cvec(density, self.n)
        check(lib().ifgf_operator_upload_density(self._h, _ptr(phi)), "upload_density")

    def time_applies(self, iters: int, flush_l2: bool = True) -> float:
        ms = C.c_double()
        check(lib().ifgf_operator_time_applies(self._h, iters, int(flush_l2), C.byref(ms)), "time_applies")
        return ms.value

    def time_applies_each(self, iters: int, flush_l2: bool = True) -> np.ndarray:
        """Device time (ms) of each of `iters` graph applies (CUDA events, engine stream)."""
        out = np.zeros(max(iters, 1))
        check(lib().ifgf_operator_time_applies_each(self._h, iters, int(flush_l2), _ptr(out)), "time_applies_each")
        return out[:iters]

    def time_phases(self) -> dict:
        v = np.zeros(7)
        check(lib().ifgf_operator_time_phases(self._h, _ptr(v)), "time_phases")
        return dict(zip(["weights", "leaf", "cousin", "parent", "near", "rp", "total"], v.tolist()))

    def kernels_per_apply(self) -> int:
        return int(lib().ifgf_operator_kernels_per_apply(self._h))

    def setup_times(self) -> dict:
        v = np.zeros(5)
        check(lib().ifgf_operator_setup_times(self._h, _ptr(v)), "setup_times")
        return dict(zip(["tree", "cone_plan", "proximity", "upload", "beta"], v.tolist()))

    # ---- multi-GPU
    def partition(self, parts: int) -> np.ndarray:
        """cost-balanced, leaf-aligned Morton boundaries (parts + 1)"""
        b = np.zeros(parts + 1, dtype=np.uint32)
        check(lib().ifgf_operator_partition(self._h, parts, _ptr(b, u32_p)), "partition")
        return b

    def set_partition(self, lo: int, hi: int):
        check(lib().ifgf_operator_set_partition(self._h, int(lo), int(hi)), "set_partition")

    def set_comm(self, rank: int, world: int, unique_id: bytes):
        buf = C.create_string_buffer(bytes(unique_id), 128)
        check(lib().ifgf_operator_set_comm(self._h, rank, world, buf), "set_comm")

    def finish_owned(self, density, far_S, far_D) -> np.ndarray:
        phi, fs, fd = _cvec(density, self.n), _cvec(far_S, self.n), _cvec(far_D, self.n)
        out = np.zeros(self.n, dtype=np.complex128)
        check(lib().ifgf_operator_finish_owned(self._h, _ptr(phi), _ptr(fs), _ptr(fd), _ptr(out)), "finish_owned")
        return out

    def work(self) -> dict:
        """Algorithmic work of one apply (counts, flops, HBM bytes per phase)."""
        w = np.zeros(16)
        check(lib().ifgf_operator_work(self._h, _ptr(w)), "work")
        return _work_dict(w)


WORK_KEYS = ["leaf_interactions", "cousin_evals", "parent_evals", "near_pairs", "rp_pairs",
             "leaf_flops", "cousin_flops", "parent_flops", "near_flops", "rp_flops",
             "leaf_bytes", "cousin_bytes", "parent_bytes", "near_bytes", "rp_bytes", "total_flops"]


def _work_dict(w):
    return dict(zip(WORK_KEYS, [float(x) for x in w]))


@dataclass
class GmresResult:  # solver.hpp:86-91
    solution: np.ndarray
    residual_history: list
    iterations: int
    converged: bool


def gmres_solve(op: CombinedOperator, rhs, tol: float, max_iter: int, restart: int = 0) -> GmresResult:
    b = _cvec(rhs, op.n)
    x = np.zeros(op.n, dtype=np.complex128)
    hist = np.zeros(max_iter + 1)
    it = C.c_int()
    cv = C.c_int()
    check(lib().ifgf_gmres_solve(op._h, _ptr(b), tol, max_iter, restart, _ptr(x), _ptr(hist), len(hist),
                                 C.byref(it), C.byref(cv)), "gmres_solve")
    return GmresResult(x, hist[: it.value].tolist(), it.value, bool(cv.value))


@dataclass
class IncidentField:  # solver.hpp:17-26: plane wave (theta, phi) or point sources
    theta: float = 0.0
    phi: float = float(np.pi)
    sources: object = None  # (n, 3) point-source positions: Kind::PointSources when given

    def wave_direction(self) -> np.ndarray:
        return np.array([np.cos(self.theta) * np.sin(self.phi), np.sin(self.theta) * np.sin(self.phi),
                         np.cos(self.phi)])

    def _src(self):
        if self.sources is None:
            return np.zeros((0, 3))
        return np.ascontiguousarray(self.sources, dtype=np.float64).reshape(-1, 3)


def incident_trace(incident: IncidentField, mesh: SurfaceMesh, k: float) -> np.ndarray:
    """u^i at the surface nodes (solver.hpp:28-30)."""
    src = incident._src()
    out = np.zeros(mesh.size(), dtype=np.complex128)
    check(lib().ifgf_incident_trace(mesh._h, k, incident.theta, incident.phi, _ptr(src), src.shape[0], _ptr(out)),
          "incident_trace")
    return out


def solve(op: CombinedOperator, incident: IncidentField, tol=None, max_iter=None, restart=None) -> GmresResult:
    """solve(mesh, incident, cfg) (solver.hpp:111-112): GMRES on the device for -u^i."""
    tol = op.cfg.tol if tol is None else tol
    max_iter = op.cfg.max_iter if max_iter is None else max_iter
    restart = op.cfg.restart if restart is None else restart
    src = incident._src()
    x = np.zeros(op.n, dtype=np.complex128)
    hist = np.zeros(max_iter + 1)
    it = C.c_int()
    cv = C.c_int()
    check(lib().ifgf_solve_incident(op._h, incident.theta, incident.phi, _ptr(src), src.shape[0], tol, max_iter,
                                    restart, _ptr(x), _ptr(hist), len(hist), C.byref(it), C.byref(cv)), "solve")
    return GmresResult(x, hist[: it.value].tolist(), it.value, bool(cv.value))
