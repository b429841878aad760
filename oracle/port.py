"""TEST INFRASTRUCTURE ONLY: ctypes driver of the C restatement (oracle/ifgf_oracle.c).

It feeds the restatement with the reference's own plan objects (exported from
oracle/_ref through oracle/ref.py) and returns the IFGF far field, the near field and the
RP correction computed by plain C — an oracle independent of both the reference binary's
apply and the B200 product, pinned against the reference in tests/test_oracle.py.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

from . import ref as R

LIB = os.path.join(os.path.dirname(os.path.abspath(__file__)), "_ref", "libifgf_oracle.so")
_lib = None

d_p = C.POINTER(C.c_double)
i32_p = C.POINTER(C.c_int32)
u32_p = C.POINTER(C.c_uint32)
u64_p = C.POINTER(C.c_uint64)
i64_p = C.POINTER(C.c_int64)
int_p = C.POINTER(C.c_int)


class OracleIfgf(C.Structure):
    _fields_ = [("n", C.c_int), ("depth", C.c_int), ("k", C.c_double), ("root_min", C.c_double * 3),
                ("root_side", C.c_double), ("px", d_p), ("py", d_p), ("pz", d_p), ("nx", d_p), ("ny", d_p),
                ("nz", d_p), ("nboxes", int_p), ("cell", C.POINTER(i32_p)), ("beg", C.POINTER(u32_p)),
                ("end", C.POINTER(u32_p)), ("child", C.POINTER(i32_p)), ("cz_ptr", C.POINTER(i32_p)),
                ("cz_idx", C.POINTER(i32_p)), ("ns", int_p), ("nc", int_p), ("nseg", int_p),
                ("seg_box", C.POINTER(i32_p)), ("seg_gamma", C.POINTER(i32_p)), ("npipes", int_p),
                ("pipes", int_p), ("ps", C.c_int), ("pang", C.c_int)]


class OracleNear(C.Structure):
    _fields_ = [("n", C.c_int), ("k", C.c_double), ("x", d_p), ("y", d_p), ("z", d_p), ("nx", d_p), ("ny", d_p),
                ("nz", d_p), ("jw", d_p), ("patch_of", i32_p), ("leaf_of", i32_p), ("perm", u32_p),
                ("leaf_beg", u32_p), ("leaf_end", u32_p), ("nb_ptr", i32_p), ("nb_idx", i32_p), ("tpb", u32_p),
                ("pair_patch", i32_p), ("far_begin", u32_p), ("far_end", u32_p), ("far_nodes", u32_p)]


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            raise RuntimeError(f"C oracle not built: {LIB} (make -C oracle)")
        L = C.CDLL(LIB)
        L.oracle_ifgf_apply.argtypes = [C.POINTER(OracleIfgf), d_p, d_p, d_p]
        L.oracle_level_d_fill.argtypes = [C.POINTER(OracleIfgf), d_p, d_p]
        L.oracle_near_field.argtypes = [C.POINTER(OracleNear), d_p, d_p, d_p]
        L.oracle_rp_apply.argtypes = [C.c_int, C.c_int, i32_p, i32_p, i64_p, u32_p, i32_p, u64_p, d_p, d_p, d_p,
                                      d_p, d_p]
        _lib = L
    return _lib


def _p(a, t=d_p):
    return a.ctypes.data_as(t)


def _pipes(strategy, depth, lam, side):
    """pipes_at for both layers (ifgf.cpp:132-140, 193-207)"""
    out = []
    for d in range(1, depth + 1):
        if strategy == 0:
            dl = [4]
        elif strategy == 1:
            dl = [2, 3]
        else:
            dl = [2, 3] if side(d) / lam < 0.5 - 1e-12 else [4]
        out.append([1] + dl)
    return out


class Restatement:
    """The C restatement bound to one reference operator's plan."""

    def __init__(self, ro: "R.RefOperator"):
        self.ro = ro
        self.keep = []
        mesh = ro.mesh
        D = ro.depth
        perm = ro.perm()
        rm, side = ro.tree_geom()
        self.perm = perm
        self.n = n = mesh.n
        pos = np.ascontiguousarray(mesh.pos[perm])
        nrm = np.ascontiguousarray(mesh.normal[perm])
        cols = [np.ascontiguousarray(pos[:, i]) for i in range(3)] + [np.ascontiguousarray(nrm[:, i]) for i in range(3)]
        self.keep += cols
        o = OracleIfgf()
        o.n, o.depth, o.k = n, D, ro.k
        o.root_min = (C.c_double * 3)(*rm)
        o.root_side = side
        o.px, o.py, o.pz, o.nx, o.ny, o.nz = (_p(c) for c in cols)
        nboxes = np.zeros(D, dtype=np.int32)
        ns = np.zeros(D, dtype=np.int32)
        nc = np.zeros(D, dtype=np.int32)
        nseg = np.zeros(D, dtype=np.int32)
        P = {key: (C.POINTER(t) * D)() for key, t in
             [("cell", C.c_int32), ("beg", C.c_uint32), ("end", C.c_uint32), ("child", C.c_int32),
              ("cz_ptr", C.c_int32), ("cz_idx", C.c_int32), ("seg_box", C.c_int32), ("seg_gamma", C.c_int32)]}
        lam = 2 * np.pi / ro.k
        pipes = _pipes(ro.strategy, D, lam, lambda d: side / float(1 << (d - 1)))
        npipes = np.array([len(p) for p in pipes], dtype=np.int32)
        pipe_arr = np.zeros(3 * D, dtype=np.int32)
        ps = pang = 0
        for d in range(1, D + 1):
            bx = ro.boxes(d)
            nboxes[d - 1] = len(bx["key"])
            arrs = {"cell": np.ascontiguousarray(bx["coords"].reshape(-1)), "beg": bx["begin"], "end": bx["end"],
                    "child": np.ascontiguousarray(bx["children"].reshape(-1))}
            ptr, idx = ro.relation(d, 1)
            arrs["cz_ptr"], arrs["cz_idx"] = ptr, np.ascontiguousarray(idx) if len(idx) else np.zeros(1, np.int32)
            if d >= 3:
                lc = ro.level_cones(d)
                ns[d - 1], nc[d - 1] = lc["ns"], lc["nc"]
                nseg[d - 1] = len(lc["seg_box"])
                ps, pang = lc["ps"], lc["pang"]
                arrs["seg_box"] = lc["seg_box"] if nseg[d - 1] else np.zeros(1, np.int32)
                arrs["seg_gamma"] = lc["seg_gamma"] if nseg[d - 1] else np.zeros(1, np.int32)
            for key, a in arrs.items():
                a = np.ascontiguousarray(a)
                self.keep.append(a)
                P[key][d - 1] = a.ctypes.data_as(C.POINTER(C.c_int32 if a.dtype == np.int32 else C.c_uint32))
            pipe_arr[3 * (d - 1): 3 * (d - 1) + len(pipes[d - 1])] = pipes[d - 1]
        for a in (nboxes, ns, nc, nseg, npipes, pipe_arr):
            self.keep.append(a)
        o.nboxes, o.ns, o.nc, o.nseg = (_p(a, int_p) for a in (nboxes, ns, nc, nseg))
        o.npipes, o.pipes = _p(npipes, int_p), _p(pipe_arr, int_p)
        for key, arr in P.items():
            setattr(o, key, arr)
        self.keep.append(P)
        o.ps, o.pang = ps, pang
        self.o = o
        self.nseg_leaf = int(nseg[D - 1])
        self.P = ps * pang * pang
        self.pipes = pipes

    def ifgf_apply(self, a):
        """a in original order -> (single, dbl) in original order (ifgf_apply)"""
        ap = np.ascontiguousarray(np.asarray(a, dtype=np.complex128)[self.perm])
        S = np.zeros(self.n, dtype=np.complex128)
        Dd = np.zeros(self.n, dtype=np.complex128)
        rc = lib().oracle_ifgf_apply(C.byref(self.o), _p(ap.view(np.float64)), _p(S.view(np.float64)),
                                     _p(Dd.view(np.float64)))
        if rc:
            raise RuntimeError(f"oracle_ifgf_apply failed ({rc})")
        outS = np.zeros_like(S)
        outD = np.zeros_like(Dd)
        outS[self.perm] = S
        outD[self.perm] = Dd
        return outS, outD

    def level_d_fill(self, a_perm):
        ap = np.ascontiguousarray(a_perm, dtype=np.complex128)
        out = np.zeros(self.nseg_leaf * len(self.pipes[-1]) * self.P, dtype=np.complex128)
        lib().oracle_level_d_fill(C.byref(self.o), _p(ap.view(np.float64)), _p(out.view(np.float64)))
        return out

    def near_field(self, phi):
        ro, mesh = self.ro, self.ro.mesh
        D = ro.depth
        leaf = ro.boxes(D)
        nbp, nbi = ro.relation(D, 0)
        pr = ro.proximity()
        leaf_of = np.zeros(self.n, dtype=np.int32)
        R.lib().ref_op_leaf_of_point(ro.h, _p(leaf_of, i32_p))
        arrs = dict(x=mesh.pos[:, 0], y=mesh.pos[:, 1], z=mesh.pos[:, 2], nx=mesh.normal[:, 0],
                    ny=mesh.normal[:, 1], nz=mesh.normal[:, 2], jw=mesh.jac * mesh.weight)
        arrs = {k: np.ascontiguousarray(v) for k, v in arrs.items()}
        ints = dict(patch_of=mesh.patch_of, leaf_of=leaf_of, perm=self.perm, leaf_beg=leaf["begin"],
                    leaf_end=leaf["end"], nb_ptr=nbp, nb_idx=nbi, tpb=pr["target_pair_begin"],
                    pair_patch=pr["patch"], far_begin=pr["far_begin"], far_end=pr["far_end"],
                    far_nodes=pr["far_nodes"] if len(pr["far_nodes"]) else np.zeros(1, np.uint32))
        ints = {k: np.ascontiguousarray(v) for k, v in ints.items()}
        o = OracleNear()
        o.n, o.k = self.n, ro.k
        for k, v in arrs.items():
            setattr(o, k, _p(v))
        for k, v in ints.items():
            setattr(o, k, v.ctypes.data_as(C.POINTER(C.c_int32 if v.dtype == np.int32 else C.c_uint32)))
        phi = np.ascontiguousarray(phi, dtype=np.complex128)
        S = np.zeros(self.n, dtype=np.complex128)
        Dd = np.zeros(self.n, dtype=np.complex128)
        lib().oracle_near_field(C.byref(o), _p(phi.view(np.float64)), _p(S.view(np.float64)),
                                _p(Dd.view(np.float64)))
        return S, Dd

    def rp_apply(self, phi):
        ro, mesh = self.ro, self.ro.mesh
        pr = ro.proximity()
        off, bs, bd = ro.beta()
        nu = np.array([p.nu for p in mesh.patches], dtype=np.int32)
        nv = np.array([p.nv for p in mesh.patches], dtype=np.int32)
        start = np.concatenate([[0], np.cumsum(nu.astype(np.int64) * nv)]).astype(np.int64)
        phi = np.ascontiguousarray(phi, dtype=np.complex128)
        S = np.zeros(self.n, dtype=np.complex128)
        Dd = np.zeros(self.n, dtype=np.complex128)
        tpb = np.ascontiguousarray(pr["target_pair_begin"])
        pp = np.ascontiguousarray(pr["patch"])
        lib().oracle_rp_apply(self.n, len(nu), _p(nu, i32_p), _p(nv, i32_p), _p(start, i64_p), _p(tpb, u32_p),
                              _p(pp, i32_p), _p(off, u64_p), _p(bs.view(np.float64)), _p(bd.view(np.float64)),
                              _p(phi.view(np.float64)), _p(S.view(np.float64)), _p(Dd.view(np.float64)))
        return S, Dd

    def apply(self, phi):
        """out = 1/2 phi + D - i gamma S from the restated far, near and RP parts"""
        mesh = self.ro.mesh
        a = phi * mesh.jac * mesh.weight
        S, Dd = self.ifgf_apply(a)
        nS, nD = self.near_field(phi)
        rS, rD = self.rp_apply(phi)
        S, Dd = S + nS + rS, Dd + nD + rD
        return 0.5 * phi + Dd - 1j * self.ro.gamma * S, S, Dd
