"""The C-ABI library loads without a GPU and exports every symbol include/ifgf_b200.h declares;
host-only entry points report errors with the reference's exception taxonomy."""
import ctypes
import re

import numpy as np
import pytest

import paper_2112_06316_b200 as P
from paper_2112_06316_b200 import _lib


def declared_symbols():
    txt = open(_lib.HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(ifgf_[a-z0-9_]+)\s*\(", txt)))


def test_library_loads_and_exports_header_symbols():
    L = P.lib()
    names = declared_symbols()
    assert len(names) > 50
    missing = [n for n in names if not hasattr(L, n)]
    assert not missing, missing
    # the Python binding covers exactly the header
    assert sorted(_lib.exported_symbols()) == names


def test_shared_object_is_sm100a_cuda_build():
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_error_taxonomy_host_side():
    with pytest.raises(P.InvalidArgument):
        P.SurfaceMesh.sphere(-1.0, 0, 4, 4)
    mesh = P.SurfaceMesh.sphere(1.0, 0, 4, 4)
    # the reference's messages (solver.cpp:45, ifgf.cpp plan_cones, rp.cpp classify_targets)
    with pytest.raises(P.InvalidArgument, match="wavenumber must be positive"):
        P.HostPlan(mesh, P.SolveConfig(k=0.0))
    with pytest.raises(P.InvalidArgument, match="interpolation orders must lie in"):
        P.HostPlan(mesh, P.SolveConfig(k=2 * np.pi, cone=P.ConeConfig(ps=13)))
    assert "interpolation orders" in P.lib().ifgf_last_error().decode()
    with pytest.raises(P.InvalidArgument, match="n_beta >= 2 and cov_d >= 2"):
        P.HostPlan(mesh, P.SolveConfig(k=2 * np.pi, rp=P.RpConfig(n_beta=1)))
    assert "classify_targets" in P.lib().ifgf_last_error().decode()


def test_config_defaults_match_reference():
    c = _lib.IfgfConfig()
    P.lib().ifgf_config_default(ctypes.byref(c))
    # solver.hpp:32-45, ifgf.hpp:12-17, rp.hpp:14-19
    assert (c.gamma, c.strategy, c.finest_box_lambda) == (-1.0, 2, 0.5)
    assert (c.n_c0, c.n_s0, c.ps, c.pang) == (2, 1, 3, 5)
    assert (c.delta_rel, c.delta_abs, c.n_beta, c.cov_d) == (1.0, -1.0, 96, 6)
