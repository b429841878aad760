"""The multi-GPU data plane executed on hardware: bench.py's torchrun path at world 1.

DistributedCombinedOperator always creates its NCCL communicator, so on one GPU the whole
distributed apply runs — ncclReduceScatter of the padded far-field partials, the owned-target
combine, ncclAllGather + un-permute, NCCL captured inside the CUDA graph — and so does the
Morton-sharded GMRES (allreduce per inner product). At world 1 the collectives are identities,
so the apply must equal the single-GPU apply bit for bit and GMRES must take the same
iterations (the local Morton-order partial sums round differently: the relative-residual
histories agree to 1e-12 absolute).
The N > 1 layout logic is covered on CPU with gloo (tests/test_distributed_cpu.py)."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

HERE = os.path.dirname(os.path.abspath(__file__))


def _port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_torchrun_world1_collective_path():
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node=1", "--master-addr",
           "127.0.0.1", "--master-port", str(_port()), os.path.join(HERE, "dist", "torchrun_worker.py")]
    p = subprocess.run(cmd, capture_output=True, text=True, timeout=900)
    lines = [l for l in p.stdout.splitlines() if l.startswith("RESULT ")]
    assert p.returncode == 0 and lines, p.stdout[-3000:] + p.stderr[-3000:]
    r = json.loads(lines[0][len("RESULT "):])
    print(r)
    assert r["world"] == 1
    assert all(r["apply_bitwise"]), r["apply_rel"]
    assert r["apply_after_timing_bitwise"]
    # pack + reduce-scatter unpack + pad + all-gather un-permute on top of the single-GPU kernels
    assert r["kernels_per_apply"] == r["single_kernels_per_apply"] + 4
    for key in ("gmres_r0", "gmres_r5"):
        g = r[key]
        assert g["iters"][0] == g["iters"][1] and g["converged"][0] and g["converged"][1], g
        assert g["hist_max_abs"] is not None and g["hist_max_abs"] <= 1e-12, g
        assert g["x_rel"] <= 1e-10, g
