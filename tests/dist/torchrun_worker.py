"""Worker for tests/test_gpu_torchrun.py: runs under torch.distributed.run (NCCL), builds the
DistributedCombinedOperator (the multi-GPU path: per-rank plan, set_comm, ncclReduceScatter
of the far-field partials, ncclAllGather of the outputs, NCCL captured in the apply graph,
Morton-sharded GMRES) and, on every rank, a plain single-GPU CombinedOperator of the same
mesh, then prints one JSON line per rank with the comparisons."""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2112_06316_b200 as P  # noqa: E402
from paper_2112_06316_b200.distributed import DistributedCombinedOperator  # noqa: E402


def main():
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    rank, world = dist.get_rank(), dist.get_world_size()
    splits, nu, k = (int(sys.argv[1]), int(sys.argv[2]), float(sys.argv[3])) if len(sys.argv) > 3 else (2, 16, 4 * np.pi)
    mesh = P.SurfaceMesh.sphere(1.0, splits, nu, nu)
    cfg = P.SolveConfig(k=k, gamma=k, device=local)
    single = P.CombinedOperator(mesh, cfg)
    op = DistributedCombinedOperator(mesh, cfg)
    n = mesh.size()
    phi = P.random_density(n, 1)
    ref = single.apply(phi)
    outs = [op.apply(phi) for _ in range(3)]  # eager, capture, graph replay
    res = {"rank": rank, "world": world, "n": n, "kernels_per_apply": op.kernels_per_apply(),
           "single_kernels_per_apply": single.kernels_per_apply()}
    res["apply_bitwise"] = [bool(np.array_equal(o, ref)) for o in outs]
    res["apply_rel"] = [float(np.linalg.norm(o - ref) / np.linalg.norm(ref)) for o in outs]
    # device-resident graph replays (NCCL inside the graph)
    op.upload_density(phi)
    res["ms_per_apply"] = float(op.time_applies(3, flush_l2=False))
    res["apply_after_timing_bitwise"] = bool(np.array_equal(op.apply(phi), ref))
    # sharded GMRES vs the single-GPU GMRES (restarted and not)
    rhs = -P.incident_trace(P.IncidentField(theta=0.0, phi=0.0), mesh, k)
    for restart in (0, 5):
        a = P.gmres_solve(single, rhs, 1e-8, 40, restart)
        b = P.gmres_solve(op, rhs, 1e-8, 40, restart)
        h1, h2 = np.array(a.residual_history), np.array(b.residual_history)
        res[f"gmres_r{restart}"] = {
            "iters": [a.iterations, b.iterations], "converged": [a.converged, b.converged],
            # the history is the relative residual |r_j| / |b|: differences are absolute in it
            "hist_max_abs": float(np.max(np.abs(h1 - h2))) if len(h1) == len(h2) and len(h1) else None,
            "x_rel": float(np.linalg.norm(a.solution - b.solution) / np.linalg.norm(a.solution))}
    print("RESULT " + json.dumps(res), flush=True)
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
