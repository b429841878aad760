"""Multi-GPU operator: one process per GPU (torch.distributed for the rendezvous only),
NCCL inside the engine for the per-apply exchange.

Each rank owns the sources and targets of a cost-balanced, leaf-aligned Morton range:
  1. IFGF far field of the owned sources onto ALL targets (leaf fill of owned leaves,
     parent fill and cousin evaluation only for boxes holding owned sources);
  2. one ncclReduceScatter of the far-field partials (every rank's range padded to the
     longest) to the owner of each target range;
  3. near field + RP + combine for the owned targets (every rank holds the full phi; the
     beta tables hold only the owned targets' pairs);
  4. one ncclAllGather of the owned outputs, so every rank returns the full out.
The NCCL calls are captured into the apply's CUDA graph with the kernels. gmres_solve on
this operator keeps only the owned Morton segment of every Krylov vector (one allreduce of
2 doubles per inner product). At world 1 the same collective path runs (NCCL over a
single-rank communicator), which is how it is exercised on one GPU.
Each rank partitions with the same deterministic, plan-free cost model and then builds
only its share of the cone plan, so the partition needs no communication; only the
128-byte ncclUniqueId is broadcast.
"""
from __future__ import annotations

import ctypes as C
import dataclasses

import numpy as np

from ._lib import check, lib, u32_p
from .operator import CombinedOperator, HostPlan, SolveConfig, SurfaceMesh, nccl_unique_id


def plan_partition(plan: HostPlan, parts: int) -> np.ndarray:
    """cost-balanced, leaf-aligned Morton boundaries (host only, no GPU)"""
    b = np.zeros(parts + 1, dtype=np.uint32)
    check(lib().ifgf_plan_partition(plan._h, parts, b.ctypes.data_as(u32_p)), "plan_partition")
    return b


def broadcast_unique_id(rank: int) -> bytes:
    """rank 0 creates the ncclUniqueId, torch.distributed carries it to the others"""
    import torch
    import torch.distributed as dist

    uid = nccl_unique_id() if rank == 0 else bytes(128)
    t = torch.tensor(list(uid), dtype=torch.uint8)
    if dist.get_backend() == "nccl":
        t = t.cuda()
    dist.broadcast(t, src=0)
    return bytes(t.cpu().tolist())


class DistributedCombinedOperator(CombinedOperator):
    """CombinedOperator over torch.distributed's world: same apply(), full in/out on every rank."""

    def __init__(self, mesh: SurfaceMesh, cfg: SolveConfig):
        import torch.distributed as dist

        self.rank = dist.get_rank()
        self.world = dist.get_world_size()
        # per-rank plan (only boxes holding this rank's sources) and beta tables sharded by
        # target owner, built once the partition is set
        if self.world > 1:
            cfg = dataclasses.replace(cfg, part_rank=self.rank, part_world=self.world)
        super().__init__(mesh, cfg, compute_beta=False)
        uid = broadcast_unique_id(self.rank)
        self.set_comm(self.rank, self.world, uid)
        self.compute_beta()
        self.bounds = self.partition(self.world)

    @property
    def owned(self):
        return int(self.bounds[self.rank]), int(self.bounds[self.rank + 1])
