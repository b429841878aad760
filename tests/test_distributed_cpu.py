"""Host side of the multi-GPU path on CPU with torch.distributed (gloo, world size 2):
every rank builds the same plan and derives the same cost-balanced, leaf-aligned
partition without communicating; the NCCL unique id travels through the process group."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2112_06316_b200 as P
    from paper_2112_06316_b200.distributed import broadcast_unique_id, plan_partition

    mesh = P.SurfaceMesh.sphere(1.0, 2, 16, 16)
    plan = P.HostPlan(mesh, P.SolveConfig(k=4 * np.pi, gamma=4 * np.pi))
    b = plan_partition(plan, world)
    uid = broadcast_unique_id(rank)
    gathered = [None] * world
    dist.all_gather_object(gathered, (b.tolist(), uid))
    q.put((rank, gathered, plan.boxes(plan.depth)["begin"].tolist(), mesh.size()))
    dist.destroy_process_group()


def test_partition_agrees_across_ranks_and_is_leaf_aligned():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    _, gathered, leaf_begin, n = res[0]
    bounds = [g[0] for g in gathered]
    uids = [g[1] for g in gathered]
    assert bounds[0] == bounds[1]  # identical partition on both ranks
    assert uids[0] == uids[1] and len(uids[0]) == 128  # the NCCL id reached every rank
    b = bounds[0]
    assert b[0] == 0 and b[-1] == n and b[0] < b[1] < b[2]
    assert set(b[1:-1]) <= set(leaf_begin) | {n}  # cuts at leaf-box boundaries


def test_partition_balance_single_process():
    import paper_2112_06316_b200 as P
    from paper_2112_06316_b200.distributed import plan_partition

    mesh = P.SurfaceMesh.sphere(1.0, 3, 16, 16)
    plan = P.HostPlan(mesh, P.SolveConfig(k=8 * np.pi))
    for parts in (1, 2, 4, 8):
        b = plan_partition(plan, parts).astype(np.int64)
        sizes = np.diff(b)
        assert b[0] == 0 and b[-1] == mesh.size() and np.all(sizes > 0)
        assert sizes.max() <= 2.0 * sizes.mean()  # cost-balanced, so roughly point-balanced


def _worker_per_rank(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2112_06316_b200 as P
    from paper_2112_06316_b200.distributed import plan_partition

    mesh = P.SurfaceMesh.sphere(1.0, 2, 16, 16)
    cfg = P.SolveConfig(k=4 * np.pi, gamma=4 * np.pi, device=-1, part_rank=rank, part_world=world)
    plan = P.HostPlan(mesh, cfg)  # this rank's share only
    b = plan_partition(plan, world)
    segs = {d: sorted(zip(plan.level_cones(d)["seg_box"].tolist(), plan.level_cones(d)["seg_gamma"].tolist()))
            for d in range(3, plan.depth + 1)}
    npairs = len(plan.proximity()["target"])
    gathered = [None] * world
    dist.all_gather_object(gathered, (b.tolist(), segs, npairs))
    q.put((rank, gathered))
    dist.destroy_process_group()


def test_per_rank_plans_over_gloo():
    # each rank builds only its share of the plan (SolveConfig.part_rank / part_world) with a
    # partition derived identically on every rank; together the shares cover the full plan
    import paper_2112_06316_b200 as P

    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker_per_rank, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    gathered = res[0][1]
    assert gathered[0][0] == gathered[1][0]  # same partition on both ranks
    mesh = P.SurfaceMesh.sphere(1.0, 2, 16, 16)
    full = P.HostPlan(mesh, P.SolveConfig(k=4 * np.pi, gamma=4 * np.pi, device=-1))
    for d in range(3, full.depth + 1):
        F = set(zip(full.level_cones(d)["seg_box"].tolist(), full.level_cones(d)["seg_gamma"].tolist()))
        union = set(gathered[0][1][d]) | set(gathered[1][1][d])
        assert union == F, d
    # pairs are classified for the owned targets only: the shares add up to the full list
    assert gathered[0][2] + gathered[1][2] == len(full.proximity()["target"])
