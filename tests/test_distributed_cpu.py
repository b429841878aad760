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


# ---- the per-apply exchange layout of the NCCL path (engine.cu reduce_far_to_owners /
# allgather_to_original, exchange_kernels.cu), restated in numpy and run over gloo at world 2
# with the real plan partition: each rank's Morton range padded to the longest range C;
# reduce-scatter send [rank][S | D][C]; all-gather of the owned outputs, then
# out[perm[t]] = recv[r(t) C + t - bounds[r(t)]]. (gloo has no reduce_scatter: all_reduce +
# the rank's chunk is the same sum.)
def _pack_ranges(Sp, Dp, bounds, C):
    world = len(bounds) - 1
    send = np.zeros((world, 2, C), complex)
    for r in range(world):
        lo, hi = bounds[r], bounds[r + 1]
        send[r, 0, : hi - lo] = Sp[lo:hi]
        send[r, 1, : hi - lo] = Dp[lo:hi]
    return send


def _exchange_worker(rank, world, port, q):
    import torch

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    import paper_2112_06316_b200 as P
    from paper_2112_06316_b200.distributed import plan_partition

    mesh = P.SurfaceMesh.sphere(1.0, 2, 8, 8)
    plan = P.HostPlan(mesh, P.SolveConfig(k=4 * np.pi, device=-1))
    bounds = [int(x) for x in plan_partition(plan, world)]
    perm = plan.perm().astype(np.int64)
    n = mesh.size()
    C = max(bounds[r + 1] - bounds[r] for r in range(world))
    rng = np.random.default_rng(100 + rank)
    Sp = rng.standard_normal(n) + 1j * rng.standard_normal(n)  # this rank's far partials (Morton)
    Dp = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    send = _pack_ranges(Sp, Dp, bounds, C)
    t = torch.from_numpy(send.view(np.float64).copy())
    dist.all_reduce(t)
    mine = t.numpy().view(complex).reshape(world, 2, C)[rank]
    lo, hi = bounds[rank], bounds[rank + 1]
    S_owned, D_owned = mine[0, : hi - lo], mine[1, : hi - lo]
    # owned outputs (here: S + D), padded, all-gathered, un-permuted into original order
    seg = np.zeros(C, complex)
    seg[: hi - lo] = S_owned + D_owned
    out_t = [torch.zeros(2 * C, dtype=torch.float64) for _ in range(world)]
    dist.all_gather(out_t, torch.from_numpy(seg.view(np.float64).copy()))
    recv = np.concatenate([x.numpy().view(complex) for x in out_t])
    out = np.zeros(n, complex)
    for tt in range(n):
        r = max(i for i in range(world) if bounds[i] <= tt) if tt < bounds[-1] else world - 1
        out[perm[tt]] = recv[r * C + tt - bounds[r]]
    q.put((rank, Sp, Dp, S_owned, D_owned, out, bounds, perm))
    dist.destroy_process_group()


def test_exchange_layout_world2():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_exchange_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=300) for _ in range(world)], key=lambda x: x[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    bounds, perm = res[0][6], res[0][7]
    S_sum = sum(x[1] for x in res)
    D_sum = sum(x[2] for x in res)
    for r, Sp, Dp, S_owned, D_owned, out, _, _ in res:
        lo, hi = bounds[r], bounds[r + 1]
        assert np.allclose(S_owned, S_sum[lo:hi], rtol=0, atol=1e-12)  # every partial reached its owner
        assert np.allclose(D_owned, D_sum[lo:hi], rtol=0, atol=1e-12)
    want = np.zeros(len(perm), complex)
    want[perm] = S_sum + D_sum  # original order
    for x in res:
        assert np.allclose(x[5], want, rtol=0, atol=1e-12)  # every rank holds the full output


def test_bench_gives_each_local_rank_its_share_of_the_cores():
    # torch.distributed.run exports OMP_NUM_THREADS=1 to its workers; bench.py replaces it
    # before any OpenMP runtime loads (the host setup is OpenMP code), and leaves a
    # single-rank run alone
    import os
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = "import os, sys; sys.argv = ['bench.py'] + sys.argv[1:]; import bench; print(os.environ.get('OMP_NUM_THREADS'))"
    cores = os.cpu_count() or 1

    def run(env_extra, *argv):
        env = dict(os.environ, **env_extra)
        out = subprocess.run([sys.executable, "-c", code, *argv], cwd=root, env=env, capture_output=True, text=True)
        assert out.returncode == 0, out.stderr
        return out.stdout.strip().splitlines()[-1]

    assert run({"LOCAL_WORLD_SIZE": "2", "OMP_NUM_THREADS": "1"}) == str(max(1, cores // 2))
    assert run({"LOCAL_WORLD_SIZE": "2", "OMP_NUM_THREADS": "1"}, "--impl", "reference") == str(cores)
    assert run({"LOCAL_WORLD_SIZE": "1", "OMP_NUM_THREADS": "3"}) == "3"
